"""Throughput and SM clock of the tcgen05 GEMM vs cuBLAS on one shape,
each back to back for ~3 s with nvidia-smi sampling: under the B200 power cap
TFLOP/s per MHz separates kernel efficiency from energy per FLOP.

    python scripts/bench_gemm_clock.py [M N K]
"""
import json
import statistics
import subprocess
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2409_01143_b200 import _lib as L  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (8192, 8192, 8192)
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)


def ours():
    assert L.hexexec_k_gemm(M, N, K, 1, 1, A.data_ptr(), 0, K, 0, 0, B.data_ptr(), 0, K, 0, 0,
                            C.data_ptr(), N, 0, 0, 0, 0, 1.0, 0, None) == 0


def cublas():
    torch.matmul(A, B.t(), out=C)


def run(fn, secs=3.0):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                          "--format=csv,noheader,nounits", "-lms", "100"],
                         stdout=subprocess.PIPE, text=True)
    time.sleep(0.5)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    s.record()
    n = 0
    while time.time() - t0 < secs:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    p.terminate()
    out = p.communicate()[0].strip().splitlines()
    rows = [[float(v) for v in r.split(",")] for r in out if r.strip()]
    rows = rows[len(rows) // 4:]  # steady part
    ms = s.elapsed_time(e) / n
    tf = 2.0 * M * N * K / ms / 1e9
    mhz = statistics.median(r[0] for r in rows)
    w = statistics.median(r[1] for r in rows)
    return {"tflops": round(tf, 1), "sm_mhz": mhz, "power_w": w,
            "tflops_per_ghz": round(tf / mhz * 1e3, 1), "gflop_per_joule": round(tf * 1e3 / w, 1)}


print(json.dumps({"shape": [M, N, K], "ours": run(ours), "cublas": run(cublas)}))
