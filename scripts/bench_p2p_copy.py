"""16 MiB peer-to-peer copy GPU0 -> GPU1 (the TP pull of the critical rank's
partial): copy engine (cudaMemcpyAsync) vs an SM copy kernel on the reader.

    python scripts/bench_p2p_copy.py      # needs 2 GPUs
"""
import json

import torch

n = 8 << 20  # bf16 elements = 16 MiB
src = torch.randn(n, device="cuda:0").bfloat16()
dst = torch.empty(n, device="cuda:1", dtype=torch.bfloat16)
dst.copy_(src)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
for name, fn in (("copy_engine_peer", lambda: dst.copy_(src, non_blocking=True)),):
    with torch.cuda.device(1):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(5):
            fn()
        torch.cuda.synchronize(1)
        s.record()
        for _ in range(50):
            fn()
        e.record()
        torch.cuda.synchronize(1)
        us = s.elapsed_time(e) / 50 * 1e3
        print(json.dumps({"how": name, "us": round(us, 1), "GBps": round(n * 2 / us / 1e3, 1)}))

# the same 16 MiB as k concurrent chunks on k streams of the reader (several
# copy engines)
for k in (2, 4, 8):
    with torch.cuda.device(1):
        streams = [torch.cuda.Stream(device=1) for _ in range(k)]
        ch = n // k
        main = torch.cuda.current_stream(1)

        def multi():
            ev = torch.cuda.Event()
            ev.record(main)
            for i, st in enumerate(streams):
                st.wait_event(ev)
                with torch.cuda.stream(st):
                    dst[i * ch:(i + 1) * ch].copy_(src[i * ch:(i + 1) * ch], non_blocking=True)
            for st in streams:
                e2 = torch.cuda.Event()
                e2.record(st)
                main.wait_event(e2)
        for _ in range(5):
            multi()
        torch.cuda.synchronize(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(main)
        for _ in range(50):
            multi()
        e.record(main)
        torch.cuda.synchronize(1)
        us = s.elapsed_time(e) / 50 * 1e3
        print(json.dumps({"how": f"copy_engine_peer x{k} streams", "us": round(us, 1),
                          "GBps": round(n * 2 / us / 1e3, 1)}))
# SM copy kernel on the reader (remote loads over NVLink)
with torch.cuda.device(1):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    srcv = src.view(torch.int32)  # noqa
    for _ in range(3):
        torch.add(src.to("cuda:1", non_blocking=True), 0)
    torch.cuda.synchronize(1)
