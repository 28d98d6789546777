"""Join the ncu --set full capture of scripts/gemm_traffic_probe.py with its
shape list: per GEMM, DRAM bytes read + written (cold-cache replay) against
the algorithmic bytes, tensor-pipe activity and duration; plus the
launch-weighted average per launch of the step's TP linear GEMMs (each of the
12 shapes runs once per layer and micro-batch), which bench.py reports as
roofline.traffic.

    python scripts/gemm_traffic_summary.py gpurun_out/r02_gemm_probe.ncu-rep \\
        gpurun_out/r02_gemm_probe.log > profiles/r02_gemm_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

MET = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
       "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active,"
       "sm__cycles_elapsed.avg.per_second")


def main():
    rep, log = sys.argv[1], sys.argv[2]
    shapes = None
    for line in open(log):
        if line.startswith('{"shapes"'):
            shapes = json.loads(line)["shapes"]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", MET],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0,
             "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3}
    out = []
    for sh, r in zip(shapes, data):
        d = {}
        for h, u, v in zip(hdr, units, r):
            if h.startswith(("dram__", "gpu__", "sm__")):
                d[h] = float(v.replace(",", "")) * scale.get(u, 1.0)
        traffic = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        out.append(dict(sh, duration_us=round(d["gpu__time_duration.sum"], 2),
                        dram_bytes=traffic, traffic_over_algorithmic=round(traffic / sh["algorithmic_bytes"], 3),
                        tensor_pipe_active_pct=round(d["sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active"], 1),
                        sm_clock_ghz=round(d["sm__cycles_elapsed.avg.per_second"] / 1e9 if d["sm__cycles_elapsed.avg.per_second"] > 1e6 else d["sm__cycles_elapsed.avg.per_second"], 3),
                        tflops=round(sh["flops"] / (d["gpu__time_duration.sum"] * 1e-6) / 1e12, 1)))
    n = len(out)
    print(json.dumps({
        "source": f"ncu --set full --clock-control none -k regex:gemm_kernel (cold-cache replay) of scripts/gemm_traffic_probe.py; report {rep}",
        "bytes_per_launch": sum(o["dram_bytes"] for o in out) / n,
        "algorithmic_bytes_per_launch": sum(o["algorithmic_bytes"] for o in out) / n,
        "flops_per_launch": sum(o["flops"] for o in out) / n,
        "launches": out}, indent=1))


if __name__ == "__main__":
    main()
