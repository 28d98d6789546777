"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``) into
per-kernel shares over the last ``--window`` launches (one step).

    python scripts/launch_summary.py gpurun_out/launches.csv --window 805 \
        --command "..." > profiles/r01_launches_1gpu_v4.json

ncu times are cold-cache and serialised: compare shares, not absolutes.
"""
import argparse
import csv
import json
from collections import OrderedDict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--window", type=int, default=0, help="launches in one step (last N)")
    ap.add_argument("--tick", default="step_tick_kernel",
                    help="kernel launched once per step: with --window 0 the window is the "
                         "launches between its last two complete occurrences")
    ap.add_argument("--command", default="")
    a = ap.parse_args()
    rows = []
    with open(a.csv) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1.0)
        rows.append((int(r["ID"]), r["Kernel Name"], v * scale))
    rows.sort()
    where = ""
    if a.window:
        win = rows[-a.window:]
    else:
        ticks = [i for i, (_, k, _) in enumerate(rows) if a.tick in k]
        win = rows[ticks[-2]:ticks[-1]]
    where = f"launches {rows.index(win[0])}..{rows.index(win[-1])}" if not a.window else f"last {len(win)}"
    total = sum(t for _, _, t in win)
    agg = OrderedDict()
    for _, k, t in win:
        e = agg.setdefault(k, [0, 0.0])
        e[0] += 1
        e[1] += t
    kernels = [{"kernel": k, "launches": n, "total_ns": t, "share": round(t / total, 3)}
               for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    print(json.dumps({"command": a.command,
                      "window": f"{where} of {len(rows)} launches = one step ({len(win)} launches)",
                      "note": "cold-cache, serialised launches: compare SHARES, not absolutes",
                      "unit": "ns", "total_ms": total / 1e6, "kernels": kernels}, indent=1))


if __name__ == "__main__":
    main()
