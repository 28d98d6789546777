"""Collect the PARITY / PIN / SMCAP / BF16FLOOR lines printed by the GPU
parity tests (pytest -s) and scripts/bf16_floor.py from gpurun logs into one
JSON summary for profiles/.

    python scripts/parity_summary.py gpurun_out/r02_*.log > profiles/r02_parity_shapes.json
"""
import json
import sys


def main():
    out = {"sources": sys.argv[1:], "parity": {}, "oracle_pin": {}, "sm_cap": [], "bf16_floor": {}}
    for path in sys.argv[1:]:
        for line in open(path, errors="replace"):
            line = line.strip()
            for tag in ("PARITY ", "PIN ", "SMCAP ", "BF16FLOOR "):
                i = line.find(tag)
                if i < 0 or not line[i + len(tag):].startswith("{"):
                    continue
                try:
                    d = json.loads(line[i + len(tag):])
                except json.JSONDecodeError:
                    continue
                if tag == "PARITY ":
                    out["parity"][d["plan"]] = dict(d, log=path)
                elif tag == "PIN ":
                    out["oracle_pin"][d["plan"]] = dict(d, log=path)
                elif tag == "SMCAP ":
                    out["sm_cap"].append(dict(d, log=path))
                else:
                    out["bf16_floor"][d["plan"]] = dict(
                        {k: v for k, v in d.items() if k != "variants"},
                        variants=[{k: v for k, v in x.items() if not k.startswith("per_tensor")}
                                  for x in d["variants"]], log=path)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
