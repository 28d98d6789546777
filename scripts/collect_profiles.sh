#!/bin/bash
# Copy the round's GPU evidence from gpurun_out/ (scratch) into profiles/ (tracked).
#   bash scripts/collect_profiles.sh r02
set -e
R=${1:-r02}
cd "$(dirname "$0")/.."
for n in 1 2 4; do
  [ -f gpurun_out/${R}_gputests${n}.log ] && cp gpurun_out/${R}_gputests${n}.log profiles/
done
: > profiles/${R}_bench_lines.jsonl
for f in gpurun_out/${R}_bench1_final.json gpurun_out/${R}_bench1_ref.json gpurun_out/${R}_bench2_final.json gpurun_out/${R}_bench4_final.json; do
  [ -f "$f" ] && grep -h '^{' "$f" | tail -1 >> profiles/${R}_bench_lines.jsonl
done
python scripts/parity_summary.py gpurun_out/${R}_gputests*.log gpurun_out/${R}_bf16_floor2.log > profiles/${R}_parity_shapes.json
[ -f gpurun_out/${R}_bench_attn_final.log ] && cp gpurun_out/${R}_bench_attn_final.log profiles/${R}_bench_attn.log
echo collected
