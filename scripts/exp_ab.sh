#!/bin/bash
# A/B of -D flag sets in one box: bench fps (16 in flight, graphs), stage split, pruned fps.
#   gpurun -- 'bash scripts/exp_ab.sh "-DA=1" "-DA=0" ...'   (each variant run twice, interleaved)
mkdir -p gpurun_out
for R in 1 2; do
for V in "$@"; do
  NVCC_APPEND_FLAGS="$V" python -m paper_2412_00578_b200.build --force > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  timeout 400 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --no-configs --steps 10 2>/dev/null > gpurun_out/ab.json
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); s=d['stages_ms']; print('$V', round(d['value'],1), 'pruned', round(d['pruned']['value'],1), {k: round(v,4) for k,v in s.items()})"
done
done
python -m paper_2412_00578_b200.build --force > /dev/null
