#!/bin/bash
# Like exp_flags.sh, also reporting the pruned-regime (config 5) fps.
i=0
for V in "$@"; do
  i=$((i+1))
  NVCC_APPEND_FLAGS="$V" python -m paper_2412_00578_b200.build --force > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  timeout 400 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --steps 10 > gpurun_out/xp$i.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/xp$i.json')); print('$V', round(d['value'],1), 'pruned', round(d['pruned']['value'],1), {k: round(v,4) for k,v in d['stages_ms'].items()})" || echo "run failed: $V"
done
python -m paper_2412_00578_b200.build --force > /dev/null
