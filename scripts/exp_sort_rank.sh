#!/bin/bash
# Experiment: onesweep ranking by match.any (1) or ballots (0), bench bin stage.
for V in "$@"; do
  NVCC_APPEND_FLAGS="-DSS_SORT_MATCH=$V" python -m paper_2412_00578_b200.build --force > /dev/null 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --steps 10 > gpurun_out/sm$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sm$V.json')); print('$V', round(d['value'],1), round(d['stages_ms']['bin'],4))"
done
python -m paper_2412_00578_b200.build --force > /dev/null
