#!/bin/bash
# Experiment: onesweep look-back back-off (ns) x depth, bench bin stage.
for V in "$@"; do
  S=${V%x*}; L=${V#*x}
  NVCC_APPEND_FLAGS="-DSS_SORT_SLEEP=$S -DSS_SORT_LB=$L" python -m paper_2412_00578_b200.build --force > /dev/null 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --steps 10 > gpurun_out/ss$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ss$V.json')); print('$V', round(d['value'],1), round(d['stages_ms']['bin'],4))"
done
python -m paper_2412_00578_b200.build --force > /dev/null
