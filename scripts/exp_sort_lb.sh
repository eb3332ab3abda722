#!/bin/bash
# Experiment: onesweep look-back depth (predecessors read per round trip), bench bin stage.
for V in "$@"; do
  NVCC_APPEND_FLAGS="-DSS_SORT_LB=$V" python -m paper_2412_00578_b200.build --force --verbose 2>&1 | grep -A2 "k_onesweepIjLb0ELb0ELb1E" | grep -i "regis"
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --steps 10 > gpurun_out/slb$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/slb$V.json')); print($V, round(d['value'],1), round(d['stages_ms']['bin'],4))"
done
python -m paper_2412_00578_b200.build --force > /dev/null
