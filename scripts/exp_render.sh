#!/bin/bash
# Experiment: k_render CTAs per SM x pairs per loop iteration (bench render stage + fps).
for V in "$@"; do
  B=${V%x*}; U=${V#*x}
  NVCC_APPEND_FLAGS="-DSS_RENDER_MINB=$B -DSS_RENDER_UNROLL=$U" python -m paper_2412_00578_b200.build --force > /dev/null 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --steps 10 > gpurun_out/rv$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/rv$V.json')); print('$V', round(d['value'],1), round(d['stages_ms']['render'],4))"
done
python -m paper_2412_00578_b200.build --force > /dev/null
