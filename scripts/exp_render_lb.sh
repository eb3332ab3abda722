#!/bin/bash
# Experiment: k_render minimum CTAs per SM in __launch_bounds__.
F=paper_2412_00578_b200/csrc/ss_render.cu
cp $F /tmp/exp_orig.cu
for V in "$@"; do
  cp /tmp/exp_orig.cu $F
  sed -i "s/__global__ void __launch_bounds__(256, [0-9]) k_render(const uint2/__global__ void __launch_bounds__(256, $V) k_render(const uint2/" $F
  python -m paper_2412_00578_b200.build --force --verbose 2>&1 | grep -A2 "k_renderILb0" | grep -i "regis"
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --steps 10 > gpurun_out/lb$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/lb$V.json')); print($V, round(d['value'],1), round(d['stages_ms']['render'],4))"
done
cp /tmp/exp_orig.cu $F
