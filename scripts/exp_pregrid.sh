#!/bin/bash
# Experiment: k_preprocess grid size (rounds of resident CTAs); frames/s and preprocess time.
for R in "$@"; do
  sed -i "s/const int resident = sms \* kPreBlocks \* [0-9]*;/const int resident = sms * kPreBlocks * $R;/" paper_2412_00578_b200/csrc/ss_geometry.cu
  python -m paper_2412_00578_b200.build --force > /dev/null 2>&1 || { echo "build failed $R"; continue; }
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --steps 10 > gpurun_out/pg$R.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/pg$R.json')); print($R, round(d['value'],1), round(d['stages_ms']['preprocess'],4))"
done
