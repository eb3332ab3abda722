#!/bin/bash
# Experiment: k_render batch size (kBatch) sweep; prints frames/s and the render stage time.
for B in "$@"; do
  sed -i "s/^constexpr int kBatch = [0-9]*;/constexpr int kBatch = $B;/" paper_2412_00578_b200/csrc/ss_render.cu
  python -m paper_2412_00578_b200.build --force > /dev/null 2>&1 || { echo "build failed $B"; continue; }
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --steps 10 > gpurun_out/kb$B.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/kb$B.json')); print($B, round(d['value'],1), round(d['stages_ms']['render'],4))"
done
