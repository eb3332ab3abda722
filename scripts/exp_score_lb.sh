#!/bin/bash
# Experiment: k_prune_score minimum CTAs per SM in __launch_bounds__ (score-pass views/s).
F=paper_2412_00578_b200/csrc/ss_render.cu
cp $F /tmp/exp_orig.cu
for V in "$@"; do
  cp /tmp/exp_orig.cu $F
  [ "$V" != "0" ] && sed -i "s/__global__ void __launch_bounds__(256) k_prune_score(/__global__ void __launch_bounds__(256, $V) k_prune_score(/" $F
  python -m paper_2412_00578_b200.build --force --verbose 2>&1 | grep -A2 "k_prune_score" | grep -i "regis"
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --steps 10 > gpurun_out/sl$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sl$V.json')); print($V, round(d['prune_score']['views_per_s'],1))"
done
cp /tmp/exp_orig.cu $F
