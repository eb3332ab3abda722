#!/bin/bash
# Experiment: level-1 kernels (k_l1_count, k_l1_emit) minimum CTAs per SM.
F=paper_2412_00578_b200/csrc/ss_bin.cu
cp $F /tmp/exp_orig.cu
for V in "$@"; do
  cp /tmp/exp_orig.cu $F
  sed -i "s/__launch_bounds__(kBinWarps \* 32, 3)/__launch_bounds__(kBinWarps * 32, $V)/g" $F
  python -m paper_2412_00578_b200.build --force --verbose 2>&1 | grep -E "Compiling entry function|Used [0-9]+ registers|spill" | grep -A2 "k_l1_emitILi9" | grep -i "regis\|spill" | head -2
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --steps 10 > gpurun_out/l1$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/l1$V.json')); print($V, round(d['value'],1), round(d['stages_ms']['bin'],4))"
done
cp /tmp/exp_orig.cu $F
