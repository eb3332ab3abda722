#!/bin/bash
# Experiment: onesweep resident CTAs per SM (launch bounds + persistent grid cap).
F=paper_2412_00578_b200/csrc/ss_sort.cu
cp $F /tmp/exp_orig.cu
for V in "$@"; do
  cp /tmp/exp_orig.cu $F
  sed -i "s/__launch_bounds__(kSortThreads, [0-9]*) k_onesweep/__launch_bounds__(kSortThreads, $V) k_onesweep/; s/const uint32_t cap = (uint32_t)sms \* [0-9]*;/const uint32_t cap = (uint32_t)sms * $V;/" $F
  python -m paper_2412_00578_b200.build --force --verbose 2>&1 | grep -A2 "k_onesweepIjLb0ELb0ELb1E" | grep -i "regis"
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --steps 10 > gpurun_out/sr$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sr$V.json')); print($V, round(d['value'],1), round(d['stages_ms']['bin'],4))"
done
cp /tmp/exp_orig.cu $F
