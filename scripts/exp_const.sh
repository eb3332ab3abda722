#!/bin/bash
# Experiment: sweep one integer constexpr.  usage: exp_const.sh <file> <name> <values...>
F=paper_2412_00578_b200/csrc/$1; N=$2; shift 2
cp $F /tmp/exp_orig.cu
for V in "$@"; do
  cp /tmp/exp_orig.cu $F
  sed -i "s/constexpr int $N = [0-9]*;/constexpr int $N = $V;/" $F
  grep -q "constexpr int $N = $V;" $F || { echo "not applied $V"; continue; }
  python -m paper_2412_00578_b200.build --force > /dev/null 2>&1 || { echo "build failed $V"; continue; }
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --steps 10 > gpurun_out/c$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c$V.json')); print('$N', $V, round(d['value'],1), {k: round(v,4) for k,v in d['stages_ms'].items()})"
done
cp /tmp/exp_orig.cu $F
python -m paper_2412_00578_b200.build --force > /dev/null 2>&1
