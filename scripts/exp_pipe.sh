#!/bin/bash
# Experiment: -D flag sets -> bench fps (16 in flight) and the pipelined stage costs.
for V in "$@"; do
  NVCC_APPEND_FLAGS="$V" python -m paper_2412_00578_b200.build --force > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  F=$(timeout 400 python bench.py --no-cpu-baseline --no-e2e --no-backward --no-train --no-score --no-configs --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['pruned']['value'],1))")
  D=$(timeout 400 python scripts/diag_pipelined_stages.py | tail -1)
  echo "$V | $F | $D"
done
python -m paper_2412_00578_b200.build --force > /dev/null
