#!/bin/bash
# Pipelined cost of the parts of ss_bin (diagnostic builds that stop ss_bin early; a1-a2 rows).
for F in "-DSS_DIAG_BIN_STAGES" "-DSS_DIAG_BIN_UPTO=2" "-DSS_DIAG_BIN_UPTO=3" "-DSS_DIAG_BIN_UPTO=4" ""; do
  NVCC_APPEND_FLAGS="$F" python -m paper_2412_00578_b200.build --force > /dev/null 2>&1
  echo "== $F"; timeout 600 python scripts/diag_pipelined_stages.py 2>&1 | grep "^a1-a2 "
done
python -m paper_2412_00578_b200.build --force > /dev/null
