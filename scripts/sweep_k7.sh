#!/bin/bash
# K7 variant sweep at n = m = N (default 1e6): rows per thread x interleaved
# columns of the dot-product kernel, and the difference-form kernel.
#   scripts/sweep_k7.sh N OUT "RPT list" "CU list"
N=${1:-1000000}
OUT=${2:-gpurun_out/sweep_k7.txt}
RPTS=${3:-"4 2 1"}
CUS=${4:-"1 2 4"}
: > "$OUT"
for rpt in $RPTS; do
  for cu in $CUS; do
    echo -n "dot rpt=$rpt cu=$cu: " >> "$OUT"
    RPLU_GEMV_RPT=$rpt RPLU_GEMV_CU=$cu python scripts/profile_gauss.py $N 2>&1 | tail -1 >> "$OUT"
  done
done
echo -n "diff rpt=4: " >> "$OUT"
RPLU_GEMV_DOT=0 python scripts/profile_gauss.py $N 2>&1 | tail -1 >> "$OUT"
cat "$OUT"
