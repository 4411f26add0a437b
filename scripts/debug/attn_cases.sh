#!/bin/bash
OUT=gpurun_out/${1:-dbg}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
for c in "390 2 0 0" "390 2 1 0" "390 2 0 2" "390 2 1 2" "1000 4 0 3" "1000 4 1 3" "4680 40 0 4" "4680 40 1 4"; do
  echo "case $c" >> $OUT/cases.log
  timeout 60 python scripts/debug/attn_case.py $c >> $OUT/cases.log 2>&1
  echo "rc=$?" >> $OUT/cases.log
done
cat $OUT/cases.log
