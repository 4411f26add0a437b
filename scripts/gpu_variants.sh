#!/bin/bash
# Bench several builds of the library (LIVEPIPE_LIB) back to back: attention avg ms per variant.
OUT=gpurun_out/${1:-var}
shift
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); a=torch.randn(64,64,device='cuda'); a@a" > /dev/null 2>&1
for v in "$@"; do
  LIVEPIPE_LIB=$PWD/paper_2512_04677_b200/$v timeout 400 python bench.py --no-cpu-baseline --steps 3 > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  python -c "import json,sys; d=json.load(open('$OUT/bench_$v.json')); print('$v', round(d['value'],3), {k: round(x['avg_ms'],4) for k,x in d['kernels'].items()})" >> $OUT/summary.txt 2>&1
done
cat $OUT/summary.txt
