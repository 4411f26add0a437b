#!/bin/bash
OUT=gpurun_out/${1:-a4}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_wan.py -x -q --timeout 200 > $OUT/pytest_attn.log 2>&1
echo "rc=$?" >> $OUT/pytest_attn.log
if grep -q " passed" $OUT/pytest_attn.log && ! grep -q "failed\|Timeout\|rc=[1-9]" $OUT/pytest_attn.log; then
  for v in default nonpersist default nonpersist; do
    if [ $v = default ]; then E=""; elif [ $v = single ]; then E="LP_ATTN_SINGLE=1"; elif [ $v = nonpersist ]; then E="LP_ATTN_NONPERSIST=1"; else E="LIVEPIPE_LIB=$PWD/paper_2512_04677_b200/$v.so"; fi
    env $E timeout 420 python bench.py --no-cpu-baseline --no-decode --steps 4 > $OUT/bench_$v.json 2> $OUT/bench_$v.err
    python -c "import json; d=json.loads(open('$OUT/bench_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],3), d['clocks']['sm_mhz'], {k: round(x['avg_ms'],4) for k,x in d['kernels'].items()})" >> $OUT/summary.txt 2>&1
  done
  timeout 420 python bench.py --history-sigma 0.1 --no-cpu-baseline --no-decode --steps 4 > $OUT/bench_sigma.json 2> $OUT/bench_sigma.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe --no-decode > $OUT/bench_ncu.log 2>&1
fi
tail -3 $OUT/pytest_attn.log; cat $OUT/summary.txt
