#!/bin/bash
# Attention kernel iteration: unit tests (pair kernel default, then the single-CTA A/B), bench, ncu of the pair kernel.
OUT=gpurun_out/${1:-a2}
mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_attn.py -x -q --timeout 120 > $OUT/pytest_attn.log 2>&1
echo "rc=$?" >> $OUT/pytest_attn.log
export AB
if grep -q " passed" $OUT/pytest_attn.log && ! grep -q "failed\|Timeout\|rc=[1-9]" $OUT/pytest_attn.log; then
  timeout 420 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
  env ${AB:-LP_ATTN_SINGLE=1} timeout 420 python bench.py --no-cpu-baseline --steps 3 > $OUT/bench_single.json 2> $OUT/bench_single.err
  if [ -n "$2" ]; then
    timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s 700 -c 1 \
      -o $OUT/attn python bench.py --steps 1 --warmup 5 --no-cpu-baseline --no-probe > $OUT/ncu_attn.log 2>&1
  fi
fi
tail -4 $OUT/pytest_attn.log; tail -c 300 $OUT/bench.json
