#!/bin/bash
# Iteration check: kernel unit tests + selected tests + bench (+ optional ncu of one kernel).
# Usage: gpurun -- 'bash scripts/gpu_iter.sh <tag> "<pytest -k expr>" [kernel-regex]'
TAG=${1:-it}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_attn.py tests/test_gpu_gemm.py -x -q --timeout 200 > $OUT/pytest_kern.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_kern.log
if [ -n "$2" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -k "$2" --timeout 1200 -rf > $OUT/pytest_sel.log 2>&1
  echo "pytest rc=$?" >> $OUT/pytest_sel.log
fi
timeout 420 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
if [ -n "$3" ]; then
  timeout 500 ncu --set full --clock-control none --import-source on -k regex:$3 -s ${4:-700} -c 1 \
    -o $OUT/prof python bench.py --steps 1 --warmup 5 --no-cpu-baseline --no-probe > $OUT/ncu.log 2>&1
fi
tail -3 $OUT/pytest_kern.log; tail -5 $OUT/pytest_sel.log 2>/dev/null; tail -c 600 $OUT/bench.json
