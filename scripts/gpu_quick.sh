#!/bin/bash
# Quick GPU iteration: attention/GEMM unit tests + bench (+ optional ncu of one kernel).
# Usage: gpurun -- 'bash scripts/gpu_quick.sh <tag> [kernel-regex]'
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_gemm.py -x -q > $OUT/pytest_kern.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
if [ -n "$2" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${3:-700} -c 1 \
    -o $OUT/prof python bench.py --steps 1 --warmup 5 --no-cpu-baseline --no-probe > $OUT/ncu.log 2>&1
fi
tail -3 $OUT/pytest_kern.log
