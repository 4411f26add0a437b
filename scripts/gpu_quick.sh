#!/bin/bash
# Quick GPU iteration: attention/GEMM unit tests + bench (+ optional ncu of one kernel).
# Usage: gpurun --timeout 1800 -- 'bash scripts/gpu_quick.sh <tag> [kernel-regex] [skip-launches]'
# Per-step timeouts sum below the gpurun limit (a hung kernel is killed by us).
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_attn.py tests/test_gpu_gemm.py -x -q --timeout 120 > $OUT/pytest_kern.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_kern.log
if grep -q "passed" $OUT/pytest_kern.log && ! grep -q "failed\|Timeout" $OUT/pytest_kern.log; then
  timeout 420 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
  if [ -n "$2" ]; then
    timeout 500 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${3:-700} -c 1 \
      -o $OUT/prof python bench.py --steps 1 --warmup 5 --no-cpu-baseline --no-probe > $OUT/ncu.log 2>&1
  fi
fi
tail -3 $OUT/pytest_kern.log
