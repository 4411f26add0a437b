#!/bin/bash
OUT=gpurun_out/${1:-r2d}
mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_attn.py -x -q --timeout 200 > $OUT/pytest_attn.log 2>&1
PYTHONPATH=. timeout 500 python scripts/debug/run_1p3b.py bf16 > $OUT/run_bf16.log 2>&1
PYTHONPATH=. CUDA_LAUNCH_BLOCKING=1 timeout 900 python scripts/debug/run_1p3b.py fp32 2 > $OUT/run_fp32.log 2>&1
timeout 420 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
B="python bench.py --steps 1 --warmup 5 --no-cpu-baseline --no-probe"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:attn_tc_kernel<\(bool\)1>' -s 350 -c 1 -o $OUT/attn $B > $OUT/ncu_attn.log 2>&1
tail -3 $OUT/pytest_attn.log; tail -5 $OUT/run_bf16.log; tail -30 $OUT/run_fp32.log; tail -3 $OUT/ncu_attn.log
