#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list + full captures.
# Usage (from this container): gpurun --timeout 2400 -- 'bash scripts/gpu_check.sh [tag]'
set -x
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
# launch list: one steady block (3 warm-up blocks + 1 timed + 1 e2e, eager probe pass)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/bench_ncu.log 2>&1
# full captures of the top kernels (one launch each)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 120 -c 1 \
  -o $OUT/attn python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe > $OUT/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 500 -c 5 \
  -o $OUT/gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe > $OUT/ncu_gemm.log 2>&1
ls -la $OUT
