#!/bin/bash
# Round-end validation on one B200: every GPU test (no -x), smoke, the headline bench (with the
# CPU baseline), the reference arm, the drop-in and sigma bench lines, and ncu captures of the
# persistent and per-item attention kernels in a steady block.
OUT=gpurun_out/${1:-final}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
LP_PARITY_LOG=$OUT/parity.jsonl timeout 3000 python -m pytest tests -m gpu -q --timeout 1500 -rf --durations=20 > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 python bench.py --api dropin --config 1.3b --steps 5 --warmup 5 > $OUT/bench_dropin.json 2> $OUT/bench_dropin.err
timeout 420 python bench.py --history-sigma 0.1 --no-cpu-baseline > $OUT/bench_sigma.json 2> $OUT/bench_sigma.err
B="python bench.py --steps 1 --warmup 5 --no-cpu-baseline --no-probe --no-decode"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc2p_kernel -s 700 -c 1 -o $OUT/attn_p $B > $OUT/ncu_attn_p.log 2>&1
LP_ATTN_NONPERSIST=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc2_kernel -s 700 -c 1 -o $OUT/attn_np $B > $OUT/ncu_attn_np.log 2>&1
tail -8 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; tail -c 400 $OUT/bench.json
