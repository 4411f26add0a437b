#!/bin/bash
# Round-end validation (round 2, second pass): every GPU test, smoke, the headline bench (with the
# CPU baseline), the reference arm, drop-in and sigma lines, the ncu launch list of a steady block
# and --set full captures of the attention, the norm apply pass and the history-noise kernel.
OUT=gpurun_out/${1:-final2}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
LP_PARITY_LOG=$OUT/parity.jsonl timeout 2700 python -m pytest tests -m gpu -q --timeout 1500 -rfs --durations=15 > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 python bench.py --api dropin --config 1.3b --steps 5 --warmup 5 > $OUT/bench_dropin.json 2> $OUT/bench_dropin.err
timeout 420 python bench.py --history-sigma 0.1 --no-cpu-baseline > $OUT/bench_sigma.json 2> $OUT/bench_sigma.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe --no-decode > $OUT/ncu_launches.log 2>&1
B="python bench.py --steps 1 --warmup 5 --no-cpu-baseline --no-probe --no-decode"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc2p_kernel -s 700 -c 1 -o $OUT/attn_p $B > $OUT/ncu_attn_p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:history_noise_bm -s 1000 -c 1 -o $OUT/hist $B --history-sigma 0.1 > $OUT/ncu_hist.log 2>&1
LP_NORM_STATS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"norm_apply|norm_mod" -s 700 -c 2 -o $OUT/norm $B > $OUT/ncu_norm.log 2>&1
timeout 1200 python bench.py --long-horizon 834 --history-sigma 0.1 --no-cpu-baseline > $OUT/bench_long_horizon_834.json 2> $OUT/bench_long.err
tail -8 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; tail -c 400 $OUT/bench.json
