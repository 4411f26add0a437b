#!/bin/bash
# Last HEAD certification: every GPU test, smoke, and the bench lines (headline with the CPU
# baseline, reference arm, sigma 0.1, drop-in).
OUT=gpurun_out/${1:-final4}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
LP_PARITY_LOG=$OUT/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -rfs --durations=10 > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 420 python bench.py --history-sigma 0.1 --no-cpu-baseline > $OUT/bench_sigma.json 2> $OUT/bench_sigma.err
timeout 600 python bench.py --api dropin --config 1.3b --steps 5 --warmup 5 > $OUT/bench_dropin.json 2> $OUT/bench_dropin.err
tail -6 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; tail -c 300 $OUT/bench.json
