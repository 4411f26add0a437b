#!/bin/bash
# Full validation: all GPU tests (no -x), smoke, bench, drop-in bench (1.3B), short long-horizon stream.
OUT=gpurun_out/${1:-val}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
LP_PARITY_LOG=$OUT/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -rf > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 420 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --api dropin --config 1.3b --steps 5 --warmup 5 > $OUT/bench_dropin.json 2> $OUT/bench_dropin.err
timeout 600 python bench.py --long-horizon ${2:-60} --history-sigma 0.1 > $OUT/bench_long.json 2> $OUT/bench_long.err
tail -6 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; tail -c 300 $OUT/bench.json; tail -c 400 $OUT/bench_dropin.json; tail -c 600 $OUT/bench_long.json; tail -3 $OUT/bench_long.err
