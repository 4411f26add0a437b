#!/bin/bash
# Validate HEAD on one B200: every GPU test, smoke, the headline bench.
OUT=gpurun_out/${1:-head}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
LP_PARITY_LOG=$OUT/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -rf --durations=10 > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
tail -8 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; tail -c 400 $OUT/bench.json
