#!/bin/bash
# Extra bench lines at HEAD: BASELINE config 2 (1.3B) and a repeat of the 14B headline.
OUT=gpurun_out/${1:-lines}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
timeout 600 python bench.py --config 1.3b --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_1p3b.json 2> $OUT/bench_1p3b.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_14b_repeat.json 2> $OUT/bench_14b_repeat.err
tail -c 300 $OUT/bench_1p3b.json; tail -c 300 $OUT/bench_14b_repeat.json
