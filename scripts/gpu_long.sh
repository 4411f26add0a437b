#!/bin/bash
# BASELINE config 4 at shape: a 10k-frame (834-block) 14B stream with RSFM, the rolling window and
# history noise (sigma 0.1), from a cold start; plus the headline and sigma bench lines.
OUT=gpurun_out/${1:-long}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
timeout 1500 python bench.py --long-horizon 834 --history-sigma 0.1 > $OUT/bench_long834.json 2> $OUT/bench_long834.err
timeout 420 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
timeout 420 python bench.py --history-sigma 0.1 --no-cpu-baseline --no-decode > $OUT/bench_sigma.json 2> $OUT/bench_sigma.err
tail -c 1500 $OUT/bench_long834.json; tail -3 $OUT/bench_long834.err
