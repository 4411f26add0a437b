#!/bin/bash
# Full GPU validation: all gpu tests, smoke, bench (headline + history-noise variant).
TAG=${1:-full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); a=torch.randn(64,64,device='cuda'); a@a" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 420 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 420 python bench.py --history-sigma 0.1 --no-cpu-baseline > $OUT/bench_sigma.json 2> $OUT/bench_sigma.err
tail -3 $OUT/pytest_gpu.log; cat $OUT/smoke.log | tail -2; tail -c 300 $OUT/bench.json; grep -v "^frame" $OUT/bench.err | tail -5
