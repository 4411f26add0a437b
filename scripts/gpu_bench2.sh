#!/bin/bash
OUT=gpurun_out/${1:-b2}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); a=torch.randn(64,64,device='cuda'); a@a" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > $OUT/pytest_gemm.log 2>&1; tail -1 $OUT/pytest_gemm.log
timeout 420 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
timeout 420 python bench.py --no-cpu-baseline --config 1.3b > $OUT/bench13.json 2> $OUT/bench13.err
for f in bench bench13; do python -c "import json; d=json.load(open('$OUT/$f.json')); print('$f', round(d['value'],3), {k: round(x['avg_ms'],4) for k,x in d['kernels'].items()})"; done
