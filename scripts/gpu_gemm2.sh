#!/bin/bash
OUT=gpurun_out/${1:-g2}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); a=torch.randn(64,64,device='cuda'); a@a" > /dev/null 2>&1
timeout 240 python -m pytest tests/test_gpu_gemm.py -x -q > $OUT/pytest_gemm.log 2>&1; echo "gemm rc=$?" >> $OUT/pytest_gemm.log; tail -3 $OUT/pytest_gemm.log
if grep -q " passed" $OUT/pytest_gemm.log && ! grep -q "failed" $OUT/pytest_gemm.log; then
  timeout 420 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
  LP_NO_GEMM2=1 timeout 420 python bench.py --no-cpu-baseline > $OUT/bench_1cta.json 2> $OUT/bench_1cta.err
  for f in bench bench_1cta; do python -c "import json; d=json.load(open('$OUT/$f.json')); print('$f', round(d['value'],3), {k: round(x['avg_ms'],4) for k,x in d['kernels'].items()})"; done
  timeout 300 python -m pytest tests/test_gpu_wan.py -x -q > $OUT/pytest_wan.log 2>&1; tail -1 $OUT/pytest_wan.log
fi
