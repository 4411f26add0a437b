OUT=gpurun_out/g3; mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); a=torch.randn(64,64,device='cuda'); a@a" > /dev/null 2>&1
LP_GEMM2_ALL=1 timeout 420 python bench.py --no-cpu-baseline > $OUT/bench_all.json 2> $OUT/bench_all.err
python -c "import json; d=json.load(open('$OUT/bench_all.json')); print('all2', round(d['value'],3), {k: round(x['avg_ms'],4) for k,x in d['kernels'].items()})"
