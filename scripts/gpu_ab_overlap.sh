#!/bin/bash
# History noise on a side stream beside the GEMMs (default) vs in line (LP_HIST_OVERLAP=0):
# the noise / TPP GPU tests, then sigma = 0.1 and sigma = 0 bench lines, interleaved.
OUT=gpurun_out/${1:-ov}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_wan.py tests/test_gpu_attn.py tests/test_gpu_tpp_dist.py tests/test_gpu_reference_engine.py -q -k "noise or sigma or corrupt or history or tpp or abi" --timeout 400 -rf > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
B="python bench.py --no-cpu-baseline --no-decode --steps 5 --warmup 3"
for rep in 1 2; do
  timeout 400 $B --history-sigma 0.1 > $OUT/bench_sigma_ov_$rep.json 2> $OUT/bench_sigma_ov_$rep.err
  LP_HIST_OVERLAP=0 timeout 400 $B --history-sigma 0.1 > $OUT/bench_sigma_inline_$rep.json 2> $OUT/bench_sigma_inline_$rep.err
  timeout 400 $B > $OUT/bench_sigma0_$rep.json 2> $OUT/bench_sigma0_$rep.err
done
tail -3 $OUT/pytest.log
for f in $OUT/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels']
print('$f', round(d['value'],3), d['clocks']['sm_mhz'], {n:round(v['avg_ms'],4) for n,v in k.items() if n in ('attention','qkv','history_noise','ffn_down','o_proj')})"; done
