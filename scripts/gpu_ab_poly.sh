#!/bin/bash
# A/B: degree of the bounded-exponent attention's FMA-pipe 2^f polynomial (library variants via
# LIVEPIPE_LIB), interleaved to average out clock drift; parity of the degree-2 build.
OUT=gpurun_out/${1:-poly}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
D=$PWD/paper_2512_04677_b200
LIVEPIPE_LIB=$D/lib_deg2.so timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_wan_shapes.py -q -k "not 1p3b_full and not fp32" --timeout 400 -rf > $OUT/pytest_deg2.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_deg2.log
for rep in 1 2; do
  for v in lib_base lib_deg2 lib_deg2w4; do
    LIVEPIPE_LIB=$D/$v.so timeout 400 python bench.py --no-cpu-baseline --no-decode --steps 5 --warmup 3 > $OUT/bench_${v}_$rep.json 2> $OUT/bench_${v}_$rep.err
  done
done
tail -3 $OUT/pytest_deg2.log
for f in $OUT/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],3), d['clocks']['sm_mhz'], round(d['kernels']['attention']['avg_ms'],4))"; done
