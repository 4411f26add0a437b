#!/bin/bash
# Round-2 evidence on one B200: ncu launch list of a steady block, --set full captures of the
# pair attention, the four GEMMs of a layer, the norm / history-noise row kernels and a VAE conv.
TAG=${1:-ev2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe > $OUT/bench_ncu.log 2>&1
B="python bench.py --steps 1 --warmup 5 --no-cpu-baseline --no-probe"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:attn_tc2_kernel" -s 700 -c 1 -o $OUT/attn $B > $OUT/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3000 -c 6 -o $OUT/gemm $B > $OUT/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:norm_mod_kernel -s 1000 -c 1 -o $OUT/norm $B > $OUT/ncu_norm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:history_noise -s 700 -c 1 -o $OUT/hist $B --history-sigma 0.1 > $OUT/ncu_hist.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 16 -c 2 -o $OUT/vae python -c "
import torch, paper_2512_04677_b200 as lp
d = lp.VaeDecoder(16, 60, 104, 'cuda:0'); x = torch.randn(3, 16*60*104, device='cuda'); f = torch.empty(12, 3*480*832, device='cuda')
d.decode_into(x, f); torch.cuda.synchronize()" > $OUT/ncu_vae.log 2>&1
ls -la $OUT
# GEMM dispatch A/B (O-proj / FFN-down): pair + tail split (default), no split, pairs everywhere
for ab in "" "LP_NO_PAIR_SPLIT=1" "LP_GEMM2_ALL=1"; do
  env $ab timeout 420 python bench.py --no-cpu-baseline --steps 3 > $OUT/bench_ab_${ab:-default}.json 2> $OUT/bench_ab_${ab:-default}.err
  python -c "import json; d=json.loads(open('$OUT/bench_ab_${ab:-default}.json').read().strip().splitlines()[-1]); print('${ab:-default}', round(d['value'],3), d['clocks']['sm_mhz'], {k: round(x['avg_ms'],4) for k,x in d['kernels'].items()})" >> $OUT/gemm_ab.txt 2>&1
done
timeout 420 python bench.py --history-sigma 0.1 --no-cpu-baseline > $OUT/bench_sigma.json 2> $OUT/bench_sigma.err
cat $OUT/gemm_ab.txt
