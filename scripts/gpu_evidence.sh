#!/bin/bash
# Round evidence on one B200: bench lines (headline + history-noise variant + reference arm),
# ncu launch list of a steady block, --set full captures of the attention, a GEMM and the
# HBM-bound row kernels.  Usage: gpurun --timeout 3000 -- 'bash scripts/gpu_evidence.sh <tag>'
TAG=${1:-ev}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda(); a=torch.randn(64,64,device='cuda'); a@a" > /dev/null 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --history-sigma 0.1 --no-cpu-baseline > $OUT/bench_sigma.json 2> $OUT/bench_sigma.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 0 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 python bench.py --config 1.3b --no-cpu-baseline > $OUT/bench_1p3b.json 2> $OUT/bench_1p3b.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/bench_ncu.log 2>&1
B="python bench.py --steps 1 --warmup 5 --no-cpu-baseline --no-probe"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 700 -c 1 -o $OUT/attn $B > $OUT/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2000 -c 4 -o $OUT/gemm $B > $OUT/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:norm_mod_kernel -s 1000 -c 1 -o $OUT/norm $B > $OUT/ncu_norm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sink_refresh_t_kernel -s 2 -c 1 -o $OUT/sink $B > $OUT/ncu_sink.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:history_noise -s 700 -c 1 -o $OUT/hist $B --history-sigma 0.1 > $OUT/ncu_hist.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:codec_patch_decode -c 1 -o $OUT/codec $B > $OUT/ncu_codec.log 2>&1
ls -la $OUT
