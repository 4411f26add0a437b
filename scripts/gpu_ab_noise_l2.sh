#!/bin/bash
# A/B session: norm statistics from the RESID epilogue (default) vs the full-row norm
# (LP_NO_NORM_STATS=1); history noise (Box-Muller kernel vs the round-2 x8 kernel,
# LP_HIST_X8=1); persistent attention L2 hints (LP_ATTN_L2POL 0/1/3) with DRAM bytes per launch.
OUT=gpurun_out/${1:-ab}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_gemm.py tests/test_gpu_wan.py tests/test_gpu_wan_shapes.py \
  -q -k "(noise or row_stats or resid or wan or bf16) and not 1p3b_full" --timeout 400 -rf > $OUT/pytest_sel.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_sel.log
B="python bench.py --no-cpu-baseline --no-decode --steps 5 --warmup 3"
timeout 400 $B > $OUT/bench_default.json 2> $OUT/bench_default.err
LP_NO_NORM_STATS=1 timeout 400 $B > $OUT/bench_nostats.json 2> $OUT/bench_nostats.err
timeout 400 $B --history-sigma 0.1 > $OUT/bench_sigma_bm.json 2> $OUT/bench_sigma_bm.err
LP_HIST_X8=1 timeout 400 $B --history-sigma 0.1 > $OUT/bench_sigma_x8.json 2> $OUT/bench_sigma_x8.err
for pol in 1 3; do
  LP_ATTN_L2POL=$pol timeout 400 $B > $OUT/bench_l2pol$pol.json 2> $OUT/bench_l2pol$pol.err
done
LP_ATTN_DYN=1 timeout 300 python -m pytest tests/test_gpu_attn.py -q --timeout 300 -rf > $OUT/pytest_attn_dyn.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_attn_dyn.log
LP_ATTN_DYN=1 timeout 400 $B > $OUT/bench_dyn.json 2> $OUT/bench_dyn.err
for pol in 0 1 3 dyn; do
  [ $pol = dyn ] && export LP_ATTN_DYN=1 LP_ATTN_L2POL=0 || export LP_ATTN_L2POL=$pol
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_requests_srcunit_ltcfabric_lookup_miss.sum \
    --clock-control none -k regex:attn_tc2p_kernel -s 300 -c 3 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe --no-decode > $OUT/ncu_l2pol$pol.csv 2> $OUT/ncu_l2pol$pol.err
done
unset LP_ATTN_DYN LP_ATTN_L2POL
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"history_noise|norm_apply" -s 200 -c 2 -o $OUT/rows_full \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe --no-decode --history-sigma 0.1 > $OUT/ncu_rows.log 2>&1
tail -3 $OUT/pytest_sel.log $OUT/pytest_attn_dyn.log
for f in $OUT/bench_*.json; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d.get('kernels',{})
print(round(d['value'],3), d['clocks'], {n:(round(v.get('avg_ms',0),4), round(v.get('gbs',v.get('tflops',0)),1)) for n,v in k.items() if n in ('attention','history_noise','norm_mod','o_proj','ffn_down')})"; done
