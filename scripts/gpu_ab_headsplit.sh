#!/bin/bash
# A/B: persistent attention with the dynamic queue, single queue vs head-split queues by SM id
# (LP_ATTN_HEADSPLIT=T): DRAM / L2-fabric bytes per steady-state launch and the bench.
OUT=gpurun_out/${1:-hs}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
LP_ATTN_DYN=1 LP_ATTN_HEADSPLIT=74 timeout 300 python -m pytest tests/test_gpu_attn.py -q --timeout 200 -rf > $OUT/pytest_attn_hs.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_attn_hs.log
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_sectors_srcunit_ltcfabric.sum
for v in static dyn 70 74 78; do
  unset LP_ATTN_DYN LP_ATTN_HEADSPLIT
  [ $v != static ] && export LP_ATTN_DYN=1
  [ $v != static ] && [ $v != dyn ] && export LP_ATTN_HEADSPLIT=$v
  timeout 300 ncu --metrics $M --clock-control none -k regex:attn_tc2p_kernel -s 700 -c 2 --csv \
    python bench.py --steps 1 --warmup 5 --no-cpu-baseline --no-probe --no-decode > $OUT/ncu_$v.csv 2> $OUT/ncu_$v.err
  timeout 400 python bench.py --no-cpu-baseline --no-decode --steps 5 --warmup 3 > $OUT/bench_$v.json 2> $OUT/bench_$v.err
done
tail -3 $OUT/pytest_attn_hs.log
