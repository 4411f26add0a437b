#!/bin/bash
OUT=gpurun_out/${1:-vae}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_vae.py -q --timeout 300 > $OUT/pytest_vae.log 2>&1
echo "rc=$?" >> $OUT/pytest_vae.log
for e in "" "LP_CONV_ROWSHIFT=1"; do
  env $e timeout 300 python -c "
import torch, time, paper_2512_04677_b200 as lp
d = lp.VaeDecoder(16, 60, 104, 'cuda:0'); x = torch.randn(3, 16*60*104, device='cuda'); f = torch.empty(12, 3*480*832, device='cuda')
for _ in range(2): d.decode_into(x, f)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): d.decode_into(x, f)
b.record(); torch.cuda.synchronize(); ms = a.elapsed_time(b) / 5
print('${e:-halo}', round(ms, 2), 'ms', round(d.flops_per_block() / ms / 1e9, 1), 'TFLOP/s')
" >> $OUT/vae_time.txt 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:conv_tc -s 15 -c 2 -o $OUT/conv python -c "
import torch, paper_2512_04677_b200 as lp
d = lp.VaeDecoder(16, 60, 104, 'cuda:0'); x = torch.randn(3, 16*60*104, device='cuda'); f = torch.empty(12, 3*480*832, device='cuda')
d.decode_into(x, f); torch.cuda.synchronize()" > $OUT/ncu_conv.log 2>&1
tail -3 $OUT/pytest_vae.log; cat $OUT/vae_time.txt
