#!/bin/bash
# Quick HEAD check after the final validation: the kernel-count test, the wan/attention/gemm
# tests, smoke and one bench line.
OUT=gpurun_out/${1:-head2}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_wan.py tests/test_gpu_attn.py tests/test_gpu_gemm.py tests/test_gpu_toy.py -q --timeout 400 -rf > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
tail -3 $OUT/pytest.log; tail -2 $OUT/smoke.log; tail -c 300 $OUT/bench.json
