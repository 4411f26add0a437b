#!/bin/bash
# compute-sanitizer memcheck / synccheck over the round-2 kernels: persistent attention with the
# dynamic item queue (cluster-scope smem ring), Box-Muller history noise, RESID row statistics +
# norm apply pass, and a Wan bf16 rollout.
OUT=gpurun_out/${1:-san}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
T="tests/test_gpu_attn.py::test_flash_attention_matches_reference tests/test_gpu_attn.py::test_segment_order_modes tests/test_gpu_attn.py::test_exponent_window_fallback tests/test_gpu_attn.py::test_device_history_noise_streams_independent"
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest $T -q -x --timeout 800 > $OUT/${tool}_attn.log 2>&1
  echo "rc=$?" >> $OUT/${tool}_attn.log
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_gemm.py -q -x -k "row_stats and 300" --timeout 800 > $OUT/memcheck_rowstats.log 2>&1
echo "rc=$?" >> $OUT/memcheck_rowstats.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest "tests/test_gpu_wan.py::test_wan_rollout_matches_oracle" -q -x -k bf16 --timeout 800 > $OUT/memcheck_wan.log 2>&1
echo "rc=$?" >> $OUT/memcheck_wan.log
tail -3 $OUT/*.log
