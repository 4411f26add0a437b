mkdir -p gpurun_out/dbg2
for args in "3 0 w14" "3 1 w14" "5 1 1p3b"; do
  PYTHONPATH=. CUDA_LAUNCH_BLOCKING=1 timeout 500 python scripts/debug/run_w14_fp32.py $args > gpurun_out/dbg2/log_${args// /_}.txt 2>&1
  echo "$args rc=$?"; grep -v "^frame" gpurun_out/dbg2/log_${args// /_}.txt | grep -E "ok|Error|error" | head -3
done
