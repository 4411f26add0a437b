mkdir -p gpurun_out/dbg3
PYTHONPATH=. timeout 300 python scripts/debug/run_w14_fp32.py 5 1 1p3b_l1 > gpurun_out/dbg3/plain.txt 2>&1
echo "plain rc=$?"; grep -E " ok |Error" gpurun_out/dbg3/plain.txt | head -2
PYTHONPATH=. timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/debug/run_w14_fp32.py 5 0 1p3b_l1 > gpurun_out/dbg3/memcheck.txt 2>&1
echo "memcheck rc=$?"; grep -v "^frame" gpurun_out/dbg3/memcheck.txt | head -60
