mkdir -p gpurun_out/fp32p
PYTHONPATH=. timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fp32p/launches.csv python scripts/debug/run_w14_fp32.py 2 0 1p3b > gpurun_out/fp32p/log.txt 2>&1
tail -2 gpurun_out/fp32p/log.txt
