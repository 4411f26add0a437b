#!/bin/bash
# All GPU tests without -x (full failure picture), then the given pytest -k filter repeated.
TAG=${1:-t}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -rf > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
if [ -n "$2" ]; then
  for i in 1 2 3; do
    timeout 300 python -m pytest tests -m gpu -q -k "$2" --timeout 200 >> $OUT/pytest_rep.log 2>&1
  done
fi
tail -8 $OUT/pytest_gpu.log; grep -E "passed|failed" $OUT/pytest_rep.log 2>/dev/null
