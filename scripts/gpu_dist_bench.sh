#!/bin/bash
# Functional check of bench.py's N>1 path on a 1-GPU box: ranks share cuda:0 (gloo process group,
# CUDA-IPC latent links).  Timings are meaningless (the ranks time-slice one GPU).
OUT=gpurun_out/${1:-dist}
mkdir -p $OUT
python -c "import torch; torch.zeros(1).cuda()" > /dev/null 2>&1
for n in 2 4 8; do
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus $n --steps 3 --warmup 3 --config 1.3b --dist-backend gloo --no-probe > $OUT/bench_n$n.json 2> $OUT/bench_n$n.err
  echo "n=$n rc=$?" >> $OUT/summary.txt
done
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus 3 --steps 3 --warmup 3 --config 1.3b --dist-backend gloo --no-probe --decode-gpu > $OUT/bench_n3_decode.json 2> $OUT/bench_n3_decode.err
echo "n=3 decode rc=$?" >> $OUT/summary.txt
timeout 600 python -m pytest tests/test_gpu_tpp_dist.py -x -q > $OUT/pytest_dist.log 2>&1; tail -2 $OUT/pytest_dist.log >> $OUT/summary.txt
timeout 300 python bench.py --config 1.3b --steps 3 > $OUT/bench_1p3b_n1.json 2> $OUT/bench_1p3b_n1.err
echo "1.3b n=1 rc=$?" >> $OUT/summary.txt
cat $OUT/summary.txt; tail -c 600 $OUT/bench_n2.json; tail -5 $OUT/bench_n2.err
