#!/bin/bash
# Page in torch / CUDA libraries on a fresh box before any timed or timeout-bounded step.
OUT=gpurun_out/${1:-warm}
mkdir -p $OUT
( time python -c "import torch; torch.zeros(1).cuda(); print('torch ok')" ) > $OUT/warm.log 2>&1
( time CUDA_MODULE_LOADING=EAGER python -c "import torch; torch.zeros(1).cuda(); print('eager ok')" ) >> $OUT/warm.log 2>&1
( time CUDA_MODULE_LOADING=LAZY python -c "import torch; torch.zeros(1).cuda(); print('lazy ok')" ) >> $OUT/warm.log 2>&1
( time CUDA_MODULE_LOADING=EAGER python -c "import torch; torch.zeros(1).cuda(); print('eager ok')" ) >> $OUT/warm.log 2>&1
