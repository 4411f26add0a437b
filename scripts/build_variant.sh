#!/bin/bash
# Build a variant of liblivepipe_b200.so with extra nvcc defines for lp_attn_tc.cu only.
# Usage: scripts/build_variant.sh <name> -DFOO=1 ...   -> paper_2512_04677_b200/<name>.so
set -e
NAME=$1; shift
D=paper_2512_04677_b200
mkdir -p /tmp/variant_$NAME
cp $D/build/*.o /tmp/variant_$NAME/
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -I include "$@" -c $D/csrc/lp_attn_tc.cu -o /tmp/variant_$NAME/lp_attn_tc.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static /tmp/variant_$NAME/*.o -o $D/$NAME.so
echo $D/$NAME.so
