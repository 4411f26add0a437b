// Host-side TMA tensor-map encoding (cuTensorMapEncodeTiled resolved through
// cudaGetDriverEntryPoint, so the library does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "lp_common.cuh"

namespace lp {

int tma_init();
// 2-D bf16 tensor map over a row-major [rows, cols] matrix with leading
// dimension ld (elements).  Box = box_cols x box_rows, 128-byte swizzle when
// box_cols * 2 == 128.  Out-of-bounds boxes are zero-filled.
int make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                      uint32_t box_rows, uint32_t box_cols);

}  // namespace lp
