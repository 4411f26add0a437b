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

// 4-D bf16 tensor map over a dense [d3][d2][d1][d0] array (d0 innermost),
// box b0 x b1 x b2 x b3, 128-byte swizzle when b0 * 2 == 128.
int make_tmap_bf16_4d(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint32_t box[4]);

}  // namespace lp
