// Shared helpers for the livepipe B200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>

#include "../../include/livepipe_b200.h"

namespace lp {

// Thread-local last error string, surfaced through lp_last_error().
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define LP_CHECK_ARG(cond, msg)                                  \
  do {                                                           \
    if (!(cond)) return ::lp::fail(LP_EINVAL, std::string(msg)); \
  } while (0)

#define LP_CUDA_TRY(expr)                                                               \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return ::lp::fail(LP_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

inline int launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return LP_OK;
}

int num_sms();

// ---- element access ------------------------------------------------------
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

__device__ __forceinline__ float gelu_tanh_f(float x) {
  // 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float u = k0 * (x + k1 * x * x * x);
  return 0.5f * x * (1.0f + tanhf(u));
}

// Rotary angle tables for token `tok` and pair `p` of a head.
struct RopeTab {
  const float* tcos;   // temporal pairs (from the block descriptor)
  const float* tsin;
  lp_rope_geom g;
  __device__ __forceinline__ void get(int tok, int p, float& c, float& s) const {
    if (p < g.t_pairs) {
      c = tcos[p];
      s = tsin[p];
    } else {
      int q = (tok % g.tokens_per_frame) * g.spatial_pairs + (p - g.t_pairs);
      c = g.spatial_cos[q];
      s = g.spatial_sin[q];
    }
  }
};

// Rotation of an interleaved pair with the reference's rounding
// (numerics.py:110-114): x*c - y*s and x*s + y*c, each product rounded.
__device__ __forceinline__ void rotate_pair(float x, float y, float c, float s, float& xo, float& yo) {
  xo = __fsub_rn(__fmul_rn(x, c), __fmul_rn(y, s));
  yo = __fadd_rn(__fmul_rn(x, s), __fmul_rn(y, c));
}

// lp_fork_create handle: a side stream and fork/join events for a launch
// that runs part of its grid concurrently (GEMM pair + tail split, the
// attention's ragged query tails).
struct ForkCtx {
  cudaStream_t side;
  cudaEvent_t fork, join;
};

}  // namespace lp
