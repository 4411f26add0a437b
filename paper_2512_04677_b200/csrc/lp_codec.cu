// Decode stage: the per-location patch codec that stands
// in for the video VAE on patched (wan-shaped) profiles.
//
// A latent frame is (C, H, W) fp32.  Decoding maps every latent location
// (h, w) through r matrices M_u (Q x C, Q = pc*s*s) to an s x s patch of pc
// pixel channels in each of the r output frames of that latent frame:
//   pix[f*r+u][ch][h*s+dy][w*s+dx] = sum_c M_u[(ch*s+dy)*s+dx][c] * x[f][c][h][w]
// Encoding applies E = pinv(M_0) (C x Q) to the patches of one pixel frame.
// This is the ToyVideoCodec contract (latent.py:150-193: r decode maps, the
// encoder the float64 pseudo-inverse of the first) restricted to a block-
// diagonal map, i.e. the shape of a stride-s transposed convolution.  Every
// sum keeps the reference matmul's pinned order (numerics.py:50-64): ascending
// inner index, one rounding for the product and one for the add, so the
// NumPy restatement in oracle/ reproduces it bit for bit.
//
// Both kernels are HBM-bound (decode writes F*r*pc*H*s*W*s fp32 per block,
// ~57.5 MB at 480p, F=3, r=4); the maps sit in shared memory and are read
// as warp-wide broadcasts, the latent is read once, the pixel rows are
// written as coalesced float4 runs.
#include "lp_common.cuh"

namespace lp {

constexpr int CODEC_MAX_C = 32;
constexpr int CODEC_THREADS = 128;

// grid (ceil(W / 128), H * pc, frames * r); one thread per (latent location,
// pixel channel): s x s outputs.  The
// map is staged transposed (c-major) so that four adjacent dx outputs take
// one 16-byte shared load per channel.
template <int VEC, int NC>
__global__ void __launch_bounds__(CODEC_THREADS, 4) codec_patch_decode_kernel(const float* __restrict__ x, int C, int H,
                                                                           int W, const float* __restrict__ maps,
                                                                           int r, int pc, int s,
                                                                           float* __restrict__ out) {
  extern __shared__ __align__(16) float sm_map[];  // C x (s*s): rows of map u for channel ch
  const int SS = s * s;
  const int fu = blockIdx.z, u = fu % r, f = fu / r;
  const int h = blockIdx.y / pc, ch = blockIdx.y - h * pc, w = blockIdx.x * CODEC_THREADS + threadIdx.x;
  const float* mu = maps + ((int64_t)u * pc + ch) * SS * C;
  for (int e = threadIdx.x; e < SS * C; e += CODEC_THREADS) {
    const int q = e / C, c = e - q * C;
    sm_map[c * SS + q] = mu[e];
  }
  __syncthreads();
  if (w >= W) return;

  float xr[NC];
  const float* xf = x + (int64_t)f * C * H * W + (int64_t)h * W + w;
#pragma unroll
  for (int c = 0; c < NC; ++c) xr[c] = (c < C) ? xf[(int64_t)c * H * W] : 0.0f;

  const int64_t ow = (int64_t)W * s, oh = (int64_t)H * s;
  float* of = out + (int64_t)fu * pc * oh * ow;
  {
#pragma unroll 1
    for (int dy = 0; dy < s; ++dy) {
      float* orow = of + ((int64_t)ch * oh + (int64_t)h * s + dy) * ow + (int64_t)w * s;
      const int q0 = dy * s;
#pragma unroll 1
      for (int dx = 0; dx < s; dx += VEC) {
        if constexpr (VEC == 4) {
          // scalar mul.rn / add.rn: ptxas contracts the packed f32x2 forms
          // (mul.rn.f32x2 + add.rn.f32x2 -> FFMA2, checked in the SASS),
          // which would break the pinned rounding
          float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            if (c < C) {
              const float4 m = *reinterpret_cast<const float4*>(sm_map + c * SS + q0 + dx);
              a0 = __fadd_rn(a0, __fmul_rn(m.x, xr[c]));
              a1 = __fadd_rn(a1, __fmul_rn(m.y, xr[c]));
              a2 = __fadd_rn(a2, __fmul_rn(m.z, xr[c]));
              a3 = __fadd_rn(a3, __fmul_rn(m.w, xr[c]));
            }
          }
          *reinterpret_cast<float4*>(orow + dx) = make_float4(a0, a1, a2, a3);
        } else {
          float acc = 0.0f;
#pragma unroll
          for (int c = 0; c < NC; ++c)
            if (c < C) acc = __fadd_rn(acc, __fmul_rn(sm_map[c * SS + q0 + dx], xr[c]));
          orow[dx] = acc;
        }
      }
    }
  }
}

// grid (ceil(W / 128), H); one thread per latent location, q ascending.
__global__ void __launch_bounds__(CODEC_THREADS) codec_patch_encode_kernel(const float* __restrict__ frame, int C,
                                                                           int H, int W,
                                                                           const float* __restrict__ enc, int pc,
                                                                           int s, float* __restrict__ out) {
  extern __shared__ float sm_enc[];  // C x Q
  const int Q = pc * s * s;
  for (int e = threadIdx.x; e < Q * C; e += CODEC_THREADS) sm_enc[e] = enc[e];
  __syncthreads();
  const int h = blockIdx.y, w = blockIdx.x * CODEC_THREADS + threadIdx.x;
  if (w >= W) return;
  float acc[CODEC_MAX_C];
#pragma unroll
  for (int c = 0; c < CODEC_MAX_C; ++c) acc[c] = 0.0f;
  const int64_t ow = (int64_t)W * s, oh = (int64_t)H * s;
  int q = 0;
  for (int ch = 0; ch < pc; ++ch)
    for (int dy = 0; dy < s; ++dy)
      for (int dx = 0; dx < s; ++dx, ++q) {
        const float p = frame[((int64_t)ch * oh + (int64_t)h * s + dy) * ow + (int64_t)w * s + dx];
#pragma unroll
        for (int c = 0; c < CODEC_MAX_C; ++c)
          if (c < C) acc[c] = __fadd_rn(acc[c], __fmul_rn(sm_enc[c * Q + q], p));
      }
#pragma unroll
  for (int c = 0; c < CODEC_MAX_C; ++c)
    if (c < C) out[(int64_t)c * H * W + (int64_t)h * W + w] = acc[c];
}

static int codec_check(int C, int H, int W, int pc, int s) {
  LP_CHECK_ARG(C >= 1 && C <= CODEC_MAX_C, "codec: latent channels must be in [1, 32]");
  LP_CHECK_ARG(H >= 1 && W >= 1 && pc >= 1 && s >= 1, "codec: bad geometry");
  LP_CHECK_ARG((int64_t)pc * s * s * C * 4 <= 200 * 1024, "codec: map does not fit in shared memory");
  return LP_OK;
}

int codec_patch_decode(const float* x, int frames, int C, int H, int W, const float* maps, int r, int pc, int s,
                       float* out, cudaStream_t st) {
  int rc = codec_check(C, H, W, pc, s);
  if (rc) return rc;
  LP_CHECK_ARG(frames >= 1 && r >= 1 && frames * r <= 65535, "codec: bad frame count");
  LP_CHECK_ARG(H <= 65535, "codec: H too large");
  const size_t smem = (size_t)s * s * C * sizeof(float);
  LP_CHECK_ARG((int64_t)H * pc <= 65535, "codec: H * pixel channels too large");
  dim3 grid((W + CODEC_THREADS - 1) / CODEC_THREADS, H * pc, frames * r);
  auto launch = [&](auto kern) -> int {
    if (smem > 48 * 1024)
      LP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, CODEC_THREADS, smem, st>>>(x, C, H, W, maps, r, pc, s, out);
    return LP_OK;
  };
  const bool v4 = s % 4 == 0;
  if (C <= 16) rc = v4 ? launch(codec_patch_decode_kernel<4, 16>) : launch(codec_patch_decode_kernel<1, 16>);
  else rc = v4 ? launch(codec_patch_decode_kernel<4, CODEC_MAX_C>) : launch(codec_patch_decode_kernel<1, CODEC_MAX_C>);
  if (rc) return rc;
  return launch_status("codec_patch_decode");
}

int codec_patch_encode(const float* frame, int C, int H, int W, const float* enc, int pc, int s, float* out,
                       cudaStream_t st) {
  int rc = codec_check(C, H, W, pc, s);
  if (rc) return rc;
  LP_CHECK_ARG(H <= 65535, "codec: H too large");
  const size_t smem = (size_t)pc * s * s * C * sizeof(float);
  if (smem > 48 * 1024)
    LP_CUDA_TRY(cudaFuncSetAttribute(codec_patch_encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  dim3 grid((W + CODEC_THREADS - 1) / CODEC_THREADS, H);
  codec_patch_encode_kernel<<<grid, CODEC_THREADS, smem, st>>>(frame, C, H, W, enc, pc, s, out);
  return launch_status("codec_patch_encode");
}

int preload_codec() {
  cudaFuncAttributes a;
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, codec_patch_decode_kernel<4, 16>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, codec_patch_decode_kernel<1, 16>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, codec_patch_decode_kernel<4, CODEC_MAX_C>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, codec_patch_decode_kernel<1, CODEC_MAX_C>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, codec_patch_encode_kernel));
  return LP_OK;
}

}  // namespace lp
