// Decode stage, VAE stand-in (reference decode worker
// engine.py:465-480, codec latent.py:150-193): the row kernels around the
// implicit-GEMM 3-D convolutions (lp_gemm + lp_conv_taps) of a Wan-VAE-like
// decoder.  Activations live as [T][H+2][W+2][C] rows with a one-pixel zero
// border, so a conv tap is a constant row shift of the GEMM's A operand.
#include "lp_common.cuh"

namespace lp {

// latent [F, C, H, W] fp32 -> [F][H+2][W+2][cpad] bf16 (zero border, zero pad channels)
__global__ void vae_pack_latent_kernel(const float* __restrict__ x, int F, int C, int H, int W, int cpad,
                                       __nv_bfloat16* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)F * (H + 2) * (W + 2) * cpad;
  if (i >= total) return;
  const int c = (int)(i % cpad);
  int64_t px = i / cpad;
  const int xx = (int)(px % (W + 2)) - 1;
  px /= (W + 2);
  const int yy = (int)(px % (H + 2)) - 1;
  const int f = (int)(px / (H + 2));
  float v = 0.0f;
  if (c < C && xx >= 0 && xx < W && yy >= 0 && yy < H) v = x[(((int64_t)f * C + c) * H + yy) * W + xx];
  out[i] = __float2bfloat16_rn(v);
}

// One warp per pixel row of C channels: mode 1 = RMS norm over channels
// (x / sqrt(mean(x^2) + eps) * gamma) then SiLU; mode 0 = plain cast.  Border
// pixels are written as zeros (the next conv's padding).
template <int PER>
__global__ void vae_norm_silu_kernel(const float* __restrict__ h, const float* __restrict__ gamma, int T, int H,
                                     int W, int C, int mode, float eps, __nv_bfloat16* __restrict__ out) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int64_t rows = (int64_t)T * (H + 2) * (W + 2);
  if (row >= rows) return;
  const int xx = (int)(row % (W + 2)), yy = (int)((row / (W + 2)) % (H + 2));
  __nv_bfloat16* o = out + row * C;
  if (xx == 0 || yy == 0 || xx == W + 1 || yy == H + 1) {
    for (int c = lane; c < C; c += 32) o[c] = __float2bfloat16_rn(0.0f);
    return;
  }
  const float* x = h + row * C;
  float v[PER];
  float ss = 0.0f;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int c = k * 32 + lane;
    v[k] = c < C ? x[c] : 0.0f;
    ss += v[k] * v[k];
  }
  float scale = 1.0f;
  if (mode == 1) {
#pragma unroll
    for (int s = 16; s; s >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, s);
    scale = rsqrtf(ss / C + eps);
  }
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int c = k * 32 + lane;
    if (c >= C) continue;
    float y = v[k];
    if (mode == 1) {
      y = y * scale * gamma[c];
      y = y / (1.0f + __expf(-y));
    }
    o[c] = __float2bfloat16_rn(y);
  }
}

// Same, float4 per lane (C a multiple of 128: 128 -> 1, 256 -> 2, 384 -> 3
// float4 per lane): one 16-byte load and one 8-byte store per 4 channels.
template <int PER4>
__global__ void vae_norm_silu4_kernel(const float* __restrict__ h, const float* __restrict__ gamma, int T, int H,
                                      int W, int C, int mode, float eps, __nv_bfloat16* __restrict__ out) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int64_t rows = (int64_t)T * (H + 2) * (W + 2);
  if (row >= rows) return;
  const int xx = (int)(row % (W + 2)), yy = (int)((row / (W + 2)) % (H + 2));
  uint2* o = reinterpret_cast<uint2*>(out + row * C);
  if (xx == 0 || yy == 0 || xx == W + 1 || yy == H + 1) {
#pragma unroll
    for (int k = 0; k < PER4; ++k) o[k * 32 + lane] = make_uint2(0u, 0u);
    return;
  }
  const float4* x = reinterpret_cast<const float4*>(h + row * C);
  float4 v[PER4];
  float ss = 0.0f;
#pragma unroll
  for (int k = 0; k < PER4; ++k) {
    v[k] = x[k * 32 + lane];
    ss += (v[k].x * v[k].x + v[k].y * v[k].y) + (v[k].z * v[k].z + v[k].w * v[k].w);
  }
  float scale = 1.0f;
  if (mode == 1) {
#pragma unroll
    for (int s = 16; s; s >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, s);
    scale = rsqrtf(ss / C + eps);
  }
#pragma unroll
  for (int k = 0; k < PER4; ++k) {
    float y[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
    if (mode == 1) {
      const float4 g = reinterpret_cast<const float4*>(gamma)[k * 32 + lane];
      const float gg[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float t = y[e] * scale * gg[e];
        y[e] = t / (1.0f + __expf(-t));
      }
    }
    __nv_bfloat162 p0 = __floats2bfloat162_rn(y[0], y[1]), p1 = __floats2bfloat162_rn(y[2], y[3]);
    o[k * 32 + lane] = make_uint2(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1));
  }
}

// Nearest upsampling x2 in space (and x ft in time) between bordered layouts:
// in [T][H+2][W+2][C] -> out [T*ft][2H+2][2W+2][C], 8 channels per thread.
__global__ void vae_upsample_kernel(const __nv_bfloat16* __restrict__ in, int T, int H, int W, int C, int ft,
                                    __nv_bfloat16* __restrict__ out) {
  const int H2 = 2 * H, W2 = 2 * W, c8 = C / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)T * ft * (H2 + 2) * (W2 + 2) * c8;
  if (i >= total) return;
  const int c = (int)(i % c8) * 8;
  int64_t px = i / c8;
  const int xx = (int)(px % (W2 + 2));
  px /= (W2 + 2);
  const int yy = (int)(px % (H2 + 2));
  const int t = (int)(px / (H2 + 2));
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  if (xx > 0 && yy > 0 && xx <= W2 && yy <= H2) {
    const int sx = (xx - 1) / 2 + 1, sy = (yy - 1) / 2 + 1, st = t / ft;
    v = *reinterpret_cast<const uint4*>(in + (((int64_t)st * (H + 2) + sy) * (W + 2) + sx) * C + c);
  }
  *reinterpret_cast<uint4*>(out + i * 8) = v;
}

// Interior pixels, first cout channels of [T][H+2][W+2][cpad] fp32 -> frames [T][cout][H][W]
__global__ void vae_frames_kernel(const float* __restrict__ h, int T, int H, int W, int cpad, int cout,
                                  float* __restrict__ frames) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)T * cout * H * W;
  if (i >= total) return;
  const int xx = (int)(i % W);
  int64_t r = i / W;
  const int yy = (int)(r % H);
  r /= H;
  const int c = (int)(r % cout);
  const int t = (int)(r / cout);
  frames[i] = h[(((int64_t)t * (H + 2) + yy + 1) * (W + 2) + xx + 1) * cpad + c];
}

static inline unsigned nblocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

int preload_vae() {
  cudaFuncAttributes a;
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, vae_pack_latent_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, vae_norm_silu_kernel<2>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, vae_norm_silu_kernel<4>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, vae_norm_silu_kernel<8>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, vae_norm_silu_kernel<16>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, vae_norm_silu4_kernel<1>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, vae_norm_silu4_kernel<2>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, vae_norm_silu4_kernel<3>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, vae_upsample_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, vae_frames_kernel));
  return LP_OK;
}

int vae_pack_latent(const float* x, int F, int C, int H, int W, int cpad, void* out, cudaStream_t st) {
  LP_CHECK_ARG(x && out && C <= cpad, "lp_vae_pack_latent: bad arguments");
  const int64_t n = (int64_t)F * (H + 2) * (W + 2) * cpad;
  vae_pack_latent_kernel<<<nblocks(n, 256), 256, 0, st>>>(x, F, C, H, W, cpad, (__nv_bfloat16*)out);
  return launch_status("vae_pack_latent");
}

int vae_norm_silu(const float* h, const float* gamma, int T, int H, int W, int C, int mode, float eps, void* out,
                  cudaStream_t st) {
  LP_CHECK_ARG(h && out && (mode == 0 || gamma) && C > 0 && C <= 512, "lp_vae_norm_silu: bad arguments");
  const int64_t rows = (int64_t)T * (H + 2) * (W + 2);
  const unsigned blocks = nblocks(rows, 8);
  auto* o = (__nv_bfloat16*)out;
  if (C == 128 || C == 256 || C == 384) {
    if (C == 128)
      vae_norm_silu4_kernel<1><<<blocks, 256, 0, st>>>(h, gamma, T, H, W, C, mode, eps, o);
    else if (C == 256)
      vae_norm_silu4_kernel<2><<<blocks, 256, 0, st>>>(h, gamma, T, H, W, C, mode, eps, o);
    else
      vae_norm_silu4_kernel<3><<<blocks, 256, 0, st>>>(h, gamma, T, H, W, C, mode, eps, o);
    return launch_status("vae_norm_silu");
  }
  if (C <= 64)
    vae_norm_silu_kernel<2><<<blocks, 256, 0, st>>>(h, gamma, T, H, W, C, mode, eps, o);
  else if (C <= 128)
    vae_norm_silu_kernel<4><<<blocks, 256, 0, st>>>(h, gamma, T, H, W, C, mode, eps, o);
  else if (C <= 256)
    vae_norm_silu_kernel<8><<<blocks, 256, 0, st>>>(h, gamma, T, H, W, C, mode, eps, o);
  else
    vae_norm_silu_kernel<16><<<blocks, 256, 0, st>>>(h, gamma, T, H, W, C, mode, eps, o);
  return launch_status("vae_norm_silu");
}

int vae_upsample(const void* in, int T, int H, int W, int C, int ft, void* out, cudaStream_t st) {
  LP_CHECK_ARG(in && out && C % 8 == 0 && (ft == 1 || ft == 2), "lp_vae_upsample: bad arguments");
  const int64_t n = (int64_t)T * ft * (2 * H + 2) * (2 * W + 2) * (C / 8);
  vae_upsample_kernel<<<nblocks(n, 256), 256, 0, st>>>((const __nv_bfloat16*)in, T, H, W, C, ft,
                                                       (__nv_bfloat16*)out);
  return launch_status("vae_upsample");
}

int vae_frames(const float* h, int T, int H, int W, int cpad, int cout, float* frames, cudaStream_t st) {
  LP_CHECK_ARG(h && frames && cout <= cpad, "lp_vae_frames: bad arguments");
  const int64_t n = (int64_t)T * cout * H * W;
  vae_frames_kernel<<<nblocks(n, 256), 256, 0, st>>>(h, T, H, W, cpad, cout, frames);
  return launch_status("vae_frames");
}

}  // namespace lp
