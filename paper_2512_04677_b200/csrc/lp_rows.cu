// HBM-bound row kernels around the projections: conditioning row, norm +
// AdaLN modulation, sink-frame refresh (RSFM), patch (un)embedding + Euler
// step, history-noise injection and the device RNG.
#include "lp_common.cuh"

namespace lp {

__global__ void oracle_step_kernel(const float* __restrict__, const float* __restrict__, float, float,
                                   float* __restrict__, float* __restrict__, int64_t);

// ------------------------------------------------------------ cond row -----
// c[col] = a.Wa[:,col] ; c += p.Wp[:,col] ; c += tau.Wt[:,col]
// (denoiser.py:178-185: three pinned-order products summed in this order).
__device__ __forceinline__ float dot_col(const float* x, int n, const float* w, int ldw, int col) {
  float acc = 0.0f;
  for (int k = 0; k < n; ++k) acc = __fadd_rn(acc, __fmul_rn(x[k], w[(int64_t)k * ldw + col]));
  return acc;
}

__global__ void cond_row_kernel(const float* audio, int na, const float* wa, const float* prompt, int np,
                                const float* wp, const float* tau, int nt, const float* wt, float* out,
                                int d) {
  int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= d) return;
  float c = audio ? dot_col(audio, na, wa, d, col) : 0.0f;
  c = __fadd_rn(c, dot_col(prompt, np, wp, d, col));
  c = __fadd_rn(c, dot_col(tau, nt, wt, d, col));
  out[col] = c;
}

// h[r,c] = x[r,c] + cond[c]   (denoiser.py:236)
__global__ void add_row_kernel(const float* x, const float* c, float* h, int rows, int d) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)rows * d) return;
  h[i] = __fadd_rn(x[i], c[i % d]);
}

// ------------------------------------------------------ norm + modulate ----
template <int THREADS>
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.0f;
  if (threadIdx.x < THREADS / 32) t = red[threadIdx.x];
  if (w == 0) {
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (l == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

// One CTA per row, float4 loads, two-pass mean/variance in fp32.  The row
// is read from HBM once: up to NV float4 per thread stay in registers
// (d <= THREADS*4*NV, the 14B/1.3B widths), wider rows re-read through L1/L2.
template <typename OutT>
__device__ __forceinline__ void store4(OutT* o, const float* y) {
  if constexpr (sizeof(OutT) == 2) {
    __nv_bfloat162 p0 = __floats2bfloat162_rn(y[0], y[1]);
    __nv_bfloat162 p1 = __floats2bfloat162_rn(y[2], y[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&p0);
    u.y = *reinterpret_cast<uint32_t*>(&p1);
    *reinterpret_cast<uint2*>(o) = u;
  } else {
    *reinterpret_cast<float4*>(o) = make_float4(y[0], y[1], y[2], y[3]);
  }
}

template <typename OutT, int THREADS, int NV = 8>
__global__ void __launch_bounds__(THREADS) norm_mod_kernel(const float* __restrict__ h, int d, int mode,
                                                           float eps, const float* __restrict__ shift,
                                                           const float* __restrict__ scale,
                                                           OutT* __restrict__ out) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const float* x = h + row * d;
  OutT* o = out + row * d;
  if (mode == 0) {
    for (int c = threadIdx.x; c < d; c += THREADS) o[c] = from_f32<OutT>(x[c]);
    return;
  }
  const bool cached = d <= THREADS * 4 * NV;
  float4 v[NV];
  float s = 0.0f;
  if (cached) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * THREADS + threadIdx.x) * 4;
      v[i] = c < d ? *reinterpret_cast<const float4*>(x + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
  } else {
    for (int c = threadIdx.x * 4; c < d; c += THREADS * 4) {
      float4 t = *reinterpret_cast<const float4*>(x + c);
      s += (t.x + t.y) + (t.z + t.w);
    }
  }
  const float mu = block_sum<THREADS>(s, red) / d;
  float q = 0.0f;
  if (cached) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * THREADS + threadIdx.x) * 4;
      if (c < d) {
        float a = v[i].x - mu, b = v[i].y - mu, e = v[i].z - mu, f = v[i].w - mu;
        q += (a * a + b * b) + (e * e + f * f);
      }
    }
  } else {
    for (int c = threadIdx.x * 4; c < d; c += THREADS * 4) {
      float4 t = *reinterpret_cast<const float4*>(x + c);
      float a = t.x - mu, b = t.y - mu, e = t.z - mu, f = t.w - mu;
      q += (a * a + b * b) + (e * e + f * f);
    }
  }
  const float rstd = rsqrtf(block_sum<THREADS>(q, red) / d + eps);
  auto emit = [&](int c, float4 t) {
    float y[4] = {(t.x - mu) * rstd, (t.y - mu) * rstd, (t.z - mu) * rstd, (t.w - mu) * rstd};
    if (mode == 2) {
      const float4 sc = __ldg(reinterpret_cast<const float4*>(scale + c));
      const float4 sh = __ldg(reinterpret_cast<const float4*>(shift + c));
      y[0] = y[0] * (1.0f + sc.x) + sh.x;
      y[1] = y[1] * (1.0f + sc.y) + sh.y;
      y[2] = y[2] * (1.0f + sc.z) + sh.z;
      y[3] = y[3] * (1.0f + sc.w) + sh.w;
    }
    store4<OutT>(o + c, y);
  };
  if (cached) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * THREADS + threadIdx.x) * 4;
      if (c < d) emit(c, v[i]);
    }
  } else {
    for (int c = threadIdx.x * 4; c < d; c += THREADS * 4) emit(c, *reinterpret_cast<const float4*>(x + c));
  }
}

// Software-pipelined form of norm_mod_kernel (modes 1/2, d <= 128 * 4 * NV):
// a resident grid (a few CTAs per SM) walks the rows, and while a CTA
// reduces and writes row r its loads of row r + G are already in flight
// (two register buffers, ping-pong).  The one-row-per-CTA kernel runs its
// waves in lock step -- every CTA of a wave loads, then reduces, then
// writes -- so HBM idles during the reductions (3.6 TB/s at 14B).  Same
// per-thread and block-reduction order as norm_mod_kernel: bitwise equal.
template <typename OutT, int NV>
__global__ void __launch_bounds__(128) norm_mod_pipe_kernel(const float* __restrict__ h, int rows, int d, int mode,
                                                            float eps, const float* __restrict__ shift,
                                                            const float* __restrict__ scale,
                                                            OutT* __restrict__ out) {
  constexpr int THREADS = 128;
  __shared__ float red[32];
  const int G = gridDim.x;
  float4 a[NV], b[NV];
  auto load = [&](float4(&v)[NV], int r) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * THREADS + threadIdx.x) * 4;
      v[i] = (r < rows && c < d) ? __ldcs(reinterpret_cast<const float4*>(h + (int64_t)r * d + c))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto process = [&](const float4(&v)[NV], int r) {
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < NV; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    const float mu = block_sum<THREADS>(s, red) / d;
    float q = 0.0f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * THREADS + threadIdx.x) * 4;
      if (c < d) {
        float x0 = v[i].x - mu, x1 = v[i].y - mu, x2 = v[i].z - mu, x3 = v[i].w - mu;
        q += (x0 * x0 + x1 * x1) + (x2 * x2 + x3 * x3);
      }
    }
    const float rstd = rsqrtf(block_sum<THREADS>(q, red) / d + eps);
    OutT* o = out + (int64_t)r * d;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * THREADS + threadIdx.x) * 4;
      if (c >= d) continue;
      float y[4] = {(v[i].x - mu) * rstd, (v[i].y - mu) * rstd, (v[i].z - mu) * rstd, (v[i].w - mu) * rstd};
      if (mode == 2) {
        const float4 sc = __ldg(reinterpret_cast<const float4*>(scale + c));
        const float4 sh = __ldg(reinterpret_cast<const float4*>(shift + c));
        y[0] = y[0] * (1.0f + sc.x) + sh.x;
        y[1] = y[1] * (1.0f + sc.y) + sh.y;
        y[2] = y[2] * (1.0f + sc.z) + sh.z;
        y[3] = y[3] * (1.0f + sc.w) + sh.w;
      }
      store4<OutT>(o + c, y);
    }
  };
  int row = blockIdx.x;
  load(a, row);
  for (; row < rows; row += 2 * G) {
    load(b, row + G);
    process(a, row);
    if (row + G >= rows) break;
    load(a, row + 2 * G);
    process(b, row + G);
  }
}

// LayerNorm(+AdaLN) apply pass whose row statistics were produced by the
// RESID GEMM epilogue that wrote h (lp_gemm_args.row_stats): per row, d/32
// partials (mean, M2) of 32-column chunks.  One warp per row (grid-stride):
// the lanes merge the partials (Chan et al.: fixed order in-lane, then a
// shfl_down tree into lane 0, broadcast), then stream the row -- no second
// read of h for the variance, no block-wide barriers, 8 float4 loads in
// flight per lane.  Same math as norm_mod_kernel up to the fp32 rounding of
// the merged moments.
__device__ __forceinline__ void chan_merge(float& n, float& m, float& q, float nb, float mb, float qb) {
  const float nt = n + nb;
  if (nb == 0.0f) return;
  const float dl = mb - m, f = nb / nt;
  m = fmaf(dl, f, m);
  q = q + qb + dl * dl * n * f;
  n = nt;
}

template <typename OutT>
__global__ void __launch_bounds__(256) norm_apply_kernel(const float* __restrict__ h,
                                                         const float2* __restrict__ stats, int rows, int d,
                                                         int mode, float eps, const float* __restrict__ shift,
                                                         const float* __restrict__ scale, OutT* __restrict__ out) {
  const int lane = threadIdx.x % 32;
  const int nwarps = gridDim.x * (blockDim.x / 32);
  const int np = d / 32;  // partials per row
  for (int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; row < rows; row += nwarps) {
    const float2* st = stats + (int64_t)row * np;
    float n = 0.0f, m = 0.0f, q = 0.0f;
    for (int i = lane; i < np; i += 32) {
      const float2 t = st[i];
      chan_merge(n, m, q, 32.0f, t.x, t.y);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float nb = __shfl_down_sync(0xffffffffu, n, o);
      const float mb = __shfl_down_sync(0xffffffffu, m, o);
      const float qb = __shfl_down_sync(0xffffffffu, q, o);
      if (lane < o) chan_merge(n, m, q, nb, mb, qb);
    }
    const float mu = __shfl_sync(0xffffffffu, m, 0);
    const float rstd = rsqrtf(__shfl_sync(0xffffffffu, q, 0) / d + eps);
    const float* x = h + (int64_t)row * d;
    OutT* o = out + (int64_t)row * d;
    for (int c0 = lane * 4; c0 < d; c0 += 32 * 4 * 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * 128;
        if (c < d) v[u] = __ldcs(reinterpret_cast<const float4*>(x + c));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * 128;
        if (c >= d) break;
        float y[4] = {(v[u].x - mu) * rstd, (v[u].y - mu) * rstd, (v[u].z - mu) * rstd, (v[u].w - mu) * rstd};
        if (mode == 2) {
          const float4 sc = __ldg(reinterpret_cast<const float4*>(scale + c));
          const float4 sh = __ldg(reinterpret_cast<const float4*>(shift + c));
          y[0] = y[0] * (1.0f + sc.x) + sh.x;
          y[1] = y[1] * (1.0f + sc.y) + sh.y;
          y[2] = y[2] * (1.0f + sc.z) + sh.z;
          y[3] = y[3] * (1.0f + sc.w) + sh.w;
        }
        store4<OutT>(o + c, y);
      }
    }
  }
}

// ----------------------------------------------------------- sink refresh --
// One warp per (sink token, head): optional RMSNorm(k) then rotation at the
// sink position i + delta (kvcache.py:86-90, denoiser.py:249); v copied.
template <typename T>
__global__ void sink_refresh_kernel(const float* __restrict__ kraw, const float* __restrict__ vraw, int s_tok,
                                    int d, int n_heads, int qk_norm, const float* __restrict__ g_k, float eps,
                                    const lp_block_desc* __restrict__ desc, lp_rope_geom geom,
                                    T* __restrict__ karena, T* __restrict__ varena, int64_t raw_stride,
                                    int64_t arena_stride, float* __restrict__ inv_out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int tok = warp / n_heads, head = warp % n_heads;
  if (tok >= s_tok) return;
  const int layer = blockIdx.y;
  kraw += layer * raw_stride;
  karena += layer * arena_stride;
  if (g_k) g_k += (int64_t)layer * d;
  const int hd = geom.head_dim;
  const int row = desc->seg_row[0] + tok;
  const float* k = kraw + (int64_t)tok * d + head * hd;
  float inv = 1.0f;
  if (qk_norm) {
    float ss = 0.0f;
    for (int c = lane * 2; c < hd; c += 64) {
      const float2 t = *reinterpret_cast<const float2*>(k + c);
      ss += t.x * t.x + t.y * t.y;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    inv = rsqrtf(ss / hd + eps);
    if (inv_out && lane == 0) inv_out[((int64_t)layer * s_tok + tok) * n_heads + head] = inv;
  }
  RopeTab rt{desc->sink_cos, desc->sink_sin, geom};
  T* ko = karena + (int64_t)row * d + head * hd;
  // 4 consecutive elements (2 rotary pairs) per lane: one 16-byte load, one
  // 8-byte (bf16) store
  for (int c = lane * 4; c < hd; c += 128) {
    const float4 t = *reinterpret_cast<const float4*>(k + c);
    float v[4] = {t.x, t.y, t.z, t.w};
    if (qk_norm) {
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = v[e] * inv * (g_k ? g_k[head * hd + c + e] : 1.0f);
    }
    float o[4];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float cs, sn;
      rt.get(tok, c / 2 + q, cs, sn);
      rotate_pair(v[2 * q], v[2 * q + 1], cs, sn, o[2 * q], o[2 * q + 1]);
    }
    store4(ko + c, o);
  }
  if (vraw == nullptr) return;  // V rows are position-independent: written once per sink content
  vraw += layer * raw_stride;
  varena += layer * arena_stride;
  const float* v = vraw + (int64_t)tok * d + head * hd;
  T* vo = varena + (int64_t)row * d + head * hd;
  for (int c = lane; c < hd; c += 32) vo[c] = from_f32<T>(v[c]);
}

// Temporal rotary pairs of the sink K only (the only part that moves with the
// sink position): one thread per (layer, token, head, temporal pair), same
// arithmetic and order as sink_refresh_kernel, RMS factor from its table.
template <typename T>
__global__ void sink_refresh_t_kernel(const float* __restrict__ kraw, const float* __restrict__ inv_rms, int s_tok,
                                      int d, int n_heads, int qk_norm, const float* __restrict__ g_k,
                                      const lp_block_desc* __restrict__ desc, int hd, int t_pairs,
                                      T* __restrict__ karena, int64_t raw_stride, int64_t arena_stride) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // < s_tok * n_heads * t_pairs (32-bit)
  const int layer = blockIdx.y;
  const int p = idx % t_pairs;
  const int th = idx / t_pairs;
  const int head = th % n_heads, tok = th / n_heads;
  if (tok >= s_tok) return;
  const int c = head * hd + 2 * p;
  const float2 t = *reinterpret_cast<const float2*>(kraw + layer * raw_stride + (int64_t)tok * d + c);
  float x = t.x, y = t.y;
  if (qk_norm) {
    const float inv = inv_rms[((int64_t)layer * s_tok + tok) * n_heads + head];
    const float* g = g_k ? g_k + (int64_t)layer * d : nullptr;
    x = x * inv * (g ? g[c] : 1.0f);
    y = y * inv * (g ? g[c + 1] : 1.0f);
  }
  float xo, yo;
  rotate_pair(x, y, desc->sink_cos[p], desc->sink_sin[p], xo, yo);
  T* ko = karena + layer * arena_stride + (int64_t)(desc->seg_row[0] + tok) * d + c;
  if constexpr (sizeof(T) == 2) {
    *reinterpret_cast<__nv_bfloat162*>(ko) = __floats2bfloat162_rn(xo, yo);  // one 4-byte store
  } else {
    *reinterpret_cast<float2*>(ko) = make_float2(xo, yo);
  }
}

// ------------------------------------------------------- patch embedding ---
// x frames [F, C, H, W] -> tokens [(f, hp, wp), (c, py, px)]
template <typename T>
__global__ void patchify_kernel(const float* __restrict__ x, int frames, int C, int H, int W, int ph, int pw,
                                T* __restrict__ tok) {
  const int hp = H / ph, wp = W / pw, pd = C * ph * pw;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)frames * hp * wp * pd;
  if (i >= total) return;
  int e = (int)(i % pd);
  int64_t t = i / pd;
  int px = e % pw, py = (e / pw) % ph, c = e / (pw * ph);
  int w = (int)(t % wp), hh = (int)((t / wp) % hp), f = (int)(t / ((int64_t)wp * hp));
  tok[i] = from_f32<T>(x[(((int64_t)f * C + c) * H + hh * ph + py) * W + w * pw + px]);
}

// x_out = x + unpatchify(v) * dt   (latent.py:140-147: v*fp32(dt), then add)
__global__ void unpatchify_euler_kernel(const float* __restrict__ x, const float* __restrict__ v, int frames,
                                        int C, int H, int W, int ph, int pw,
                                        const lp_block_desc* __restrict__ desc, float* __restrict__ xo) {
  const int64_t total = (int64_t)frames * C * H * W;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const float dt = desc->dt;
  float vv;
  if (ph == 0) {
    vv = v[i];
  } else {
    int xx = (int)(i % W), yy = (int)((i / W) % H), c = (int)((i / ((int64_t)W * H)) % C);
    int f = (int)(i / ((int64_t)W * H * C));
    const int hp = H / ph, wp = W / pw, pd = C * ph * pw;
    int64_t t = ((int64_t)f * hp + yy / ph) * wp + xx / pw;
    int e = (c * ph + yy % ph) * pw + xx % pw;
    vv = v[t * pd + e];
  }
  xo[i] = __fadd_rn(x[i], __fmul_rn(vv, dt));
  __threadfence_system();  // xo may be a peer's receive slot (fused TPP send)
}

// ------------------------------------------------------------------- RNG ---
// Philox4x32-10 (Salmon et al. 2011) + Box-Muller; counter = element / 4.
struct Philox {
  __device__ __forceinline__ static uint4 round(uint4 c, uint2 k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  template <int ROUNDS = 10>
  __device__ __forceinline__ static uint4 gen(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < ROUNDS; ++r) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

__device__ __forceinline__ float4 normal4(uint64_t seed, uint64_t stream, uint64_t ctr) {
  uint4 c = make_uint4((uint32_t)ctr, (uint32_t)(ctr >> 32), (uint32_t)stream, (uint32_t)(stream >> 32));
  uint2 k = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  uint4 r = Philox::gen(c, k);
  const float inv = 2.3283064365386963e-10f;  // 2^-32
  float u0 = (r.x + 0.5f) * inv, u1 = (r.y + 0.5f) * inv, u2 = (r.z + 0.5f) * inv, u3 = (r.w + 0.5f) * inv;
  float r0 = sqrtf(-2.0f * logf(u0)), r1 = sqrtf(-2.0f * logf(u2));
  float s0, c0, s1, c1;
  sincospif(2.0f * u1, &s0, &c0);
  sincospif(2.0f * u3, &s1, &c1);
  return make_float4(r0 * c0, r0 * s0, r1 * c1, r1 * s1);
}

template <typename T>
__global__ void randn_kernel(T* out, int64_t n, uint64_t seed, uint64_t stream, float scale) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t i = q * 4;
  if (i >= n) return;
  float4 g = normal4(seed, stream, (uint64_t)q);
  float v[4] = {g.x, g.y, g.z, g.w};
  for (int j = 0; j < 4 && i + j < n; ++j) out[i + j] = from_f32<T>(v[j] * scale);
}

// History noise over the descriptor's history segments (kvcache.py:121-137):
// dst rows = src rows + z * sigma (noise*sigma rounded, then the add).
// Grid: x covers max history rows * d / 4 elements (packed over segments);
// each thread moves 4 contiguous elements with one vector load / store.
// Device noise (perf runs) is Philox4x32-7 + Box-Muller on the fast
// intrinsics (__logf, __sincosf); parity runs pass the reference's draws.
// Philox4x32-7: the fewest rounds Salmon et al. (SC'11) report as passing
// BigCrush; the history noise is perf-run noise checked by its moments.
__device__ __forceinline__ float4 normal4_fast(uint64_t seed, uint64_t stream, uint64_t ctr) {
  uint4 c = make_uint4((uint32_t)ctr, (uint32_t)(ctr >> 32), (uint32_t)stream, (uint32_t)(stream >> 32));
  uint2 k = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  uint4 r = Philox::gen<7>(c, k);
  const float inv = 2.3283064365386963e-10f;  // 2^-32
  const float u0 = (r.x + 0.5f) * inv, u1 = (r.y + 0.5f) * inv, u2 = (r.z + 0.5f) * inv, u3 = (r.w + 0.5f) * inv;
  const float r0 = sqrtf(-2.0f * __logf(u0)), r1 = sqrtf(-2.0f * __logf(u2));
  float s0, c0, s1, c1;
  __sincosf(6.283185307179586f * u1, &s0, &c0);
  __sincosf(6.283185307179586f * u3, &s1, &c1);
  return make_float4(r0 * c0, r0 * s0, r1 * c1, r1 * s1);
}

template <typename T>
__device__ __forceinline__ void load4(const T* p, float* v);
template <>
__device__ __forceinline__ void load4<float>(const float* p, float* v) {
  const float4 t = *reinterpret_cast<const float4*>(p);
  v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
}
template <>
__device__ __forceinline__ void load4<__nv_bfloat16>(const __nv_bfloat16* p, float* v) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
  const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
  v[0] = __low2float(a), v[1] = __high2float(a), v[2] = __low2float(b), v[3] = __high2float(b);
}

template <typename T>
__global__ void history_noise_kernel(T* __restrict__ arena, int d, const float* __restrict__ noise,
                                     int n_layers, int layer, int kv, const lp_block_desc* __restrict__ desc) {
  const float sigma = desc->sigma;
  const int n_hist = desc->n_seg - 2;
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t i = q * 4;  // element index within the packed history
  int64_t base = 0;
  for (int e = 0; e < n_hist; ++e) {
    const int s = e + 1;
    const int64_t len = (int64_t)desc->seg_len[s] * d;
    if (i < base + len) {
      const int64_t off = i - base;  // multiple of 4, len multiple of d (of 4): 4 elements in range
      T* dst = arena + (int64_t)desc->seg_row[s] * d + off;
      const T* src = arena + (int64_t)desc->src_row[s] * d + off;
      float z[4];
      if (noise) {
        const float4 t = *reinterpret_cast<const float4*>(noise + ((((int64_t)e * 2 + kv) * n_layers + layer) * len) + off);
        z[0] = t.x, z[1] = t.y, z[2] = t.z, z[3] = t.w;
      } else {
        const float4 g =
            normal4_fast(desc->noise_key, ((uint64_t)(layer * 2 + kv) << 8) | (uint64_t)e, (uint64_t)(off >> 2));
        z[0] = g.x, z[1] = g.y, z[2] = g.z, z[3] = g.w;
      }
      float x[4], o[4];
      load4<T>(src, x);
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] = __fadd_rn(x[j], __fmul_rn(z[j], sigma));
      store4<T>(dst, o);
      return;
    }
    base += len;
  }
}

// Perf-run variant (device RNG, bf16 arena): 8 elements per thread from four
// hash words, one 16-byte load and store and 32-bit index math.  Half the RNG and index work
// per element of history_noise_kernel; the parity path (host draws) is above.
// Perf-run noise source (device RNG, bf16 arena): a counter hash instead of
// Philox -- the Philox4x32-7 rounds made the kernel integer-bound (ALU pipe
// 56 %, issue 75 %, ncu r2 ev2).  Two murmur3 fmix32 finalisers over a unique
// (key, stream, counter) word: bijective with full avalanche, ~10 integer ops
// per 32-bit word.  Each word drives one Box-Muller pair (20-bit radius
// uniform, 12-bit angle) on the MUFU pipe; perf-run noise is checked by its
// moments (tests/test_gpu_attn.py), parity runs upload the reference's draws.
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

__device__ __forceinline__ void normal8_fast(uint64_t seed, uint64_t stream, uint32_t ctr, float* z) {
  const uint64_t sk = seed ^ (stream * 0x9E3779B97F4A7C15ull);
  const uint32_t k0 = (uint32_t)sk, k1 = (uint32_t)(sk >> 32);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t w = fmix32(fmix32((ctr * 4u + (uint32_t)j) ^ k0) + k1);
    const float u = ((float)(w >> 12) + 0.5f) * 9.5367431640625e-07f;  // 2^-20
    const float a = ((float)(w & 0xFFFu) + 0.5f) * 1.5339807878856412e-03f;  // 2 pi / 4096
    float rad;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rad) : "f"(-2.0f * __logf(u)));  // one MUFU op, no IEEE fix-up
    float sn, cs;
    __sincosf(a, &sn, &cs);
    z[2 * j] = rad * cs;
    z[2 * j + 1] = rad * sn;
  }
}

__global__ void history_noise_bf16x8_kernel(__nv_bfloat16* __restrict__ arena, int d, int layer, int kv,
                                            const lp_block_desc* __restrict__ desc) {
  const float sigma = desc->sigma;
  const int n_hist = desc->n_seg - 2;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  int base = 0;
  for (int e = 0; e < n_hist; ++e) {
    const int s = e + 1;
    const int len = desc->seg_len[s] * d;
    if (i < base + len) {
      const int off = i - base;  // multiple of 8; len is a multiple of d (of 8)
      __nv_bfloat16* dst = arena + (int64_t)desc->seg_row[s] * d + off;
      const __nv_bfloat16* src = arena + (int64_t)desc->src_row[s] * d + off;
      float z[8];
      normal8_fast(desc->noise_key, ((uint64_t)(layer * 2 + kv) << 8) | (uint64_t)e, (uint32_t)(off >> 3), z);
      uint4 raw = *reinterpret_cast<const uint4*>(src);
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 x = __bfloat1622float2(h[j]);
        h[j] = __floats2bfloat162_rn(__fadd_rn(x.x, __fmul_rn(z[2 * j], sigma)),
                                     __fadd_rn(x.y, __fmul_rn(z[2 * j + 1], sigma)));
      }
      *reinterpret_cast<uint4*>(dst) = raw;
      return;
    }
    base += len;
  }
}

// Perf-run noise, round 2b: the x8 kernel above spends 6 XU-pipe ops per
// Box-Muller pair (2 I2F, LG2, SQRT, SIN, COS; 16/clk/SM) and two fmix32
// rounds per word, which caps it near 2.5 TB/s.  Here each 32-bit word
// w = fmix32(c * m + k) (one round; m odd and k per stream, so c -> w is a
// bijection within a stream) drives one pair:
//   radius  u = 2 - float(1.[w >> 12]) in (0, 1]  (20 bits, mantissa trick, no I2F)
//           r = sqrt(-2 ln u) = sqrt(-2 ln2 * lg2 u)  (LG2 + SQRT: the only XU ops)
//   angle   theta = (f + 1/2) / 1024 * pi/2 from 10 bits, sin/cos by one packed
//           degree-4 Horner in theta^2 on the FMA pipe (|err| < 3e-5),
//           and the quadrant by two independent sign bits: (+-r cos, +-r sin)
//           with theta uniform on [0, pi/2) is (r cos phi, r sin phi) with phi
//           uniform on [0, 2 pi) (the four sign patterns are the reflections
//           into the four quadrants), i.e. exact Box-Muller.
// Grid-stride over 16-byte chunks, two chunks per iteration with both loads
// issued before the RNG work (memory-level parallelism).
__device__ __forceinline__ uint64_t f32x2p(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpack_f32x2p(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2p(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

__device__ __forceinline__ void bm_pair(uint32_t w, float& z0, float& z1) {
  const float x = __uint_as_float(0x3F800000u | ((w >> 9) & 0x007FFFF8u));  // [1, 2), 20 random bits
  const float u = 2.0f - x;                                                 // (0, 1]
  float l2, r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(u));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(-1.3862943611198906f * l2));
  const float y = __uint_as_float(0x3F800000u | ((w << 13) & 0x007FE000u));  // [1, 2), 10 bits
  const float th = fmaf(y, 1.5707963267948966f, -1.5707963267948966f * (1.0f - 1.0f / 2048.0f));
  const float t = th * th;
  // (sin(th)/th, cos(th)) as polynomials in t, packed
  uint64_t q = f32x2p(2.7557319e-06f, 2.4801587e-05f);
  q = ffma2p(q, f32x2p(t, t), f32x2p(-1.9841270e-04f, -1.3888889e-03f));
  q = ffma2p(q, f32x2p(t, t), f32x2p(8.3333333e-03f, 4.1666667e-02f));
  q = ffma2p(q, f32x2p(t, t), f32x2p(-1.6666667e-01f, -0.5f));
  q = ffma2p(q, f32x2p(t, t), f32x2p(1.0f, 1.0f));
  float sn, cs;
  unpack_f32x2p(q, sn, cs);
  sn *= th;
  z0 = __uint_as_float(__float_as_uint(r * cs) ^ ((w << 21) & 0x80000000u));  // sign: bit 10
  z1 = __uint_as_float(__float_as_uint(r * sn) ^ ((w << 20) & 0x80000000u));  // sign: bit 11
}

__device__ __forceinline__ void noise8_bm(uint32_t m, uint32_t k, uint32_t ctr, float* z) {
#pragma unroll
  for (int j = 0; j < 4; ++j) bm_pair(fmix32((ctr * 4u + (uint32_t)j) * m + k), z[2 * j], z[2 * j + 1]);
}

__device__ __forceinline__ uint4 add_noise8(uint4 raw, const float* z, float sigma) {
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 x = __bfloat1622float2(h[j]);
    h[j] = __floats2bfloat162_rn(fmaf(z[2 * j], sigma, x.x), fmaf(z[2 * j + 1], sigma, x.y));
  }
  return raw;
}

// THREADS / MINB: 256 / 5 standalone (<= 48 registers); 128 / 12 for the co-resident form
// (<= 40 registers: two CTAs fit beside a tcgen05 GEMM CTA's 168 x 320).
template <int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) history_noise_bm_kernel(__nv_bfloat16* __restrict__ arena, int d,
                                                                         int layer, int kv,
                                                                         const lp_block_desc* __restrict__ desc) {
  // per-segment tables, once per CTA: chunk base (cumulative), source and
  // destination element offsets, and the stream's multiplier / offset
  // (splitmix64 finaliser of (key, layer, kv, entry))
  __shared__ int s_base[LP_MAX_SEG];
  __shared__ int64_t s_src[LP_MAX_SEG], s_dst[LP_MAX_SEG];
  __shared__ uint32_t s_m[LP_MAX_SEG], s_k[LP_MAX_SEG];
  __shared__ int s_total;
  const int n_hist = desc->n_seg - 2;
  if (n_hist <= 0) return;
  const int cpr = d / 8;  // 16-byte chunks per row
  if (threadIdx.x == 0) {
    int base = 0;
    for (int e = 0; e < n_hist; ++e) {
      s_base[e] = base;
      base += desc->seg_len[e + 1] * cpr;
    }
    s_total = base;
  }
  if (threadIdx.x < n_hist) {
    const int e = threadIdx.x;
    s_src[e] = (int64_t)desc->src_row[e + 1] * d;
    s_dst[e] = (int64_t)desc->seg_row[e + 1] * d;
    uint64_t z = desc->noise_key ^ ((((uint64_t)(layer * 2 + kv) << 8) | (uint64_t)e) * 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    s_m[e] = (uint32_t)z | 1u;
    s_k[e] = (uint32_t)(z >> 32);
  }
  __syncthreads();
  const float sigma = desc->sigma;
  const int total = s_total;
  const int stride = gridDim.x * blockDim.x;
  // chunks only grow along the grid-stride walk, so each of the two lanes of
  // work keeps its segment index and advances it (usually zero steps)
  int e0 = 0, e1 = 0;
  for (int c0 = blockIdx.x * blockDim.x + threadIdx.x; c0 < total; c0 += 2 * stride) {
    const int c1 = c0 + stride;
    while (e0 + 1 < n_hist && c0 >= s_base[e0 + 1]) ++e0;
    while (e1 + 1 < n_hist && c1 >= s_base[e1 + 1]) ++e1;
    const int r0 = c0 - s_base[e0], r1 = c1 - s_base[e1];
    const bool has1 = c1 < total;
    // both loads unconditional (the second re-reads chunk 0 past the end) so
    // they issue back to back ahead of the RNG work
    const uint4 raw0 = *reinterpret_cast<const uint4*>(arena + s_src[e0] + (int64_t)r0 * 8);
    const uint4 raw1 =
        *reinterpret_cast<const uint4*>(arena + (has1 ? s_src[e1] + (int64_t)r1 * 8 : s_src[e0] + (int64_t)r0 * 8));
    float z[8];
    noise8_bm(s_m[e0], s_k[e0], (uint32_t)r0, z);
    *reinterpret_cast<uint4*>(arena + s_dst[e0] + (int64_t)r0 * 8) = add_noise8(raw0, z, sigma);
    if (has1) {
      noise8_bm(s_m[e1], s_k[e1], (uint32_t)r1, z);
      *reinterpret_cast<uint4*>(arena + s_dst[e1] + (int64_t)r1 * 8) = add_noise8(raw1, z, sigma);
    }
  }
}

// ---------------------------------------------------------------- launch ---
static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

int preload_rows() {
  cudaFuncAttributes a;
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, cond_row_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, add_row_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, norm_mod_kernel<float, 256>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, norm_mod_kernel<float, 128, 4>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, norm_mod_kernel<__nv_bfloat16, 128, 4>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, norm_mod_kernel<__nv_bfloat16, 256>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, norm_mod_kernel<__nv_bfloat16, 128, 10>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, norm_mod_kernel<float, 128, 10>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, oracle_step_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, sink_refresh_kernel<float>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, sink_refresh_kernel<__nv_bfloat16>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, sink_refresh_t_kernel<float>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, sink_refresh_t_kernel<__nv_bfloat16>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, patchify_kernel<float>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, patchify_kernel<__nv_bfloat16>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, unpatchify_euler_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, history_noise_kernel<float>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, history_noise_kernel<__nv_bfloat16>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, history_noise_bf16x8_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, history_noise_bm_kernel<256, 5>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, history_noise_bm_kernel<128, 12>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, norm_apply_kernel<__nv_bfloat16>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, norm_mod_pipe_kernel<__nv_bfloat16, 4>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, norm_mod_pipe_kernel<__nv_bfloat16, 10>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, norm_mod_pipe_kernel<float, 4>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, norm_mod_pipe_kernel<float, 10>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, norm_apply_kernel<float>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, randn_kernel<float>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, randn_kernel<__nv_bfloat16>));
  return LP_OK;
}

int cond_row(const float* audio, int na, const float* wa, const float* prompt, int np, const float* wp,
             const float* tau, int nt, const float* wt, float* out, int d, cudaStream_t st) {
  cond_row_kernel<<<nblk(d, 128), 128, 0, st>>>(audio, na, wa, prompt, np, wp, tau, nt, wt, out, d);
  return launch_status("cond_row");
}

int add_row(const float* x, const float* c, float* h, int rows, int d, cudaStream_t st) {
  int64_t n = (int64_t)rows * d;
  if (n == 0) return LP_OK;
  add_row_kernel<<<nblk(n, 256), 256, 0, st>>>(x, c, h, rows, d);
  return launch_status("add_row");
}

int norm_mod(const float* h, int rows, int d, int mode, float eps, const float* shift, const float* scale,
             void* out, int out_dtype, cudaStream_t st) {
  LP_CHECK_ARG(mode == 0 || d % 4 == 0, "norm_mod: d must be a multiple of 4");
  LP_CHECK_ARG(mode != 2 || (shift && scale), "norm_mod: modulation needs shift and scale");
  if (rows == 0) return LP_OK;
  // LP_NORM_PIPE=1: the resident-grid pipelined kernel (measured slower: 43.6 vs 39.1 us at 14B,
  // profiles/r2b/hs1_summary.md), kept for A/B
  static const bool pipe = getenv("LP_NORM_PIPE") != nullptr;
  if (pipe && mode != 0 && d % 4 == 0 && d <= 128 * 4 * 10) {
    // resident grid: 4 CTAs per SM (two row buffers per thread: ~100 registers)
    const int cap = 4 * num_sms(), grid = rows < cap ? rows : cap;
    if (d <= 2048) {
      if (out_dtype == LP_BF16)
        norm_mod_pipe_kernel<__nv_bfloat16, 4><<<grid, 128, 0, st>>>(h, rows, d, mode, eps, shift, scale,
                                                                    (__nv_bfloat16*)out);
      else
        norm_mod_pipe_kernel<float, 4><<<grid, 128, 0, st>>>(h, rows, d, mode, eps, shift, scale, (float*)out);
    } else {
      if (out_dtype == LP_BF16)
        norm_mod_pipe_kernel<__nv_bfloat16, 10><<<grid, 128, 0, st>>>(h, rows, d, mode, eps, shift, scale,
                                                                     (__nv_bfloat16*)out);
      else
        norm_mod_pipe_kernel<float, 10><<<grid, 128, 0, st>>>(h, rows, d, mode, eps, shift, scale, (float*)out);
    }
    return launch_status("norm_mod");
  }
  if (d <= 2048) {  // narrow rows (1.3B: d = 1536): 128 threads, 4 float4 per thread
    if (out_dtype == LP_BF16)
      norm_mod_kernel<__nv_bfloat16, 128, 4><<<rows, 128, 0, st>>>(h, d, mode, eps, shift, scale,
                                                                   (__nv_bfloat16*)out);
    else
      norm_mod_kernel<float, 128, 4><<<rows, 128, 0, st>>>(h, d, mode, eps, shift, scale, (float*)out);
  } else if (d <= 128 * 4 * 10) {  // 14B (d = 5120): 128 threads, 10 float4 per thread (6-8 % over 256 x 5)
    if (out_dtype == LP_BF16)
      norm_mod_kernel<__nv_bfloat16, 128, 10><<<rows, 128, 0, st>>>(h, d, mode, eps, shift, scale,
                                                                     (__nv_bfloat16*)out);
    else
      norm_mod_kernel<float, 128, 10><<<rows, 128, 0, st>>>(h, d, mode, eps, shift, scale, (float*)out);
  } else if (out_dtype == LP_BF16) {
    norm_mod_kernel<__nv_bfloat16, 256><<<rows, 256, 0, st>>>(h, d, mode, eps, shift, scale,
                                                               (__nv_bfloat16*)out);
  } else {
    norm_mod_kernel<float, 256><<<rows, 256, 0, st>>>(h, d, mode, eps, shift, scale, (float*)out);
  }
  return launch_status("norm_mod");
}

int norm_mod_stats(const float* h, const float* stats, int rows, int d, int mode, float eps, const float* shift,
                   const float* scale, void* out, int out_dtype, cudaStream_t st) {
  LP_CHECK_ARG(mode == 1 || mode == 2, "norm_mod_stats: mode must be 1 (LayerNorm) or 2 (AdaLN)");
  LP_CHECK_ARG(d % 32 == 0, "norm_mod_stats: d must be a multiple of 32");
  LP_CHECK_ARG(h && stats && out, "norm_mod_stats: null pointer");
  LP_CHECK_ARG(mode != 2 || (shift && scale), "norm_mod_stats: modulation needs shift and scale");
  if (rows == 0) return LP_OK;
  // 8 rows per 256-thread CTA, up to 8 CTAs per SM resident (grid-stride beyond)
  const int want = nblk(rows, 8), cap = 8 * num_sms();
  const int grid = want < cap ? want : cap;
  const float2* s2 = reinterpret_cast<const float2*>(stats);
  if (out_dtype == LP_BF16)
    norm_apply_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(h, s2, rows, d, mode, eps, shift, scale,
                                                           (__nv_bfloat16*)out);
  else
    norm_apply_kernel<float><<<grid, 256, 0, st>>>(h, s2, rows, d, mode, eps, shift, scale, (float*)out);
  return launch_status("norm_mod_stats");
}

int sink_refresh(const float* kraw, const float* vraw, int s_tok, int d, int n_heads, int qk_norm,
                 const float* g_k, float eps, const lp_block_desc* desc, const lp_rope_geom& geom, void* karena,
                 void* varena, int dtype, int n_layers, int64_t raw_stride, int64_t arena_stride, float* inv_out,
                 cudaStream_t st) {
  const int warps = s_tok * n_heads;
  if (warps == 0 || n_layers == 0) return LP_OK;
  dim3 grid(nblk((int64_t)warps * 32, 128), n_layers);
  if (dtype == LP_BF16)
    sink_refresh_kernel<__nv_bfloat16><<<grid, 128, 0, st>>>(kraw, vraw, s_tok, d, n_heads, qk_norm, g_k, eps,
                                                             desc, geom, (__nv_bfloat16*)karena,
                                                             (__nv_bfloat16*)varena, raw_stride, arena_stride,
                                                             inv_out);
  else
    sink_refresh_kernel<float><<<grid, 128, 0, st>>>(kraw, vraw, s_tok, d, n_heads, qk_norm, g_k, eps, desc, geom,
                                                     (float*)karena, (float*)varena, raw_stride, arena_stride,
                                                     inv_out);
  return launch_status("sink_refresh");
}

template <typename T>
__global__ void silu_kernel(const float* x, T* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = from_f32<T>(x[i] / (1.0f + expf(-x[i])));
}

int sink_refresh_temporal(const float* kraw, const float* inv_rms, int s_tok, int d, int n_heads, int qk_norm,
                          const float* g_k, const lp_block_desc* desc, const lp_rope_geom& geom, void* karena,
                          int dtype, int n_layers, int64_t raw_stride, int64_t arena_stride, cudaStream_t st) {
  const int tp = geom.t_pairs;
  const int64_t n = (int64_t)s_tok * n_heads * tp;
  if (n == 0 || n_layers == 0) return LP_OK;
  LP_CHECK_ARG(n < (1ll << 31), "sink_refresh_temporal: too many sink rows");
  dim3 grid(nblk(n, 256), n_layers);
  if (dtype == LP_BF16)
    sink_refresh_t_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(kraw, inv_rms, s_tok, d, n_heads, qk_norm, g_k, desc,
                                                               geom.head_dim, tp, (__nv_bfloat16*)karena, raw_stride,
                                                               arena_stride);
  else
    sink_refresh_t_kernel<float><<<grid, 256, 0, st>>>(kraw, inv_rms, s_tok, d, n_heads, qk_norm, g_k, desc,
                                                       geom.head_dim, tp, (float*)karena, raw_stride, arena_stride);
  return launch_status("sink_refresh_temporal");
}

int silu(const float* x, void* out, int n, int dtype, cudaStream_t st) {
  if (n == 0) return LP_OK;
  if (dtype == LP_BF16)
    silu_kernel<__nv_bfloat16><<<nblk(n, 256), 256, 0, st>>>(x, (__nv_bfloat16*)out, n);
  else
    silu_kernel<float><<<nblk(n, 256), 256, 0, st>>>(x, (float*)out, n);
  return launch_status("silu");
}

int patchify(const float* x, int frames, int C, int H, int W, int ph, int pw, void* tok, int dtype,
             cudaStream_t st) {
  LP_CHECK_ARG(ph > 0 && pw > 0 && H % ph == 0 && W % pw == 0, "patchify: bad patch");
  int64_t n = (int64_t)frames * C * H * W;
  if (dtype == LP_BF16)
    patchify_kernel<__nv_bfloat16><<<nblk(n, 256), 256, 0, st>>>(x, frames, C, H, W, ph, pw, (__nv_bfloat16*)tok);
  else
    patchify_kernel<float><<<nblk(n, 256), 256, 0, st>>>(x, frames, C, H, W, ph, pw, (float*)tok);
  return launch_status("patchify");
}

// The reference's analytic test denoiser (OracleDenoiser, denoiser.py:294-343)
// fused with the flow step (latent.py:140-147):
//   v = (x - target) / s ;  x' = x + v * dt   -- IEEE ops in numpy's order, no FMA.
__global__ void oracle_step_kernel(const float* __restrict__ x, const float* __restrict__ target, float s, float dt,
                                   float* __restrict__ vel, float* __restrict__ x_out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float v = __fdiv_rn(__fsub_rn(x[i], target[i]), s);
  if (vel) vel[i] = v;
  x_out[i] = __fadd_rn(x[i], __fmul_rn(v, dt));
}

int oracle_step(const float* x, const float* target, float s, float dt, float* vel, float* x_out, int64_t n,
                cudaStream_t st) {
  LP_CHECK_ARG(x && target && x_out, "lp_oracle_step: null pointer");
  LP_CHECK_ARG(s != 0.0f, "lp_oracle_step: oracle velocity undefined at s = 0");
  if (n <= 0) return LP_OK;
  oracle_step_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, target, s, dt, vel, x_out, n);
  return launch_status("oracle_step");
}

int unpatchify_euler(const float* x, const float* v, int frames, int C, int H, int W, int ph, int pw,
                     const lp_block_desc* desc, float* xo, cudaStream_t st) {
  int64_t n = (int64_t)frames * C * H * W;
  unpatchify_euler_kernel<<<nblk(n, 256), 256, 0, st>>>(x, v, frames, C, H, W, ph, pw, desc, xo);
  return launch_status("unpatchify_euler");
}

int history_noise(void* arena, int dtype, int d, const float* noise, int n_layers, int layer, int kv,
                  const lp_block_desc* desc, int max_rows, cudaStream_t st) {
  LP_CHECK_ARG(d % 4 == 0, "history_noise: d must be a multiple of 4");
  int64_t n = (int64_t)max_rows * d;
  if (n == 0) return LP_OK;
  if (!noise && dtype == LP_BF16 && d % 8 == 0 && n < (1ll << 31)) {
    static const bool x8 = getenv("LP_HIST_X8") != nullptr;  // round-2 kernel, A/B
    if (x8) {
      history_noise_bf16x8_kernel<<<nblk(n / 8, 256), 256, 0, st>>>((__nv_bfloat16*)arena, d, layer, kv, desc);
    } else {
      // two 16-byte chunks per thread and iteration; at most 8 CTAs per SM resident
      const int want = nblk(n / 16, 256), cap = 8 * num_sms();
      history_noise_bm_kernel<256, 5><<<want < cap ? want : cap, 256, 0, st>>>((__nv_bfloat16*)arena, d, layer, kv,
                                                                              desc);
    }
    return launch_status("history_noise");
  }
  int blocks = nblk((n + 3) / 4, 256);
  if (dtype == LP_BF16)
    history_noise_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>((__nv_bfloat16*)arena, d, noise, n_layers, layer,
                                                                kv, desc);
  else
    history_noise_kernel<float><<<blocks, 256, 0, st>>>((float*)arena, d, noise, n_layers, layer, kv, desc);
  return launch_status("history_noise");
}

// Co-resident form for a side stream beside the tensor-bound GEMMs: two
// 128-thread CTAs per SM (the registers and shared memory a tcgen05 GEMM CTA
// leaves free), grid-stride over the whole history.
int history_noise_co(void* arena, int d, int layer, int kv, const lp_block_desc* desc, int max_rows, cudaStream_t st) {
  LP_CHECK_ARG(d % 8 == 0, "history_noise_co: d must be a multiple of 8");
  const int64_t n = (int64_t)max_rows * d;
  if (n == 0) return LP_OK;
  LP_CHECK_ARG(n < (1ll << 31), "history_noise_co: history too large");
  const int want = nblk(n / 16, 128), cap = 2 * num_sms();
  history_noise_bm_kernel<128, 12><<<want < cap ? want : cap, 128, 0, st>>>((__nv_bfloat16*)arena, d, layer, kv,
                                                                              desc);
  return launch_status("history_noise_co");
}

int randn(void* out, int64_t n, uint64_t seed, uint64_t stream, float scale, int dtype, cudaStream_t st) {
  if (n == 0) return LP_OK;
  int blocks = nblk((n + 3) / 4, 256);
  if (dtype == LP_BF16)
    randn_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>((__nv_bfloat16*)out, n, seed, stream, scale);
  else
    randn_kernel<float><<<blocks, 256, 0, st>>>((float*)out, n, seed, stream, scale);
  return launch_status("randn");
}

}  // namespace lp
