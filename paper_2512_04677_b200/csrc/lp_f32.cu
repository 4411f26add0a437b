// fp32 validation-mode kernels: SIMT, no FMA contraction, reference order.
//
// GEMM: numerics.matmul (numerics.py:50-64) accumulates rank-1 updates in
// ascending k with one rounding for the product and one for the sum; the
// kernel below keeps exactly that order per output element, so its result is
// bit-identical to the reference for any shape.
//
// Attention: _attend_head (denoiser.py:152-158) + softmax (numerics.py:67-78).
// The logits and P.V products keep the pinned order; the row sum follows
// NumPy's pairwise summation (the reduction np.sum uses along a contiguous
// axis), so the only remaining difference to the reference is expf's ulp.
#include "lp_common.cuh"

namespace lp {

// ---------------------------------------------------------------- GEMM ----
constexpr int FBM = 64, FBN = 64, FBK = 16;

template <int EPI, typename OutT>
__global__ void __launch_bounds__(256) gemm_f32_pinned(const float* __restrict__ A, int64_t lda,
                                                       const float* __restrict__ W, int64_t ldw,
                                                       void* __restrict__ Cv, int64_t ldc, int m, int n,
                                                       int k, const float* __restrict__ bias,
                                                       const float* __restrict__ gate) {
  __shared__ float As[FBK][FBM + 1];
  __shared__ float Ws[FBK][FBN];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int row0 = blockIdx.y * FBM, col0 = blockIdx.x * FBN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

  for (int k0 = 0; k0 < k; k0 += FBK) {
    for (int e = threadIdx.x; e < FBM * FBK; e += 256) {
      int r = e / FBK, kk = e % FBK;
      int gr = row0 + r, gk = k0 + kk;
      As[kk][r] = (gr < m && gk < k) ? A[(int64_t)gr * lda + gk] : 0.0f;
    }
    for (int e = threadIdx.x; e < FBN * FBK; e += 256) {
      int kk = e / FBN, c = e % FBN;
      int gk = k0 + kk, gc = col0 + c;
      Ws[kk][c] = (gk < k && gc < n) ? W[(int64_t)gk * ldw + gc] : 0.0f;
    }
    __syncthreads();
    const int kmax = min(FBK, k - k0);
    for (int kk = 0; kk < kmax; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = row0 + ty * 4 + i;
    if (r >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int c = col0 + tx * 4 + j;
      if (c >= n) continue;
      float v = acc[i][j];
      if (EPI == LP_EPI_RESID) {
        float* H = reinterpret_cast<float*>(Cv);
        float g = gate ? gate[c] : 1.0f;
        float upd = gate ? __fmul_rn(g, v) : v;
        H[(int64_t)r * ldc + c] = __fadd_rn(H[(int64_t)r * ldc + c], upd);
      } else {
        if (EPI == LP_EPI_STORE && bias) v = __fadd_rn(v, bias[c]);
        if (EPI == LP_EPI_RELU) v = fmaxf(v, 0.0f);
        if (EPI == LP_EPI_GELU) v = gelu_tanh_f(v);
        reinterpret_cast<OutT*>(Cv)[(int64_t)r * ldc + c] = from_f32<OutT>(v);
      }
    }
  }
}

// ------------------------------------------------- QKV post-processing ----
// One warp per (row, head): optional per-head RMSNorm of q and k, rotary
// embedding (denoiser.py:192-197, numerics.py:104-115), then q -> q_out,
// k/v -> the current block's rows of the KV arena.
template <typename OutT>
__global__ void qkv_post_kernel(const float* __restrict__ qkv, int m, lp_qkv_epi e) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int row = warp / e.n_heads, head = warp % e.n_heads;
  if (row >= m) return;
  const int hd = e.head_dim, d = e.d;
  const float* src = qkv + (int64_t)row * 3 * d;
  const int cur = e.desc->cur_row;
  RopeTab rt{e.desc->rope_cos, e.desc->rope_sin, e.geom};
  OutT* qo = reinterpret_cast<OutT*>(e.q_out) + (int64_t)row * d + head * hd;
  OutT* ko = reinterpret_cast<OutT*>(e.k_arena) + (int64_t)(cur + row) * d + head * hd;
  OutT* vo = reinterpret_cast<OutT*>(e.v_arena) + (int64_t)(cur + row) * d + head * hd;
  for (int which = 0; which < 2; ++which) {
    const float* x = src + which * d + head * hd;
    float inv = 1.0f;
    const float* g = which == 0 ? e.g_q : e.g_k;
    if (e.qk_norm) {
      float ss = 0.0f;
      for (int c = lane; c < hd; c += 32) ss += x[c] * x[c];
#pragma unroll
      for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      inv = rsqrtf(ss / hd + e.eps);
    }
    OutT* dst = which == 0 ? qo : ko;
    for (int p = lane; p < hd / 2; p += 32) {
      float xv = x[2 * p], yv = x[2 * p + 1];
      if (e.qk_norm) {
        xv = xv * inv * (g ? g[head * hd + 2 * p] : 1.0f);
        yv = yv * inv * (g ? g[head * hd + 2 * p + 1] : 1.0f);
      }
      float c, s, xo, yo;
      rt.get(row, p, c, s);
      rotate_pair(xv, yv, c, s, xo, yo);
      dst[2 * p] = from_f32<OutT>(xo);
      dst[2 * p + 1] = from_f32<OutT>(yo);
    }
  }
  const float* v = src + 2 * d + head * hd;
  for (int c = lane; c < hd; c += 32) vo[c] = from_f32<OutT>(v[c]);
}

// ------------------------------------------------------------ attention ---
// NumPy pairwise sum of a contiguous fp32 run (8 accumulators below 128
// elements, recursive halving above) -- the order np.sum(..., axis=-1) uses.
// The halving recursion runs on an explicit stack: device recursion over
// 24,960 logits overflowed the 1 KB per-thread call stack (compute-sanitizer
// "Stack overflow", an illegal-address fault at the benched N_kv in fp32 mode).
__device__ __forceinline__ float pairwise_leaf(const float* a, int n) {
  if (n < 8) {
    float r = 0.0f;  // NumPy starts from -0.0 only for empty input; 0.0 + x == x for x != -0
    for (int i = 0; i < n; ++i) r = __fadd_rn(r, a[i]);
    return r;
  }
  float r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], a[i + j]);
  float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                        __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __fadd_rn(res, a[i]);
  return res;
}

__device__ float pairwise_sum(const float* a, int n) {
  // frames of the halving recursion: (offset, length, state: 0 new, 1 left
  // pending, 2 right pending, left partial)
  int off[26], len[26], state[26];
  float left[26];
  int sp = 0;
  off[0] = 0, len[0] = n, state[0] = 0;
  for (;;) {
    if (len[sp] <= 128) {
      float v = pairwise_leaf(a + off[sp], len[sp]);
      for (;;) {  // deliver v to the parents
        if (sp == 0) return v;
        --sp;
        if (state[sp] == 1) {  // left half done: descend into the right half
          left[sp] = v;
          state[sp] = 2;
          int n2 = len[sp] / 2;
          n2 -= n2 % 8;
          off[sp + 1] = off[sp] + n2, len[sp + 1] = len[sp] - n2, state[sp + 1] = 0;
          ++sp;
          break;
        }
        v = __fadd_rn(left[sp], v);  // both halves done
      }
      continue;
    }
    int n2 = len[sp] / 2;
    n2 -= n2 % 8;
    state[sp] = 1;
    off[sp + 1] = off[sp], len[sp + 1] = n2, state[sp + 1] = 0;
    ++sp;
  }
}

// One 128-thread CTA per (query row, head); the logits row in shared memory.
// Every value is produced in the reference's order (bit-identical to the
// round-1 one-warp-per-row kernel, 4x its parallelism): logit j = ascending-c
// fp32 dot product * scale (thread j % 128), row max, exp, NumPy pairwise row
// sum (thread 0), normalise, then out[c] = ascending-key chain (thread c).
template <typename T>
__global__ void __launch_bounds__(128) attn_f32_kernel(const T* __restrict__ q, const T* __restrict__ karena,
                                                       const T* __restrict__ varena, T* __restrict__ out, int n_q,
                                                       int n_heads, int hd, float scale,
                                                       const lp_block_desc* __restrict__ desc, int n_kv_max) {
  extern __shared__ float logit[];
  __shared__ float red[4];
  __shared__ float total_sum;
  const int tid = threadIdx.x, lane = tid % 32, wid = tid / 32;
  const int row = blockIdx.x / n_heads, head = blockIdx.x % n_heads;
  if (row >= n_q) return;
  const int d = n_heads * hd;
  const T* qr = q + (int64_t)row * d + head * hd;
  // logits in reference key order: segments as listed in the descriptor
  int total = 0;
  for (int s = 0; s < desc->n_seg; ++s) total += desc->seg_len[s];
  if (total > n_kv_max) __trap();  // host bound violated: fail loudly, never overrun smem
  int base = 0;
  for (int s = 0; s < desc->n_seg; ++s) {
    const int r0 = desc->seg_row[s], len = desc->seg_len[s];
    for (int j = tid; j < len; j += blockDim.x) {
      const T* kr = karena + (int64_t)(r0 + j) * d + head * hd;
      float acc = 0.0f;
      for (int c = 0; c < hd; ++c) acc = __fadd_rn(acc, __fmul_rn(to_f32(qr[c]), to_f32(kr[c])));
      logit[base + j] = __fmul_rn(acc, scale);
    }
    base += len;
  }
  const int n_kv = base;
  __syncthreads();
  float mx = -INFINITY;
  for (int j = tid; j < n_kv; j += blockDim.x) mx = fmaxf(mx, logit[j]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[wid] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  for (int j = tid; j < n_kv; j += blockDim.x) logit[j] = expf(__fsub_rn(logit[j], mx));
  __syncthreads();
  if (tid == 0) total_sum = pairwise_sum(logit, n_kv);
  __syncthreads();
  const float sum = total_sum;
  for (int j = tid; j < n_kv; j += blockDim.x) logit[j] = __fdiv_rn(logit[j], sum);
  __syncthreads();
  // out = P . V, ascending key order (pinned), one thread per head column
  for (int c = tid; c < hd; c += blockDim.x) {
    float acc = 0.0f;
    int kb = 0;
    for (int s = 0; s < desc->n_seg; ++s) {
      const int r0 = desc->seg_row[s], len = desc->seg_len[s];
      const T* vc = varena + (int64_t)r0 * d + head * hd + c;
      for (int j = 0; j < len; ++j) acc = __fadd_rn(acc, __fmul_rn(logit[kb + j], to_f32(vc[(int64_t)j * d])));
      kb += len;
    }
    out[(int64_t)row * d + head * hd + c] = from_f32<T>(acc);
  }
}

// --------------------------------------------------------------- launch ---
int preload_f32() {
  cudaFuncAttributes a;
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, gemm_f32_pinned<LP_EPI_RESID, float>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, gemm_f32_pinned<LP_EPI_STORE, float>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, gemm_f32_pinned<LP_EPI_STORE, __nv_bfloat16>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, gemm_f32_pinned<LP_EPI_RELU, float>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, gemm_f32_pinned<LP_EPI_RELU, __nv_bfloat16>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, gemm_f32_pinned<LP_EPI_GELU, float>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, gemm_f32_pinned<LP_EPI_GELU, __nv_bfloat16>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, qkv_post_kernel<float>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, qkv_post_kernel<__nv_bfloat16>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, attn_f32_kernel<float>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, attn_f32_kernel<__nv_bfloat16>));
  return LP_OK;
}

int gemm_f32(const lp_gemm_args* a, cudaStream_t st) {
  LP_CHECK_ARG(a->in_dtype == LP_F32, "gemm_f32: in_dtype must be LP_F32");
  dim3 grid((a->n + FBN - 1) / FBN, (a->m + FBM - 1) / FBM);
  if (grid.x == 0 || grid.y == 0) return LP_OK;
  const float* A = static_cast<const float*>(a->a);
  const float* W = static_cast<const float*>(a->w);
  switch (a->epilogue) {
    case LP_EPI_RESID:
      gemm_f32_pinned<LP_EPI_RESID, float><<<grid, 256, 0, st>>>(A, a->lda, W, a->ldw, a->c, a->ldc, a->m,
                                                                  a->n, a->k, nullptr, a->gate);
      break;
    case LP_EPI_STORE:
    case LP_EPI_RELU:
    case LP_EPI_GELU: {
      bool bf = a->out_dtype == LP_BF16;
#define LP_F32_EPI(E)                                                                                  \
  if (bf)                                                                                              \
    gemm_f32_pinned<E, __nv_bfloat16><<<grid, 256, 0, st>>>(A, a->lda, W, a->ldw, a->c, a->ldc, a->m, \
                                                            a->n, a->k, a->bias, nullptr);             \
  else                                                                                                 \
    gemm_f32_pinned<E, float><<<grid, 256, 0, st>>>(A, a->lda, W, a->ldw, a->c, a->ldc, a->m, a->n,   \
                                                    a->k, a->bias, nullptr);
      if (a->epilogue == LP_EPI_STORE) { LP_F32_EPI(LP_EPI_STORE) }
      else if (a->epilogue == LP_EPI_RELU) { LP_F32_EPI(LP_EPI_RELU) }
      else { LP_F32_EPI(LP_EPI_GELU) }
#undef LP_F32_EPI
      break;
    }
    default:
      return fail(LP_EUNSUPPORTED, "gemm_f32: epilogue not handled here");
  }
  return launch_status("gemm_f32");
}

int qkv_post(const float* qkv, int m, const lp_qkv_epi& e, int out_dtype, cudaStream_t st) {
  const int warps = m * e.n_heads;
  const int threads = 128;
  const int blocks = (warps * 32 + threads - 1) / threads;
  if (blocks == 0) return LP_OK;
  if (out_dtype == LP_BF16)
    qkv_post_kernel<__nv_bfloat16><<<blocks, threads, 0, st>>>(qkv, m, e);
  else
    qkv_post_kernel<float><<<blocks, threads, 0, st>>>(qkv, m, e);
  return launch_status("qkv_post");
}

int attention_simt(const lp_attn_args* a, int n_kv_max, cudaStream_t st) {
  LP_CHECK_ARG(n_kv_max > 0, "attention: empty key set");
  const size_t smem = (size_t)n_kv_max * sizeof(float);
  LP_CHECK_ARG(smem <= 200 * 1024, "attention_simt: too many keys for validation mode");
  const int64_t blocks = (int64_t)a->n_q * a->n_heads;
  if (blocks == 0) return LP_OK;
  if (a->dtype == LP_BF16) {
    auto k = attn_f32_kernel<__nv_bfloat16>;
    LP_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)blocks, 128, smem, st>>>(
        (const __nv_bfloat16*)a->q, (const __nv_bfloat16*)a->k_arena, (const __nv_bfloat16*)a->v_arena,
        (__nv_bfloat16*)a->out, a->n_q, a->n_heads, a->head_dim, a->scale, a->desc, n_kv_max);
  } else {
    auto k = attn_f32_kernel<float>;
    LP_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)blocks, 128, smem, st>>>((const float*)a->q, (const float*)a->k_arena, (const float*)a->v_arena,
                                           (float*)a->out, a->n_q, a->n_heads, a->head_dim, a->scale, a->desc,
                                           n_kv_max);
  }
  return launch_status("attention_simt");
}

}  // namespace lp
