// tcgen05 flash attention over the RSFM key set [sink | history ring | current]
// (denoiser.py:246-264, _attend_head :152-158, softmax numerics.py:67-78).
//
// One CTA per (128-query tile, head).  Head dim 128, bf16 Q/K/V, fp32 S/O in
// TMEM, online softmax in fp32.  KV tiles of 128 keys walk the descriptor's
// segments in reference order (sink, oldest -> newest history, current); the
// ragged tail of each segment is masked to -inf, so segments need no padding
// and no K/V is gathered or copied.
//
//   warp 0      TMA producer: Q once, then K_j (2-stage ring) and V_{j-1}
//               (2-stage ring; V lags K by one tile so K never waits on V)
//   warp 1      TMEM allocator + MMA issuer: S_{j+1} = Q K_{j+1}^T is issued
//               before P_j V_j so the tensor core works on the next tile while
//               the softmax warps process this one (S double-buffered in TMEM)
//   warps 2..5  softmax / correction / epilogue: thread = query row; S row
//               from TMEM (two passes: max, then exp2), P (bf16) -> smem in
//               the UMMA K-major SW128 layout, O rescaled in TMEM when the
//               running max grows, O / l -> bf16 output at the end
//
// TMEM columns: S0 [0,128) S1 [128,256) O [256,384).
#include "lp_common.cuh"
#include "lp_sm100.cuh"
#include "lp_tma.cuh"

namespace lp {

using namespace sm100;

constexpr int AT_M = 128;      // query rows per CTA
constexpr int AT_N = 128;      // keys per tile
constexpr int AT_D = 128;      // head dim
constexpr int AT_THREADS = 192;
constexpr int AT_TILE_BYTES = AT_N * AT_D * 2;  // 32 KB: K tile, V tile, Q tile, P tile
constexpr int AT_HALF = AT_TILE_BYTES / 2;      // one 64-column SW128 block

struct AttnSmem {
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + AT_TILE_BYTES;
  static constexpr int V_OFF = K_OFF + 2 * AT_TILE_BYTES;
  static constexpr int P_OFF = V_OFF + 2 * AT_TILE_BYTES;
  static constexpr int BAR_OFF = P_OFF + AT_TILE_BYTES;
  static constexpr int SEG_OFF = BAR_OFF + 256;
  static constexpr int TOTAL = SEG_OFF + 2 * LP_MAX_SEG * 4 + 16 + 1024;
};

struct AttnParams {
  int n_q, n_heads;
  float scale_log2;  // scale * log2(e)
  __nv_bfloat16* out;
  int64_t ldo;
  const lp_block_desc* desc;
};

// Walks the KV tiles of the descriptor's segments in order.
struct TileCursor {
  const int* row;
  const int* len;
  int n_seg, seg, off;
  __device__ void init(const int* r, const int* l, int n) {
    row = r; len = l; n_seg = n; seg = 0; off = 0;
    while (seg < n_seg && len[seg] == 0) ++seg;
  }
  __device__ bool valid() const { return seg < n_seg; }
  __device__ int cur_row() const { return row[seg] + off; }
  __device__ int cur_valid() const { return min(AT_N, len[seg] - off); }
  __device__ void next() {
    off += AT_N;
    if (off >= len[seg]) {
      off = 0;
      ++seg;
      while (seg < n_seg && len[seg] == 0) ++seg;
    }
  }
};

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + AttnSmem::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2]
  uint64_t* s_free = bars + 11;  // [2]
  uint64_t* p_full = bars + 13;
  uint64_t* o_done = bars + 14;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  int* seg_row = reinterpret_cast<int*>(smem + AttnSmem::SEG_OFF);
  int* seg_len = seg_row + LP_MAX_SEG;
  int* n_seg_s = seg_len + LP_MAX_SEG;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int head = blockIdx.y;
  const int q0 = blockIdx.x * AT_M;

  const int nseg = min(p.desc->n_seg, LP_MAX_SEG);
  for (int s = threadIdx.x; s < nseg; s += blockDim.x) {
    seg_row[s] = p.desc->seg_row[s];
    seg_len[s] = p.desc->seg_len[s];
  }
  if (threadIdx.x == 0) {
    int nt = 0;
    for (int s = 0; s < nseg; ++s) nt += (p.desc->seg_len[s] + AT_N - 1) / AT_N;
    n_seg_s[0] = nseg;
    n_seg_s[1] = nt;
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
      mbar_init(&o_done[i], 1);
    }
    mbar_init(p_full, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int n_tiles = n_seg_s[1];
  const int col0 = head * AT_D;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      uint8_t* sq = smem + AttnSmem::Q_OFF;
      mbar_arrive_expect_tx(q_full, AT_TILE_BYTES);
      tma_load_2d(sq, &tmQ, q_full, col0, q0);
      tma_load_2d(sq + AT_HALF, &tmQ, q_full, col0 + 64, q0);
      TileCursor ck, cv;
      ck.init(seg_row, seg_len, n_seg_s[0]);
      cv.init(seg_row, seg_len, n_seg_s[0]);
      const uint64_t pol = l2_policy_evict_last();
      for (int t = 0; t <= n_tiles; ++t) {
        if (t < n_tiles) {
          const int b = t & 1;
          mbar_wait(&k_empty[b], ((t >> 1) & 1) ^ 1);
          uint8_t* sk = smem + AttnSmem::K_OFF + b * AT_TILE_BYTES;
          mbar_arrive_expect_tx(&k_full[b], AT_TILE_BYTES);
          tma_load_2d_hint(sk, &tmK, &k_full[b], col0, ck.cur_row(), pol);
          tma_load_2d_hint(sk + AT_HALF, &tmK, &k_full[b], col0 + 64, ck.cur_row(), pol);
          ck.next();
        }
        if (t >= 1) {
          const int u = t - 1, b = u & 1;
          mbar_wait(&v_empty[b], ((u >> 1) & 1) ^ 1);
          uint8_t* sv = smem + AttnSmem::V_OFF + b * AT_TILE_BYTES;
          mbar_arrive_expect_tx(&v_full[b], AT_TILE_BYTES);
          tma_load_2d_hint(sv, &tmV, &v_full[b], col0, cv.cur_row(), pol);
          tma_load_2d_hint(sv + AT_HALF, &tmV, &v_full[b], col0 + 64, cv.cur_row(), pol);
          cv.next();
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    constexpr uint32_t IDESC_S = idesc_bf16_f32(AT_M, AT_N);                 // Q K^T: both K-major
    constexpr uint32_t IDESC_O = idesc_bf16_f32(AT_M, AT_D, false, true);    // P V: V is MN-major
    const uint32_t sq = smem_u32(smem + AttnSmem::Q_OFF);
    const uint32_t sp = smem_u32(smem + AttnSmem::P_OFF);
    const uint32_t t_o = tmem_base + 256;
    auto issue_s = [&](int t) {
      const int b = t & 1;
      mbar_wait(&k_full[b], (t >> 1) & 1);
      if (t >= 2) mbar_wait(&s_free[b], ((t >> 1) - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sk = smem_u32(smem + AttnSmem::K_OFF + b * AT_TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < AT_D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * AT_HALF + (kk & 3) * 32;
          mma_bf16_ss(tmem_base + b * AT_N, sdesc_kmajor_sw128(sq + off), sdesc_kmajor_sw128(sk + off), IDESC_S,
                      kk != 0);
        }
        mma_commit(&k_empty[b]);
        mma_commit(&s_full[b]);
      }
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    if (n_tiles > 0) issue_s(0);
    for (int j = 0; j < n_tiles; ++j) {
      if (j + 1 < n_tiles) issue_s(j + 1);
      const int b = j & 1;
      mbar_wait(p_full, j & 1);
      mbar_wait(&v_full[b], (j >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sv = smem_u32(smem + AttnSmem::V_OFF + b * AT_TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < AT_N / 16; ++kk) {
          const uint32_t aoff = (kk >> 2) * AT_HALF + (kk & 3) * 32;  // P: K-major over keys
          const uint32_t boff = kk * 16 * 128;                         // V: 16 key rows of 128 B
          mma_bf16_ss(t_o, sdesc_kmajor_sw128(sp + aoff), sdesc_mnmajor_sw128(sv + boff, AT_HALF), IDESC_O,
                      (j | kk) != 0);
        }
        mma_commit(&v_empty[b]);
        mma_commit(&o_done[b]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------ softmax warps
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // row within the tile == TMEM lane
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t t_o = tmem_base + lane_base + 256;
    uint8_t* sp = smem + AttnSmem::P_OFF;
    float m_run = -INFINITY, l_run = 0.0f;
    TileCursor cs;
    cs.init(seg_row, seg_len, n_seg_s[0]);
    for (int j = 0; j < n_tiles; ++j, cs.next()) {
      const int b = j & 1;
      const int nvalid = cs.cur_valid();
      const uint32_t t_s = tmem_base + lane_base + b * AT_N;
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_fence_after();
      // pass 1: row max of the valid columns
      float mx = -INFINITY;
#pragma unroll 1
      for (int c0 = 0; c0 < AT_N; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(t_s + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (c0 + i < nvalid) mx = fmaxf(mx, __uint_as_float(v[i]));
      }
      const float m_new = fmaxf(m_run, mx * p.scale_log2);
      const float alpha = exp2f(m_run - m_new);  // 0 on the first tile (m_run = -inf)
      // pass 2: p = exp2(s*scale*log2e - m_new), packed bf16
      uint32_t pk[64];
      float rs = 0.0f;
#pragma unroll
      for (int c0 = 0; c0 < AT_N; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(t_s + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float e0 = (c0 + i < nvalid) ? exp2f(__uint_as_float(v[i]) * p.scale_log2 - m_new) : 0.0f;
          float e1 = (c0 + i + 1 < nvalid) ? exp2f(__uint_as_float(v[i + 1]) * p.scale_log2 - m_new) : 0.0f;
          __nv_bfloat162 h2 = __floats2bfloat162_rn(e0, e1);
          rs += __low2float(h2) + __high2float(h2);
          pk[(c0 + i) / 2] = *reinterpret_cast<uint32_t*>(&h2);
        }
      }
      // S buffer b may now be overwritten by S_{j+2}
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[b]);
      l_run = l_run * alpha + rs;
      m_run = m_new;
      // PV_{j-1} must be complete before O is rescaled and P is overwritten
      if (j >= 1) {
        mbar_wait(&o_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.0f)) {
#pragma unroll 1
          for (int c0 = 0; c0 < AT_D; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(t_o + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            tmem_st32(t_o + c0, v);
          }
          tmem_st_wait();
        }
      }
      // P row r -> smem, UMMA K-major SW128: block kb = keys [64kb, 64kb+64),
      // row r at 128 B, 16-byte chunk c stored at chunk c ^ (r % 8)
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        uint8_t* rowp = sp + kb * AT_HALF + r * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int src = kb * 32 + c * 4;
          *reinterpret_cast<uint4*>(rowp + ((c ^ (r & 7)) * 16)) =
              make_uint4(pk[src], pk[src + 1], pk[src + 2], pk[src + 3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16
    if (n_tiles > 0) {
      mbar_wait(&o_done[(n_tiles - 1) & 1], ((n_tiles - 1) >> 1) & 1);
      tc_fence_after();
    }
    const float inv_l = l_run > 0.0f ? 1.0f / l_run : 0.0f;
    const int row = q0 + r;
#pragma unroll 1
    for (int c0 = 0; c0 < AT_D; c0 += 32) {
      uint32_t v[32];
      tmem_ld32(t_o + c0, v);
      tmem_ld_wait();
      if (row < p.n_q) {
        uint4* o = reinterpret_cast<uint4*>(p.out + (int64_t)row * p.ldo + col0 + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          o[q] = make_uint4(pack_bf16(__uint_as_float(v[8 * q]) * inv_l, __uint_as_float(v[8 * q + 1]) * inv_l),
                            pack_bf16(__uint_as_float(v[8 * q + 2]) * inv_l, __uint_as_float(v[8 * q + 3]) * inv_l),
                            pack_bf16(__uint_as_float(v[8 * q + 4]) * inv_l, __uint_as_float(v[8 * q + 5]) * inv_l),
                            pack_bf16(__uint_as_float(v[8 * q + 6]) * inv_l, __uint_as_float(v[8 * q + 7]) * inv_l));
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

int preload_attn_tc() {
  cudaFuncAttributes a;
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, attn_tc_kernel));
  return LP_OK;
}

int attention_tc(const lp_attn_args* a, cudaStream_t st) {
  LP_CHECK_ARG(num_sms() > 0, "lp_init() must be called before lp_attention");
  LP_CHECK_ARG(a->head_dim == AT_D, "attention_tc: head_dim must be 128");
  if (a->n_q == 0) return LP_OK;
  const int d = a->n_heads * a->head_dim;
  CUtensorMap tq, tk, tv;
  int rc = make_tmap_bf16_2d(&tq, a->q, (uint64_t)a->n_q, (uint64_t)d, (uint64_t)d, AT_M, 64);
  if (rc) return rc;
  rc = make_tmap_bf16_2d(&tk, a->k_arena, (uint64_t)a->arena_rows, (uint64_t)d, (uint64_t)d, AT_N, 64);
  if (rc) return rc;
  rc = make_tmap_bf16_2d(&tv, a->v_arena, (uint64_t)a->arena_rows, (uint64_t)d, (uint64_t)d, AT_N, 64);
  if (rc) return rc;
  AttnParams p;
  p.n_q = a->n_q;
  p.n_heads = a->n_heads;
  p.scale_log2 = a->scale * 1.4426950408889634f;
  p.out = static_cast<__nv_bfloat16*>(a->out);
  p.ldo = d;
  p.desc = a->desc;
  dim3 grid((a->n_q + AT_M - 1) / AT_M, a->n_heads);
  const int smem = AttnSmem::TOTAL;
  LP_CUDA_TRY(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  attn_tc_kernel<<<grid, AT_THREADS, smem, st>>>(tq, tk, tv, p);
  return launch_status("attention_tc");
}

}  // namespace lp
