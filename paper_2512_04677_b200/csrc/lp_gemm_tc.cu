// tcgen05 bf16 GEMM with fused epilogues (the projections of denoise_block:
// QKV denoiser.py:240-242 + rotary :192-197, O :265, FFN :266, head :268).
//
//   C[M, N] = A[M, K] . W^T[N, K]^T     A, W^T bf16 K-major, fp32 accumulate
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer (elected lane): A/B tiles -> 4-stage smem ring
//   warp 1      TMEM allocator + MMA issuer (elected lane): tcgen05.mma
//               128 x BN x 16 per instruction, accumulator in TMEM, double
//               buffered (2 x BN columns) so the epilogue of tile t overlaps
//               the main loop of tile t+1
//   warps 2..9  epilogue (two warps per TMEM lane quarter, one column half
//               each): tcgen05.ld 32 rows x 32 columns per warp-load,
//               fused STORE / RELU / GELU / gated RESIDUAL / QKV (per-head
//               RMSNorm + rotary + scatter of k, v into the KV ring slot)
#include <algorithm>
#include <cstdlib>

#include "lp_common.cuh"
#include "lp_sm100.cuh"
#include "lp_tma.cuh"

namespace lp {

using namespace sm100;

constexpr int GBM = 128, GBK = 64, GSTAGES = 4;
constexpr int G_THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (2 per TMEM lane quarter)

struct GemmParams {
  int m, n, k;
  int m_begin, m_end;  // tiles cover rows [m_begin, m_end); rows >= m are discarded
  int epilogue, out_dtype;
  void* c;
  int64_t ldc;
  const float* bias;
  const float* gate;
  lp_qkv_epi qkv;
  lp_euler_epi euler;
  // implicit-GEMM conv (lp_conv_taps): k-chunk kb reads A rows m0 + tap_row[kb / conv_kpt],
  // columns (kb % conv_kpt) * GBK; conv_kpt = 0 for a plain GEMM
  int conv_kpt;
  int tap_row[27];
  int conv_t, conv_h, conv_w;  // halo conv (conv_tc_kernel): interior frames, height, width
  float2* stats;  // RESID: per-row (mean, M2) of each 32-column chunk of the new h, [m][n/32]
};

__device__ __forceinline__ void a_coords(const GemmParams& p, int kb, int m0, int& col, int& row) {
  if (p.conv_kpt) {
    const int t = kb / p.conv_kpt;
    col = (kb - t * p.conv_kpt) * GBK;
    row = m0 + p.tap_row[t];
  } else {
    col = kb * GBK;
    row = m0;
  }
}


// Tile raster: groups of LP_GEMM_GROUP row blocks, column-major inside a
// group, so a wave of ~148 (74 pair) tiles covers a compact block of rows x
// columns and both operands are re-read from L2 rather than DRAM.
#ifndef LP_GEMM_GROUP
#define LP_GEMM_GROUP 16
#endif
__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int& mb, int& nb) {
  const int per = LP_GEMM_GROUP * tiles_n;
  const int g = tile / per, r = tile - g * per;
  const int gm = min(LP_GEMM_GROUP, tiles_m - g * LP_GEMM_GROUP);
  mb = g * LP_GEMM_GROUP + r % gm;
  nb = r / gm;
}

template <int BN>
struct GemmSmem {
  static constexpr int A_BYTES = GBM * GBK * 2;
  static constexpr int B_BYTES = BN * GBK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = GSTAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;  // barriers + alignment slack
};

__device__ __forceinline__ void store_row32(void* out, int out_dtype, const float* v) {
  if (out_dtype == LP_BF16) {
    uint4* o = reinterpret_cast<uint4*>(out);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      o[q] = make_uint4(pack_bf16(v[8 * q + 0], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                        pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
  } else {
    float4* o = reinterpret_cast<float4*>(out);
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
}

// Epilogue of one accumulator tile for this thread's row: TMEM (tbase: lane
// quarter + accumulator buffer) -> fused QKV / EULER / RESID / activation.
// n0: first output column of the tile; half: which column half this warp
// owns (two epilogue warps per TMEM lane quarter).
template <int BN>
__device__ __forceinline__ void gemm_epilogue_tile(const GemmParams& p, int row, bool valid, uint32_t tbase,
                                                   int n0, int half, int lane) {
  constexpr int HALF_N = BN / 2;
  if (p.epilogue == LP_EPI_QKV) {
    const lp_qkv_epi& e = p.qkv;
    const int hd = e.head_dim;
    const int section = n0 / e.d;  // 0 q, 1 k, 2 v
    const int col0 = n0 - section * e.d;
    int cur = e.desc->cur_row;
    __nv_bfloat16* dst_base =
        section == 0 ? reinterpret_cast<__nv_bfloat16*>(e.q_out) + (int64_t)row * e.d
                     : reinterpret_cast<__nv_bfloat16*>(section == 1 ? e.k_arena : e.v_arena) +
                           (int64_t)(cur + row) * e.d;
    RopeTab rt{e.desc->rope_cos, e.desc->rope_sin, e.geom};
    const float* g = section == 0 ? e.g_q : e.g_k;
    // one head per warp when the column half holds whole heads, else the
    // half-0 warps take the whole tile
    const bool split = HALF_N % hd == 0;
    const int hb = split ? half * HALF_N : 0, he = split ? hb + HALF_N : (half ? 0 : BN);
    for (int h0 = hb; h0 < he; h0 += hd) {
      float inv = 1.0f;
      if (section < 2 && e.qk_norm) {
        float ss[4] = {0.f, 0.f, 0.f, 0.f};  // 4 independent chains, not one 128-long FMA chain
        for (int c0 = 0; c0 < hd; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(tbase + h0 + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float v = __uint_as_float(r[j]);
            ss[j & 3] = fmaf(v, v, ss[j & 3]);
          }
        }
        inv = rsqrtf(((ss[0] + ss[1]) + (ss[2] + ss[3])) / hd + e.eps);
      }
      for (int c0 = 0; c0 < hd; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + h0 + c0, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        const int col = col0 + h0 + c0;  // column within the section
        if (section < 2) {
          float cs[16], sn[16], gg[32];
#pragma unroll
          for (int j = 0; j < 16; ++j) rt.get(row, c0 / 2 + j, cs[j], sn[j]);
          if (e.qk_norm) {
#pragma unroll
            for (int j = 0; j < 32; ++j) gg[j] = g ? __ldg(g + col + j) * inv : inv;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= gg[j];
          }
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float xo, yo;
            rotate_pair(v[j], v[j + 1], cs[j / 2], sn[j / 2], xo, yo);
            v[j] = xo;
            v[j + 1] = yo;
          }
        }
        if (valid) store_row32(dst_base + col, LP_BF16, v);
      }
    }
  } else {
    for (int c0 = half * HALF_N; c0 < (half + 1) * HALF_N; c0 += 32) {
      uint32_t r[32];
      tmem_ld32(tbase + c0, r);
      tmem_ld_wait();
      const int col = n0 + c0;
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
      if (!valid) continue;
      if (p.epilogue == LP_EPI_EULER) {
        const lp_euler_epi& e = p.euler;
        // a failed wait on the consumer's free counter: leave its slot alone
        if (e.gate_status && *(const volatile int32_t*)e.gate_status != 0) continue;
        const float dt = e.desc->dt;
        int64_t base;
        int gy = 0, gx = 0;
        if (e.ph == 0) {
          base = (int64_t)row * p.n;
        } else {
          const int hp = e.height / e.ph, wp = e.width / e.pw, tpf = hp * wp;
          const int f = row / tpf, tok = row % tpf;
          gy = tok / wp;
          gx = tok % wp;
          base = (int64_t)f * e.channels * e.height * e.width;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int c = col + j;
          int64_t idx;
          if (e.ph == 0) {
            idx = base + c;
          } else {
            const int pp = e.ph * e.pw, ch = c / pp, py = (c % pp) / e.pw, px = c % e.pw;
            idx = base + ((int64_t)ch * e.height + gy * e.ph + py) * e.width + gx * e.pw + px;
          }
          e.x_out[idx] = __fadd_rn(e.x_in[idx], __fmul_rn(v[j], dt));
        }
        __threadfence_system();  // x_out may be a peer's receive slot: visible before the ready flag
        continue;
      }
      if (p.epilogue == LP_EPI_RESID) {
        // all loads first (h and gate may alias as far as the compiler
        // knows; interleaving loads with stores serialises DRAM round trips)
        float4* h = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.c) + (int64_t)row * p.ldc + col);
        float4 o[8], g[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = __ldcs(h + q);
        if (p.gate) {
#pragma unroll
          for (int q = 0; q < 8; ++q) g[q] = __ldg(reinterpret_cast<const float4*>(p.gate + col) + q);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) g[q] = make_float4(1.f, 1.f, 1.f, 1.f);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          o[q].x = fmaf(g[q].x, v[4 * q], o[q].x);
          o[q].y = fmaf(g[q].y, v[4 * q + 1], o[q].y);
          o[q].z = fmaf(g[q].z, v[4 * q + 2], o[q].z);
          o[q].w = fmaf(g[q].w, v[4 * q + 3], o[q].w);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) __stcs(h + q, o[q]);
        if (p.stats) {
          // LayerNorm partials of the updated row chunk for the next norm pass
          // (two-pass on the registers: exact mean, then the squared deviations)
          float s4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) s4[j] = (o[2 * j].x + o[2 * j].y) + (o[2 * j].z + o[2 * j].w) +
                                              ((o[2 * j + 1].x + o[2 * j + 1].y) + (o[2 * j + 1].z + o[2 * j + 1].w));
          const float mc = ((s4[0] + s4[1]) + (s4[2] + s4[3])) * (1.0f / 32.0f);
          float q4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float a = o[q].x - mc, b = o[q].y - mc, e = o[q].z - mc, f = o[q].w - mc;
            q4[q & 3] = fmaf(a, a, fmaf(b, b, fmaf(e, e, fmaf(f, f, q4[q & 3]))));
          }
          p.stats[(int64_t)row * (p.n / 32) + col / 32] = make_float2(mc, (q4[0] + q4[1]) + (q4[2] + q4[3]));
        }
      } else {
        if (p.epilogue == LP_EPI_STORE && p.bias) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += p.bias[col + j];
        } else if (p.epilogue == LP_EPI_RELU) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.0f);
        } else if (p.epilogue == LP_EPI_GELU) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = gelu_tanh_f(v[j]);
        }
        const int esz = p.out_dtype == LP_BF16 ? 2 : 4;
        store_row32(reinterpret_cast<uint8_t*>(p.c) + ((int64_t)row * p.ldc + col) * esz, p.out_dtype, v);
      }
    }
  }
}

template <int BN>
__global__ void __launch_bounds__(G_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmParams p) {
  using SM = GemmSmem<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  uint64_t* empty = full + GSTAGES;
  uint64_t* tfull = empty + GSTAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles_m = (p.m_end - p.m_begin + GBM - 1) / GBM, tiles_n = p.n / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int num_kb = p.k / GBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < GSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    fence_barrier_init();
  }
  constexpr uint32_t TMEM_COLS = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);  // power of 2
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t pol_a = l2_policy_evict_last();
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int mb, nb;
        tile_coords(tile, tiles_m, tiles_n, mb, nb);
        const int m0 = p.m_begin + mb * GBM, n0 = nb * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * SM::STAGE_BYTES;
          uint8_t* sb = sa + SM::A_BYTES;
          mbar_arrive_expect_tx(&full[stage], SM::STAGE_BYTES);
          int ac, ar;
          a_coords(p, kb, m0, ac, ar);
          tma_load_2d_hint(sa, &tmA, &full[stage], ac, ar, pol_a);
          tma_load_2d(sb, &tmB, &full[stage], kb * GBK, n0);
          if (++stage == GSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t IDESC = idesc_bf16_f32(GBM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t aphase = (local >> 1) & 1;
      mbar_wait(&tempty[acc], aphase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(smem + stage * SM::STAGE_BYTES);
          const uint32_t sb = sa + SM::A_BYTES;
          const uint64_t da = sdesc_kmajor_sw128(sa), db = sdesc_kmajor_sw128(sb);
#pragma unroll
          for (int k = 0; k < GBK / 16; ++k)
            mma_bf16_ss(d_tmem, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), IDESC, (kb | k) != 0);
          mma_commit(&empty[stage]);
          if (kb == num_kb - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == GSTAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..9) ----------------
    const int quarter = warp & 3;  // TMEM lanes [32*quarter, +32) are addressable by this warp
    const int half = (warp - 2) >> 2;  // the two warps of a lane quarter split the tile's columns
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t aphase = (local >> 1) & 1;
      int mb, nb;
      tile_coords(tile, tiles_m, tiles_n, mb, nb);
      const int m0 = p.m_begin + mb * GBM, n0 = nb * BN;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const int row = m0 + quarter * 32 + lane;
      const bool valid = row < p.m;
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;

      gemm_epilogue_tile<BN>(p, row, valid, tbase, n0, half, lane);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// Halo-tile causal 3x3x3 convolution (the decode stage's VAE stand-in):
// output tile = 8 image rows x 16 pixels of one frame (128 TMEM lanes) x BN
// channels.  For every (dt, dx) and 64-channel chunk one 4-D TMA box brings
// the 10 x 16-pixel window (rows y0-1 .. y0+8 of the bordered layout) whose
// three 8-row views at 16-row offsets are the A operands of the dy = -1, 0, +1
// taps -- 2.4x less A traffic than one row-shifted box per tap -- plus the
// three taps' weight chunks.  Frames before 0 (causal padding) and the window
// rows past the last frame are TMA zero fill; the bordered layout supplies the
// spatial padding.  Same warp roles and double-buffered TMEM accumulator as
// gemm_tc_kernel; the epilogue maps lane r to pixel (y0 + r/16, x0 + r%16).
template <int BN>
struct ConvSmem {
  static constexpr int A_BYTES = 10 * 16 * 128;  // 20 KB window
  static constexpr int B_BYTES = 3 * BN * GBK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN >= 128 ? 3 : 4;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

template <int BN>
__global__ void __launch_bounds__(G_THREADS, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmParams p) {
  using SM = ConvSmem<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  uint64_t* empty = full + SM::STAGES;
  uint64_t* tfull = empty + SM::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int T = p.conv_t, H = p.conv_h, W = p.conv_w, cin = p.conv_kpt * GBK;
  const int ty = (H + 7) / 8, tx = (W + 15) / 16, tiles_n = p.n / BN;
  const int num_tiles = T * ty * tx * tiles_n;
  const int num_kb = 9 * p.conv_kpt;  // (dt, dx) x 64-channel chunks; 3 dy taps per block
  // order: N fastest, then time, then x, then y -- the tiles in flight share
  // their A windows in L2 across output channels and across the three
  // frames each causal tap reads (frame-major order re-read every frame
  // from DRAM three times: 7.5 GB per stage-3 conv)
  auto coords = [&](int tile, int& t, int& y0, int& x0, int& n0) {
    n0 = (tile % tiles_n) * BN;
    int r = tile / tiles_n;
    t = r % T;
    r /= T;
    x0 = (r % tx) * 16;
    y0 = (r / tx) * 8;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < SM::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    fence_barrier_init();
  }
  constexpr uint32_t TMEM_COLS = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int t, y0, x0, n0;
        coords(tile, t, y0, x0, n0);
        for (int kb = 0; kb < num_kb; ++kb) {
          const int tdx = kb / p.conv_kpt, kc = (kb - tdx * p.conv_kpt) * GBK;
          const int dt = tdx / 3 - 2, dx = tdx % 3 - 1;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * SM::STAGE_BYTES;
          uint8_t* sb = sa + SM::A_BYTES;
          mbar_arrive_expect_tx(&full[stage], SM::STAGE_BYTES);
          // window: bordered columns x0+1+dx .. +15, bordered rows y0 .. y0+9, frame t+dt
          tma_load_4d(sa, &tmA, &full[stage], kc, x0 + 1 + dx, y0, t + dt);
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)  // tap (dt, dy-1, dx) weights: K chunk of tap index (dt+2)*9 + dy*3 + dx+1
            tma_load_2d(sb + dy * BN * GBK * 2, &tmB, &full[stage], ((dt + 2) * 9 + dy * 3 + dx + 1) * cin + kc,
                        n0);
          if (++stage == SM::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t IDESC = idesc_bf16_f32(GBM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t aphase = (local >> 1) & 1;
      mbar_wait(&tempty[acc], aphase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(smem + stage * SM::STAGE_BYTES);
          const uint32_t sb = sa + SM::A_BYTES;
#pragma unroll
          for (int dy = 0; dy < 3; ++dy) {
            const uint64_t da = sdesc_kmajor_sw128(sa + dy * 16 * 128);  // window rows 16*dy ..: the dy tap
            const uint64_t db = sdesc_kmajor_sw128(sb + dy * BN * GBK * 2);
#pragma unroll
            for (int k = 0; k < GBK / 16; ++k)
              mma_bf16_ss(d_tmem, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), IDESC, (kb | dy | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (kb == num_kb - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == SM::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t aphase = (local >> 1) & 1;
      int t, y0, x0, n0;
      coords(tile, t, y0, x0, n0);
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const int r = quarter * 32 + lane, yy = y0 + r / 16, xx = x0 + r % 16;
      const bool valid = yy < H && xx < W;
      const int row = (t * (H + 2) + yy + 1) * (W + 2) + xx + 1;
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
      gemm_epilogue_tile<BN>(p, valid ? row : 0, valid, tbase, n0, half, lane);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// 2-CTA variant (cluster pair, tcgen05.mma.cta_group::2): tile 256 x BN per
// pair, each CTA loads its 128 rows of A and its BN/2 rows of B, the leader
// issues M = 256 MMAs whose accumulator halves land in each CTA's TMEM.  Per
// CTA a k-block costs 32 KB of shared memory instead of 48 KB, so 6 stages
// buffer 1.5x more time against TMA latency.
constexpr int G2_STAGES = 6;

template <int BN>
struct Gemm2Smem {
  static constexpr int A_BYTES = GBM * GBK * 2;
  static constexpr int B_BYTES = (BN / 2) * GBK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = G2_STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G_THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmParams p) {
  using SM = Gemm2Smem<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  uint64_t* empty = full + G2_STAGES;
  uint64_t* tfull = empty + G2_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int tiles_m = (p.m_end - p.m_begin + 2 * GBM - 1) / (2 * GBM), tiles_n = p.n / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int num_kb = p.k / GBK;
  const int cid = blockIdx.x >> 1, nclu = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < G2_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 16);  // 8 epilogue warps x 2 CTAs (the leader's copy is used)
    }
    fence_barrier_init();
  }
  cluster_sync_all();  // barriers initialised in both CTAs before any remote arrive / TMA
  if (warp == 1) tmem_alloc_2cta(tmem_slot, 2 * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t pol = l2_policy_evict_last();
      for (int tile = cid; tile < num_tiles; tile += nclu) {
        int mb, nb;
        tile_coords(tile, tiles_m, tiles_n, mb, nb);
        int m0 = p.m_begin + mb * 2 * GBM + rank * GBM;
        if (m0 >= p.m) m0 = p.m > GBM ? p.m - GBM : 0;  // wholly past M: load valid rows, results discarded
        const int n0 = nb * BN + rank * (BN / 2);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * SM::STAGE_BYTES;
          uint8_t* sb = sa + SM::A_BYTES;
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * SM::STAGE_BYTES);
          tma_load_2d_2sm(sa, &tmA, &full[stage], kb * GBK, m0, pol);
          tma_load_2d_2sm(sb, &tmB, &full[stage], kb * GBK, n0, pol);
          if (++stage == G2_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only) ----------------
    if (rank == 0) {
      constexpr uint32_t IDESC = idesc_bf16_f32(2 * GBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int tile = cid; tile < num_tiles; tile += nclu, ++local) {
        const int acc = local & 1;
        const uint32_t aphase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = smem_u32(smem + stage * SM::STAGE_BYTES);
            const uint32_t sb = sa + SM::A_BYTES;
            const uint64_t da = sdesc_kmajor_sw128(sa), db = sdesc_kmajor_sw128(sb);
#pragma unroll
            for (int k = 0; k < GBK / 16; ++k)
              mma_bf16_ss_2cta(d_tmem, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), IDESC, (kb | k) != 0);
            mma_commit_2cta_mc(&empty[stage]);
            if (kb == num_kb - 1) mma_commit_2cta_mc(&tfull[acc]);
          }
          __syncwarp();
          if (++stage == G2_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..9, both CTAs) ----------------
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    int local = 0;
    for (int tile = cid; tile < num_tiles; tile += nclu, ++local) {
      const int acc = local & 1;
      const uint32_t aphase = (local >> 1) & 1;
      int mb, nb;
      tile_coords(tile, tiles_m, tiles_n, mb, nb);
      const int m0 = p.m_begin + mb * 2 * GBM + rank * GBM, n0 = nb * BN;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const int row = m0 + quarter * 32 + lane;
      const bool valid = row < p.m;
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
      gemm_epilogue_tile<BN>(p, row, valid, tbase, n0, half, lane);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's smem / TMEM are in use until the leader's last MMA is consumed
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2cta(tmem_base, 2 * BN);
  }
}

template <int BN>
static int launch_gemm_tc2(const lp_gemm_args* a, const GemmParams& p, cudaStream_t st) {
  CUtensorMap ta, tb;
  int rc = make_tmap_bf16_2d(&ta, a->a, (uint64_t)a->m, (uint64_t)a->k, (uint64_t)a->lda, GBM, GBK);
  if (rc) return rc;
  rc = make_tmap_bf16_2d(&tb, a->w, (uint64_t)a->n, (uint64_t)a->k, (uint64_t)a->ldw, BN / 2, GBK);
  if (rc) return rc;
  const int tiles = ((p.m_end - p.m_begin + 2 * GBM - 1) / (2 * GBM)) * (a->n / BN);
  const int clusters = std::min(tiles, std::max(1, num_sms() / 2));
  const int smem = Gemm2Smem<BN>::TOTAL;
  auto kern = gemm_tc2_kernel<BN>;
  LP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<2 * clusters, G_THREADS, smem, st>>>(ta, tb, p);
  return launch_status("gemm_tc2");
}

template <int BN>
static int launch_conv_tc(const lp_gemm_args* a, const GemmParams& p, cudaStream_t st) {
  CUtensorMap ta, tb;
  const uint64_t dims[4] = {(uint64_t)p.conv_kpt * GBK, (uint64_t)p.conv_w + 2, (uint64_t)p.conv_h + 2,
                            (uint64_t)p.conv_t};
  const uint32_t box[4] = {GBK, 16, 10, 1};
  int rc = make_tmap_bf16_4d(&ta, a->a, dims, box);
  if (rc) return rc;
  rc = make_tmap_bf16_2d(&tb, a->w, (uint64_t)a->n, (uint64_t)a->k, (uint64_t)a->ldw, BN, GBK);
  if (rc) return rc;
  const int tiles = p.conv_t * ((p.conv_h + 7) / 8) * ((p.conv_w + 15) / 16) * (a->n / BN);
  const int grid = std::min(tiles, std::max(1, num_sms()));
  const int smem = ConvSmem<BN>::TOTAL;
  auto kern = conv_tc_kernel<BN>;
  LP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, G_THREADS, smem, st>>>(ta, tb, p);
  return launch_status("conv_tc");
}

template <int BN>
static int launch_gemm_tc(const lp_gemm_args* a, const GemmParams& p, cudaStream_t st) {
  CUtensorMap ta, tb;
  const uint64_t a_cols = p.conv_kpt ? (uint64_t)p.conv_kpt * GBK : (uint64_t)a->k;  // conv: A is [rows, cin]
  int rc = make_tmap_bf16_2d(&ta, a->a, (uint64_t)a->m, a_cols, (uint64_t)a->lda, GBM, GBK);
  if (rc) return rc;
  rc = make_tmap_bf16_2d(&tb, a->w, (uint64_t)a->n, (uint64_t)a->k, (uint64_t)a->ldw, BN, GBK);
  if (rc) return rc;
  const int tiles = ((p.m_end - p.m_begin + GBM - 1) / GBM) * (a->n / BN);
  const int grid = std::min(tiles, std::max(1, num_sms()));
  const int smem = GemmSmem<BN>::TOTAL;
  auto kern = gemm_tc_kernel<BN>;
  LP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, G_THREADS, smem, st>>>(ta, tb, p);
  return launch_status("gemm_tc");
}

int fork_create(void** out) {
  LP_CHECK_ARG(out, "lp_fork_create: null argument");
  ForkCtx* f = new ForkCtx();
  // lowest priority: the side branch's CTAs are scheduled only when no CTA of
  // the main branch's grid is waiting (they fill its last wave instead of
  // taking, and fragmenting, SMs a cluster pair of the main grid needs)
  int least = 0, greatest = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&f->side, cudaStreamNonBlocking, least);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->join, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete f;
    return fail(LP_ECUDA, std::string("lp_fork_create: ") + cudaGetErrorString(e));
  }
  *out = f;
  return LP_OK;
}

int fork_destroy(void* h) {
  if (!h) return LP_OK;
  ForkCtx* f = static_cast<ForkCtx*>(h);
  cudaEventDestroy(f->fork);
  cudaEventDestroy(f->join);
  cudaStreamDestroy(f->side);
  delete f;
  return LP_OK;
}

int preload_gemm_tc() {
  cudaFuncAttributes a;
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, gemm_tc_kernel<64>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, gemm_tc_kernel<128>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, gemm_tc_kernel<256>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, gemm_tc2_kernel<256>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, conv_tc_kernel<128>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, conv_tc_kernel<64>));
  return LP_OK;
}

static bool g_gemm2 = getenv("LP_NO_GEMM2") == nullptr;      // LP_NO_GEMM2=1 forces 1-CTA tiles
static bool g_gemm2_all = getenv("LP_GEMM2_ALL") != nullptr;  // LP_GEMM2_ALL=1: pairs whenever N % 256 == 0
static bool g_gemm2_qkv = getenv("LP_NO_GEMM2_QKV") == nullptr;  // LP_NO_GEMM2_QKV=1: 1-CTA QKV tiles
static bool g_split = getenv("LP_NO_PAIR_SPLIT") == nullptr;     // LP_NO_PAIR_SPLIT=1: no pair + tail split

// Cluster pairs on the rows [0, m_pair) that whole 256-row pair tiles cover,
// and the ragged last rows (m - m_pair < 256) as single-CTA tiles on the
// fork context's side stream, concurrently: the pair kernel's last wave
// leaves 2 * (pairs * waves - tiles) SMs idle, and the tail tiles run there.
// At 14B (m = 4680) this turns O-proj / FFN-down from 5 single-CTA waves
// into 5 pair waves (whose tiles read half of B per CTA) and QKV from 16 to
// 15 pair waves.  Returns 1 when the split does not apply.
// Wave costs in the comparison: a pair wave 100, a single-CTA wave 115 (the
// 14B GEMMs run at 96 % vs 81-84 % of the tensor pipe: single-CTA tiles read
// all of B per CTA and are L2-feed bound).  LP_PAIR_SPLIT_ALL forces the split
// whenever the shape allows it (tests of small shapes).
static int launch_pair_split(const lp_gemm_args* a, const GemmParams& p, cudaStream_t st, long waves_now,
                             bool pair_now) {
  if (!a->fork || !g_gemm2 || !g_split || a->n % 256 != 0) return 1;
  const long sms = std::max(1, num_sms()), pairs = std::max(1L, sms / 2);
  const long m_pair = (a->m / 256) * 256;
  if (m_pair < 256 || m_pair == a->m) return 1;
  const long tiles2 = (m_pair / 256) * (a->n / 256), waves2 = (tiles2 + pairs - 1) / pairs;
  const long idle = 2 * (pairs * waves2 - tiles2), tail = ((a->m - m_pair + GBM - 1) / GBM) * (a->n / 256);
  const long t_now = waves_now * (pair_now ? 100 : 115);
  const long t_split = waves2 * 100 + (tail > idle ? 115 * ((tail - idle + sms - 1) / sms) : 0) + 2;
  if (getenv("LP_PAIR_SPLIT_ALL") == nullptr && t_split >= t_now) return 1;
  const ForkCtx* f = static_cast<const ForkCtx*>(a->fork);
  GemmParams pp = p, pt = p;
  pp.m_end = (int)m_pair;
  pt.m_begin = (int)m_pair;
  LP_CUDA_TRY(cudaEventRecord(f->fork, st));
  LP_CUDA_TRY(cudaStreamWaitEvent(f->side, f->fork, 0));
  int rc = launch_gemm_tc2<256>(a, pp, st);  // launched first: its CTAs take every SM
  if (rc) return rc;
  rc = launch_gemm_tc<256>(a, pt, f->side);
  if (rc) return rc;
  LP_CUDA_TRY(cudaEventRecord(f->join, f->side));
  LP_CUDA_TRY(cudaStreamWaitEvent(st, f->join, 0));
  return LP_OK;
}

int gemm_tc(const lp_gemm_args* a, cudaStream_t st) {
  LP_CHECK_ARG(num_sms() > 0, "lp_init() must be called before the tcgen05 GEMM");
  LP_CHECK_ARG(a->k % GBK == 0, "gemm_tc: k must be a multiple of 64");
  LP_CHECK_ARG(a->lda % 8 == 0 && a->ldw % 8 == 0, "gemm_tc: leading dims must be 16-byte aligned");
  if (a->m == 0) return LP_OK;
  GemmParams p;
  p.m = a->m;
  p.m_begin = 0;
  p.m_end = a->m;
  p.n = a->n;
  p.k = a->k;
  p.epilogue = a->epilogue;
  p.out_dtype = a->out_dtype;
  p.c = a->c;
  p.ldc = a->ldc;
  p.bias = a->bias;
  p.gate = a->gate;
  p.stats = nullptr;
  if (a->row_stats) {
    LP_CHECK_ARG(a->epilogue == LP_EPI_RESID && a->n % 32 == 0 && !a->conv,
                 "gemm_tc: row_stats needs a RESID epilogue with n % 32 == 0");
    p.stats = reinterpret_cast<float2*>(a->row_stats);
  }
  memset(&p.qkv, 0, sizeof(p.qkv));
  memset(&p.euler, 0, sizeof(p.euler));
  p.conv_kpt = 0;
  if (a->conv) {
    const lp_conv_taps& cv = *a->conv;
    LP_CHECK_ARG(cv.n_taps >= 1 && cv.n_taps <= 27 && cv.cin % GBK == 0 && a->k == cv.n_taps * cv.cin,
                 "gemm_tc: conv needs 1..27 taps, cin % 64 == 0 and k == n_taps * cin");
    LP_CHECK_ARG(a->epilogue == LP_EPI_STORE || a->epilogue == LP_EPI_RESID, "gemm_tc: conv epilogue STORE/RESID");
    LP_CHECK_ARG(a->lda == cv.cin, "gemm_tc: conv A is [rows, cin] (lda == cin)");
    p.conv_kpt = cv.cin / GBK;
    for (int t = 0; t < cv.n_taps; ++t) p.tap_row[t] = cv.tap_row[t];
    p.conv_t = cv.frames, p.conv_h = cv.height, p.conv_w = cv.width;
    if (cv.n_taps == 27 && cv.frames > 0 && cv.height > 0 && cv.width > 0 && getenv("LP_CONV_ROWSHIFT") == nullptr) {
      LP_CHECK_ARG((int64_t)cv.frames * (cv.height + 2) * (cv.width + 2) == a->m, "gemm_tc: conv geometry vs m");
      if (a->n % 128 == 0) return launch_conv_tc<128>(a, p, st);
      if (a->n % 64 == 0) return launch_conv_tc<64>(a, p, st);
    }
    // single-CTA tiles: the A box of a tap is one row-shifted 128-row window
    if (a->n % 256 == 0) return launch_gemm_tc<256>(a, p, st);
    if (a->n % 128 == 0) return launch_gemm_tc<128>(a, p, st);
    if (a->n % 64 == 0) return launch_gemm_tc<64>(a, p, st);
    return fail(LP_EUNSUPPORTED, "gemm_tc: conv n must be a multiple of 64");
  }
  if (a->epilogue == LP_EPI_EULER) {
    LP_CHECK_ARG(a->euler != nullptr && a->euler->x_in && a->euler->x_out && a->euler->desc,
                 "gemm_tc: EULER epilogue needs euler args");
    p.euler = *a->euler;
    LP_CHECK_ARG(p.euler.ph == 0 || a->n == p.euler.channels * p.euler.ph * p.euler.pw, "gemm_tc: EULER shape");
  }
  if (a->epilogue == LP_EPI_QKV) {
    LP_CHECK_ARG(a->qkv != nullptr, "gemm_tc: QKV epilogue needs qkv args");
    p.qkv = *a->qkv;
    LP_CHECK_ARG(a->n == 3 * p.qkv.d && p.qkv.head_dim % 32 == 0, "gemm_tc: QKV shape");
    LP_CHECK_ARG(p.qkv.d % 256 == 0 || p.qkv.d % 128 == 0, "gemm_tc: QKV needs d % 128 == 0");
    if (p.qkv.d % 256 == 0 && p.qkv.head_dim <= 256 && 256 % p.qkv.head_dim == 0) {
      // cluster pairs under the same wave rule as the plain GEMMs below (each
      // CTA of a pair runs the per-row epilogue on its own 128 rows)
      const long sms = std::max(1, num_sms()), pairs = std::max(1L, sms / 2);
      const long waves2 = (((a->m + 255) / 256) * (a->n / 256) + pairs - 1) / pairs;
      const long waves1 = (((a->m + GBM - 1) / GBM) * (a->n / 256) + sms - 1) / sms;
      const bool pair = g_gemm2 && g_gemm2_qkv && a->m >= 256 && (g_gemm2_all || waves2 * 23 < waves1 * 25);
      if (g_gemm2_qkv) {
        const int rc = launch_pair_split(a, p, st, pair ? waves2 : waves1, pair);
        if (rc != 1) return rc;
      }
      if (pair) return launch_gemm_tc2<256>(a, p, st);
      return launch_gemm_tc<256>(a, p, st);
    }
    LP_CHECK_ARG(128 % p.qkv.head_dim == 0, "gemm_tc: head_dim must divide the tile");
    return launch_gemm_tc<128>(a, p, st);
  }
  LP_CHECK_ARG(a->ldc % 4 == 0, "gemm_tc: ldc alignment");
  // Widest tile that divides N, unless halving it removes more than 10% of
  // the makespan in whole waves (the 1.3B shape's N = 1536 GEMMs: 1.5 waves
  // of 256-wide tiles vs 3 full waves of 128).  Narrower tiles read more
  // operand bytes per FLOP, so small wave gains are not worth it (a 192-wide
  // tile for FFN-up at 14B: 18 full waves instead of 13.5, measured slower).
  const long tiles_m = (a->m + GBM - 1) / GBM, sms = std::max(1, num_sms());
  auto makespan = [&](int bn) { return ((tiles_m * (a->n / bn) + sms - 1) / sms) * bn; };
  // (only for short K: with K = 8960 the 128-wide tile measured slower even at 3 vs 1.5 waves)
  if (a->n % 256 == 0 && !(a->k <= 4096 && makespan(128) * 10 < makespan(256) * 9)) {
    // cluster-pair (2-CTA) tiles unless their waves lose more than the ~8%
    // per-wave gain (O-proj / FFN-down at 14B: 6 pair waves vs 5 single waves)
    const long pairs = std::max(1L, sms / 2), tiles2 = ((a->m + 255) / 256) * (a->n / 256);
    const long waves2 = (tiles2 + pairs - 1) / pairs, waves1 = (tiles_m * (a->n / 256) + sms - 1) / sms;
    const bool pair = g_gemm2 && a->m >= 256 && (g_gemm2_all || waves2 * 23 < waves1 * 25);
    const int rc = launch_pair_split(a, p, st, pair ? waves2 : waves1, pair);
    if (rc != 1) return rc;
    if (pair) return launch_gemm_tc2<256>(a, p, st);
    return launch_gemm_tc<256>(a, p, st);
  }
  if (a->n % 128 == 0) return launch_gemm_tc<128>(a, p, st);
  if (a->n % 64 == 0) return launch_gemm_tc<64>(a, p, st);
  return fail(LP_EUNSUPPORTED, "gemm_tc: n must be a multiple of 64");
}

// ------------------------------------------------------------------- TMA ---
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn g_encode = nullptr;

int tma_init() {
  if (g_encode) return LP_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  LP_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return fail(LP_ECUDA, "cuTensorMapEncodeTiled not available");
  g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  return LP_OK;
}

int make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                      uint32_t box_rows, uint32_t box_cols) {
  if (!g_encode) return fail(LP_EINVAL, "TMA not initialised (call lp_init)");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle sw = box_cols * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : box_cols * 2 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                               : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LP_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return LP_OK;
}

int make_tmap_bf16_4d(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint32_t box[4]) {
  if (!g_encode) return fail(LP_EINVAL, "TMA not initialised (call lp_init)");
  cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t strides[3] = {dims[0] * 2, dims[0] * dims[1] * 2, dims[0] * dims[1] * dims[2] * 2};
  cuuint32_t b[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUtensorMapSwizzle sw = box[0] * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), d, strides, b, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LP_ECUDA, "cuTensorMapEncodeTiled (4-D) failed: " + std::to_string((int)r));
  return LP_OK;
}

}  // namespace lp
