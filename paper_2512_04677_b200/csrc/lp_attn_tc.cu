// tcgen05 flash attention over the RSFM key set [sink | history ring | current]
// (denoiser.py:246-264, _attend_head :152-158, softmax numerics.py:67-78).
//
// One CTA per work unit = (256 queries, head[, KV range]): two 128-row Q
// tiles (A, B) share every K/V tile.  Wave quantisation: the host orders the
// units regular-first and splits the last few (the ragged query tail of each
// head plus as many regular units as the makespan model asks for) into S
// KV-range pieces whose (O, m, l) partials are merged by attn_combine_kernel
// in a fixed order (deterministic).  A unit whose tile B lies wholly past
// n_q skips B's MMAs and softmax.  Head dim 128, bf16 Q/K/V, fp32 S/O in TMEM, online softmax in
// fp32.  KV tiles of 128 keys walk the descriptor's segments in reference
// order (sink, oldest -> newest history, current); the ragged tail of a
// segment is masked to -inf, so segments need no padding and nothing is
// gathered or copied.
//
//   warp 0      TMA producer: Q_A, Q_B once, then K_j (2-stage ring) and
//               V_{j-1} (2-stage ring, lagging K by one tile)
//   warp 1      TMEM allocator + MMA issuer (one elected lane):
//                 S_A(j+1) and S_B(j+1) = Q K^T are issued right after
//                 P_A(j) V_j / P_B(j) V_j, so the tensor core always has the
//                 other tile's work while a softmax warpgroup runs
//   warps 2-5   softmax warpgroup A, warps 6-9 softmax warpgroup B: thread =
//               query row; S row from TMEM in one pass, exp2 with a lazily
//               updated running max (O is rescaled in TMEM only when the max
//               grows by more than 2^8; 1/4 of the exponentials run as a
//               degree-3 polynomial on the FMA pipe so MUFU is not the
//               co-bottleneck with the tensor core), P written back to TMEM as bf16 over
//               its own S columns and consumed from TMEM by the P.V MMA
//               (A-operand-in-TMEM form), O / l -> bf16 at the end
//
// TMEM columns: S_A|P_A [0,128)  S_B|P_B [128,256)  O_A [256,384)  O_B [384,512).
// In-order completion of one thread's tcgen05.mma stream makes the S(j+1)
// write after P(j).V safe, and s_full(j) imply P(j-1).V done.
#include <algorithm>
#include <map>
#include <mutex>
#include <queue>
#include <tuple>
#include <vector>

#include "lp_common.cuh"
#include "lp_sm100.cuh"
#include "lp_tma.cuh"

namespace lp {

using namespace sm100;

#ifndef LP_ATTN_POLY
#define LP_ATTN_POLY 3  // pairs of every 8 whose exp2 runs as the FMA-pipe polynomial (sweep: r1c, r1j)
#endif
#ifndef LP_ATTN_POLY_WIN
#define LP_ATTN_POLY_WIN 3  // ... in the bounded-exponent kernel (cheaper polynomial: no clamps)
#endif
#ifndef LP_ATTN_POLY_DEG
#define LP_ATTN_POLY_DEG 3  // degree of the bounded-exponent kernel's 2^f polynomial (A/B: 2)
#endif

constexpr int AT_M = 128;      // query rows per softmax warpgroup
constexpr int AT_N = 128;      // keys per tile
constexpr int AT_D = 128;      // head dim
constexpr int AT_THREADS = 384;  // WG0: TMA warp, MMA warp, 2 idle; WG1, WG2: softmax of Q tiles A, B
constexpr int AT_REG_CTRL = 56;  // setmaxnreg budget of the control warpgroup
constexpr int AT_REG_SOFTMAX = 224;  // ... and of each softmax warpgroup (56*128 + 224*256 <= 64K)
constexpr int AT_TILE_BYTES = AT_N * AT_D * 2;  // 32 KB
constexpr int AT_HALF = AT_TILE_BYTES / 2;      // one 64-column SW128 block
constexpr float AT_RESCALE_THRESH = 8.0f;       // log2 units: rescale O when the max grows > 2^8

struct AttnSmem {
  static constexpr int Q_OFF = 0;                           // Q_A, Q_B
  static constexpr int K_OFF = Q_OFF + 2 * AT_TILE_BYTES;   // 2 stages
  static constexpr int V_OFF = K_OFF + 2 * AT_TILE_BYTES;   // 2 stages
  static constexpr int BAR_OFF = V_OFF + 2 * AT_TILE_BYTES;
  static constexpr int SEG_OFF = BAR_OFF + 256;
  static constexpr int TOTAL = SEG_OFF + 2 * LP_MAX_SEG * 4 + 16 + 1024;
  static_assert(2 * LP_MAX_SEG * 4 + 16 >= 2 * LP_MAX_SEG * 4 + 3 * 4, "segment scratch");
};

struct AttnParams {
  int n_q, n_heads;
  float scale_log2;  // scale * log2(e)
  __nv_bfloat16* out;
  int64_t ldo;
  const lp_block_desc* desc;
  // work decomposition (see AttnPlan)
  int pairs;      // 256-query units per head
  int reg_pairs;  // units per head whose both tiles hold valid rows
  int n_whole;    // leading units run whole (grid prefix)
  int split;      // KV pieces per split unit
  float* part_o;  // [piece][256][128] unnormalised O of split units
  float* part_ml; // [piece][256][2]   (running max in log2 units, row sum)
  int* flags;     // bounded-exponent kernels: 1 = a row left the exponent window,
                  // rerun exactly; exact kernel: non-null = rerun only those
  int flag_pairs; // flags written per CTA of a cluster pair (2 per work unit)
  int unit_base;  // first unit of this launch (the ragged tail runs as its own launch)
  int l2pol;      // persistent kernel L2 hints (A/B, LP_ATTN_L2POL): bit 0 = Q evict_first,
                  // bit 1 = K/V evict_normal (default 0: everything evict_last)
  int* sched;     // persistent kernel: global item counters (zeroed before the launch) for
                  // dynamic item assignment, or NULL: static round robin
  // head-split queues (LP_ATTN_HEADSPLIT=T): clusters whose leader SM id is < T
  // take the items of heads [0, H/2) first, the others heads [H/2, H); each
  // queue is a list of item-index runs; an exhausted queue steals from the other
  int hs_smid;       // T, or 0: one queue in item order.  sched[0..1]: queue counters,
                     // sched[2..3]: items per queue, sched[4..5]: runs per queue,
                     // sched[8 + 16 q + 2 r]: (first item, length) of run r of queue q
};

// Written into the workspace before each dynamic launch by sched_init_kernel
// (by-value kernel argument, so a captured graph replays it unchanged).
struct SchedTable {
  int v[40];
};

// Unit u -> (head, pair): regular units (both Q tiles valid) first, head-major
// so concurrently running CTAs share K/V in L2, then the ragged tail unit of
// every head.
__device__ __forceinline__ void unit_coords(const AttnParams& p, int u, int& head, int& pair) {
  const int n_reg = p.reg_pairs * p.n_heads;
  if (u < n_reg) {
    head = u / p.reg_pairs;
    pair = u % p.reg_pairs;
  } else {
    head = u - n_reg;
    pair = p.pairs - 1;
  }
}

// packed fp32x2 helpers (FFMA2 / FADD2 on sm_100)
__device__ __forceinline__ uint64_t f32x2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpack_f32x2(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fadd2_rm(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// Packed version of ex2_poly (below) for a pair.
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t xv) {
  float x0, x1;
  unpack_f32x2(xv, x0, x1);
  xv = f32x2(fmaxf(x0, -127.0f), fmaxf(x1, -127.0f));
  const uint64_t magic = f32x2(12582912.0f, 12582912.0f);
  const uint64_t t = fadd2_rm(xv, magic);
  const uint64_t f = fsub2(xv, fsub2(t, magic));
  uint64_t q = ffma2(f32x2(0.07706641f, 0.07706641f), f, f32x2(0.2276457f, 0.2276457f));
  q = ffma2(q, f, f32x2(0.69511662f, 0.69511662f));
  q = ffma2(q, f, f32x2(1.0f, 1.0f));
  float q0, q1, t0, t1;
  unpack_f32x2(q, q0, q1);
  unpack_f32x2(t, t0, t1);
  return f32x2(__int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23)),
               __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23)));
}

// fma.f32x2 has no .sat form: two scalar FFMA.SAT (still no FMNMX clamps)
__device__ __forceinline__ uint64_t ffma2_sat(uint64_t a, uint64_t b, uint64_t c) {
  float a0, a1, b0, b1, c0, c1;
  unpack_f32x2(a, a0, a1);
  unpack_f32x2(b, b0, b1);
  unpack_f32x2(c, c0, c1);
  return f32x2(__saturatef(fmaf(a0, b0, c0)), __saturatef(fmaf(a1, b1, c1)));
}
__device__ __forceinline__ uint64_t ffma2_rm(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// 2^x for a pair of raw scores s with x = s*scale*log2e - m clamped to
// [-127, 65] for free: the first FMA computes y = (x + 127) / 192 with .sat
// (y in [0, 1]), so no FMNMX clamps are needed.  floor(x) comes from a
// round-down FMA into the 1.5*2^23 magic range, the fraction from one more
// FMA, 2^f from the degree-3 polynomial and the exponent is added as an
// integer.  At x = -127 the result is exactly +0 (masked keys); at the upper
// clamp 2^65 is returned and the caller's window check (row sum < 2^64) fails.
__device__ __forceinline__ uint64_t ex2_poly2_win(uint64_t s2, uint64_t a2, uint64_t b2) {
  const uint64_t y = ffma2_sat(s2, a2, b2);
  const uint64_t k192 = f32x2(192.0f, 192.0f), cm = f32x2(12582912.0f - 127.0f, 12582912.0f - 127.0f);
  const uint64_t t = ffma2_rm(y, k192, cm);
  const uint64_t f = ffma2(y, k192, fsub2(cm, t));
#if LP_ATTN_POLY_DEG == 2
  // minimax quadratic (max rel. error 1.7e-3, under the bf16 rounding of P)
  uint64_t q = ffma2(f32x2(0.33718635f, 0.33718635f), f, f32x2(0.65763494f, 0.65763494f));
  q = ffma2(q, f, f32x2(1.00172607f, 1.00172607f));
#else
  uint64_t q = ffma2(f32x2(0.07706641f, 0.07706641f), f, f32x2(0.2276457f, 0.2276457f));
  q = ffma2(q, f, f32x2(0.69511662f, 0.69511662f));
  q = ffma2(q, f, f32x2(1.0f, 1.0f));
#endif
  float q0, q1, t0, t1;
  unpack_f32x2(q, q0, q1);
  unpack_f32x2(t, t0, t1);
  return f32x2(__int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23)),
               __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23)));
}

// 2^x for x <= 8 on the FMA pipe: Cody-Waite split x = j + f, degree-3
// minimax polynomial for 2^f on [0, 1) (max rel. error 8.6e-5, far below the
// bf16 rounding of P), exponent added as an integer.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -127.0f);
  const float t = __fadd_rd(x, 12582912.0f);  // 1.5 * 2^23: floor(x) lands in the low mantissa bits
  const float f = __fsub_rn(x, __fsub_rn(t, 12582912.0f));
  const float q = fmaf(fmaf(fmaf(0.07706641f, f, 0.2276457f), f, 0.69511662f), f, 1.0f);
  return __int_as_float(__float_as_int(q) + (__float_as_int(t) << 23));
}

// Walks the KV tiles of the (merged, arena-ordered) segments.  The segment
// table lives in shared memory and is read through 32-bit shared addresses
// (ld.shared): a generic int* here compiled to LD.E through a 64-bit pointer
// that the softmax warpgroups spilled and reloaded every tile.
__device__ __forceinline__ int lds_s32(uint32_t addr) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

struct TileCursor {
  uint32_t row_s, len_s;  // shared addresses of seg_row[0], seg_len[0]
  int n_seg, seg, off, len, row;
  __device__ void load() {
    row = lds_s32(row_s + 4u * seg);
    len = lds_s32(len_s + 4u * seg);
  }
  __device__ void init(const int* r, const int* l, int n) {
    row_s = (uint32_t)__cvta_generic_to_shared(r);
    len_s = (uint32_t)__cvta_generic_to_shared(l);
    n_seg = n; seg = 0; off = 0; len = 0; row = 0;
    if (n_seg > 0) load();
  }
  __device__ void skip(int tiles) {
    for (int i = 0; i < tiles; ++i) next();
  }
  __device__ int cur_row() const { return row + off; }
  __device__ int cur_valid() const { return min(AT_N, len - off); }
  __device__ void next() {
    off += AT_N;
    if (off >= len) {
      off = 0;
      if (++seg < n_seg) load();
    }
  }
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void tmem_st32_x(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}

// Thread 0: the descriptor's segments (merged in arena-row order when the
// descriptor says so) and this CTA's KV tile range -> shared memory.
__device__ void plan_segments(const AttnParams& p, int piece, int* seg_row, int* seg_len, int* n_seg_s) {
  // Key order does not change softmax(QK^T)V, so with desc->arena_order
  // the segments are visited in arena-row order with physically adjacent
  // ones merged: in steady state [sink | L+1 ring slots] is one contiguous
  // range and only its last tile is ragged (24,960 keys: 195 tiles instead
  // of 198 segment-by-segment).  Deterministic for a given row placement
  // (the engines' ring slots depend only on the block index: TPP == seq);
  // without it, logical order, so the drop-in's pool placement is invisible.
  const int n_in = min(p.desc->n_seg, LP_MAX_SEG);
  const bool by_row = p.desc->arena_order != 0;
  int nseg = 0;
  for (int s = 0; s < n_in; ++s) {
    const int r = p.desc->seg_row[s], l = p.desc->seg_len[s];
    if (l <= 0) continue;
    int i = nseg++;
    while (by_row && i > 0 && seg_row[i - 1] > r) {
      seg_row[i] = seg_row[i - 1];
      seg_len[i] = seg_len[i - 1];
      --i;
    }
    seg_row[i] = r;
    seg_len[i] = l;
  }
  int merged = 0;
  for (int s = 0; s < nseg; ++s) {
    if (by_row && merged > 0 && seg_row[merged - 1] + seg_len[merged - 1] == seg_row[s]) {
      seg_len[merged - 1] += seg_len[s];
    } else {
      seg_row[merged] = seg_row[s];
      seg_len[merged] = seg_len[s];
      ++merged;
    }
  }
  nseg = merged;
  int nt = 0;
  for (int s = 0; s < nseg; ++s) nt += (seg_len[s] + AT_N - 1) / AT_N;
  n_seg_s[0] = nseg;
  // this CTA's KV tile range: all tiles, or piece `piece` of `split`
  const int t0 = piece < 0 ? 0 : (int)((int64_t)nt * piece / p.split);
  const int t1 = piece < 0 ? nt : (int)((int64_t)nt * (piece + 1) / p.split);
  n_seg_s[1] = t1 - t0;
  n_seg_s[2] = t0;
}

// FAST = the bounded-exponent form: each row's exponent offset m is the exact
// max of its FIRST KV tile and is never updated, so the per-tile row max, the
// O rescale and the exponent clamps leave the softmax critical path.  This is
// exact softmax (the offset cancels in O / l) whenever every later score stays
// within 2^64 of 2^m; a row that leaves that window shows up as a row sum
// >= 2^64 (or inf), flags its CTA, and the exact kernel (!FAST, running only
// the flagged CTAs) recomputes that work unit with the online max.  Wan's
// q/k RMSNorm bounds |s| by |q||k|/sqrt(d), far inside the window.
template <bool FAST>
__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  if (!FAST && p.flags != nullptr &&
      (p.flag_pairs ? (p.flags[2 * blockIdx.x] | p.flags[2 * blockIdx.x + 1]) : p.flags[blockIdx.x]) == 0)
    return;  // rerun only flagged units
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + AttnSmem::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2] per Q tile
  uint64_t* p_full = bars + 11;  // [2] per Q tile: all of P(j) in TMEM
  uint64_t* p_half = bars + 13;  // [2] per Q tile: keys [0, 64) of P(j) in TMEM (O rescaled)
  uint64_t* o_done = bars + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  int* seg_row = reinterpret_cast<int*>(smem + AttnSmem::SEG_OFF);
  int* seg_len = seg_row + LP_MAX_SEG;
  int* n_seg_s = seg_len + LP_MAX_SEG;
  int* win_flag = n_seg_s + 3;  // FAST: some row left the exponent window

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int unit, piece = -1;
  if ((int)blockIdx.x < p.n_whole) {
    unit = blockIdx.x;
  } else {
    const int v = blockIdx.x - p.n_whole;
    unit = p.n_whole + v / p.split;
    piece = v % p.split;
  }
  int head, pair;
  unit_coords(p, p.unit_base + unit, head, pair);
  const int q0 = pair * (2 * AT_M);
  const bool two = q0 + AT_M < p.n_q;  // tile B holds valid rows

  if (threadIdx.x == 0) {
    plan_segments(p, piece, seg_row, seg_len, n_seg_s);
    *win_flag = 0;
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
      mbar_init(&p_full[i], 4);
      mbar_init(&p_half[i], 4);
    }
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int n_tiles = n_seg_s[1];
  const int t_first = n_seg_s[2];
  const int col0 = head * AT_D;

  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(AT_REG_CTRL));
  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      uint8_t* sq = smem + AttnSmem::Q_OFF;
      mbar_arrive_expect_tx(q_full, (two ? 2 : 1) * AT_TILE_BYTES);
      for (int t = 0; t < (two ? 2 : 1); ++t) {
        tma_load_2d(sq + t * AT_TILE_BYTES, &tmQ, q_full, col0, q0 + t * AT_M);
        tma_load_2d(sq + t * AT_TILE_BYTES + AT_HALF, &tmQ, q_full, col0 + 64, q0 + t * AT_M);
      }
      TileCursor ck, cv;
      ck.init(seg_row, seg_len, n_seg_s[0]);
      cv.init(seg_row, seg_len, n_seg_s[0]);
      ck.skip(t_first);
      cv.skip(t_first);
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
    constexpr uint32_t IDESC_S = idesc_bf16_f32(AT_M, AT_N);               // Q K^T: both K-major
    constexpr uint32_t IDESC_O = idesc_bf16_f32(AT_M, AT_D, false, true);  // P V: P in TMEM, V MN-major
    const uint32_t sq = smem_u32(smem + AttnSmem::Q_OFF);
    auto issue_s = [&](int t, int x) {  // S_x(t) = Q_x K_t^T
      const uint32_t sk = smem_u32(smem + AttnSmem::K_OFF + (t & 1) * AT_TILE_BYTES);
      const uint32_t sqx = sq + x * AT_TILE_BYTES;
#pragma unroll
      for (int kk = 0; kk < AT_D / 16; ++kk) {
        const uint32_t off = (kk >> 2) * AT_HALF + (kk & 3) * 32;
        mma_bf16_ss(tmem_base + x * AT_N, sdesc_kmajor_sw128(sqx + off), sdesc_kmajor_sw128(sk + off), IDESC_S,
                    kk != 0);
      }
    };
    auto issue_pv = [&](int t, int x, int h) {  // O_x += P_x(t)[keys 64h..] V_t[64h..]
      const uint32_t sv = smem_u32(smem + AttnSmem::V_OFF + (t & 1) * AT_TILE_BYTES);
      const uint32_t tp = tmem_base + x * AT_N;        // P_x: 64 columns of packed bf16 pairs
      const uint32_t to = tmem_base + 256 + x * AT_D;  // O_x
#pragma unroll
      for (int kk = 4 * h; kk < 4 * h + 4; ++kk)
        mma_bf16_ts(to, tp + kk * 8, sdesc_mnmajor_sw128(sv + kk * 16 * 128, AT_HALF), IDESC_O, (t | kk) != 0);
    };
    mbar_wait(q_full, 0);
    if (n_tiles > 0) {
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      if (elect_one()) {
        issue_s(0, 0);
        mma_commit(&s_full[0]);
        if (two) {
          issue_s(0, 1);
          mma_commit(&s_full[1]);
        }
        mma_commit(&k_empty[0]);
      }
      __syncwarp();
    }
    for (int j = 0; j < n_tiles; ++j) {
      const bool more = j + 1 < n_tiles;
      // tile A: P_A(j) V_j in two key halves (the first overlaps the softmax
      // of the second), then S_A(j+1)
      mbar_wait(&p_half[0], j & 1);
      mbar_wait(&v_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      if (elect_one()) issue_pv(j, 0, 0);
      __syncwarp();
      mbar_wait(&p_full[0], j & 1);
      if (more) mbar_wait(&k_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        issue_pv(j, 0, 1);
        if (more) {
          issue_s(j + 1, 0);
          mma_commit(&s_full[0]);
        }
        if (!two) {
          mma_commit(&v_empty[j & 1]);
          if (more) mma_commit(&k_empty[(j + 1) & 1]);
        }
      }
      __syncwarp();
      if (two) {
        // tile B: P_B(j) V_j, then S_B(j+1)
        mbar_wait(&p_half[1], j & 1);
        tc_fence_after();
        if (elect_one()) issue_pv(j, 1, 0);
        __syncwarp();
        mbar_wait(&p_full[1], j & 1);
        tc_fence_after();
        if (elect_one()) {
          issue_pv(j, 1, 1);
          mma_commit(&v_empty[j & 1]);
          if (more) {
            issue_s(j + 1, 1);
            mma_commit(&s_full[1]);
            mma_commit(&k_empty[(j + 1) & 1]);
          }
        }
        __syncwarp();
      }
    }
    if (elect_one()) mma_commit(o_done);
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax warpgroups
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(AT_REG_SOFTMAX));
    const int x = (warp - 4) / 4;        // Q tile: 0 = A (warps 4-7), 1 = B (warps 8-11)
    const int quarter = warp & 3;        // TMEM lane quarter accessible to this warp
    const int r = quarter * 32 + lane;   // row within the Q tile == TMEM lane
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t t_s = tmem_base + lane_base + x * AT_N;
    const uint32_t t_o = tmem_base + lane_base + 256 + x * AT_D;
    const float sc = p.scale_log2;
    float m_run = -INFINITY, l_run = 0.0f;
    TileCursor cs;
    cs.init(seg_row, seg_len, n_seg_s[0]);
    cs.skip(t_first);
    const bool active = x == 0 || two;
    for (int j = 0; j < (active ? n_tiles : 0); ++j, cs.next()) {
      const int nvalid = cs.cur_valid();
      mbar_wait(&s_full[x], j & 1);
      tc_fence_after();
      uint32_t s[128];
      tmem_ld32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
      tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
      tmem_ld32(t_s + 64, *reinterpret_cast<uint32_t(*)[32]>(&s[64]));
      tmem_ld32(t_s + 96, *reinterpret_cast<uint32_t(*)[32]>(&s[96]));
      tmem_ld_wait();
      if (nvalid < AT_N) {  // ragged segment tail (warp-uniform)
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i >= nvalid) s[i] = __float_as_uint(-INFINITY);
      }
      float alpha = 1.0f;
      bool rescale = false;
      if (!FAST || j == 0) {
      // row max as a tree: 8 independent 3-input max chains, then 8 -> 1
      float mq[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mq[k] = fmaxf(__uint_as_float(s[k]), __uint_as_float(s[k + 8]));
#pragma unroll
      for (int i = 16; i < 128; i += 16)
#pragma unroll
        for (int k = 0; k < 8; ++k) mq[k] = fmaxf(mq[k], fmaxf(__uint_as_float(s[i + k]), __uint_as_float(s[i + 8 + k])));
      const float mx = fmaxf(fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])),
                             fmaxf(fmaxf(mq[4], mq[5]), fmaxf(mq[6], mq[7])));
      const float m_tile = mx * sc;
      if (j == 0) {
        m_run = m_tile;
      } else {
        const bool need = m_tile > m_run + AT_RESCALE_THRESH;
        rescale = __any_sync(0xffffffffu, need);
        if (need) {
          alpha = ex2(m_run - m_tile);
          m_run = m_tile;
        }
      }
      }
      // p = 2^(s*scale*log2e - m), packed to bf16 pairs in key order.
      // Pairs go through the packed fp32x2 FMA pipe (FFMA2/FADD2); 3 of
      // every 8 pairs take the polynomial exp2, the rest MUFU.EX2.
      const uint64_t sc2 = f32x2(sc, sc), nm2 = f32x2(-m_run, -m_run);
      const float wa = sc * (1.0f / 192.0f), wb = (127.0f - m_run) * (1.0f / 192.0f);
      const uint64_t wa2 = f32x2(wa, wa), wb2 = f32x2(wb, wb);
      uint64_t rs2[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) rs2[k] = f32x2(0.f, 0.f);
      uint32_t* pk = s;  // packed P overwrites the consumed front of s in place
      auto exp_pairs = [&](int i0) {
#pragma unroll
        for (int i = i0; i < i0 + 64; i += 2) {
          const bool poly = ((i >> 1) & 7) >= 8 - (FAST ? LP_ATTN_POLY_WIN : LP_ATTN_POLY);
          const uint64_t sv2 = f32x2(__uint_as_float(s[i]), __uint_as_float(s[i + 1]));
          uint64_t e;
          if (FAST && poly) {
            e = ex2_poly2_win(sv2, wa2, wb2);
          } else if (poly) {
            e = ex2_poly2(ffma2(sv2, sc2, nm2));
          } else {
            const uint64_t a = ffma2(sv2, sc2, nm2);
            float a0, a1;
            unpack_f32x2(a, a0, a1);
            e = f32x2(ex2(a0), ex2(a1));
          }
          rs2[(i >> 1) & 3] = fadd2(rs2[(i >> 1) & 3], e);
          float e0, e1;
          unpack_f32x2(e, e0, e1);
          pk[i / 2] = pack_bf16(e0, e1);
        }
      };
      // keys [0, 64): P columns [0, 32); O is rescaled before P(j).V starts
      exp_pairs(0);
      tmem_st32_x(t_s + 0, &s[0]);
      if (!FAST && rescale) {
        // P(j-1).V is complete (implied by s_full(j)); O_x is idle until p_half(j)
#pragma unroll 1
        for (int c0 = 0; c0 < AT_D; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(t_o + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
          tmem_st32(t_o + c0, v);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_half[x]);
      // keys [64, 128): P columns [32, 64)
      exp_pairs(64);
      float r[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) unpack_f32x2(rs2[k], r[2 * k], r[2 * k + 1]);
      const float rsum = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      l_run = FAST ? l_run + rsum : l_run * alpha + rsum;
      tmem_st32_x(t_s + 32, &s[32]);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[x]);
    }
    if (FAST && active && __any_sync(0xffffffffu, !(l_run < 0x1p64f)) && lane == 0) atomicOr(win_flag, 1);
    // epilogue: O / l -> bf16 (whole unit) or unnormalised (O, m, l) partials
    if (active) {
    mbar_wait(o_done, 0);
    tc_fence_after();
    const int row = q0 + x * AT_M + r;
    if (piece >= 0) {
      const int64_t slot = (int64_t)(blockIdx.x - p.n_whole) * (2 * AT_M) + x * AT_M + r;
      float* po = p.part_o + slot * AT_D;
#pragma unroll 1
      for (int c0 = 0; c0 < AT_D; c0 += 32) {
        uint32_t v[32];
        if (n_tiles > 0) {
          tmem_ld32(t_o + c0, v);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0u;
        }
        float4* o = reinterpret_cast<float4*>(po + c0);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          o[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                             __uint_as_float(v[4 * q + 3]));
      }
      reinterpret_cast<float2*>(p.part_ml)[slot] = make_float2(n_tiles > 0 ? m_run : -INFINITY, l_run);
    } else {
    const float inv_l = l_run > 0.0f ? 1.0f / l_run : 0.0f;
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
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
  if (FAST && threadIdx.x == 0) p.flags[blockIdx.x] = *win_flag;
}

// ---------------------------------------------------------------------------
// Cluster-pair attention (tcgen05.mma.cta_group::2), the product kernel.
//
// A work unit (256 queries of one head[, one KV range]) runs on a CTA pair:
// each CTA owns 128 query rows (its TMEM lanes) and loads HALF of every K/V
// tile -- K: 64 of the 128 keys, all 128 dims; V: all 128 keys, 64 of the
// dims -- so each SM streams half the K/V bytes of the single-CTA kernel, and
// the leader issues M = 256 MMAs for the pair.  With one Q tile per SM the
// TMEM holds two S buffers, O and two P buffers:
//   S0 [0,128)  S1 [128,256)  O [256,384)  P0 [384,448)  P1 [448,512)
// so S(j+2) is issued as soon as the softmax has LOADED S(j) (s_free), before
// its exponentials: the tensor core runs S(j+2) while softmax(j) computes and
// PV(j) once P(j) is stored.  Nothing on the tensor pipe waits on the softmax
// latency, only on its throughput.  Two softmax warpgroups per CTA take the
// KV tiles alternately (S_b / P_b belong to warpgroup b), so the two warps
// sharing an SM sub-partition are half a tile out of phase and hide each
// other's TMEM-load and barrier latency; with the bounded-exponent offset
// (max of tile 0, handed to warpgroup 1 once) they share one offset and never
// synchronise per tile; their row sums are added at the end.
//   warp 0      TMA producer (both CTAs): Q once, the K halves (4-stage ring)
//   warp 3      TMA producer (both CTAs): the V halves (4-stage ring); both
//               count completion on the leader's barriers
//   warp 1      TMEM allocation (both); leader: issues the S = Q K^T MMAs
//   warp 2      leader: issues the O += P V MMAs
//   warps 4-7   softmax of tiles 0, 2, 4, ...    warps 8-11  tiles 1, 3, 5, ...
#ifndef LP_ATTN2_KS
#define LP_ATTN2_KS 4
#endif
constexpr int A2_KS = LP_ATTN2_KS, A2_VS = 4;  // K / V ring stages
constexpr int A2_KT = 64 * AT_D * 2;         // 16 KB: this CTA's 64 keys x 128 dims
constexpr int A2_KHALF = 64 * 64 * 2;        // 8 KB: one 64-dim SW128 block of it
constexpr int A2_VT = AT_N * 64 * 2;         // 16 KB: 128 keys x this CTA's 64 dims

struct Attn2Smem {
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + AT_TILE_BYTES;
  static constexpr int V_OFF = K_OFF + A2_KS * A2_KT;
  static constexpr int BAR_OFF = V_OFF + A2_VS * A2_VT;
  static constexpr int XCH_OFF = BAR_OFF + 512;
  static constexpr int SEG_OFF = XCH_OFF + 2 * AT_M * 4;
  static constexpr int TOTAL = SEG_OFF + 2 * LP_MAX_SEG * 4 + 16 + 1024;
};

__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(AT_THREADS, 1)
    attn_tc2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Attn2Smem::BAR_OFF);
  uint64_t* q_full = bars;               // leader's copy used
  uint64_t* k_full = bars + 1;           // [KS] leader
  uint64_t* k_empty = k_full + A2_KS;    // [KS] both (multicast commit)
  uint64_t* v_full = k_empty + A2_KS;    // [VS] leader
  uint64_t* v_empty = v_full + A2_VS;    // [VS] both
  uint64_t* s_full = v_empty + A2_VS;    // [2] both
  uint64_t* s_free = s_full + 2;         // [2] leader: warpgroup b's 4 warps x 2 CTAs loaded S_b
  uint64_t* p_lo = s_free + 2;           // [2] leader: P(j) of buffer j&1 stored (4 warps x 2 CTAs)
  uint64_t* pv_done = p_lo + 2;          // [2] both: P buffer consumed
  uint64_t* o_done = pv_done + 2;        // both
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);
  float* xch = reinterpret_cast<float*>(smem + Attn2Smem::XCH_OFF);  // [2][128] per-row exchange
  int* seg_row = reinterpret_cast<int*>(smem + Attn2Smem::SEG_OFF);
  int* seg_len = seg_row + LP_MAX_SEG;
  int* n_seg_s = seg_len + LP_MAX_SEG;
  int* win_flag = n_seg_s + 3;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int c = blockIdx.x >> 1;
  int unit, piece = -1;
  if (c < p.n_whole) {
    unit = c;
  } else {
    const int v = c - p.n_whole;
    unit = p.n_whole + v / p.split;
    piece = v % p.split;
  }
  int head, pair;
  unit_coords(p, p.unit_base + unit, head, pair);
  const int q0 = pair * (2 * AT_M) + (int)rank * AT_M;  // this CTA's first query row

  if (threadIdx.x == 0) {
    plan_segments(p, piece, seg_row, seg_len, n_seg_s);
    *win_flag = 0;
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < A2_KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < A2_VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
      mbar_init(&p_lo[i], 8);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive / TMA
  if (warp == 1) tmem_alloc_2cta(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int n_tiles = n_seg_s[1];
  const int t_first = n_seg_s[2];
  const int col0 = head * AT_D;

  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(AT_REG_CTRL));
  if (warp == 0 || warp == 3) {
    // ------------------------------------------------ TMA producers (both CTAs):
    // warp 0 loads Q and the K ring, warp 3 the V ring, so a K load never
    // queues behind a V stage that PV has not released yet (S(t+2) needs
    // K(t+2) early; V(t) is needed only after softmax(t))
    if (elect_one()) {
      const uint64_t pol = l2_policy_evict_last();
      TileCursor cur;
      cur.init(seg_row, seg_len, n_seg_s[0]);
      cur.skip(t_first);
      if (warp == 0) {
        uint8_t* sq = smem + Attn2Smem::Q_OFF;
        if (rank == 0) mbar_arrive_expect_tx(q_full, 2 * AT_TILE_BYTES);
        tma_load_2d_2sm(sq, &tmQ, q_full, col0, q0, pol);
        tma_load_2d_2sm(sq + AT_HALF, &tmQ, q_full, col0 + 64, q0, pol);
        for (int t = 0; t < n_tiles; ++t, cur.next()) {
          const int ks = t % A2_KS;
          mbar_wait(&k_empty[ks], ((t / A2_KS) & 1) ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&k_full[ks], 2 * A2_KT);
          uint8_t* sk = smem + Attn2Smem::K_OFF + ks * A2_KT;
          const int krow = cur.cur_row() + 64 * (int)rank;  // this CTA's 64 keys of the tile
          tma_load_2d_2sm(sk, &tmK, &k_full[ks], col0, krow, pol);
          tma_load_2d_2sm(sk + A2_KHALF, &tmK, &k_full[ks], col0 + 64, krow, pol);
        }
      } else {
        for (int t = 0; t < n_tiles; ++t, cur.next()) {
          const int vs = t % A2_VS;
          mbar_wait(&v_empty[vs], ((t / A2_VS) & 1) ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&v_full[vs], 2 * A2_VT);
          tma_load_2d_2sm(smem + Attn2Smem::V_OFF + vs * A2_VT, &tmV, &v_full[vs], col0 + 64 * (int)rank,
                          cur.cur_row(), pol);
        }
      }
    }
  } else if ((warp == 1 || warp == 2) && rank == 0) {
    // ------------------------------------------------ MMA issue (leader), two
    // independent in-order streams so neither waits behind the other's
    // dependency: warp 1 issues S(t) as soon as S_{t&1} is free (softmax(t-2)
    // has loaded it) and K_t has landed; warp 2 issues PV(j) as soon as P(j)
    // is stored.  O is only written by warp 2's stream (in order); S and P
    // live in separate TMEM columns.
    constexpr uint32_t IDESC_S = idesc_bf16_f32(2 * AT_M, AT_N);               // Q K^T, both K-major
    constexpr uint32_t IDESC_O = idesc_bf16_f32(2 * AT_M, AT_D, false, true);  // P V: P in TMEM, V MN-major
    if (warp == 1) {
      const uint32_t sq = smem_u32(smem + Attn2Smem::Q_OFF);
      mbar_wait(q_full, 0);
      for (int t = 0; t < n_tiles; ++t) {
        if (t >= 2) mbar_wait(&s_free[t & 1], ((t - 2) >> 1) & 1);
        mbar_wait(&k_full[t % A2_KS], (t / A2_KS) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sk = smem_u32(smem + Attn2Smem::K_OFF + (t % A2_KS) * A2_KT);
#pragma unroll
          for (int kk = 0; kk < AT_D / 16; ++kk)
            mma_bf16_ss_2cta(tmem_base + (t & 1) * AT_N,
                             sdesc_kmajor_sw128(sq + (kk >> 2) * AT_HALF + (kk & 3) * 32),
                             sdesc_kmajor_sw128(sk + (kk >> 2) * A2_KHALF + (kk & 3) * 32), IDESC_S, kk != 0);
          mma_commit_2cta_mc(&s_full[t & 1]);
          mma_commit_2cta_mc(&k_empty[t % A2_KS]);
        }
        __syncwarp();
      }
    } else {
      for (int j = 0; j < n_tiles; ++j) {
        const int b = j & 1;
        mbar_wait(&v_full[j % A2_VS], (j / A2_VS) & 1);
        mbar_wait(&p_lo[b], (j >> 1) & 1);  // P(j) stored by warpgroup b (both CTAs)
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sv = smem_u32(smem + Attn2Smem::V_OFF + (j % A2_VS) * A2_VT);
          const uint32_t tp = tmem_base + 384 + b * 64;
#pragma unroll
          for (int kk = 0; kk < AT_N / 16; ++kk)
            mma_bf16_ts_2cta(tmem_base + 256, tp + kk * 8, sdesc_mnmajor_sw128(sv + kk * 16 * 128, A2_VT), IDESC_O,
                             (j | kk) != 0);
          mma_commit_2cta_mc(&pv_done[b]);
          mma_commit_2cta_mc(&v_empty[j % A2_VS]);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit_2cta_mc(o_done);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax (both CTAs)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(AT_REG_SOFTMAX));
    const int x = (warp - 4) / 4;        // this warpgroup's tiles: j = x, x + 2, ...
    const int w = x;                     // (epilogue: output column half)
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;   // row within this CTA's 128 == TMEM lane
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t t_s = tmem_base + lane_base + x * AT_N;
    const uint32_t t_p = tmem_base + lane_base + 384 + x * 64;
    const uint32_t t_o = tmem_base + lane_base + 256;
    const float sc = p.scale_log2;
    float m_run = 0.0f, l_run = 0.0f;
    uint64_t wa2 = 0, wb2 = 0, sc2 = f32x2(sc, sc), nm2 = 0;
    auto set_offset = [&](float m) {
      m_run = m;
      const float wa = sc * (1.0f / 192.0f), wb = (127.0f - m_run) * (1.0f / 192.0f);
      wa2 = f32x2(wa, wa);
      wb2 = f32x2(wb, wb);
      nm2 = f32x2(-m_run, -m_run);
    };
    // the shared exponent offset (max of tile 0) reaches warpgroup 1 once
    if (x == 1 && n_tiles > 0) {
      softmax_bar();
      set_offset(xch[r]);
    }
    TileCursor cs;
    cs.init(seg_row, seg_len, n_seg_s[0]);
    cs.skip(t_first + x);
    for (int j = x; j < n_tiles; j += 2, cs.next(), cs.next()) {
      const uint32_t ph = (j >> 1) & 1;
      const int nvalid = cs.cur_valid();
      mbar_wait(&s_full[x], ph);
      tc_fence_after();
      uint32_t s[128];
      tmem_ld32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
      tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
      tmem_ld32(t_s + 64, *reinterpret_cast<uint32_t(*)[32]>(&s[64]));
      tmem_ld32(t_s + 96, *reinterpret_cast<uint32_t(*)[32]>(&s[96]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&s_free[x], 0);  // S_x may take S(j+2)
      if (nvalid < AT_N) {  // ragged segment tail (warp-uniform)
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i >= nvalid) s[i] = __float_as_uint(-INFINITY);
      }
      if (j == 0) {  // tile 0: the row's exponent offset for the whole unit
        float mq[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mq[k] = fmaxf(__uint_as_float(s[k]), __uint_as_float(s[k + 8]));
#pragma unroll
        for (int i = 16; i < 128; i += 16)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            mq[k] = fmaxf(mq[k], fmaxf(__uint_as_float(s[i + k]), __uint_as_float(s[i + 8 + k])));
        const float mx = fmaxf(fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])),
                               fmaxf(fmaxf(mq[4], mq[5]), fmaxf(mq[6], mq[7]))) * sc;
        xch[r] = mx;
        softmax_bar();
        set_offset(mx);
      }
      uint64_t rs2[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) rs2[k] = f32x2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 128; i += 2) {
        const bool poly = ((i >> 1) & 7) >= 8 - LP_ATTN_POLY_WIN;
        const uint64_t sv2 = f32x2(__uint_as_float(s[i]), __uint_as_float(s[i + 1]));
        uint64_t e;
        if (poly) {
          e = ex2_poly2_win(sv2, wa2, wb2);
        } else {
          const uint64_t a = ffma2(sv2, sc2, nm2);
          float a0, a1;
          unpack_f32x2(a, a0, a1);
          e = f32x2(ex2(a0), ex2(a1));
        }
        rs2[(i >> 1) & 3] = fadd2(rs2[(i >> 1) & 3], e);
        float e0, e1;
        unpack_f32x2(e, e0, e1);
        s[i / 2] = pack_bf16(e0, e1);
      }
      if (j >= 2) {  // P_x of tile j-2 consumed (the exps above did not wait for it)
        mbar_wait(&pv_done[x], ph ^ 1);
        tc_fence_after();
      }
      tmem_st32_x(t_p, &s[0]);
      tmem_st32_x(t_p + 32, &s[32]);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&p_lo[x], 0);
      float rr[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) unpack_f32x2(rs2[k], rr[2 * k], rr[2 * k + 1]);
      l_run += ((rr[0] + rr[1]) + (rr[2] + rr[3])) + ((rr[4] + rr[5]) + (rr[6] + rr[7]));
    }
    // epilogue: the row sums of both warpgroups' tiles, then O / l (or partials);
    // each warpgroup stores 64 of the 128 output columns of its rows
    mbar_wait(o_done, 0);
    tc_fence_after();
    softmax_bar();  // every read of xch (first-tile max) is done
    xch[w * AT_M + r] = l_run;
    softmax_bar();
    const float l_tot = xch[r] + xch[AT_M + r];
    const int row = q0 + r;
    const bool valid = row < p.n_q;
    if (w == 0 && __any_sync(0xffffffffu, valid && !(l_tot < 0x1p64f)) && lane == 0) atomicOr(win_flag, 1);
    if (piece >= 0) {
      const int64_t slot = (int64_t)(c - p.n_whole) * (2 * AT_M) + (int)rank * AT_M + r;
      float* po = p.part_o + slot * AT_D;
#pragma unroll 1
      for (int c0 = 64 * w; c0 < 64 * w + 64; c0 += 32) {
        uint32_t v[32];
        if (n_tiles > 0) {
          tmem_ld32(t_o + c0, v);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0u;
        }
        float4* o = reinterpret_cast<float4*>(po + c0);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          o[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                             __uint_as_float(v[4 * q + 3]));
      }
      if (w == 0) reinterpret_cast<float2*>(p.part_ml)[slot] = make_float2(n_tiles > 0 ? m_run : -INFINITY, l_tot);
    } else {
      const float inv_l = l_tot > 0.0f ? 1.0f / l_tot : 0.0f;
#pragma unroll 1
      for (int c0 = 64 * w; c0 < 64 * w + 64; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(t_o + c0, v);
        tmem_ld_wait();
        if (valid) {
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
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's smem / TMEM are read by the leader's MMAs until o_done
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2cta(tmem_base, 512);
  }
  if (threadIdx.x == 0) p.flags[blockIdx.x] = *win_flag;
}

// Persistent form of the cluster-pair kernel: one cluster per SM pair walks
// the work items c, c + G, c + 2G, ... (G = clusters), so the next item's Q,
// K/V loads and first S MMAs run while the softmax warps finish the previous
// item's epilogue, and there is no per-item CTA launch, barrier init, TMEM
// allocation or pipeline fill/drain.  Every ring runs on counters that
// continue across items (K/V stages, the S/P buffer of global tile g = g & 1
// and its softmax warpgroup), Q is double-buffered, and the first PV of an
// item waits for the previous item's epilogue to have read O (o_free).
struct Attn2pSmem {
  static constexpr int Q_OFF = 0;                                  // 2 x 32 KB
  static constexpr int K_OFF = Q_OFF + 2 * AT_TILE_BYTES;
  static constexpr int V_OFF = K_OFF + A2_KS * A2_KT;
  static constexpr int BAR_OFF = V_OFF + A2_VS * A2_VT;
  static constexpr int XM_OFF = BAR_OFF + 512;                     // [128] first-tile max
  static constexpr int XL_OFF = XM_OFF + AT_M * 4;                 // [2][128] row sums
  static constexpr int SEG_OFF = XL_OFF + 2 * AT_M * 4;
  static constexpr int TOTAL = SEG_OFF + 2 * LP_MAX_SEG * 4 + 16 + 1024;
};

// sched_empty arrivals per item: leader warps 1, 2, 3 + 8 softmax warps;
// partner warps 0, 3 + 8 softmax warps
constexpr int SCHED_CONSUMERS = 11 + 10;

struct Item {  // one work unit or KV piece, as every role derives it
  int head, pair, piece, t_first, n_tiles;
};
__device__ __forceinline__ Item item_of(const AttnParams& p, int it, int nt_total) {
  Item r;
  int unit;
  r.piece = -1;
  if (it < p.n_whole) {
    unit = it;
  } else {
    const int v = it - p.n_whole;
    unit = p.n_whole + v / p.split;
    r.piece = v % p.split;
  }
  unit_coords(p, p.unit_base + unit, r.head, r.pair);
  const int t0 = r.piece < 0 ? 0 : (int)((int64_t)nt_total * r.piece / p.split);
  const int t1 = r.piece < 0 ? nt_total : (int)((int64_t)nt_total * (r.piece + 1) / p.split);
  r.t_first = t0;
  r.n_tiles = t1 - t0;
  return r;
}

// Head-split queues: this SM's queue first, then steal from the other one
// (out of line: it runs once per item on the leader's producer thread and
// must not add to the 56-register control warps' pressure).
__device__ __noinline__ int claim_head_split(int* sched, int smid_split) {
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const int q0 = (int)smid < smid_split ? 0 : 1;
  for (int t = 0; t < 2; ++t) {
    const int q = t ? 1 - q0 : q0;
    int j = atomicAdd(sched + q, 1);
    if (j >= sched[2 + q]) continue;
    const int* run = sched + 8 + 16 * q;
    for (int r = 0; r < sched[4 + q]; ++r) {
      if (j < run[2 * r + 1]) return run[2 * r] + j;
      j -= run[2 * r + 1];
    }
  }
  return -1;
}

__global__ void sched_init_kernel(int* sched, SchedTable t) {
  if (threadIdx.x < 40) sched[threadIdx.x] = t.v[threadIdx.x];
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(AT_THREADS, 1)
    attn_tc2p_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const AttnParams p, int n_items) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Attn2pSmem::BAR_OFF);
  uint64_t* q_full = bars;               // [2] leader
  uint64_t* q_empty = q_full + 2;        // [2] both (multicast commit after an item's last S)
  uint64_t* k_full = q_empty + 2;        // [KS] leader
  uint64_t* k_empty = k_full + A2_KS;    // [KS] both
  uint64_t* v_full = k_empty + A2_KS;    // [VS] leader
  uint64_t* v_empty = v_full + A2_VS;    // [VS] both
  uint64_t* s_full = v_empty + A2_VS;    // [2] both
  uint64_t* s_free = s_full + 2;         // [2] leader: 4 warps x 2 CTAs
  uint64_t* p_full = s_free + 2;         // [2] leader: 4 warps x 2 CTAs
  uint64_t* pv_done = p_full + 2;        // [2] both
  uint64_t* o_done = pv_done + 2;        // both: an item's last PV complete
  uint64_t* o_free = o_done + 1;         // leader: the epilogue read O (8 warps x 2 CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 1);
  int* win_flag = reinterpret_cast<int*>(tmem_slot + 1);
  // dynamic item queue (p.sched): a 4-slot ring of item indices per CTA,
  // filled by the leader's Q/K producer thread (one atomicAdd per item) and
  // released by every consumer role of both CTAs on the leader's sched_empty
  uint64_t* sched_full = reinterpret_cast<uint64_t*>(smem + Attn2pSmem::BAR_OFF + 384);  // [4] both
  uint64_t* sched_empty = sched_full + 4;                                                  // [4] leader
  int* sched_item = reinterpret_cast<int*>(sched_empty + 4);                               // [4] both
  float* xm = reinterpret_cast<float*>(smem + Attn2pSmem::XM_OFF);
  float* xl = reinterpret_cast<float*>(smem + Attn2pSmem::XL_OFF);
  int* seg_row = reinterpret_cast<int*>(smem + Attn2pSmem::SEG_OFF);
  int* seg_len = seg_row + LP_MAX_SEG;
  int* n_seg_s = seg_len + LP_MAX_SEG;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int c = blockIdx.x >> 1, G = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    plan_segments(p, -1, seg_row, seg_len, n_seg_s);  // the whole range; items take slices of it
    *win_flag = 0;
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
      mbar_init(&p_full[i], 8);
      mbar_init(&pv_done[i], 1);
    }
    for (int i = 0; i < A2_KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < A2_VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    mbar_init(o_done, 1);
    mbar_init(o_free, 16);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&sched_full[i], 1);
      mbar_init(&sched_empty[i], SCHED_CONSUMERS);
    }
    fence_barrier_init();
  }
  cluster_sync_all();
  if (warp == 1) tmem_alloc_2cta(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nt_total = n_seg_s[1];
  const bool dyn = p.sched != nullptr;
  // the cluster's k-th item: static round robin, or from the queue (consumer
  // side; `single` = a one-thread role, else the whole warp reads the slot)
  auto take_item = [&](int k, bool single) -> int {
    if (!dyn) {
      const int it = c + k * G;
      return it < n_items ? it : -1;
    }
    mbar_wait(&sched_full[k & 3], (k >> 2) & 1);
    if (rank) fence_acquire_cluster();
    const int it = *reinterpret_cast<volatile int*>(&sched_item[k & 3]);
    if (it >= 0) {  // the slot is released (the final -1 slot is never reused)
      if (!single) __syncwarp();
      if (single || lane == 0) {
        if (rank) mbar_arrive_remote(&sched_empty[k & 3], 0);
        else mbar_arrive(&sched_empty[k & 3]);
      }
    }
    return it;
  };
  // producer side (leader's Q/K thread): claim the next item, publish it to both CTAs
  auto claim_item = [&](int k) -> int {
    if (!dyn) return take_item(k, true);
    if (k >= 4) mbar_wait(&sched_empty[k & 3], ((k >> 2) - 1) & 1);
    int it;
    if (p.hs_smid > 0) {
      it = claim_head_split(p.sched, p.hs_smid);
    } else {
      it = atomicAdd(p.sched, 1);
      if (it >= n_items) it = -1;
    }
    sched_item[k & 3] = it;
    st_shared_remote_s32(&sched_item[k & 3], 1, it);
    mbar_arrive(&sched_full[k & 3]);
    mbar_arrive_remote_release(&sched_full[k & 3], 1);
    return it;
  };

  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(AT_REG_CTRL));
  if (warp == 0 || warp == 3) {
    // ------------------------------------------------ TMA producers (both CTAs)
    if (elect_one()) {
      const uint64_t pol = (p.l2pol & 2) ? l2_policy_evict_normal() : l2_policy_evict_last();
      const uint64_t pol_q = (p.l2pol & 1) ? l2_policy_evict_first() : pol;
      uint32_t g = 0;  // global K (warp 0) or V (warp 3) tile counter
      for (int k = 0;; ++k) {  // k: item count of this cluster
        const int it = (warp == 0 && rank == 0) ? claim_item(k) : take_item(k, true);
        if (it < 0) break;
        const Item im = item_of(p, it, nt_total);
        const int col0 = im.head * AT_D;
        TileCursor cur;
        cur.init(seg_row, seg_len, n_seg_s[0]);
        cur.skip(im.t_first);
        if (warp == 0) {
          const int qb = k & 1;
          mbar_wait(&q_empty[qb], ((k >> 1) & 1) ^ 1);
          uint8_t* sq = smem + Attn2pSmem::Q_OFF + qb * AT_TILE_BYTES;
          const int q0 = im.pair * (2 * AT_M) + (int)rank * AT_M;
          if (rank == 0) mbar_arrive_expect_tx(&q_full[qb], 2 * AT_TILE_BYTES);
          tma_load_2d_2sm(sq, &tmQ, &q_full[qb], col0, q0, pol_q);
          tma_load_2d_2sm(sq + AT_HALF, &tmQ, &q_full[qb], col0 + 64, q0, pol_q);
          for (int t = 0; t < im.n_tiles; ++t, ++g, cur.next()) {
            const int ks = g % A2_KS;
            mbar_wait(&k_empty[ks], ((g / A2_KS) & 1) ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&k_full[ks], 2 * A2_KT);
            uint8_t* sk = smem + Attn2pSmem::K_OFF + ks * A2_KT;
            const int krow = cur.cur_row() + 64 * (int)rank;
            tma_load_2d_2sm(sk, &tmK, &k_full[ks], col0, krow, pol);
            tma_load_2d_2sm(sk + A2_KHALF, &tmK, &k_full[ks], col0 + 64, krow, pol);
          }
        } else {
          for (int t = 0; t < im.n_tiles; ++t, ++g, cur.next()) {
            const int vs = g % A2_VS;
            mbar_wait(&v_empty[vs], ((g / A2_VS) & 1) ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&v_full[vs], 2 * A2_VT);
            tma_load_2d_2sm(smem + Attn2pSmem::V_OFF + vs * A2_VT, &tmV, &v_full[vs], col0 + 64 * (int)rank,
                            cur.cur_row(), pol);
          }
        }
      }
    }
  } else if ((warp == 1 || warp == 2) && rank == 0) {
    // ------------------------------------------------ MMA issue (leader): S (warp 1), PV (warp 2)
    constexpr uint32_t IDESC_S = idesc_bf16_f32(2 * AT_M, AT_N);
    constexpr uint32_t IDESC_O = idesc_bf16_f32(2 * AT_M, AT_D, false, true);
    uint32_t g = 0;
    for (int k = 0;; ++k) {
      const int it = take_item(k, false);
      if (it < 0) break;
      const Item im = item_of(p, it, nt_total);
      if (warp == 1) {
        const int qb = k & 1;
        const uint32_t sq = smem_u32(smem + Attn2pSmem::Q_OFF + qb * AT_TILE_BYTES);
        mbar_wait(&q_full[qb], (k >> 1) & 1);
        for (int t = 0; t < im.n_tiles; ++t, ++g) {
          if (g >= 2) mbar_wait(&s_free[g & 1], ((g - 2) >> 1) & 1);
          mbar_wait(&k_full[g % A2_KS], (g / A2_KS) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sk = smem_u32(smem + Attn2pSmem::K_OFF + (g % A2_KS) * A2_KT);
#pragma unroll
            for (int kk = 0; kk < AT_D / 16; ++kk)
              mma_bf16_ss_2cta(tmem_base + (g & 1) * AT_N,
                               sdesc_kmajor_sw128(sq + (kk >> 2) * AT_HALF + (kk & 3) * 32),
                               sdesc_kmajor_sw128(sk + (kk >> 2) * A2_KHALF + (kk & 3) * 32), IDESC_S, kk != 0);
            mma_commit_2cta_mc(&s_full[g & 1]);
            mma_commit_2cta_mc(&k_empty[g % A2_KS]);
            if (t == im.n_tiles - 1) mma_commit_2cta_mc(&q_empty[qb]);
          }
          __syncwarp();
        }
        if (im.n_tiles == 0 && elect_one()) mma_commit_2cta_mc(&q_empty[qb]);
        __syncwarp();
      } else {
        for (int t = 0; t < im.n_tiles; ++t, ++g) {
          const int b = g & 1;
          mbar_wait(&v_full[g % A2_VS], (g / A2_VS) & 1);
          mbar_wait(&p_full[b], (g >> 1) & 1);
          if (t == 0 && k >= 1) mbar_wait(o_free, (k - 1) & 1);  // the previous item's epilogue read O
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sv = smem_u32(smem + Attn2pSmem::V_OFF + (g % A2_VS) * A2_VT);
            const uint32_t tp = tmem_base + 384 + b * 64;
#pragma unroll
            for (int kk = 0; kk < AT_N / 16; ++kk)
              mma_bf16_ts_2cta(tmem_base + 256, tp + kk * 8, sdesc_mnmajor_sw128(sv + kk * 16 * 128, A2_VT),
                               IDESC_O, (t | kk) != 0);
            mma_commit_2cta_mc(&pv_done[b]);
            mma_commit_2cta_mc(&v_empty[g % A2_VS]);
          }
          __syncwarp();
        }
        if (im.n_tiles == 0 && k >= 1) mbar_wait(o_free, (k - 1) & 1);
        if (elect_one()) mma_commit_2cta_mc(o_done);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax + epilogue (both CTAs)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(AT_REG_SOFTMAX));
    const int x = (warp - 4) / 4;  // handles global tiles g with g & 1 == x
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t t_s = tmem_base + lane_base + x * AT_N;
    const uint32_t t_p = tmem_base + lane_base + 384 + x * 64;
    const uint32_t t_o = tmem_base + lane_base + 256;
    const float sc = p.scale_log2;
    const uint64_t sc2 = f32x2(sc, sc);
    uint32_t g = 0;
    for (int k = 0;; ++k) {
      const int it = take_item(k, false);
      if (it < 0) break;
      const Item im = item_of(p, it, nt_total);
      const int g0 = (int)g;
      float m_run = 0.0f, l_run = 0.0f;
      uint64_t wa2 = 0, wb2 = 0, nm2 = 0;
      auto set_offset = [&](float m) {
        m_run = m;
        const float wa = sc * (1.0f / 192.0f), wb = (127.0f - m_run) * (1.0f / 192.0f);
        wa2 = f32x2(wa, wa);
        wb2 = f32x2(wb, wb);
        nm2 = f32x2(-m_run, -m_run);
      };
      // this warpgroup's first tile of the item: the item's tile 0 (it computes
      // the shared offset) or tile 1 (it waits for the offset)
      const int first = ((g0 & 1) == x) ? 0 : 1;
      if (first == 1 && im.n_tiles > 0) {
        softmax_bar();
        set_offset(xm[r]);
      }
      TileCursor cs;
      cs.init(seg_row, seg_len, n_seg_s[0]);
      cs.skip(im.t_first + first);
      for (int t = first; t < im.n_tiles; t += 2, cs.next(), cs.next()) {
        const uint32_t gt = (uint32_t)g0 + t;
        const uint32_t ph = (gt >> 1) & 1;
        const int nvalid = cs.cur_valid();
        mbar_wait(&s_full[x], ph);
        tc_fence_after();
        uint32_t s[128];
        tmem_ld32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
        tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
        tmem_ld32(t_s + 64, *reinterpret_cast<uint32_t(*)[32]>(&s[64]));
        tmem_ld32(t_s + 96, *reinterpret_cast<uint32_t(*)[32]>(&s[96]));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&s_free[x], 0);
        if (nvalid < AT_N) {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i >= nvalid) s[i] = __float_as_uint(-INFINITY);
        }
        if (t == 0) {
          float mq[8];
#pragma unroll
          for (int kq = 0; kq < 8; ++kq) mq[kq] = fmaxf(__uint_as_float(s[kq]), __uint_as_float(s[kq + 8]));
#pragma unroll
          for (int i = 16; i < 128; i += 16)
#pragma unroll
            for (int kq = 0; kq < 8; ++kq)
              mq[kq] = fmaxf(mq[kq], fmaxf(__uint_as_float(s[i + kq]), __uint_as_float(s[i + 8 + kq])));
          const float mx = fmaxf(fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])),
                                 fmaxf(fmaxf(mq[4], mq[5]), fmaxf(mq[6], mq[7]))) * sc;
          xm[r] = mx;
          softmax_bar();
          set_offset(mx);
        }
        uint64_t rs2[4];
#pragma unroll
        for (int kq = 0; kq < 4; ++kq) rs2[kq] = f32x2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 128; i += 2) {
          const bool poly = ((i >> 1) & 7) >= 8 - LP_ATTN_POLY_WIN;
          const uint64_t sv2 = f32x2(__uint_as_float(s[i]), __uint_as_float(s[i + 1]));
          uint64_t e;
          if (poly) {
            e = ex2_poly2_win(sv2, wa2, wb2);
          } else {
            const uint64_t a = ffma2(sv2, sc2, nm2);
            float a0, a1;
            unpack_f32x2(a, a0, a1);
            e = f32x2(ex2(a0), ex2(a1));
          }
          rs2[(i >> 1) & 3] = fadd2(rs2[(i >> 1) & 3], e);
          float e0, e1;
          unpack_f32x2(e, e0, e1);
          s[i / 2] = pack_bf16(e0, e1);
        }
        if (gt >= 2) {  // P_x of global tile gt-2 consumed
          mbar_wait(&pv_done[x], ph ^ 1);
          tc_fence_after();
        }
        tmem_st32_x(t_p, &s[0]);
        tmem_st32_x(t_p + 32, &s[32]);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&p_full[x], 0);
        float rr[8];
#pragma unroll
        for (int kq = 0; kq < 4; ++kq) unpack_f32x2(rs2[kq], rr[2 * kq], rr[2 * kq + 1]);
        l_run += ((rr[0] + rr[1]) + (rr[2] + rr[3])) + ((rr[4] + rr[5]) + (rr[6] + rr[7]));
      }
      g += (uint32_t)im.n_tiles;
      // epilogue of the item: row sums of both warpgroups, then O / l (or partials)
      xl[x * AT_M + r] = l_run;
      softmax_bar();
      const float l_tot = xl[r] + xl[AT_M + r];
      const int q0 = im.pair * (2 * AT_M) + (int)rank * AT_M;
      const int row = q0 + r;
      const bool valid = row < p.n_q;
      if (x == 0 && __any_sync(0xffffffffu, valid && !(l_tot < 0x1p64f)) && lane == 0) atomicOr(win_flag, 1);
      mbar_wait(o_done, k & 1);
      tc_fence_after();
      const int col0 = im.head * AT_D;
      uint32_t v0[32], v1[32];
      tmem_ld32(t_o + 64 * x, v0);
      tmem_ld32(t_o + 64 * x + 32, v1);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(o_free, 0);  // O may take the next item's PV
      if (im.piece >= 0) {
        const int64_t slot = (int64_t)(it - p.n_whole) * (2 * AT_M) + (int)rank * AT_M + r;
        float4* o = reinterpret_cast<float4*>(p.part_o + slot * AT_D + 64 * x);
        const bool any = im.n_tiles > 0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          o[q] = any ? make_float4(__uint_as_float(v0[4 * q]), __uint_as_float(v0[4 * q + 1]),
                                   __uint_as_float(v0[4 * q + 2]), __uint_as_float(v0[4 * q + 3]))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          o[8 + q] = any ? make_float4(__uint_as_float(v1[4 * q]), __uint_as_float(v1[4 * q + 1]),
                                       __uint_as_float(v1[4 * q + 2]), __uint_as_float(v1[4 * q + 3]))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        if (x == 0) reinterpret_cast<float2*>(p.part_ml)[slot] = make_float2(any ? m_run : -INFINITY, l_tot);
      } else if (valid) {
        const float inv_l = l_tot > 0.0f ? 1.0f / l_tot : 0.0f;
        uint4* o = reinterpret_cast<uint4*>(p.out + (int64_t)row * p.ldo + col0 + 64 * x);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          o[q] = make_uint4(pack_bf16(__uint_as_float(v0[8 * q]) * inv_l, __uint_as_float(v0[8 * q + 1]) * inv_l),
                            pack_bf16(__uint_as_float(v0[8 * q + 2]) * inv_l, __uint_as_float(v0[8 * q + 3]) * inv_l),
                            pack_bf16(__uint_as_float(v0[8 * q + 4]) * inv_l, __uint_as_float(v0[8 * q + 5]) * inv_l),
                            pack_bf16(__uint_as_float(v0[8 * q + 6]) * inv_l, __uint_as_float(v0[8 * q + 7]) * inv_l));
#pragma unroll
        for (int q = 0; q < 4; ++q)
          o[4 + q] =
              make_uint4(pack_bf16(__uint_as_float(v1[8 * q]) * inv_l, __uint_as_float(v1[8 * q + 1]) * inv_l),
                         pack_bf16(__uint_as_float(v1[8 * q + 2]) * inv_l, __uint_as_float(v1[8 * q + 3]) * inv_l),
                         pack_bf16(__uint_as_float(v1[8 * q + 4]) * inv_l, __uint_as_float(v1[8 * q + 5]) * inv_l),
                         pack_bf16(__uint_as_float(v1[8 * q + 6]) * inv_l, __uint_as_float(v1[8 * q + 7]) * inv_l));
      }
      softmax_bar();  // win_flag complete; xl free for the next item
      if (warp == 4 && lane == 0) {
        p.flags[2 * it + rank] = *win_flag;
        *win_flag = 0;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2cta(tmem_base, 512);
  }
}

// Merge the KV-range partials of the split units in piece order:
// O = sum_s 2^(m_s - m) O_s / sum_s 2^(m_s - m) l_s (one warp per query row).
__global__ void __launch_bounds__(256) attn_combine_kernel(const AttnParams p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int k = warp / (2 * AT_M);  // split unit
  const int r = warp % (2 * AT_M);  // row within the unit
  const int n_units = p.pairs * p.n_heads;
  if (p.n_whole + k >= n_units) return;
  int head, pair;
  unit_coords(p, p.unit_base + p.n_whole + k, head, pair);
  const int row = pair * (2 * AT_M) + r;
  if (row >= p.n_q) return;
  const float2* ml = reinterpret_cast<const float2*>(p.part_ml);
  const int64_t base = (int64_t)k * p.split * (2 * AT_M) + r;
  float m = -INFINITY;
  for (int s = 0; s < p.split; ++s) m = fmaxf(m, ml[base + (int64_t)s * (2 * AT_M)].x);
  float l = 0.f;
  float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s = 0; s < p.split; ++s) {
    const int64_t slot = base + (int64_t)s * (2 * AT_M);
    const float2 v = ml[slot];
    const float w = v.x == -INFINITY ? 0.f : exp2f(v.x - m);
    l = fmaf(w, v.y, l);
    const float4 x = reinterpret_cast<const float4*>(p.part_o + slot * AT_D)[lane];
    o.x = fmaf(w, x.x, o.x);
    o.y = fmaf(w, x.y, o.y);
    o.z = fmaf(w, x.z, o.z);
    o.w = fmaf(w, x.w, o.w);
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
  uint2* dst = reinterpret_cast<uint2*>(p.out + (int64_t)row * p.ldo + head * AT_D + lane * 4);
  *dst = make_uint2(pack_bf16(o.x * inv, o.y * inv), pack_bf16(o.z * inv, o.w * inv));
}

int preload_attn_tc() {
  cudaFuncAttributes a;
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, attn_tc_kernel<true>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, attn_tc_kernel<false>));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, attn_tc2_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, attn_tc2p_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, attn_combine_kernel));
  LP_CUDA_TRY(cudaFuncGetAttributes(&a, sched_init_kernel));
  return LP_OK;
}

// Work decomposition for (n_q, n_heads) on `sms` SMs.  Units are 256-query
// pairs of one head; a pair whose second tile is empty costs ~0.6.  The last
// n_split units (all ragged ones first in line) are cut into `split`
// KV-range pieces.  (n_split, split) minimise the makespan of in-order
// dispatch to the earliest-free SM (the hardware block scheduler), with a
// small fixed cost per CTA and for the combine pass.
struct AttnPlan {
  int pairs = 0, reg_pairs = 0, n_units = 0, n_whole = 0, split = 1;
  int64_t pieces() const { return (int64_t)(n_units - n_whole) * split; }
  int grid() const { return n_whole + (int)pieces(); }
};

// Static round-robin assignment (the persistent kernel: cluster c runs items
// c, c + slots, ...): the largest per-slot sum.
static double makespan_rr(const std::vector<double>& costs, int slots) {
  std::vector<double> t(slots, 0.0);
  for (size_t i = 0; i < costs.size(); ++i) t[i % slots] += costs[i];
  return *std::max_element(t.begin(), t.end());
}

static double makespan(const std::vector<double>& costs, int sms) {
  std::priority_queue<double, std::vector<double>, std::greater<double>> q;
  for (int i = 0; i < sms; ++i) q.push(0.0);
  double end = 0.0;
  for (double c : costs) {
    double t = q.top() + c;
    q.pop();
    q.push(t);
    end = std::max(end, t);
  }
  return end;
}

// `slots` = concurrent work units (SMs, or SM pairs for the cluster-pair
// kernel); c_rag = relative cost of a unit whose second 128-row tile is empty
// (0.6 single-CTA: its MMAs and softmax are skipped; 1.0 for a pair, whose
// M = 256 MMAs run regardless).
static AttnPlan plan_attention(int n_q, int n_heads, int sms, double c_rag = 0.6, bool rr = false) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, bool>, AttnPlan> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(n_q, n_heads, sms, (int)(c_rag * 100), rr);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  AttnPlan pl;
  pl.pairs = (n_q + 2 * AT_M - 1) / (2 * AT_M);
  const bool ragged = (pl.pairs - 1) * 2 * AT_M + AT_M >= n_q;  // last pair has one tile
  pl.reg_pairs = pl.pairs - (ragged ? 1 : 0);
  pl.n_units = pl.pairs * n_heads;
  const int n_reg = pl.reg_pairs * n_heads;
  const double eps = 0.02;
  auto cost = [&](int u) { return u < n_reg ? 1.0 : c_rag; };
  double best = 1e300;
  AttnPlan bp = pl;
  bp.n_whole = pl.n_units;
  bp.split = 1;
  std::vector<double> costs;
  for (int n_split = 0; n_split <= std::min(pl.n_units, 2 * sms); ++n_split) {
    for (int split = (n_split ? 2 : 1); split <= (n_split ? 16 : 1); ++split) {
      const int n_whole = pl.n_units - n_split;
      costs.clear();
      for (int u = 0; u < n_whole; ++u) costs.push_back(cost(u) + eps);
      for (int u = n_whole; u < pl.n_units; ++u)
        for (int s = 0; s < split; ++s) costs.push_back(cost(u) / split + eps);
      double t = (rr ? makespan_rr(costs, sms) : makespan(costs, sms)) + (n_split ? 0.05 : 0.0);
      if (t < best - 1e-9) {
        best = t;
        bp.n_whole = n_whole;
        bp.split = split;
      }
    }
  }
  bp.pairs = pl.pairs;
  bp.reg_pairs = pl.reg_pairs;
  bp.n_units = pl.n_units;
  cache[key] = bp;
  return bp;
}

// Workspace: [KV-split partials O | (m, l)] then one window flag per CTA.
static int64_t partial_bytes(const AttnPlan& pl) { return pl.pieces() * (2 * AT_M) * (AT_D + 2) * 4; }
static int64_t flag_bytes(int grid) { return ((int64_t)grid * 4 + 255) / 256 * 256; }

static bool persistent_attention() {
  static const bool persist = getenv("LP_ATTN_NONPERSIST") == nullptr;
  return persist;
}
// Dynamic item assignment in the persistent kernel (default; LP_ATTN_STATIC=1
// keeps the round robin): every cluster claims the next item from a global
// counter, so the split plan is the greedy-list makespan rather than the
// round-robin one.  Measured 1-1.6 % faster at steady state with ~6 % less
// DRAM and ~20 % less die-to-die L2 traffic (profiles/r2b/hs1_summary.md).
static bool dynamic_attention() {
  static const bool dyn = getenv("LP_ATTN_STATIC") == nullptr;
  return dyn && persistent_attention();
}
// Head-split queues for the dynamic persistent kernel: the items of heads
// [0, H/2) and [H/2, H) as runs of consecutive item indices (host mirror of
// item_of / unit_coords).  False if a queue needs more than 8 runs.
static bool head_split_queues(const AttnParams& q, int n_items, SchedTable& t) {
  const int n_reg = q.reg_pairs * q.n_heads;
  memset(&t, 0, sizeof(t));
  for (int it = 0; it < n_items; ++it) {
    const int unit = q.unit_base + (it < q.n_whole ? it : q.n_whole + (it - q.n_whole) / q.split);
    const int head = unit < n_reg ? unit / q.reg_pairs : unit - n_reg;
    const int g = head < q.n_heads / 2 ? 0 : 1;
    int* run = t.v + 8 + 16 * g;
    const int r = t.v[4 + g] - 1;
    if (r >= 0 && run[2 * r] + run[2 * r + 1] == it) {
      ++run[2 * r + 1];
    } else {
      if (r + 1 == 8) return false;
      run[2 * (r + 1)] = it;
      run[2 * (r + 1) + 1] = 1;
      ++t.v[4 + g];
    }
    ++t.v[2 + g];
  }
  return true;
}

static AttnPlan plan_pair(int n_q, int n_heads) {
  return plan_attention(n_q, n_heads, num_sms() / 2, 1.0, persistent_attention() && !dynamic_attention());
}

// The product path: the pair kernel over every unit; with LP_ATTN_TAIL_SPLIT
// the ragged query tail of every head (one 128-row tile) runs on the
// single-CTA kernel instead (forked onto the fork handle's side stream).
struct PairLayout {
  AttnPlan main;      // regular units only
  int n_tail = 0;     // ragged units (one per head) or 0
  int64_t sched = 0;  // workspace offset of the dynamic item counter
  int64_t flags_main = 0, flags_tail = 0, bytes = 0;  // workspace offsets / total
};
static PairLayout pair_layout(int n_q, int n_heads) {
  PairLayout L;
  const int pairs = (n_q + 2 * AT_M - 1) / (2 * AT_M);
  // Default: the pair grid runs the ragged tails too (a pair spends a whole
  // M = 256 unit on 72 rows, but the alternatives measured slower: the tails
  // on the single-CTA kernel after the pair grid 2.20 vs 2.04 ms; forked onto a
  // low-priority side stream 2.16-2.19 vs 2.01 ms, profiles/r2/attn_ragged_tail_ab.txt).
  // LP_ATTN_TAIL_SPLIT=1 keeps the split path for A/B.
  static const bool split_tail = getenv("LP_ATTN_TAIL_SPLIT") != nullptr;
  const bool ragged = split_tail && (pairs - 1) * 2 * AT_M + AT_M >= n_q;
  const int reg = pairs - (ragged ? 1 : 0);
  if (reg > 0) L.main = plan_pair(reg * 2 * AT_M, n_heads);
  L.n_tail = ragged ? n_heads : 0;
  L.flags_main = partial_bytes(L.main);
  L.flags_tail = L.flags_main + flag_bytes(2 * L.main.grid());
  L.sched = L.flags_tail + flag_bytes(L.n_tail);
  L.bytes = L.sched + 256;  // dynamic item counter
  return L;
}

int64_t attention_workspace_bytes(int n_q, int n_heads) {
  if (n_q <= 0 || n_heads <= 0 || num_sms() <= 0) return 0;
  const AttnPlan p1 = plan_attention(n_q, n_heads, num_sms());
  return std::max(partial_bytes(p1) + flag_bytes(p1.grid()), pair_layout(n_q, n_heads).bytes);
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
  // cluster-pair kernel (default) or the single-CTA one (LP_ATTN_SINGLE=1, A/B)
  const bool pair_k = getenv("LP_ATTN_SINGLE") == nullptr && getenv("LP_ATTN_EXACT") == nullptr;
  const int64_t have = a->workspace ? a->workspace_bytes : 0;
  AttnParams p;
  p.n_q = a->n_q;
  p.n_heads = a->n_heads;
  p.scale_log2 = a->scale * 1.4426950408889634f;
  p.out = static_cast<__nv_bfloat16*>(a->out);
  p.ldo = d;
  p.desc = a->desc;
  p.part_o = static_cast<float*>(a->workspace);
  p.unit_base = 0;
  static const int l2pol = getenv("LP_ATTN_L2POL") ? atoi(getenv("LP_ATTN_L2POL")) : 0;
  p.l2pol = l2pol;
  p.sched = nullptr;
  p.hs_smid = 0;
  const int smem = AttnSmem::TOTAL;
  if (pair_k) {
    const PairLayout lay = pair_layout(a->n_q, a->n_heads);
    if (have >= lay.bytes) {
      char* ws = static_cast<char*>(a->workspace);
      const AttnPlan full = plan_attention(a->n_q, a->n_heads, num_sms());  // unit numbering (pairs, reg_pairs)
      p.pairs = full.pairs;
      p.reg_pairs = full.reg_pairs;
      LP_CUDA_TRY(cudaFuncSetAttribute(attn_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      // ragged query tails: single-CTA kernel (tile B skipped), on the fork's
      // side stream when there is one -- forked before the pair grid is
      // launched, so its CTAs take the SMs the pair grid's last wave leaves idle
      const ForkCtx* fk = static_cast<const ForkCtx*>(a->fork);
      cudaStream_t ts = st;
      if (fk && lay.n_tail > 0 && lay.main.n_units > 0) {
        LP_CUDA_TRY(cudaEventRecord(fk->fork, st));
        LP_CUDA_TRY(cudaStreamWaitEvent(fk->side, fk->fork, 0));
        ts = fk->side;
      }
      if (lay.main.n_units > 0) {
        const AttnPlan& pm = lay.main;
        AttnParams q = p;
        q.n_whole = pm.n_whole;
        q.split = pm.split;
        q.part_ml = q.part_o + pm.pieces() * (2 * AT_M) * AT_D;
        q.flags = reinterpret_cast<int*>(ws + lay.flags_main);
        q.flag_pairs = 1;
        CUtensorMap tk2;  // this CTA's 64 keys of a tile
        rc = make_tmap_bf16_2d(&tk2, a->k_arena, (uint64_t)a->arena_rows, (uint64_t)d, (uint64_t)d, 64, 64);
        if (rc) return rc;
        if (persistent_attention()) {  // one cluster per SM pair walks the items
          const int clusters = std::min(pm.grid(), std::max(1, num_sms() / 2));
          LP_CUDA_TRY(cudaFuncSetAttribute(attn_tc2p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           Attn2pSmem::TOTAL));
          q.sched = nullptr;
          if (dynamic_attention()) {
            q.sched = reinterpret_cast<int*>(ws + lay.sched);
            static const int hs = getenv("LP_ATTN_HEADSPLIT") ? atoi(getenv("LP_ATTN_HEADSPLIT")) : 0;
            SchedTable tab;
            if (hs > 0 && head_split_queues(q, pm.grid(), tab)) {
              q.hs_smid = hs;
            } else {
              memset(&tab, 0, sizeof(tab));
              q.hs_smid = 0;
            }
            sched_init_kernel<<<1, 64, 0, st>>>(q.sched, tab);  // counters zeroed (+ the queue table)
            if ((rc = launch_status("attention_sched_init"))) return rc;
          }
          attn_tc2p_kernel<<<2 * clusters, AT_THREADS, Attn2pSmem::TOTAL, st>>>(tq, tk2, tv, q, pm.grid());
          if ((rc = launch_status("attention_tc2p"))) return rc;
        } else {
          LP_CUDA_TRY(cudaFuncSetAttribute(attn_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           Attn2Smem::TOTAL));
          attn_tc2_kernel<<<2 * pm.grid(), AT_THREADS, Attn2Smem::TOTAL, st>>>(tq, tk2, tv, q);
          if ((rc = launch_status("attention_tc2"))) return rc;
        }
        attn_tc_kernel<false><<<pm.grid(), AT_THREADS, smem, st>>>(tq, tk, tv, q);  // rerun flagged units
        if ((rc = launch_status("attention_tc"))) return rc;
        if (pm.n_whole < pm.n_units) {
          const int64_t warps = (int64_t)(pm.n_units - pm.n_whole) * (2 * AT_M);
          attn_combine_kernel<<<(int)((warps * 32 + 255) / 256), 256, 0, st>>>(q);
          if ((rc = launch_status("attention_combine"))) return rc;
        }
      }
      if (lay.n_tail > 0) {
        AttnParams q = p;
        q.unit_base = full.reg_pairs * a->n_heads;
        q.n_whole = lay.n_tail;
        q.split = 1;
        q.part_ml = nullptr;
        q.flags = reinterpret_cast<int*>(ws + lay.flags_tail);
        q.flag_pairs = 0;
        LP_CUDA_TRY(cudaFuncSetAttribute(attn_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attn_tc_kernel<true><<<lay.n_tail, AT_THREADS, smem, ts>>>(tq, tk, tv, q);
        if ((rc = launch_status("attention_tc_window"))) return rc;
        attn_tc_kernel<false><<<lay.n_tail, AT_THREADS, smem, ts>>>(tq, tk, tv, q);
        if ((rc = launch_status("attention_tc"))) return rc;
      }
      if (ts != st) {
        LP_CUDA_TRY(cudaEventRecord(fk->join, ts));
        LP_CUDA_TRY(cudaStreamWaitEvent(st, fk->join, 0));
      }
      return LP_OK;
    }
  }
  AttnPlan pl = plan_attention(a->n_q, a->n_heads, num_sms());
  if (pl.pieces() > 0 && have < partial_bytes(pl) + flag_bytes(pl.grid())) {
    pl.n_whole = pl.n_units;  // no (or too small a) workspace: run every unit whole
    pl.split = 1;
  }
  // the bounded-exponent kernel needs the flag words (after the partials);
  // without them the exact single-CTA kernel runs every unit
  const bool fast = have >= partial_bytes(pl) + flag_bytes(pl.grid()) && getenv("LP_ATTN_EXACT") == nullptr;
  p.pairs = pl.pairs;
  p.reg_pairs = pl.reg_pairs;
  p.n_whole = pl.n_whole;
  p.split = pl.split;
  p.part_ml = p.part_o ? p.part_o + pl.pieces() * (2 * AT_M) * AT_D : nullptr;
  p.flags = fast ? reinterpret_cast<int*>(static_cast<char*>(a->workspace) + partial_bytes(pl)) : nullptr;
  p.flag_pairs = 0;
  if (fast) {
    LP_CUDA_TRY(cudaFuncSetAttribute(attn_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attn_tc_kernel<true><<<pl.grid(), AT_THREADS, smem, st>>>(tq, tk, tv, p);
    rc = launch_status("attention_tc_window");
    if (rc) return rc;
  }
  // exact online-max kernel: every unit, or (after the bounded-exponent
  // kernel) only the units it flagged -- the others exit on their first load
  LP_CUDA_TRY(cudaFuncSetAttribute(attn_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  attn_tc_kernel<false><<<pl.grid(), AT_THREADS, smem, st>>>(tq, tk, tv, p);
  rc = launch_status("attention_tc");
  if (rc || pl.n_whole == pl.n_units) return rc;
  const int64_t warps = (int64_t)(pl.n_units - pl.n_whole) * (2 * AT_M);
  attn_combine_kernel<<<(int)((warps * 32 + 255) / 256), 256, 0, st>>>(p);
  return launch_status("attention_combine");
}

}  // namespace lp
