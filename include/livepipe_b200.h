/*
 * livepipe_b200.h -- C ABI of liblivepipe_b200.so, the B200 (sm_100a) kernels
 * behind the livepipe streaming-denoiser hot path.
 *
 * The reference (Python/NumPy, /root/reference/pkg/src/livepipe) has one
 * plugin point on this path: the duck-typed denoiser object the engine calls,
 * `ToyDenoiser.denoise_block` (denoiser.py:201-276), picked by
 * `build_runtime` (engine.py:177-201).  The Python class
 * `paper_2512_04677_b200.denoiser.B200Denoiser` keeps that signature and calls
 * the entry points below through ctypes.  Every entry point takes plain
 * pointers / sizes and an explicit cudaStream_t (passed as void*), returns 0
 * on success or an LP_E* code (message via lp_last_error()), never throws, and
 * allocates nothing on the hot path (all buffers come from the caller).
 *
 * Each entry point names the reference function it replaces.
 */
#ifndef LIVEPIPE_B200_H
#define LIVEPIPE_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define LP_API __attribute__((visibility("default")))
#else
#define LP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define LP_ABI_VERSION 8

/* status codes */
#define LP_OK 0
#define LP_EINVAL 1       /* bad argument (shape, alignment, null pointer) */
#define LP_ECUDA 2        /* CUDA runtime / driver error */
#define LP_EUNSUPPORTED 3 /* shape or mode this build does not handle */
#define LP_ETIMEOUT 4     /* a stage-link wait exceeded its bound */
#define LP_EABORT 5       /* another stage raised the pipeline abort flag */

/* element types */
#define LP_F32 0
#define LP_BF16 1

/* GEMM epilogues (what happens to acc = A.W for output element (r, c)) */
#define LP_EPI_STORE 0      /* c = acc + bias[c]               (out dtype = args.out_dtype) */
#define LP_EPI_RELU 1       /* c = max(acc, 0)                                             */
#define LP_EPI_GELU 2       /* c = gelu_tanh(acc)                                          */
#define LP_EPI_RESID 3      /* h[r,c] = h[r,c] + gate[c] * acc   (h fp32; gate NULL => 1)  */
#define LP_EPI_QKV 4        /* columns [0,d)->q, [d,2d)->k ring slot, [2d,3d)->v ring slot,
                               with optional per-head RMSNorm and rotary embedding         */
#define LP_EPI_EULER 5      /* velocity head + flow step: x_out = x_in + acc * desc->dt at the
                               latent position of (token r, patch element c)  (LP_BF16)   */

#define LP_MAX_SEG 66  /* sink + up to 64 history blocks + current block */
#define LP_MAX_PAIRS 64

/*
 * Per-call block descriptor, resident in DEVICE memory and rewritten by the
 * host before each forward (one small async copy), so a captured CUDA graph
 * can replay every block of a stream.  Replaces the per-call arguments of
 * denoise_block (denoiser.py:201-211): block index, t_index, the cache view
 * (as KV-arena row segments: sink, history oldest->newest, current --
 * denoiser.py:248-253), sink_rope_index (kvcache.py:86-90) and the flow
 * step dt (latent.py:140-147).
 */
typedef struct lp_block_desc {
  int32_t block_index;    /* i: temporal rotary position of every token    */
  int32_t t_index;        /* j                                             */
  int32_t sink_pos;       /* i + delta                                     */
  int32_t n_seg;          /* number of KV segments (>= 2: sink, current)   */
  int32_t cur_row;        /* arena row where this block's K/V are written  */
  int32_t n_tokens;       /* tokens in the current block                   */
  int32_t seg_row[LP_MAX_SEG];
  int32_t seg_len[LP_MAX_SEG];
  int32_t src_row[LP_MAX_SEG]; /* history noise: uncorrupted ring rows      */
  float dt;               /* Euler step (negative)                         */
  float sigma;            /* history-noise std (0 = off)                   */
  uint64_t noise_key;     /* device-RNG key for history noise (perf runs)  */
  /* temporal-axis rotary cos/sin (pairs of the t axis), fp64 angle -> fp32 */
  float rope_cos[LP_MAX_PAIRS];
  float rope_sin[LP_MAX_PAIRS];
  float sink_cos[LP_MAX_PAIRS];
  float sink_sin[LP_MAX_PAIRS];
  /* 1: the tcgen05 attention may visit the segments in arena-row order with
     adjacent ones merged (fewer ragged tiles; the rounding then depends on
     where the rows sit -- used by the engines, whose ring slots are a
     function of the block index).  0: logical order, segment by segment,
     so the result does not depend on row placement (the drop-in denoiser,
     whose per-call K/V pool slots vary).  The fp32 path is always logical. */
  int32_t arena_order;
  int32_t reserved_;
} lp_block_desc;

/* Static rotary geometry of one model (per-head pair layout). */
typedef struct lp_rope_geom {
  int32_t head_dim;
  int32_t t_pairs;        /* pairs [0, t_pairs) use the temporal position   */
  int32_t tokens_per_frame;
  /* pairs [t_pairs, head_dim/2) use per-token spatial tables:
     cos/sin[(token % tokens_per_frame) * spatial_pairs + p]             */
  int32_t spatial_pairs;
  const float* spatial_cos;
  const float* spatial_sin;
} lp_rope_geom;

/* ---------------------------------------------------------------- setup */
LP_API int lp_abi_version(void);
LP_API const char* lp_last_error(void);
/* Select the device and resolve cuTensorMapEncodeTiled; idempotent. */
LP_API int lp_init(int device);
LP_API int lp_num_sms(void);

/* ---------------------------------------------------------------- GEMM
 * replaces numerics.matmul (numerics.py:50-64) at every projection site of
 * denoise_block: QKV :240-242, O :265, FFN :266, velocity head :268.
 *   LP_F32 : A fp32 [m,k] (lda), W fp32 [k,n] row-major (in x out, as the
 *            reference stores it, ldw); ascending-k, separately rounded
 *            mul/add (bit-faithful to the reference's pinned order).
 *   LP_BF16: A bf16 [m,k], W^T bf16 [n,k] (K-major); tcgen05.mma, fp32
 *            accumulation in TMEM, TMA-fed; k % 64 == 0, n % 16 == 0.
 */
typedef struct lp_qkv_epi {
  int32_t d;              /* model dim; GEMM n == 3*d                       */
  int32_t n_heads;
  int32_t head_dim;
  int32_t qk_norm;        /* per-head RMSNorm before rotation               */
  float eps;
  const float* g_q;       /* [d] or NULL                                    */
  const float* g_k;
  void* q_out;            /* [m, d] (dtype of the KV arena)                 */
  void* k_arena;          /* this layer's K arena base ([rows, d])          */
  void* v_arena;
  const lp_block_desc* desc; /* device: cur_row, rope_cos/sin               */
  lp_rope_geom geom;
} lp_qkv_epi;

/* Velocity-head epilogue (denoiser.py:268 + flow_step latent.py:140-147):
   token r, patch element c -> latent index of frame r / tokens_per_frame,
   channel c / (ph*pw), pixel (gy*ph + py, gx*pw + px); ph == 0 => toy layout
   (x[r * n + c]).  x_out = x_in + fp32(acc * dt), separately rounded.       */
typedef struct lp_euler_epi {
  const float* x_in;
  float* x_out;           /* may be a peer-mapped receive slot              */
  int32_t channels, height, width, ph, pw;
  const lp_block_desc* desc;
  const int32_t* gate_status; /* NULL, or a link status word: when it is
                             non-zero (a failed wait on the consumer's free
                             counter) the store is skipped, so a slot the
                             consumer has not released is never overwritten */
} lp_euler_epi;

/* Implicit-GEMM convolution over a zero-bordered row layout (the decode
 * stage's VAE stand-in, codec.py VaeDecoder): A is [rows, cin] bf16 with the
 * activation stored as [T][H+2][W+2][cin] (one zero pixel of border), and the
 * GEMM's K = n_taps * cin walks the taps: k-chunk kb reads A rows
 * m + tap_row[kb / (cin/64)] (TMA zero-fills rows outside [0, m) -- the causal
 * temporal taps of frame 0), columns (kb % (cin/64)) * 64.  W is
 * [n, n_taps*cin] (tap-major K).  Output rows are the padded grid; border
 * rows hold garbage the consumer ignores.                                    */
typedef struct lp_conv_taps {
  int32_t n_taps;         /* <= 27                                          */
  int32_t cin;            /* multiple of 64                                 */
  int32_t tap_row[27];    /* row offset of each tap in the padded layout    */
  int32_t frames, height, width; /* interior T, H, W of the bordered layout,
                             or 0: with them and the 27 causal 3x3x3 taps in
                             (dt, dy, dx) order, the conv runs as halo tiles
                             (8 x 16 pixels: one 10 x 16 window per (dt, dx)
                             feeds the three dy taps -- 2.4x less A traffic
                             than one row-shifted box per tap)             */
} lp_conv_taps;

typedef struct lp_gemm_args {
  int32_t in_dtype;       /* LP_F32 | LP_BF16                               */
  int32_t out_dtype;      /* for STORE/RELU/GELU                            */
  int32_t epilogue;       /* LP_EPI_*                                       */
  int32_t m, n, k;
  int64_t lda, ldw, ldc;
  const void* a;
  const void* w;
  void* c;                /* output (or fp32 residual h for LP_EPI_RESID)   */
  const float* bias;      /* [n] or NULL (STORE only)                       */
  const float* gate;      /* [n] or NULL (RESID only)                       */
  const lp_qkv_epi* qkv;  /* host pointer, LP_EPI_QKV only                  */
  const lp_euler_epi* euler; /* host pointer, LP_EPI_EULER only             */
  const lp_conv_taps* conv; /* host pointer or NULL: implicit-GEMM conv (bf16,
                             STORE/RESID, single-CTA tiles, no fork)        */
  void* fork;             /* lp_fork_create handle or NULL: lets a bf16 GEMM
                             whose M is not a multiple of 256 run cluster-pair
                             tiles on the whole 256-row blocks and the ragged
                             rows as single-CTA tiles on the handle's side
                             stream, concurrently (fork/join events on
                             `stream`; graph-capture safe)                   */
  float* row_stats;       /* RESID only, or NULL: LayerNorm statistics of the
                             updated h rows for the next norm (AdaLN) pass,
                             one (mean, M2) float pair per 32-column chunk,
                             [m][n/32] (ABI v8; feeds lp_norm_mod_stats)     */
} lp_gemm_args;
LP_API int lp_gemm(const lp_gemm_args* args, void* stream);

/* Side stream + fork/join events for lp_gemm_args.fork; create outside any
   stream capture, one per concurrently used stream.                        */
LP_API int lp_fork_create(void** out);
LP_API int lp_fork_destroy(void* fork);
/* Kernel nodes of a captured CUDA graph (cudaGraph_t as void*): the exact
   number of kernels one replay launches (bench.py's gpu_launches claim).  */
LP_API int lp_graph_kernel_count(void* graph, int64_t* count);

/* ---------------------------------------------------------------- attention
 * replaces the per-head loop of denoise_block (denoiser.py:246-264) and
 * _attend_head (:152-158): softmax(q K^T / sqrt(hd)) V over the visible keys
 * [sink | history oldest->newest | current] (segments from desc), no mask.
 *   LP_F32 : SIMT, reference summation order (numpy pairwise row sum).
 *   LP_BF16: tcgen05 flash attention on cluster pairs (cta_group::2, M = 256
 *            per pair, half of every K/V tile per SM), S/P/O in TMEM.  With a
 *            workspace: bounded-exponent softmax (each row's offset is the
 *            exact max of its first KV tile; the result equals exact softmax
 *            while later scores stay within 2^64 of it) and a rerun of any
 *            work unit that left that window by the exact online-max kernel,
 *            which also runs every unit when the workspace is NULL.
 *            Environment A/B: LP_ATTN_EXACT=1 (exact kernel only),
 *            LP_ATTN_SINGLE=1 (single-CTA bounded-exponent kernel).
 */
typedef struct lp_attn_args {
  int32_t dtype;
  int32_t n_q, n_heads, head_dim;
  float scale;
  const void* q;          /* [n_q, n_heads*hd]                              */
  const void* k_arena;    /* layer base, rows addressed by desc segments    */
  const void* v_arena;
  void* out;              /* [n_q, n_heads*hd]                              */
  const lp_block_desc* desc;
  int32_t arena_rows;     /* rows in the arena (bounds for TMA)             */
  int32_t n_kv_max;       /* host-known upper bound of visible keys         */
  void* workspace;        /* LP_BF16: partials of KV-split work units (the
                             tail of the grid is split to fill the last wave)
                             and one window flag per CTA; NULL or too small
                             => no splitting and the exact kernel           */
  int64_t workspace_bytes;
  void* fork;             /* lp_fork_create handle or NULL: the ragged query
                             tails (one 128-row tile per head) run on the
                             handle's side stream, concurrently with the
                             cluster-pair grid (fork/join events on `stream`;
                             graph-capture safe); NULL: after it            */
} lp_attn_args;
/* Bytes of lp_attn_args.workspace the tcgen05 attention uses for n_q queries
   and n_heads heads on this device (split partials + window flags).          */
LP_API int lp_attention_workspace(int n_q, int n_heads, int head_dim, int64_t* bytes_out);
LP_API int lp_attention(const lp_attn_args* args, void* stream);
/* SIMT reference attention for either dtype (validation tool: same math,
   reference order; used by tests to check the tcgen05 kernel on identical
   bf16 inputs).  Never used by the bf16 product path.                     */
LP_API int lp_attention_simt(const lp_attn_args* args, void* stream);

/* ---------------------------------------------------------------- row kernels */
/* cond row (denoiser.py:178-185): c = a.Wa + p.Wp + tau.Wt in that order.
   inputs fp32; tau precomputed by host (fp64 -> fp32).                     */
LP_API int lp_cond_row(const float* audio, int audio_dim, const float* w_audio,
                const float* prompt, int prompt_dim, const float* w_prompt,
                const float* tau, int tau_dim, const float* w_time,
                float* out, int d, void* stream);

/* h[r, :] = x[r, :] + c  (denoiser.py:236), toy embed (no patching)        */
LP_API int lp_add_row(const float* x, const float* c, float* h, int rows, int d, void* stream);

/* out = modulate(norm(h)) cast to out_dtype.  mode: 0 = copy (toy, no norm),
   1 = LayerNorm, 2 = LayerNorm*(1+scale)+shift.  shift/scale fp32 [d].     */
LP_API int lp_norm_mod(const float* h, int rows, int d, int mode, float eps,
                const float* shift, const float* scale, void* out, int out_dtype,
                void* stream);

/* lp_norm_mod (mode 1 or 2) with the row statistics taken from `stats`, the
   per-32-column (mean, M2) partials a RESID lp_gemm wrote for these h rows
   (lp_gemm_args.row_stats, [rows][d/32] float pairs): the pre-LN + AdaLN of
   denoiser.py's Wan profile with its reduction fused into the producing
   GEMM's epilogue, leaving one streaming apply pass.  d % 32 == 0.        */
LP_API int lp_norm_mod_stats(const float* h, const float* stats, int rows, int d, int mode, float eps,
                      const float* shift, const float* scale, void* out, int out_dtype, void* stream);

/* Sink K/V at the block's sink position (denoiser.py:187-190, :246-249) for
   n_layers layers in one launch: k_raw/v_raw fp32 [S, d] per layer
   (raw_layer_stride elements apart) are the un-rotated projections of the
   sink latent, computed once per sink content (RSFM: after the one-shot AAS
   swap); writes (optionally per-head-RMS-normed) rotated K and V into arena
   rows [desc->seg_row[0], +S) of every layer (arena_layer_stride apart).
   v_raw == NULL: K only (the V rows do not depend on the position, so a
   caller whose sink rows are fixed writes them once per sink content).     */
LP_API int lp_sink_refresh(const float* k_raw, const float* v_raw, int s_tokens, int d,
                    int n_heads, int qk_norm, const float* g_k, float eps,
                    const lp_block_desc* desc, const lp_rope_geom* geom,
                    void* k_arena, void* v_arena, int arena_dtype, int n_layers,
                    int64_t raw_layer_stride, int64_t arena_layer_stride,
                    float* inv_rms_out, void* stream);
/* Per-block sink refresh of the TEMPORAL rotary pairs only (pairs
   [0, geom->t_pairs) of every head; the spatial pairs and V do not depend on
   the sink position i + delta and were written by lp_sink_refresh once per
   sink content, which also stored the per-(layer, token, head) RMSNorm
   factors in inv_rms [n_layers, S, n_heads] (qk_norm only; NULL otherwise).
   Bitwise the same K rows as a full lp_sink_refresh at this position.      */
LP_API int lp_sink_refresh_temporal(const float* k_raw, const float* inv_rms, int s_tokens, int d,
                    int n_heads, int qk_norm, const float* g_k,
                    const lp_block_desc* desc, const lp_rope_geom* geom, void* k_arena,
                    int arena_dtype, int n_layers, int64_t raw_layer_stride,
                    int64_t arena_layer_stride, void* stream);
/* out[i] = silu(x[i]) cast to out_dtype (AdaLN input, wan profile)         */
LP_API int lp_silu(const float* x, void* out, int n, int out_dtype, void* stream);
/* QKV post-processing for the SIMT path (the tcgen05 GEMM fuses this into its
   epilogue): qkv fp32 [m, 3d] -> per-head RMSNorm (opt.), rotary, q -> q_out,
   k/v -> arena rows desc->cur_row + r.                                     */
LP_API int lp_qkv_post(const float* qkv, int m, const lp_qkv_epi* epi, int out_dtype, void* stream);

/* Patchify / embed inputs and the velocity head's scatter + Euler step.
   patchify: x frames [F, C*H*W] fp32 -> tokens [F*Hp*Wp, C*ph*pw] (dtype).  */
LP_API int lp_patchify(const float* x, int frames, int c, int h, int w, int ph, int pw,
                void* tokens, int out_dtype, void* stream);
/* x_out = x + unpatchify(v_tokens) * dt   (latent.py:140-147), fp32.
   ph == 0 => toy: tokens are frames, x_out[r,c] = x[r,c] + v[r,c]*dt.      */
LP_API int lp_unpatchify_euler(const float* x, const float* v_tokens, int frames, int c,
                        int h, int w, int ph, int pw, const lp_block_desc* desc,
                        float* x_out, void* stream);

/* Decode stage, VAE stand-in (the decode worker engine.py:465-480 runs the
   reference codec latent.py:150-193; the paper's decode GPU runs the Wan VAE,
   PAPER.md:186, :304).  Activations are [T][H+2][W+2][C] rows with a
   one-pixel zero border; the 3-D convolutions are lp_gemm with lp_conv_taps.
   pack_latent: latent [F, C, H, W] fp32 -> bordered bf16 [F][H+2][W+2][cpad].
   norm_silu:   fp32 rows -> bf16; mode 1 = RMS norm over C * gamma, SiLU;
                mode 0 = cast; border pixels written as 0 (C <= 512).
   upsample:    nearest x2 in H and W, x ft (1|2) in T, bordered bf16 -> bf16.
   frames:      interior, first cout channels of fp32 rows -> [T][cout][H][W]. */
LP_API int lp_vae_pack_latent(const float* x, int f, int c, int h, int w, int cpad, void* out, void* stream);
LP_API int lp_vae_norm_silu(const float* hbuf, const float* gamma, int t, int h, int w, int c, int mode, float eps,
                            void* out, void* stream);
LP_API int lp_vae_upsample(const void* in, int t, int h, int w, int c, int ft, void* out, void* stream);
LP_API int lp_vae_frames(const float* hbuf, int t, int h, int w, int cpad, int cout, float* frames, void* stream);

/* The reference's analytic test denoiser fused with the flow step
   (OracleDenoiser.denoise_block, denoiser.py:294-343 + flow_step,
   latent.py:140-147): vel = (x - target) / s (written when vel != NULL),
   x_out = x + vel * dt; IEEE fp32 in the reference's operation order, so the
   result is bitwise the reference's.  s == 0 -> LP_EINVAL (the reference
   raises ValueError "oracle velocity undefined at s = 0").                 */
LP_API int lp_oracle_step(const float* x, const float* target, float s, float dt, float* vel, float* x_out,
                          int64_t n, void* stream);

/* History noise (kvcache.py:121-137) for one layer and one of K/V (kv 0/1):
   for every history segment s in [1, n_seg-1) of desc, arena rows
   [seg_row[s], +seg_len[s]) = arena rows [src_row[s], +seg_len[s])
   + desc->sigma * z (the stored ring rows are never modified).  z comes from
   `noise` (host-generated in the reference draw order,
   [entry][kv][layer][rows][d], parity runs) or, when noise == NULL, from a
   device counter-hash stream keyed by desc->noise_key and (layer, kv, entry)
   (perf runs; bf16: exact Box-Muller with the sines on the FMA pipe, fp32:
   Philox4x32-7).
   max_rows bounds the history rows (grid size).                            */
LP_API int lp_history_noise(void* arena, int dtype, int d, const float* noise, int n_layers, int layer,
                     int kv, const lp_block_desc* desc, int max_rows, void* stream);

/* lp_history_noise (device counter-hash stream, bf16 arena) shaped to run on
   a side stream beside the tcgen05 GEMMs: two 128-thread CTAs per SM of
   <= 40 registers fit in what a GEMM CTA leaves free, so the corrupted-view
   copy of layer l can overlap the previous layer's O-proj / FFN and this
   layer's QKV (runtime opt-in LP_HIST_OVERLAP=1; measured slower than the
   in-line lp_history_noise at 14B).  Same noise values as lp_history_noise
   with noise == NULL.                                                      */
LP_API int lp_history_noise_co(void* arena, int d, int layer, int kv, const lp_block_desc* desc, int max_rows,
                               void* stream);

/* Device N(0,1) fp32 fill (perf-run weights / block noise), Philox4x32 +
   Box-Muller keyed by (seed, stream).  scale multiplies every sample.     */
LP_API int lp_randn(float* out, int64_t n, uint64_t seed, uint64_t stream_id, float scale,
             void* stream);
LP_API int lp_randn_bf16(void* out, int64_t n, uint64_t seed, uint64_t stream_id, float scale,
                  void* stream);

/* ---------------------------------------------------------------- codec
 * The decode stage, run on the decode GPU.  The toy
 * profile's ToyVideoCodec (latent.py:150-193) is a dense matvec per latent
 * frame in the pinned matmul order and goes through lp_gemm (LP_F32).
 * Patched (wan-shaped) profiles use a per-location patch codec standing in
 * for the video VAE: latent (frames, C, H, W) fp32 -> pixels
 * (frames*r, pc, H*s, W*s) fp32, pix[f*r+u][ch][h*s+dy][w*s+dx] =
 * sum_c maps[u][(ch*s+dy)*s+dx][c] * x[f][c][h][w]; encode applies
 * enc (C, pc*s*s) = pinv(maps[0]) to the s x s patches of one pixel frame
 * (the AAS sink round trip, kvcache.py:93-109).  Pinned ascending order,
 * no FMA contraction: bitwise equal to the NumPy restatement.  C <= 32.    */
LP_API int lp_codec_patch_decode(const float* x, int frames, int C, int H, int W, const float* maps,
                    int r, int pc, int s, float* out, void* stream);
LP_API int lp_codec_patch_encode(const float* frame, int C, int H, int W, const float* enc, int pc,
                    int s, float* out, void* stream);

/* ---------------------------------------------------------------- TPP links
 * replace _Link.send/recv (engine.py:342-388) and the one-shot sink fan-out
 * (:417, :477-478).  A link is a ring of `capacity` payload slots plus
 * monotone 32-bit flags in (peer-mapped) device memory:
 *   ready[s] = sequence+1 published by the producer (release, system scope),
 *   free[s]  = sequence+1 consumed, published by the consumer.
 * lp_link_send copies `bytes` into slot (seq % capacity) of the consumer's
 * receive buffer (peer pointer over NVLink, or local) after waiting for the
 * slot to be free, then publishes ready.  lp_link_recv waits for ready and
 * copies out.  Waits spin on the device with a bound (timeout_ns) and poll
 * the host-mapped abort word.
 * `status` (device int32, may be NULL) is STICKY: a failed wait stores
 * LP_EABORT / LP_ETIMEOUT into it, success never clears it, and every link
 * kernel that finds it already non-zero does nothing (no copy, no flag
 * publish) -- so after a failure a stage neither consumes nor forwards stale
 * data, and the host sees the first failure whenever it reads the word.  */
LP_API int lp_link_send(const void* src, void* dst_slot, int64_t bytes, volatile uint32_t* ready_flag,
                 volatile const uint32_t* free_flag, uint32_t seq, int capacity,
                 volatile const uint32_t* abort_word, uint64_t timeout_ns,
                 int32_t* status, void* stream);
LP_API int lp_link_recv(const void* src_slot, void* dst, int64_t bytes, volatile const uint32_t* ready_flag,
                 volatile uint32_t* free_flag, uint32_t seq,
                 volatile const uint32_t* abort_word, uint64_t timeout_ns,
                 int32_t* status_out, void* stream);

/* Publish `value` into a (possibly peer-mapped) flag with a system-scope
   release after all prior work on `stream` (the "ready"/"sink posted" half
   of a link, engine.py:369 / :477-478) -- unless gate_status is non-NULL and
   non-zero (the stage's sticky link status: its data is not valid).        */
LP_API int lp_signal(volatile uint32_t* flag, uint32_t value, const int32_t* gate_status, void* stream);
/* Stream-ordered bounded wait until *flag >= target (engine.py:379, :439).
   status_out (may be NULL) is sticky as for the links: set to LP_EABORT or
   LP_ETIMEOUT on failure, never cleared; a non-zero word skips the wait.   */
LP_API int lp_wait(volatile const uint32_t* flag, uint32_t target, volatile const uint32_t* abort_word,
            uint64_t timeout_ns, int32_t* status_out, void* stream);

/* CUDA IPC for the one-process-per-GPU TPP runtime: export the allocation
   containing dev_ptr as a 64-byte handle plus the pointer's offset inside it,
   and map a peer's handle into this process (peer access over NVLink is
   enabled lazily).  lp_ipc_close takes the mapped BASE (ptr - offset).      */
LP_API int lp_ipc_handle(const void* dev_ptr, uint8_t* handle_out, int64_t* offset_out);
LP_API int lp_ipc_open(const uint8_t* handle, int64_t offset, void** ptr_out);
LP_API int lp_ipc_close(void* mapped_base);
/* Let `device` address `peer`'s memory directly (NVLink P2P): the in-process
   multi-device TPP runner's link kernels run on the producer's device and
   store into the consumer's slots, and every stage polls one abort word.
   Idempotent; LP_EUNSUPPORTED when the pair cannot peer.                    */
LP_API int lp_peer_enable(int device, int peer);


/* ---------------------------------------------------------------- arenas
 * Growable KV arena on CUDA virtual memory for the drop-in denoiser
 * (Runtime.denoiser, engine.py:166-200), whose caller decides how many
 * cache entries stay alive (RollingKvCache, kvcache.py:29-59; TPP threads,
 * engine.py:431-463).  One reserved range of n_layers * layer_stride bytes;
 * the first `mapped` bytes of every layer are backed on demand.  Growth
 * never moves data (pointers stay valid) and zero-fills the new pages on
 * `stream`.                                                                */
typedef struct lp_vmm lp_vmm;
LP_API int lp_vmm_create(int device, int n_layers, int64_t layer_bytes_max, lp_vmm** out);
LP_API int lp_vmm_info(const lp_vmm* v, uint64_t* base, int64_t* layer_stride_bytes, int64_t* mapped_bytes,
                int64_t* granularity);
LP_API int lp_vmm_grow(lp_vmm* v, int64_t layer_bytes, void* stream);
LP_API int lp_vmm_destroy(lp_vmm* v);

#ifdef __cplusplus
}
#endif
#endif /* LIVEPIPE_B200_H */
