// extern "C" surface of liblivepipe_b200.so (declared in include/livepipe_b200.h).
#include <algorithm>
#include <mutex>
#include <vector>

#include "lp_common.cuh"
#include "lp_tma.cuh"

namespace lp {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

static int g_sms = 0;
int num_sms() { return g_sms; }

// defined in the other translation units
int gemm_f32(const lp_gemm_args* a, cudaStream_t st);
int qkv_post(const float* qkv, int m, const lp_qkv_epi& e, int out_dtype, cudaStream_t st);
int attention_simt(const lp_attn_args* a, int n_kv_max, cudaStream_t st);
int gemm_tc(const lp_gemm_args* a, cudaStream_t st);
int attention_tc(const lp_attn_args* a, cudaStream_t st);
int64_t attention_workspace_bytes(int n_q, int n_heads);
int cond_row(const float*, int, const float*, const float*, int, const float*, const float*, int, const float*,
             float*, int, cudaStream_t);
int add_row(const float*, const float*, float*, int, int, cudaStream_t);
int norm_mod(const float*, int, int, int, float, const float*, const float*, void*, int, cudaStream_t);
int norm_mod_stats(const float*, const float*, int, int, int, float, const float*, const float*, void*, int,
                   cudaStream_t);
int sink_refresh(const float*, const float*, int, int, int, int, const float*, float, const lp_block_desc*,
                 const lp_rope_geom&, void*, void*, int, int, int64_t, int64_t, float*, cudaStream_t);
int sink_refresh_temporal(const float*, const float*, int, int, int, int, const float*, const lp_block_desc*,
                          const lp_rope_geom&, void*, int, int, int64_t, int64_t, cudaStream_t);
int silu(const float*, void*, int, int, cudaStream_t);
int patchify(const float*, int, int, int, int, int, int, void*, int, cudaStream_t);
int unpatchify_euler(const float*, const float*, int, int, int, int, int, int, const lp_block_desc*, float*,
                     cudaStream_t);
int history_noise(void*, int, int, const float*, int, int, int, const lp_block_desc*, int, cudaStream_t);
int history_noise_co(void*, int, int, int, const lp_block_desc*, int, cudaStream_t);
int oracle_step(const float*, const float*, float, float, float*, float*, int64_t, cudaStream_t);
int randn(void*, int64_t, uint64_t, uint64_t, float, int, cudaStream_t);
int link_send(const void*, void*, int64_t, volatile uint32_t*, const volatile uint32_t*, uint32_t, int,
              const volatile uint32_t*, uint64_t, int32_t*, cudaStream_t);
int link_recv(const void*, void*, int64_t, const volatile uint32_t*, volatile uint32_t*, uint32_t,
              const volatile uint32_t*, uint64_t, int32_t*, cudaStream_t);

int signal(volatile uint32_t*, uint32_t, const int32_t*, cudaStream_t);
int wait(const volatile uint32_t*, uint32_t, const volatile uint32_t*, uint64_t, int32_t*, cudaStream_t);
int ipc_handle(const void*, uint8_t*, int64_t*);
int ipc_open(const uint8_t*, int64_t, void**);
int ipc_close(void*);

int preload_links();
int preload_f32();
int preload_rows();
int preload_gemm_tc();
int preload_attn_tc();
int preload_codec();
int preload_vae();
int vae_pack_latent(const float*, int, int, int, int, int, void*, cudaStream_t);
int vae_norm_silu(const float*, const float*, int, int, int, int, int, float, void*, cudaStream_t);
int vae_upsample(const void*, int, int, int, int, int, void*, cudaStream_t);
int vae_frames(const float*, int, int, int, int, int, float*, cudaStream_t);
int fork_create(void**);
int fork_destroy(void*);
int codec_patch_decode(const float*, int, int, int, int, const float*, int, int, int, float*, cudaStream_t);
int codec_patch_encode(const float*, int, int, int, const float*, int, int, float*, cudaStream_t);

}  // namespace lp

using namespace lp;

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

int lp_abi_version(void) { return LP_ABI_VERSION; }
const char* lp_last_error(void) { return g_err.c_str(); }

int lp_init(int device) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  LP_CUDA_TRY(cudaSetDevice(device));
  int sms = 0;
  LP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  int major = 0, minor = 0;
  LP_CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  LP_CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
  if (major != 10 || minor != 0)
    return fail(LP_EUNSUPPORTED, "liblivepipe_b200 is built for sm_100a (B200); device is sm_" +
                                     std::to_string(major) + std::to_string(minor));
  g_sms = sms;
  // Load every kernel now: stage links spin on the device, and a lazily
  // loaded kernel launched while a waiter spins can stall in the loader.
  int rc;
  if ((rc = preload_links()) || (rc = preload_f32()) || (rc = preload_rows()) || (rc = preload_gemm_tc()) ||
      (rc = preload_attn_tc()) || (rc = preload_codec()) || (rc = preload_vae()))
    return rc;
  return tma_init();
}

int lp_num_sms(void) { return g_sms; }

int lp_gemm(const lp_gemm_args* a, void* stream) {
  LP_CHECK_ARG(a && a->a && a->w && (a->c || a->epilogue == LP_EPI_QKV || a->epilogue == LP_EPI_EULER),
               "lp_gemm: null argument");
  LP_CHECK_ARG(a->m >= 0 && a->n > 0 && a->k > 0, "lp_gemm: bad shape");
  if (a->in_dtype == LP_BF16) return gemm_tc(a, S(stream));
  LP_CHECK_ARG(a->in_dtype == LP_F32, "lp_gemm: in_dtype must be LP_F32 or LP_BF16");
  if (a->conv) return fail(LP_EUNSUPPORTED, "lp_gemm: conv taps need bf16 operands");
  if (a->row_stats) return fail(LP_EUNSUPPORTED, "lp_gemm: row_stats is a bf16 (tcgen05) RESID epilogue");
  if (a->epilogue == LP_EPI_QKV)
    return fail(LP_EUNSUPPORTED, "lp_gemm: fp32 QKV epilogue is lp_gemm(STORE) + lp_qkv_post");
  if (a->epilogue == LP_EPI_EULER)
    return fail(LP_EUNSUPPORTED, "lp_gemm: fp32 EULER epilogue is lp_gemm(STORE) + lp_unpatchify_euler");
  return gemm_f32(a, S(stream));
}

int lp_qkv_post(const float* qkv, int m, const lp_qkv_epi* epi, int out_dtype, void* stream) {
  LP_CHECK_ARG(qkv && epi && epi->desc && epi->q_out && epi->k_arena && epi->v_arena, "lp_qkv_post: null");
  LP_CHECK_ARG(epi->head_dim % 2 == 0 && epi->head_dim / 2 <= 2 * LP_MAX_PAIRS, "lp_qkv_post: head_dim");
  return qkv_post(qkv, m, *epi, out_dtype, S(stream));
}

int lp_attention(const lp_attn_args* a, void* stream) {
  LP_CHECK_ARG(a && a->q && a->k_arena && a->v_arena && a->out && a->desc, "lp_attention: null argument");
  if (a->dtype == LP_BF16) return attention_tc(a, S(stream));
  LP_CHECK_ARG(a->dtype == LP_F32, "lp_attention: dtype");
  return attention_simt(a, a->n_kv_max, S(stream));
}

int lp_attention_workspace(int n_q, int n_heads, int head_dim, int64_t* bytes_out) {
  LP_CHECK_ARG(bytes_out != nullptr, "lp_attention_workspace: null argument");
  LP_CHECK_ARG(num_sms() > 0, "lp_init() must be called before lp_attention_workspace");
  *bytes_out = head_dim == 128 ? attention_workspace_bytes(n_q, n_heads) : 0;
  return LP_OK;
}

int lp_attention_simt(const lp_attn_args* a, void* stream) {
  LP_CHECK_ARG(a && a->q && a->k_arena && a->v_arena && a->out && a->desc, "lp_attention_simt: null");
  return attention_simt(a, a->n_kv_max, S(stream));
}

int lp_cond_row(const float* audio, int audio_dim, const float* w_audio, const float* prompt, int prompt_dim,
                const float* w_prompt, const float* tau, int tau_dim, const float* w_time, float* out, int d,
                void* stream) {
  LP_CHECK_ARG(prompt && w_prompt && tau && w_time && out, "lp_cond_row: null argument");
  return cond_row(audio, audio_dim, w_audio, prompt, prompt_dim, w_prompt, tau, tau_dim, w_time, out, d,
                  S(stream));
}

int lp_add_row(const float* x, const float* c, float* h, int rows, int d, void* stream) {
  return add_row(x, c, h, rows, d, S(stream));
}

int lp_norm_mod(const float* h, int rows, int d, int mode, float eps, const float* shift, const float* scale,
                void* out, int out_dtype, void* stream) {
  return norm_mod(h, rows, d, mode, eps, shift, scale, out, out_dtype, S(stream));
}

int lp_norm_mod_stats(const float* h, const float* stats, int rows, int d, int mode, float eps, const float* shift,
                      const float* scale, void* out, int out_dtype, void* stream) {
  return norm_mod_stats(h, stats, rows, d, mode, eps, shift, scale, out, out_dtype, S(stream));
}

int lp_sink_refresh(const float* k_raw, const float* v_raw, int s_tokens, int d, int n_heads, int qk_norm,
                    const float* g_k, float eps, const lp_block_desc* desc, const lp_rope_geom* geom,
                    void* k_arena, void* v_arena, int arena_dtype, int n_layers, int64_t raw_layer_stride,
                    int64_t arena_layer_stride, float* inv_rms_out, void* stream) {
  LP_CHECK_ARG(k_raw && desc && geom && k_arena && v_arena, "lp_sink_refresh: null argument");
  return sink_refresh(k_raw, v_raw, s_tokens, d, n_heads, qk_norm, g_k, eps, desc, *geom, k_arena, v_arena,
                      arena_dtype, n_layers, raw_layer_stride, arena_layer_stride, inv_rms_out, S(stream));
}

int lp_sink_refresh_temporal(const float* k_raw, const float* inv_rms, int s_tokens, int d, int n_heads,
                             int qk_norm, const float* g_k, const lp_block_desc* desc, const lp_rope_geom* geom,
                             void* k_arena, int arena_dtype, int n_layers, int64_t raw_layer_stride,
                             int64_t arena_layer_stride, void* stream) {
  LP_CHECK_ARG(k_raw && desc && geom && k_arena, "lp_sink_refresh_temporal: null argument");
  LP_CHECK_ARG(!qk_norm || inv_rms, "lp_sink_refresh_temporal: qk_norm needs inv_rms");
  return sink_refresh_temporal(k_raw, inv_rms, s_tokens, d, n_heads, qk_norm, g_k, desc, *geom, k_arena,
                               arena_dtype, n_layers, raw_layer_stride, arena_layer_stride, S(stream));
}

int lp_silu(const float* x, void* out, int n, int out_dtype, void* stream) {
  return silu(x, out, n, out_dtype, S(stream));
}

int lp_patchify(const float* x, int frames, int c, int h, int w, int ph, int pw, void* tokens, int out_dtype,
                void* stream) {
  return patchify(x, frames, c, h, w, ph, pw, tokens, out_dtype, S(stream));
}

int lp_unpatchify_euler(const float* x, const float* v_tokens, int frames, int c, int h, int w, int ph, int pw,
                        const lp_block_desc* desc, float* x_out, void* stream) {
  return unpatchify_euler(x, v_tokens, frames, c, h, w, ph, pw, desc, x_out, S(stream));
}

int lp_oracle_step(const float* x, const float* target, float s, float dt, float* vel, float* x_out, int64_t n,
                   void* stream) {
  return oracle_step(x, target, s, dt, vel, x_out, n, S(stream));
}

int lp_history_noise(void* arena, int dtype, int d, const float* noise, int n_layers, int layer, int kv,
                     const lp_block_desc* desc, int max_rows, void* stream) {
  return history_noise(arena, dtype, d, noise, n_layers, layer, kv, desc, max_rows, S(stream));
}

int lp_history_noise_co(void* arena, int d, int layer, int kv, const lp_block_desc* desc, int max_rows,
                        void* stream) {
  return history_noise_co(arena, d, layer, kv, desc, max_rows, S(stream));
}

int lp_randn(float* out, int64_t n, uint64_t seed, uint64_t stream_id, float scale, void* stream) {
  return randn(out, n, seed, stream_id, scale, LP_F32, S(stream));
}

int lp_randn_bf16(void* out, int64_t n, uint64_t seed, uint64_t stream_id, float scale, void* stream) {
  return randn(out, n, seed, stream_id, scale, LP_BF16, S(stream));
}

int lp_link_send(const void* src, void* dst_slot, int64_t bytes, volatile uint32_t* ready_flag,
                 volatile const uint32_t* free_flag, uint32_t seq, int capacity, volatile const uint32_t* abort_word,
                 uint64_t timeout_ns, int32_t* status, void* stream) {
  return link_send(src, dst_slot, bytes, ready_flag, free_flag, seq, capacity, abort_word, timeout_ns, status,
                   S(stream));
}

int lp_link_recv(const void* src_slot, void* dst, int64_t bytes, volatile const uint32_t* ready_flag,
                 volatile uint32_t* free_flag, uint32_t seq, volatile const uint32_t* abort_word, uint64_t timeout_ns,
                 int32_t* status_out, void* stream) {
  return link_recv(src_slot, dst, bytes, ready_flag, free_flag, seq, abort_word, timeout_ns, status_out,
                   S(stream));
}

int lp_fork_create(void** out) { return fork_create(out); }

int lp_fork_destroy(void* fork) { return fork_destroy(fork); }

int lp_graph_kernel_count(void* graph, int64_t* count) {
  LP_CHECK_ARG(graph && count, "lp_graph_kernel_count: null argument");
  cudaGraph_t g = static_cast<cudaGraph_t>(graph);
  size_t n = 0;
  LP_CUDA_TRY(cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  if (n) LP_CUDA_TRY(cudaGraphGetNodes(g, nodes.data(), &n));
  int64_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    cudaGraphNodeType t;
    LP_CUDA_TRY(cudaGraphNodeGetType(nodes[i], &t));
    if (t == cudaGraphNodeTypeKernel) ++k;
  }
  *count = k;
  return LP_OK;
}

int lp_codec_patch_decode(const float* x, int frames, int C, int H, int W, const float* maps, int r, int pc, int s,
                          float* out, void* stream) {
  LP_CHECK_ARG(x && maps && out, "lp_codec_patch_decode: null argument");
  return codec_patch_decode(x, frames, C, H, W, maps, r, pc, s, out, S(stream));
}

int lp_codec_patch_encode(const float* frame, int C, int H, int W, const float* enc, int pc, int s, float* out,
                          void* stream) {
  LP_CHECK_ARG(frame && enc && out, "lp_codec_patch_encode: null argument");
  return codec_patch_encode(frame, C, H, W, enc, pc, s, out, S(stream));
}

int lp_signal(volatile uint32_t* flag, uint32_t value, const int32_t* gate_status, void* stream) {
  return signal(flag, value, gate_status, S(stream));
}

int lp_wait(volatile const uint32_t* flag, uint32_t target, volatile const uint32_t* abort_word, uint64_t timeout_ns,
            int32_t* status_out, void* stream) {
  return wait(flag, target, abort_word, timeout_ns, status_out, S(stream));
}

int lp_peer_enable(int device, int peer) {
  if (device == peer) return LP_OK;
  int can = 0;
  LP_CUDA_TRY(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can)
    return fail(LP_EUNSUPPORTED, "lp_peer_enable: device " + std::to_string(device) + " cannot access device " +
                                     std::to_string(peer));
  int prev = 0;
  LP_CUDA_TRY(cudaGetDevice(&prev));
  LP_CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(prev);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return LP_OK;
  }
  if (e != cudaSuccess) return fail(LP_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
  return LP_OK;
}

int lp_ipc_handle(const void* dev_ptr, uint8_t* handle_out, int64_t* offset_out) {
  return ipc_handle(dev_ptr, handle_out, offset_out);
}

int lp_ipc_open(const uint8_t* handle, int64_t offset, void** ptr_out) { return ipc_open(handle, offset, ptr_out); }

int lp_ipc_close(void* mapped_base) { return ipc_close(mapped_base); }

}  // extern "C"

// ---- decode stage: VAE stand-in row kernels (lp_vae.cu) ----
int lp_vae_pack_latent(const float* x, int f, int c, int h, int w, int cpad, void* out, void* stream) {
  return vae_pack_latent(x, f, c, h, w, cpad, out, S(stream));
}
int lp_vae_norm_silu(const float* hbuf, const float* gamma, int t, int h, int w, int c, int mode, float eps,
                     void* out, void* stream) {
  return vae_norm_silu(hbuf, gamma, t, h, w, c, mode, eps, out, S(stream));
}
int lp_vae_upsample(const void* in, int t, int h, int w, int c, int ft, void* out, void* stream) {
  return vae_upsample(in, t, h, w, c, ft, out, S(stream));
}
int lp_vae_frames(const float* hbuf, int t, int h, int w, int cpad, int cout, float* frames, void* stream) {
  return vae_frames(hbuf, t, h, w, cpad, cout, frames, S(stream));
}
