"""ctypes binding of liblivepipe_b200.so (include/livepipe_b200.h).

The library is the only compute path: if it is missing or fails to
initialise on a CUDA device, every op raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import re
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# LIVEPIPE_LIB points at an alternative build of the same ABI (kernel variant
# sweeps, the LP_DEBUG_HANG build); default: the in-tree library
LIB_PATH = os.environ.get("LIVEPIPE_LIB") or os.path.join(HERE, "liblivepipe_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "livepipe_b200.h")

ABI_VERSION = 8  # LP_ABI_VERSION in include/livepipe_b200.h
LP_OK, LP_EINVAL, LP_ECUDA, LP_EUNSUPPORTED, LP_ETIMEOUT, LP_EABORT = range(6)
LP_F32, LP_BF16 = 0, 1
EPI_STORE, EPI_RELU, EPI_GELU, EPI_RESID, EPI_QKV, EPI_EULER = range(6)
MAX_SEG = 66
MAX_PAIRS = 64

vp = C.c_void_p
i32, i64, u32, u64, f32 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float
fp = C.POINTER(C.c_float)


class BlockDesc(C.Structure):
    _fields_ = [
        ("block_index", i32), ("t_index", i32), ("sink_pos", i32), ("n_seg", i32),
        ("cur_row", i32), ("n_tokens", i32),
        ("seg_row", i32 * MAX_SEG), ("seg_len", i32 * MAX_SEG), ("src_row", i32 * MAX_SEG),
        ("dt", f32), ("sigma", f32), ("noise_key", u64),
        ("rope_cos", f32 * MAX_PAIRS), ("rope_sin", f32 * MAX_PAIRS),
        ("sink_cos", f32 * MAX_PAIRS), ("sink_sin", f32 * MAX_PAIRS),
        ("arena_order", i32), ("reserved_", i32),
    ]


class RopeGeom(C.Structure):
    _fields_ = [("head_dim", i32), ("t_pairs", i32), ("tokens_per_frame", i32),
                ("spatial_pairs", i32), ("spatial_cos", vp), ("spatial_sin", vp)]


class QkvEpi(C.Structure):
    _fields_ = [("d", i32), ("n_heads", i32), ("head_dim", i32), ("qk_norm", i32), ("eps", f32),
                ("g_q", vp), ("g_k", vp), ("q_out", vp), ("k_arena", vp), ("v_arena", vp),
                ("desc", vp), ("geom", RopeGeom)]


class EulerEpi(C.Structure):
    _fields_ = [("x_in", vp), ("x_out", vp), ("channels", i32), ("height", i32), ("width", i32), ("ph", i32),
                ("pw", i32), ("desc", vp), ("gate_status", vp)]


class ConvTaps(C.Structure):
    _fields_ = [("n_taps", i32), ("cin", i32), ("tap_row", i32 * 27), ("frames", i32), ("height", i32),
                ("width", i32)]


class GemmArgs(C.Structure):
    _fields_ = [("in_dtype", i32), ("out_dtype", i32), ("epilogue", i32), ("m", i32), ("n", i32),
                ("k", i32), ("lda", i64), ("ldw", i64), ("ldc", i64), ("a", vp), ("w", vp), ("c", vp),
                ("bias", vp), ("gate", vp), ("qkv", C.POINTER(QkvEpi)), ("euler", C.POINTER(EulerEpi)),
                ("conv", C.POINTER(ConvTaps)), ("fork", vp), ("row_stats", vp)]


class AttnArgs(C.Structure):
    _fields_ = [("dtype", i32), ("n_q", i32), ("n_heads", i32), ("head_dim", i32), ("scale", f32),
                ("q", vp), ("k_arena", vp), ("v_arena", vp), ("out", vp), ("desc", vp),
                ("arena_rows", i32), ("n_kv_max", i32), ("workspace", vp), ("workspace_bytes", i64),
                ("fork", vp)]


_SIGS = {
    "lp_abi_version": ([], C.c_int),
    "lp_last_error": ([], C.c_char_p),
    "lp_init": ([C.c_int], C.c_int),
    "lp_num_sms": ([], C.c_int),
    "lp_gemm": ([C.POINTER(GemmArgs), vp], C.c_int),
    "lp_qkv_post": ([vp, C.c_int, C.POINTER(QkvEpi), C.c_int, vp], C.c_int),
    "lp_attention": ([C.POINTER(AttnArgs), vp], C.c_int),
    "lp_attention_simt": ([C.POINTER(AttnArgs), vp], C.c_int),
    "lp_attention_workspace": ([C.c_int, C.c_int, C.c_int, C.POINTER(i64)], C.c_int),
    "lp_cond_row": ([vp, C.c_int, vp, vp, C.c_int, vp, vp, C.c_int, vp, vp, C.c_int, vp], C.c_int),
    "lp_add_row": ([vp, vp, vp, C.c_int, C.c_int, vp], C.c_int),
    "lp_norm_mod": ([vp, C.c_int, C.c_int, C.c_int, C.c_float, vp, vp, vp, C.c_int, vp], C.c_int),
    "lp_norm_mod_stats": ([vp, vp, C.c_int, C.c_int, C.c_int, C.c_float, vp, vp, vp, C.c_int, vp], C.c_int),
    "lp_sink_refresh": ([vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_float, vp,
                         C.POINTER(RopeGeom), vp, vp, C.c_int, C.c_int, i64, i64, vp, vp], C.c_int),
    "lp_sink_refresh_temporal": ([vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, C.POINTER(RopeGeom), vp,
                                  C.c_int, C.c_int, i64, i64, vp], C.c_int),
    "lp_silu": ([vp, vp, C.c_int, C.c_int, vp], C.c_int),
    "lp_patchify": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, vp], C.c_int),
    "lp_oracle_step": ([vp, vp, C.c_float, C.c_float, vp, vp, i64, vp], C.c_int),
    "lp_vae_pack_latent": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp], C.c_int),
    "lp_vae_norm_silu": ([vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, vp, vp], C.c_int),
    "lp_vae_upsample": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp], C.c_int),
    "lp_vae_frames": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp], C.c_int),
    "lp_unpatchify_euler": ([vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp],
                            C.c_int),
    "lp_fork_create": ([C.POINTER(vp)], C.c_int),
    "lp_fork_destroy": ([vp], C.c_int),
    "lp_graph_kernel_count": ([vp, C.POINTER(C.c_int64)], C.c_int),
    "lp_codec_patch_decode": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, C.c_int, vp, vp],
                              C.c_int),
    "lp_codec_patch_encode": ([vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, vp], C.c_int),
    "lp_history_noise": ([vp, C.c_int, C.c_int, vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, vp], C.c_int),
    "lp_history_noise_co": ([vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, vp], C.c_int),
    "lp_randn": ([vp, i64, u64, u64, C.c_float, vp], C.c_int),
    "lp_randn_bf16": ([vp, i64, u64, u64, C.c_float, vp], C.c_int),
    "lp_link_send": ([vp, vp, i64, vp, vp, u32, C.c_int, vp, u64, vp, vp], C.c_int),
    "lp_link_recv": ([vp, vp, i64, vp, vp, u32, vp, u64, vp, vp], C.c_int),
    "lp_signal": ([vp, u32, vp, vp], C.c_int),
    "lp_wait": ([vp, u32, vp, u64, vp, vp], C.c_int),
    "lp_ipc_handle": ([vp, vp, C.POINTER(i64)], C.c_int),
    "lp_ipc_open": ([vp, i64, C.POINTER(vp)], C.c_int),
    "lp_ipc_close": ([vp], C.c_int),
    "lp_peer_enable": ([C.c_int, C.c_int], C.c_int),
    "lp_vmm_create": ([C.c_int, C.c_int, i64, C.POINTER(vp)], C.c_int),
    "lp_vmm_info": ([vp, C.POINTER(u64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)], C.c_int),
    "lp_vmm_grow": ([vp, i64, vp], C.c_int),
    "lp_vmm_destroy": ([vp], C.c_int),
}


class LivepipeError(RuntimeError):
    """A liblivepipe_b200 entry point returned a non-zero status."""

    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed (code {code}): {msg}")
        self.code = code


_lib = None
_lock = threading.Lock()
_inited_devices: set = set()


def header_symbols() -> list:
    """Entry points declared in include/livepipe_b200.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"LP_API\s+(?:int|const char\*)\s+(lp_\w+)\(", text)))


def load() -> C.CDLL:
    """Load the shared library (build it with `python -m paper_2512_04677_b200.build`)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing; build it with `python -m paper_2512_04677_b200.build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            if lib.lp_abi_version() != ABI_VERSION:
                raise ImportError("liblivepipe_b200 ABI version mismatch")
            _lib = lib
    return _lib


def call(name: str, *args) -> None:
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != LP_OK:
        msg = lib.lp_last_error().decode(errors="replace")
        raise LivepipeError(name, rc, msg)


def fork_create() -> int:
    """lp_fork_create: side stream + events for lp_gemm_args.fork."""
    h = C.c_void_p()
    call("lp_fork_create", C.byref(h))
    return h.value


def graph_kernel_count(graph) -> int:
    """Kernel nodes of a captured torch.cuda.CUDAGraph (exact launches per replay)."""
    n = C.c_int64(0)
    call("lp_graph_kernel_count", C.c_void_p(int(graph.raw_cuda_graph())), C.byref(n))
    return int(n.value)


def init_device(device: int) -> None:
    if device in _inited_devices:
        return
    call("lp_init", device)
    _inited_devices.add(device)
