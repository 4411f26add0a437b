"""Device runtime for one block forward: KV arena, workspace, launch sequence.

One ``Forward`` = the body of ``ToyDenoiser.denoise_block`` (denoiser.py:201-276)
plus the flow step (latent.py:140-147), as a fixed sequence of kernel
launches that reads every per-call quantity (block index, t_index, cache
view, sink position, dt, conditioning inputs) from device buffers written by
one small host->device copy.  The sequence can therefore be captured once in
a CUDA graph and replayed for every block of a stream.

HBM layout of one timestep's KV arena (``KvArena``), per layer, rows of d:

    [ sink S rows | ring slot 0 .. n_slots-1 (N rows each) | scratch hist_max*N ]

The sink rows hold the sink K/V rotated at i + delta (refreshed per block),
ring slot s holds the cache entry of some block (slot = i mod (L+1) in the
engine), the scratch rows hold the history-noise-corrupted view when
sigma > 0 (kvcache.py:121-137; the ring itself is never modified).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import time

import numpy as np
import torch

from . import _lib as L
from .model import DeviceWeights, ModelProfile, time_features
from .numerics import F32, rope_table, spatial_tables


def _p(t) -> int:
    return 0 if t is None else t.data_ptr()


def wait_event(ev) -> None:
    """Block until ``ev`` completes WITHOUT holding the GIL while the device
    works (the threaded TPP runner's stages enqueue each other's producers;
    a GIL-holding CUDA sync in one thread could starve them)."""
    if ev is None:
        return
    while not ev.query():
        time.sleep(2e-5)


def prewarm_torch(device) -> None:
    """Load the torch kernels the stage runners launch while link kernels may
    be spinning (fill / zeros / copies), so lazy module loading never happens
    concurrently with a device-side wait."""
    with torch.cuda.device(device):
        a = torch.zeros(4, dtype=torch.int32, device=device)
        a.fill_(1)
        f = torch.zeros(8, dtype=torch.float32, device=device)
        f.fill_(0.5)
        f.copy_(torch.ones(8, device=device))
        b = torch.empty(8, dtype=torch.bfloat16, device=device)
        b.copy_(f)
        f.copy_(b)
        torch.cuda.synchronize(device)


def h2d(dst: torch.Tensor, src_host, stream) -> torch.Event:
    """Asynchronous host->device copy through a fresh pinned staging tensor;
    returns the completion event (the staging tensor is kept alive by it)."""
    t = torch.as_tensor(np.ascontiguousarray(src_host)) if not isinstance(src_host, torch.Tensor) else src_host
    if not t.is_pinned():
        t = t.pin_memory()
    with torch.cuda.stream(stream):
        dst.copy_(t.reshape(dst.shape), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
    ev._keep = t  # noqa: SLF001  keep the pinned source alive until the copy completes
    return ev


def compute_stream(device) -> "torch.cuda.Stream":
    """The stream a forward is launched on: high priority, so the side
    branches it forks (lp_fork_create streams, the lowest priority) only take
    SMs its own grids leave idle."""
    return torch.cuda.Stream(device, priority=-1)


class KvArena:
    """K and V of one timestep cache: two [n_layers, rows, d] device tensors."""

    def __init__(self, prof: ModelProfile, n_tokens: int, n_slots: int, hist_max: int, dtype: torch.dtype,
                 device):
        self.prof = prof
        self.n_tokens = n_tokens
        self.s_tokens = prof.tokens_per_frame
        self.n_slots = n_slots
        self.hist_max = hist_max
        self.rows = self.s_tokens + n_slots * n_tokens + hist_max * n_tokens
        d = prof.model_dim
        self.k = torch.zeros((prof.n_layers, self.rows, d), dtype=dtype, device=device)
        self.v = torch.zeros((prof.n_layers, self.rows, d), dtype=dtype, device=device)

    @property
    def layer_stride(self) -> int:
        return self.rows * self.prof.model_dim

    def slot_row(self, slot: int) -> int:
        return self.s_tokens + slot * self.n_tokens

    def scratch_row(self, e: int) -> int:
        return self.s_tokens + self.n_slots * self.n_tokens + e * self.n_tokens

    def read_slot(self, slot: int):
        """Host copy of one ring slot: (keys, values) tuples over layers, fp32."""
        r = self.slot_row(slot)
        k = self.k[:, r:r + self.n_tokens].float().cpu().numpy()
        v = self.v[:, r:r + self.n_tokens].float().cpu().numpy()
        return tuple(k[l] for l in range(k.shape[0])), tuple(v[l] for l in range(v.shape[0]))

    def write_slot(self, slot: int, keys, values) -> None:
        r = self.slot_row(slot)
        kt = torch.from_numpy(np.stack([np.asarray(x, F32) for x in keys])).to(self.k.device, self.k.dtype)
        vt = torch.from_numpy(np.stack([np.asarray(x, F32) for x in values])).to(self.v.device, self.v.dtype)
        self.k[:, r:r + self.n_tokens].copy_(kt)
        self.v[:, r:r + self.n_tokens].copy_(vt)

    def nbytes(self) -> int:
        return 2 * self.k.numel() * self.k.element_size()


class _DeviceArray:
    """``__cuda_array_interface__`` exporter: a torch view of raw device memory."""

    def __init__(self, ptr: int, shape: tuple, strides: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": shape, "strides": strides, "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


class GrowableArena:
    """A KV arena whose ring slots are backed on demand (lp_vmm, CUDA virtual
    memory), for the drop-in denoiser.

    Same addressing as ``KvArena`` -- per layer, rows of d, one base pointer
    per layer ``layer_stride`` elements apart -- so every kernel runs on it
    unchanged.  Rows: [head_rows (sink regions) | slot 0 | slot 1 | ...].
    ``ensure_slots(n)`` maps physical HBM for slots [0, n) of every layer;
    the base never moves, so launches already enqueued (and other threads'
    workspaces) keep valid addresses while the arena grows.  ``rows`` is the
    number of backed rows (the TMA bound of the attention descriptors)."""

    def __init__(self, prof: ModelProfile, n_tokens: int, head_rows: int, dtype: torch.dtype, device,
                 max_slots: int | None = None):
        self.prof = prof
        self.n_tokens = n_tokens
        self.s_tokens = prof.tokens_per_frame
        self.head_rows = head_rows
        self.hist_max = 0
        self.n_slots = 0
        self.dtype = dtype
        self.device = torch.device(device)
        dev = self.device.index or 0
        d = prof.model_dim
        esz = torch.tensor([], dtype=dtype).element_size()
        self._row_bytes = d * esz
        if max_slots is None:
            # never more than the device could back: total HBM over K and V
            total = torch.cuda.get_device_properties(dev).total_memory
            max_slots = max(1, total // (2 * prof.n_layers * n_tokens * self._row_bytes))
        self.max_slots = int(min(max_slots, 4096, (2 ** 31 - 1 - head_rows) // n_tokens))
        self.max_rows = head_rows + self.max_slots * n_tokens
        if self.max_rows >= 2 ** 31:
            raise ValueError("arena rows exceed the int32 row index of lp_block_desc")
        lib = L.load()
        self._h = []
        views = []
        for _ in range(2):
            h = C.c_void_p()
            L.call("lp_vmm_create", dev, prof.n_layers, self.max_rows * self._row_bytes, C.byref(h))
            self._h.append(h)
            base, stride = C.c_uint64(), C.c_int64()
            lib.lp_vmm_info(h, C.byref(base), C.byref(stride), None, None)
            self._stride_bytes = int(stride.value)
            typestr = "<f4" if dtype == torch.float32 else "<i2"
            t = torch.as_tensor(_DeviceArray(int(base.value), (prof.n_layers, self.max_rows, d),
                                             (self._stride_bytes, self._row_bytes, esz), typestr),
                                device=self.device)
            views.append(t if dtype == torch.float32 else t.view(dtype))
        self.k, self.v = views
        self.rows = 0

    @property
    def layer_stride(self) -> int:
        return self._stride_bytes // self.k.element_size()

    def slot_row(self, slot: int) -> int:
        return self.head_rows + slot * self.n_tokens

    def ensure_slots(self, n: int, stream=None) -> None:
        """Back slots [0, n) of every layer (zero-filled on first mapping)."""
        if n <= self.n_slots:
            return
        if n > self.max_slots:
            raise RuntimeError(f"KV arena exhausted: {n} live slots requested, the device holds at most "
                               f"{self.max_slots} at this shape")
        rows = self.head_rows + n * self.n_tokens
        st = stream.cuda_stream if stream is not None else 0
        for h in self._h:
            L.call("lp_vmm_grow", h, rows * self._row_bytes, st)
        mapped = C.c_int64()
        L.load().lp_vmm_info(self._h[0], None, None, C.byref(mapped), None)
        self.rows = min(self.max_rows, int(mapped.value) // self._row_bytes)
        self.n_slots = n

    def nbytes(self) -> int:
        return 2 * self.rows * self._row_bytes * self.prof.n_layers

    def __del__(self):
        hs, self._h = getattr(self, "_h", []), []
        for h in hs:
            try:
                L.load().lp_vmm_destroy(h)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass


class Forward:
    """Workspace + launch sequence of one block forward on one device/stream."""

    def __init__(self, dw: DeviceWeights, n_frames: int, arena: KvArena):
        self.dw = dw
        self.prof = prof = dw.prof
        self.arena = arena
        self.device = dw.device
        self.n_frames = n_frames
        self.n_tokens = n_frames * prof.tokens_per_frame
        assert arena.n_tokens == self.n_tokens
        N, d, f = self.n_tokens, prof.model_dim, prof.ffn_dim
        dev, dt = self.device, dw.dtype
        fp = torch.float32
        self.fp32 = dw.precision == "fp32"
        self.h = torch.zeros((N, d), dtype=fp, device=dev)
        self.xa = torch.zeros((N, d), dtype=dt, device=dev)
        self.q = torch.zeros((N, d), dtype=dt, device=dev)
        self.att = torch.zeros((N, d), dtype=dt, device=dev)
        self.act = torch.zeros((N, f), dtype=dt, device=dev)
        self.qkv = torch.zeros((N, 3 * d), dtype=fp, device=dev) if self.fp32 else None
        # LP_NORM_STATS=1 (bf16 pre-LN profiles): the RESID GEMMs (O-proj,
        # FFN-down) write the LayerNorm partials of the h rows they update and
        # every later norm is one apply pass (lp_norm_mod_stats); layer 0's
        # input comes from the embedding and keeps the full lp_norm_mod.  Off
        # by default: measured 0.3 % slower at 14B (apply pass 46 us vs the
        # register-resident two-pass kernel's 39.5 us).
        self.stats_on = (not self.fp32 and prof.pre_ln and d % 32 == 0
                         and os.environ.get("LP_NORM_STATS") is not None)
        self.row_stats = torch.zeros((N, d // 32, 2), dtype=fp, device=dev) if self.stats_on else None
        self.vel = torch.zeros((N, prof.out_dim), dtype=fp, device=dev)
        self.tok = torch.zeros((N, prof.patch_dim), dtype=dt, device=dev) if prof.patched else None
        self.c = torch.zeros(d, dtype=fp, device=dev)
        self.bias_tot = torch.zeros(d, dtype=fp, device=dev)
        if prof.adaln:
            self.sc = torch.zeros((1, d), dtype=dt, device=dev)
            self.e = torch.zeros((1, 6 * d), dtype=fp, device=dev)
            self.mods = torch.zeros((prof.n_layers, 6 * d), dtype=fp, device=dev)
            self.hmod = torch.zeros(2 * d, dtype=fp, device=dev)
        lat = prof.latent_dim
        self.x_in = torch.zeros((n_frames, lat), dtype=fp, device=dev)
        self.x_out = torch.zeros((n_frames, lat), dtype=fp, device=dev)
        # inputs staged per call: [desc | tau(8) | audio | prompt]
        self._desc_bytes = C.sizeof(L.BlockDesc)
        self._in_floats = 8 + prof.audio_dim + prof.prompt_dim
        self._stage_bytes = self._desc_bytes + 4 * self._in_floats
        self.inbuf = torch.zeros(self._stage_bytes, dtype=torch.uint8, device=dev)
        self._pinned = torch.zeros(self._stage_bytes, dtype=torch.uint8, pin_memory=True)
        self._copy_done = None
        self.desc_ptr = self.inbuf.data_ptr()
        base = self.inbuf.data_ptr() + self._desc_bytes
        self.tau_ptr = base
        self.audio_ptr = base + 32
        self.prompt_ptr = base + 32 + 4 * prof.audio_dim
        self.audio_present = True
        # sink projections (un-rotated), per layer, fp32
        S = prof.tokens_per_frame
        self.k_raw = torch.zeros((prof.n_layers, S, d), dtype=fp, device=dev)
        self.v_raw = torch.zeros((prof.n_layers, S, d), dtype=fp, device=dev)
        self.sink_key = None
        self.sink_inv = torch.zeros((prof.n_layers, S, prof.n_heads), dtype=fp, device=dev) if prof.qk_norm else None
        # rotary geometry
        t_dim, dh, dw_ = prof.axes
        self.t_dim = t_dim
        sc, ss = spatial_tables(*prof.grid, dh, dw_, prof.rope_base)
        self._sp_cos = torch.from_numpy(sc).to(dev)
        self._sp_sin = torch.from_numpy(ss).to(dev)
        self.geom = L.RopeGeom(prof.head_dim, t_dim // 2, S, (dh + dw_) // 2, _p(self._sp_cos), _p(self._sp_sin))
        self.scale = float(F32(1.0) / F32(np.sqrt(prof.head_dim)))  # denoiser.py:174
        self.noise = None  # host-generated corruption noise for parity runs (device tensor)
        # partials of the KV-split tail of the tcgen05 attention grid
        self.attn_ws, self.attn_ws_bytes = None, 0
        if not self.fp32:
            nb = C.c_int64(0)
            L.call("lp_attention_workspace", N, prof.n_heads, prof.head_dim, C.byref(nb))
            self.attn_ws_bytes = int(nb.value)
            if self.attn_ws_bytes:
                self.attn_ws = torch.empty(self.attn_ws_bytes, dtype=torch.uint8, device=dev)
        # side stream + events: bf16 GEMMs with a ragged last 256-row block run
        # the pair tiles and the single-CTA tail concurrently (lp_gemm_args.fork)
        self.fork = None if self.fp32 else L.fork_create()
        self.graph = None
        self.lock = threading.Lock()
        self.probe = None  # optional callable(tag, 'begin'|'end', stream) for per-kernel timing

    def __del__(self):
        fork, self.fork = getattr(self, "fork", None), None
        if fork:
            try:
                L.load().lp_fork_destroy(fork)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass

    # ------------------------------------------------------------ inputs ----
    def write_inputs(self, block_index: int, t_index: int, steps: int, segments, cur_row: int,
                     sink_pos: int, dt: float, audio, prompt, sigma: float = 0.0, noise_key: int = 0,
                     stream=None, sink_row: int = 0, arena_order: bool = False) -> None:
        """Stage the per-call descriptor and conditioning inputs (one H2D copy).
        ``arena_order``: let the tcgen05 attention walk the view in arena-row
        order (engines with block-determined ring slots; lp_block_desc).

        ``segments``: list of (row, length, src_row) for the cache view,
        oldest first (the sink and the current block are added here)."""
        prof = self.prof
        d = L.BlockDesc()
        d.block_index, d.t_index, d.sink_pos = block_index, t_index, sink_pos
        segs = [(sink_row, prof.tokens_per_frame, sink_row)] + list(segments) + [(cur_row, self.n_tokens, cur_row)]
        if len(segs) > L.MAX_SEG:
            raise ValueError(f"cache view too long for the device descriptor ({len(segs) - 2} > {L.MAX_SEG - 2})")
        d.n_seg = len(segs)
        d.arena_order = int(bool(arena_order))
        d.cur_row = cur_row
        d.n_tokens = self.n_tokens
        for s, (r, n, src) in enumerate(segs):
            d.seg_row[s], d.seg_len[s], d.src_row[s] = r, n, src
        d.dt = float(F32(dt))
        d.sigma = float(F32(sigma))
        d.noise_key = noise_key & ((1 << 64) - 1)
        tp = self.t_dim // 2
        c, s = rope_table(block_index, self.t_dim, prof.rope_base)
        cs, ss = rope_table(sink_pos, self.t_dim, prof.rope_base)
        for p in range(tp):
            d.rope_cos[p], d.rope_sin[p] = float(c[p]), float(s[p])
            d.sink_cos[p], d.sink_sin[p] = float(cs[p]), float(ss[p])
        from .latent import level as _level

        tau = time_features(_level(steps, t_index))
        audio = np.asarray(audio, F32).reshape(-1)
        self.audio_present = audio.size != 0
        a = np.zeros(prof.audio_dim, F32)
        if audio.size:
            a[:] = audio
        buf = np.concatenate([tau, a, np.asarray(prompt, F32).reshape(-1)]).astype(F32)
        if self._copy_done is not None:
            wait_event(self._copy_done)
        pin = self._pinned.numpy()
        C.memmove(pin.ctypes.data, C.addressof(d), self._desc_bytes)
        pin[self._desc_bytes:] = buf.view(np.uint8)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):
            self.inbuf.copy_(self._pinned, non_blocking=True)
            self._copy_done = torch.cuda.Event()
            self._copy_done.record(st)

    # ------------------------------------------------------------- ops ------
    def _gemm(self, st, a, lda, m, k, w, ldw, n, c, ldc, epi, out_dtype=None, bias=0, gate=0, qkv=None,
              stats=0):
        args = L.GemmArgs()
        args.in_dtype = self.dw.ldt
        args.out_dtype = self.dw.ldt if out_dtype is None else out_dtype
        args.epilogue = epi
        args.m, args.n, args.k = m, n, k
        args.lda, args.ldw, args.ldc = lda, ldw, ldc
        args.a, args.w, args.c = a, w, c
        args.bias, args.gate = bias, gate
        args.qkv = C.pointer(qkv) if qkv is not None else None
        args.fork = self.fork
        args.row_stats = stats
        L.call("lp_gemm", C.byref(args), st)

    def _proj(self, st, a, m, k, w_t, n, c, ldc, epi, out_dtype=None, bias=0, gate=0, w_col0=0, qkv=None,
              stats=0):
        """y = a . W for a weight stored in the precision's layout.  fp32:
        W (k, n_total) row-major; bf16: W^T (n_total, k).  ``w_col0`` picks
        output columns [w_col0, w_col0 + n)."""
        esz = w_t.element_size()
        if self.fp32:
            ldw = w_t.shape[-1]
            wp = w_t.data_ptr() + w_col0 * esz
        else:
            ldw = w_t.shape[-1]
            wp = w_t.data_ptr() + w_col0 * ldw * esz
        self._gemm(st, a, k, m, k, wp, ldw, n, c, ldc, epi, out_dtype, bias, gate, qkv, stats)

    def _norm(self, st, mode, shift, scale, from_stats):
        """xa = modulate(norm(h)): the full row-reduction kernel, or the apply
        pass over the partials the last RESID GEMM left in row_stats."""
        prof, ldt = self.prof, self.dw.ldt
        N, d = self.n_tokens, prof.model_dim
        if from_stats and self.stats_on and mode >= 1:
            L.call("lp_norm_mod_stats", self.h.data_ptr(), self.row_stats.data_ptr(), N, d, mode, prof.eps,
                   shift or None, scale or None, self.xa.data_ptr(), ldt, st)
        else:
            L.call("lp_norm_mod", self.h.data_ptr(), N, d, mode, prof.eps, shift or None, scale or None,
                   self.xa.data_ptr(), ldt, st)

    # ---------------------------------------------------------- sink ---------
    def set_sink(self, sink_frame: torch.Tensor, stream=None) -> None:
        """Project the sink latent once per content (RSFM): un-rotated K/V
        rows for every layer (denoiser.py:187-190; B200: computed after the
        one-shot AAS swap instead of per call)."""
        prof, dw = self.prof, self.dw
        st = (stream if stream is not None else torch.cuda.current_stream(self.device)).cuda_stream
        d, S = prof.model_dim, prof.tokens_per_frame
        # scratch allocated on the first call (before any stream runs) and
        # reused: the RSFM swap arrives mid-stream in TPP, when another
        # stage's link kernel may be spinning, and must not allocate
        if getattr(self, "_sink_scratch", None) is None:
            dev = self.device
            self._sink_scratch = (
                torch.empty((1, prof.latent_dim), dtype=torch.float32, device=dev),
                torch.empty((S, prof.patch_dim), dtype=dw.dtype, device=dev) if prof.patched else None,
                torch.empty((S, d), dtype=torch.float32, device=dev) if prof.patched else None,
                torch.empty((S, d), dtype=dw.dtype, device=dev))
        sink, tok, sh, xs = self._sink_scratch
        s_obj = stream if stream is not None else torch.cuda.current_stream(self.device)
        if getattr(self, "_sink_ev", None) is not None:
            self._sink_ev.synchronize()
        self._sink_ev = h2d(sink, sink_frame.reshape(1, prof.latent_dim).float(), s_obj)
        self._sink_frame = sink
        if prof.patched:
            L.call("lp_patchify", sink.data_ptr(), 1, prof.channels, prof.height, prof.width, prof.patch[0],
                   prof.patch[1], tok.data_ptr(), dw.ldt, st)
            self._proj(st, tok.data_ptr(), S, prof.patch_dim, dw.w_emb, d, sh.data_ptr(), d, L.EPI_STORE,
                       L.LP_F32, bias=_p(dw.b_emb))
        else:
            sh = sink
        L.call("lp_norm_mod", sh.data_ptr(), S, d, 1 if prof.pre_ln else 0, prof.eps, None, None, xs.data_ptr(),
               dw.ldt, st)
        for l in range(prof.n_layers):
            w = dw.wqkv[l]
            self._proj(st, xs.data_ptr(), S, d, w, d, self.k_raw[l].data_ptr(), d, L.EPI_STORE, L.LP_F32,
                       w_col0=d)
            self._proj(st, xs.data_ptr(), S, d, w, d, self.v_raw[l].data_ptr(), d, L.EPI_STORE, L.LP_F32,
                       w_col0=2 * d)
        self._sink_tmp = (sh, xs)
        if self.sink_v_static:
            # V and the spatial rotary pairs of K do not depend on the sink
            # position: one full refresh per sink content (arena rows [0, S),
            # also storing the per-head RMS factors); the per-block refresh
            # (captured in the graph) rotates the temporal pairs only
            ar = self.arena
            L.call("lp_sink_refresh", self.k_raw.data_ptr(), self.v_raw.data_ptr(), S, d, prof.n_heads,
                   int(prof.qk_norm), _p(dw.g_k), prof.eps, self.desc_ptr, C.byref(self.geom), ar.k.data_ptr(),
                   ar.v.data_ptr(), dw.ldt, prof.n_layers, S * d, ar.layer_stride, _p(self.sink_inv), st)

    # ---------------------------------------------------------- forward ------
    def launch(self, stream=None, x_out=None) -> None:
        """Enqueue the whole block forward + Euler step on ``stream``.
        Reads x_in / inbuf, writes vel, x_out (default self.x_out) and the
        current block's K/V rows of the arena."""
        prof, dw, ar = self.prof, self.dw, self.arena
        st = (stream if stream is not None else torch.cuda.current_stream(self.device)).cuda_stream
        N, d, f, nl = self.n_tokens, prof.model_dim, prof.ffn_dim, prof.n_layers
        ldt = dw.ldt
        xo = self.x_out if x_out is None else x_out
        xo_ptr = xo if isinstance(xo, int) else xo.data_ptr()  # an int is a (peer-mapped) device address
        if self.oracle is not None:
            self._launch_oracle(st, xo_ptr)
            return
        # conditioning row (denoiser.py:178-185)
        L.call("lp_cond_row", self.audio_ptr if self.audio_present else None, prof.audio_dim,
               dw.w_audio.data_ptr(), self.prompt_ptr, prof.prompt_dim, dw.w_prompt.data_ptr(), self.tau_ptr, 8,
               dw.w_time.data_ptr(), self.c.data_ptr(), d, st)
        if prof.adaln:
            L.call("lp_silu", self.c.data_ptr(), self.sc.data_ptr(), d, ldt, st)
            self._proj(st, self.sc.data_ptr(), 1, d, dw.w_mod, 6 * d, self.e.data_ptr(), 6 * d, L.EPI_STORE,
                       L.LP_F32)
            L.call("lp_add_row", dw.mod.data_ptr(), self.e.data_ptr(), self.mods.data_ptr(), nl, 6 * d, st)
            L.call("lp_add_row", dw.mod_head.data_ptr(), self.e.data_ptr(), self.hmod.data_ptr(), 1, 2 * d, st)
        # embed (denoiser.py:236)
        if prof.patched:
            L.call("lp_patchify", self.x_in.data_ptr(), self.n_frames, prof.channels, prof.height, prof.width,
                   prof.patch[0], prof.patch[1], self.tok.data_ptr(), ldt, st)
            L.call("lp_add_row", dw.b_emb.data_ptr(), self.c.data_ptr(), self.bias_tot.data_ptr(), 1, d, st)
            self._proj(st, self.tok.data_ptr(), N, prof.patch_dim, dw.w_emb, d, self.h.data_ptr(), d,
                       L.EPI_STORE, L.LP_F32, bias=self.bias_tot.data_ptr())
        else:
            L.call("lp_add_row", self.x_in.data_ptr(), self.c.data_ptr(), self.h.data_ptr(), N, d, st)
        # sink K/V at i + delta for every layer (kvcache.py:86-90)
        self._tag("sink_refresh", "begin", stream)
        if self.sink_v_static:
            L.call("lp_sink_refresh_temporal", self.k_raw.data_ptr(), _p(self.sink_inv), prof.tokens_per_frame, d,
                   prof.n_heads, int(prof.qk_norm), _p(dw.g_k), self.desc_ptr, C.byref(self.geom), ar.k.data_ptr(),
                   ldt, nl, prof.tokens_per_frame * d, ar.layer_stride, st)
        else:
            L.call("lp_sink_refresh", self.k_raw.data_ptr(), self.v_raw.data_ptr(), prof.tokens_per_frame, d,
                   prof.n_heads, int(prof.qk_norm), _p(dw.g_k), prof.eps, self.desc_ptr, C.byref(self.geom),
                   ar.k.data_ptr(), ar.v.data_ptr(), ldt, nl, prof.tokens_per_frame * d, ar.layer_stride, None,
                   st)
        self._tag("sink_refresh", "end", stream)
        esz = ar.k.element_size()
        norm_mode = 2 if prof.adaln else (1 if prof.pre_ln else 0)
        # device-RNG history noise on the side stream: layer l's copy is forked
        # after attention(l-1) (layer 0: here) and joined before attention(l)
        ov = self._sigma_on and self.noise is None and self._hist_side is not None
        if ov:
            main = stream if stream is not None else torch.cuda.current_stream(self.device)
            side = self._hist_side
            hist_rows = self.hist_rows or ar.hist_max * N

            def noise_layer(l):
                self._hist_fork[l].record(main)
                side.wait_event(self._hist_fork[l])
                for kv, arena_t in ((0, ar.k), (1, ar.v)):
                    base = arena_t.data_ptr() + l * ar.layer_stride * esz
                    self._tag("history_noise", "begin", side)
                    L.call("lp_history_noise_co", base, d, l, kv, self.desc_ptr, hist_rows, side.cuda_stream)
                    self._tag("history_noise", "end", side)
                self._hist_join[l].record(side)

            noise_layer(0)
        for l in range(nl):
            kl = ar.k.data_ptr() + l * ar.layer_stride * esz
            vl = ar.v.data_ptr() + l * ar.layer_stride * esz
            mods = self.mods[l] if prof.adaln else None
            mp = (lambda k: mods.data_ptr() + k * d * 4) if prof.adaln else (lambda k: 0)
            # pre-attention norm / modulation
            self._tag("norm_mod", "begin", stream)
            self._norm(st, norm_mode, mp(0), mp(1), from_stats=l > 0)
            self._tag("norm_mod", "end", stream)
            epi = L.QkvEpi(d, prof.n_heads, prof.head_dim, int(prof.qk_norm), prof.eps,
                           _p(dw.g_q[l]) if prof.qk_norm else 0, _p(dw.g_k[l]) if prof.qk_norm else 0,
                           self.q.data_ptr(), kl, vl, self.desc_ptr, self.geom)
            if self.fp32:
                self._proj(st, self.xa.data_ptr(), N, d, dw.wqkv[l], 3 * d, self.qkv.data_ptr(), 3 * d,
                           L.EPI_STORE, L.LP_F32)
                L.call("lp_qkv_post", self.qkv.data_ptr(), N, C.byref(epi), ldt, st)
            else:
                if self.probe:
                    self.probe("qkv", "begin", stream)
                self._proj(st, self.xa.data_ptr(), N, d, dw.wqkv[l], 3 * d, 0, 0, L.EPI_QKV, qkv=epi)
                if self.probe:
                    self.probe("qkv", "end", stream)
            # history noise into the scratch rows (corrupted view)
            if ov:
                main.wait_event(self._hist_join[l])
            elif self._sigma_on:
                for kv, base in ((0, kl), (1, vl)):
                    self._tag("history_noise", "begin", stream)
                    L.call("lp_history_noise", base, ldt, d, _p(self.noise), nl, l, kv, self.desc_ptr,
                           self.hist_rows or ar.hist_max * N, st)
                    self._tag("history_noise", "end", stream)
            args = L.AttnArgs(ldt, N, prof.n_heads, prof.head_dim, self.scale, self.q.data_ptr(), kl, vl,
                              self.att.data_ptr(), self.desc_ptr, ar.rows, self.max_keys(), _p(self.attn_ws),
                              self.attn_ws_bytes, self.fork)
            if self.probe:
                self.probe("attention", "begin", stream)
            L.call("lp_attention", C.byref(args), st)
            if self.probe:
                self.probe("attention", "end", stream)
            if ov and l + 1 < nl:
                noise_layer(l + 1)  # its scratch rows were last read by this forward's predecessor
            if self.probe:
                self.probe("o_proj", "begin", stream)
            stats = self.row_stats.data_ptr() if self.stats_on else 0
            self._proj(st, self.att.data_ptr(), N, d, dw.wo[l], d, self.h.data_ptr(), d, L.EPI_RESID,
                       gate=mp(2), stats=stats)
            if self.probe:
                self.probe("o_proj", "end", stream)
            self._tag("norm_mod", "begin", stream)
            self._norm(st, norm_mode, mp(3), mp(4), from_stats=True)
            self._tag("norm_mod", "end", stream)
            if self.probe:
                self.probe("ffn_up", "begin", stream)
            self._proj(st, self.xa.data_ptr(), N, d, dw.w1[l], f, self.act.data_ptr(), f,
                       L.EPI_GELU if prof.act == "gelu_tanh" else L.EPI_RELU)
            if self.probe:
                self.probe("ffn_up", "end", stream)
            if self.probe:
                self.probe("ffn_down", "begin", stream)
            self._proj(st, self.act.data_ptr(), N, f, dw.w2[l], d, self.h.data_ptr(), d, L.EPI_RESID,
                       gate=mp(5), stats=stats)
            if self.probe:
                self.probe("ffn_down", "end", stream)
        # head + flow step (denoiser.py:268, latent.py:140-147)
        if prof.adaln:
            self._norm(st, 2, self.hmod.data_ptr(), self.hmod.data_ptr() + d * 4, from_stats=nl > 0)
        else:
            self._norm(st, 1 if prof.pre_ln else 0, 0, 0, from_stats=nl > 0)
        if self.fp32 or not self.fuse_euler:
            self._proj(st, self.xa.data_ptr(), N, d, dw.w_vel, prof.out_dim, self.vel.data_ptr(), prof.out_dim,
                       L.EPI_STORE, L.LP_F32)
            if prof.patched:
                L.call("lp_unpatchify_euler", self.x_in.data_ptr(), self.vel.data_ptr(), self.n_frames,
                       prof.channels, prof.height, prof.width, prof.patch[0], prof.patch[1], self.desc_ptr,
                       xo_ptr, st)
            else:
                L.call("lp_unpatchify_euler", self.x_in.data_ptr(), self.vel.data_ptr(), 1, 1, 1, N * d, 0, 0,
                       self.desc_ptr, xo_ptr, st)
        else:
            # velocity head with the flow step fused into the GEMM epilogue (K6)
            ph, pw = prof.patch if prof.patched else (0, 0)
            self._euler = L.EulerEpi(self.x_in.data_ptr(), xo_ptr, prof.channels, prof.height, prof.width,
                                     ph, pw, self.desc_ptr, self.euler_gate)
            args = L.GemmArgs()
            args.in_dtype, args.out_dtype, args.epilogue = self.dw.ldt, L.LP_F32, L.EPI_EULER
            args.m, args.n, args.k = N, prof.out_dim, d
            args.lda, args.ldw, args.ldc = d, d, prof.out_dim
            args.a, args.w, args.c = self.xa.data_ptr(), dw.w_vel.data_ptr(), 0
            args.euler = C.pointer(self._euler)
            L.call("lp_gemm", C.byref(args), st)

    # denoiser_kind='oracle': (target device tensor, level s, dt) of the
    # reference's analytic test denoiser (denoiser.py:294-343)
    oracle = None

    def set_oracle(self, target: np.ndarray, s: float, dt: float) -> None:
        t = torch.from_numpy(np.ascontiguousarray(target, dtype=np.float32)).to(self.device)
        self.oracle = (t.reshape(-1), float(F32(s)), float(F32(dt)))

    def _launch_oracle(self, st: int, xo_ptr: int) -> None:
        """OracleDenoiser.denoise_block + flow_step: the cache entry is the
        plain per-layer projections x.Wk (rotated at the block index) and
        x.Wv written into the ring slot (denoiser.py:307-322); the velocity
        (x - target)/s and the Euler step are one elementwise kernel."""
        prof, dw, ar = self.prof, self.dw, self.arena
        N, d = self.n_tokens, prof.model_dim
        esz = ar.k.element_size()
        a = self.x_in.data_ptr()
        if not self.fp32:  # bf16 GEMM operand
            L.call("lp_norm_mod", self.x_in.data_ptr(), N, d, 0, prof.eps, None, None, self.xa.data_ptr(), dw.ldt, st)
            a = self.xa.data_ptr()
        for l in range(prof.n_layers):
            kl = ar.k.data_ptr() + l * ar.layer_stride * esz
            vl = ar.v.data_ptr() + l * ar.layer_stride * esz
            epi = L.QkvEpi(d, prof.n_heads, prof.head_dim, 0, prof.eps, 0, 0, self.q.data_ptr(), kl, vl,
                           self.desc_ptr, self.geom)
            if self.fp32:
                self._proj(st, a, N, d, dw.wqkv[l], 3 * d, self.qkv.data_ptr(), 3 * d, L.EPI_STORE, L.LP_F32)
                L.call("lp_qkv_post", self.qkv.data_ptr(), N, C.byref(epi), dw.ldt, st)
            else:
                self._proj(st, a, N, d, dw.wqkv[l], 3 * d, 0, 0, L.EPI_QKV, qkv=epi)
        target, s, dt = self.oracle
        L.call("lp_oracle_step", self.x_in.data_ptr(), target.data_ptr(), s, dt, self.vel.data_ptr(), xo_ptr, N * d,
               st)

    _sigma_on = False
    # device address of a sticky link status word (TPP fused send): the
    # Euler epilogue skips its store into the peer slot when it is non-zero
    euler_gate = None

    def _tag(self, tag: str, phase: str, stream) -> None:
        if self.probe:
            self.probe(tag, phase, stream)
    # bf16: fuse the flow step into the velocity-head GEMM epilogue (engine
    # stages); the drop-in denoiser needs the raw velocity and turns it off
    fuse_euler = True
    # engine stages keep the sink at arena rows [0, S) (sink_row 0): sink V is
    # written by set_sink, not re-written every block
    sink_v_static = False

    # callers whose view length is known per call (the drop-in) set these:
    # an exact bound of visible keys, and of corrupted history rows
    kv_bound = None
    hist_rows = None

    def max_keys(self) -> int:
        """Upper bound of visible keys: sink + every ring slot (or the
        descriptor's history bound) + the current block."""
        if self.kv_bound:
            return self.kv_bound
        ar = self.arena
        hist = min(max(ar.n_slots - 1, ar.hist_max), L.MAX_SEG - 2)
        return ar.s_tokens + (hist + 1) * self.n_tokens

    _hist_side = None

    def set_history_noise(self, on: bool, noise: torch.Tensor | None = None) -> None:
        """Enable the corrupted-view path (graph topology changes with it).
        bf16 device-noise runs put the per-layer noise copies on a low-priority
        side stream (lp_history_noise_co) that overlaps them with the previous
        layer's O-proj / FFN and this layer's QKV when LP_HIST_OVERLAP=1; the
        stream and its events are created here, at setup, never while a TPP
        link kernel may spin.  Off by default: measured 6 % slower than the
        in-line kernel -- two 4-warp CTAs per SM beside a GEMM
        CTA cannot keep enough loads in flight to finish inside the window."""
        self._sigma_on = bool(on)
        self.noise = noise
        if on and not self.fp32 and self._hist_side is None and os.environ.get("LP_HIST_OVERLAP", "0") == "1":
            nl = self.prof.n_layers
            self._hist_side = torch.cuda.Stream(self.device, priority=0)
            self._hist_fork = [torch.cuda.Event() for _ in range(nl)]
            self._hist_join = [torch.cuda.Event() for _ in range(nl)]

    graph_kernels = None  # kernel nodes of the captured forward graph (exact, set on capture)

    def kernels_per_forward(self) -> int:
        """Number of kernel launches ``launch`` enqueues (gpu_launches claim):
        the captured graph's kernel-node count when there is one (it includes
        the side-stream tail GEMMs of lp_gemm's pair split), else the count
        of launch() call sites."""
        if self.graph_kernels is not None:
            return self.graph_kernels
        prof = self.prof
        n = 1 + 1 + 1  # cond_row, embed add (toy) or 3 (patched), sink refresh
        if prof.patched:
            n += 2
        if prof.adaln:
            n += 4
        # with a workspace the attention is the bounded-exponent kernel + the
        # exact rerun of flagged units (+ the combine of the KV-split tail),
        # and the persistent kernel's dynamic item queue adds its init kernel
        per_layer = 7 + (1 if self.fp32 else 0) + (2 if self._sigma_on else 0) + (2 if self.attn_ws_bytes else 0)
        if self.attn_ws_bytes and not self.fp32 and not any(
                os.environ.get(k) for k in ("LP_ATTN_STATIC", "LP_ATTN_NONPERSIST", "LP_ATTN_SINGLE", "LP_ATTN_EXACT")):
            per_layer += 1
        return n + prof.n_layers * per_layer + (3 if (self.fp32 or not self.fuse_euler) else 2)

    def velocity_host(self) -> np.ndarray:
        """(F, latent_dim) velocity of the last forward (host copy)."""
        v = self.vel.cpu().numpy()
        prof = self.prof
        if not prof.patched:
            return v.reshape(self.n_frames, prof.latent_dim)
        c, (ph, pw), (hp, wp) = prof.channels, prof.patch, prof.grid
        x = v.reshape(self.n_frames, hp, wp, c, ph, pw).transpose(0, 3, 1, 4, 2, 5)
        return np.ascontiguousarray(x).reshape(self.n_frames, prof.latent_dim)
