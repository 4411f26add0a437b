"""NumPy restatement of the livepipe hot path (TEST INFRASTRUCTURE ONLY).

Parity is pinned by tests/test_oracle_golden.py against vectors produced by
importing the reference (tests/golden/make_golden.py).  Every function cites
the reference file:line it restates; paths are relative to
/root/reference/pkg/src/livepipe/.

Two model profiles share one forward (``dit_forward``):

* ``toy`` (all extension flags off) -- the reference ToyDenoiser math,
  denoiser.py:201-276.  With ``mm=mm_pinned`` it is bit-identical to the
  reference (checked against the golden digests).
* ``wan`` -- builder-defined extensions (patch embed, pre-LN, AdaLN
  shift/scale/gate, per-head q/k RMSNorm, 3-axis RoPE, GELU-tanh FFN,
  modulated output head).  Not in the reference; with every flag off the
  function takes exactly the toy code path (tests/test_oracle_profiles.py).

The oracle never touches a GPU and is never imported by the product package.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32

# RNG stream namespaces (latent.py:21-24, denoiser.py:35, kvcache.py:22,
# engine.py:59).  The wan-profile extension tensors use a builder-chosen
# stream that cannot collide with any of them.
STREAM_CODEC = 1 << 40
STREAM_AUDIO = 1 << 41
STREAM_PROMPT = 1 << 42
STREAM_REFERENCE = 1 << 43
STREAM_WEIGHTS = 1 << 44
STREAM_CORRUPT = 1 << 45
STREAM_ORACLE_TARGET = 1 << 46
STREAM_WAN_EXTRA = 1 << 47
TIME_FEATURES = 8  # denoiser.py:38


# ---------------------------------------------------------------------------
# numerics (numerics.py)
# ---------------------------------------------------------------------------

def philox(seed: int, stream: int) -> np.random.Generator:
    """Counter-keyed Philox generator, key = [seed, stream] (numerics.py:118-130)."""
    return np.random.Generator(np.random.Philox(key=np.array([seed, stream], dtype=np.uint64)))


def normal(seed: int, stream: int, shape) -> np.ndarray:
    """Standard-normal float32 draw (numerics.py:132-143)."""
    return philox(seed, stream).standard_normal(shape, dtype=F32)


def mm_pinned(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """fp32 product, inner index accumulated in ascending order with one
    rounding for the product and one for the sum (numerics.py:50-64)."""
    a = np.asarray(a, dtype=F32)
    b = np.asarray(b, dtype=F32)
    assert a.ndim == 2 and b.ndim == 2 and a.shape[1] == b.shape[0]
    acc = np.zeros((a.shape[0], b.shape[1]), dtype=F32)
    for kk in range(a.shape[1]):
        acc += np.multiply.outer(a[:, kk], b[kk])
    return acc


def mm_f64(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Fast high-accuracy product (fp64 BLAS, rounded to fp32).  Used where
    parity is tolerance-based (the wan profile, bf16 kernels)."""
    return (np.asarray(a, np.float64) @ np.asarray(b, np.float64)).astype(F32)


def softmax_rows(v: np.ndarray) -> np.ndarray:
    """Row softmax with max subtraction (numerics.py:67-78)."""
    v = np.asarray(v, dtype=F32)
    m = np.max(v, axis=-1, keepdims=True)
    e = np.exp(v - m)
    return e / np.sum(e, axis=-1, keepdims=True, dtype=F32)


def rope_freqs(dim: int, base: float) -> np.ndarray:
    """theta_k = base^(-2k/dim), fp64 (numerics.py:81-86)."""
    return base ** (-2.0 * np.arange(dim // 2, dtype=np.float64) / dim)


def rope_cos_sin(pos, dim: int, base: float):
    """fp64 angles -> fp32 cos/sin (numerics.py:104-109).  ``pos`` may be an
    int or an array of per-row positions."""
    ang = np.multiply.outer(np.asarray(pos, dtype=np.float64), rope_freqs(dim, base))
    return np.cos(ang).astype(F32), np.sin(ang).astype(F32)


def rotate_pairs(x: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """Rotate interleaved pairs (2k, 2k+1) (numerics.py:110-115)."""
    x = np.asarray(x, dtype=F32)
    out = np.empty_like(x)
    ev, od = x[..., 0::2], x[..., 1::2]
    out[..., 0::2] = ev * cos - od * sin
    out[..., 1::2] = ev * sin + od * cos
    return out


def time_features(s: float) -> np.ndarray:
    """[sin(2 pi s 2^k), cos(2 pi s 2^k)], k < 4, fp64 -> fp32 (denoiser.py:141-145)."""
    ang = 2.0 * np.pi * s * (2.0 ** np.arange(TIME_FEATURES // 2, dtype=np.float64))
    return np.concatenate([np.sin(ang), np.cos(ang)]).astype(F32)


def attn_scale(head_dim: int) -> np.float32:
    """1/sqrt(hd) as the reference rounds it (denoiser.py:174)."""
    return F32(1.0) / F32(np.sqrt(head_dim))


# ---------------------------------------------------------------------------
# schedule / flow step (latent.py:54-88, :140-147)
# ---------------------------------------------------------------------------

def levels(steps: int) -> tuple:
    return tuple(j / steps for j in range(steps, 0, -1))


def level(steps: int, t_index: int) -> float:
    """s_j = j/T for j in 1..T; the reference uses 0 for j = 0 (denoiser.py:181)."""
    if t_index == 0:
        return 0.0
    return levels(steps)[steps - t_index]


def euler(x: np.ndarray, v: np.ndarray, dt: float) -> np.ndarray:
    """x + v * fp32(dt) (latent.py:140-147)."""
    return np.asarray(x, F32) + np.asarray(v, F32) * F32(dt)


# ---------------------------------------------------------------------------
# model profile and weights
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Profile:
    """Shape + extension flags.  All flags off and ``tokens_per_frame == 1``
    is the reference toy model (denoiser.py:161-276)."""

    n_layers: int = 2
    n_heads: int = 2
    head_dim: int = 8
    ffn_dim: int = 32
    audio_dim: int = 8
    prompt_dim: int = 8
    # latent geometry: a frame is (channels, height, width); toy uses a flat
    # latent vector of size model_dim and one token per frame.
    channels: int = 0
    height: int = 1
    width: int = 1
    patch: tuple = (1, 1)  # (ph, pw); spatial (1,2,2)-style patch embed when channels > 0
    pre_ln: bool = False
    adaln: bool = False
    qk_norm: bool = False
    act: str = "relu"  # relu | gelu_tanh
    rope_axes: tuple | None = None  # per-head (t, h, w) rotary dims; None = all temporal
    rope_base: float = 10000.0
    eps: float = 1e-6

    @property
    def model_dim(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def patched(self) -> bool:
        return self.channels > 0

    @property
    def grid(self) -> tuple:
        if not self.patched:
            return (1, 1)
        return (self.height // self.patch[0], self.width // self.patch[1])

    @property
    def tokens_per_frame(self) -> int:
        g = self.grid
        return g[0] * g[1]

    @property
    def patch_dim(self) -> int:
        return self.channels * self.patch[0] * self.patch[1] if self.patched else self.model_dim

    @property
    def latent_dim(self) -> int:
        """Per-frame latent size (LatentBlock.values has shape (F, latent_dim))."""
        return self.channels * self.height * self.width if self.patched else self.model_dim

    @property
    def axes(self) -> tuple:
        return self.rope_axes if self.rope_axes is not None else (self.head_dim, 0, 0)


TOY = Profile()


def wan_profile(n_layers, n_heads, head_dim=128, ffn_dim=None, channels=16, height=60,
                width=104, audio_dim=8, prompt_dim=8) -> Profile:
    """Wan-shaped profile: (1,2,2) patches, pre-LN + AdaLN, per-head q/k RMSNorm,
    3-axis RoPE split (hd - 4*(hd//6), 2*(hd//6), 2*(hd//6)), GELU-tanh FFN."""
    third = head_dim // 6
    return Profile(
        n_layers=n_layers, n_heads=n_heads, head_dim=head_dim,
        ffn_dim=ffn_dim if ffn_dim is not None else 2 * n_heads * head_dim,
        audio_dim=audio_dim, prompt_dim=prompt_dim,
        channels=channels, height=height, width=width, patch=(2, 2),
        pre_ln=True, adaln=True, qk_norm=True, act="gelu_tanh",
        rope_axes=(head_dim - 4 * third, 2 * third, 2 * third),
    )


@dataclass
class Weights:
    """Row-major (in, out) matrices, y = x @ W, as the reference stores them
    (denoiser.py:75-97).  Extension tensors are None for the toy profile."""

    wq: list
    wk: list
    wv: list
    wo: list
    w1: list
    w2: list
    w_audio: np.ndarray
    w_prompt: np.ndarray
    w_time: np.ndarray
    w_vel: np.ndarray  # toy head (d, d); wan: (d, patch_dim)
    w_emb: np.ndarray | None = None  # (patch_dim, d)
    b_emb: np.ndarray | None = None  # (d,)
    w_mod: np.ndarray | None = None  # (d, 6d)
    mod: np.ndarray | None = None  # (L, 6, d)
    g_q: np.ndarray | None = None  # (L, d)
    g_k: np.ndarray | None = None  # (L, d)
    mod_head: np.ndarray | None = None  # (2, d)


def build_weights(seed: int, prof: Profile) -> Weights:
    """Seeded weights.  The toy part is drawn from one Philox stream (1<<44)
    in the reference order wq,wk,wv,wo,w1,w2 per layer, then w_audio,
    w_prompt, w_time, w_vel, each N(0,1)*gain/sqrt(rows)
    (denoiser.py:100-138).  Extension tensors come from stream 1<<47."""
    g = philox(seed, STREAM_WEIGHTS)
    d = prof.model_dim

    def mat(rows, cols, gain=1.0):
        return g.standard_normal((rows, cols), dtype=F32) * F32(gain / np.sqrt(rows))

    wq, wk, wv, wo, w1, w2 = [], [], [], [], [], []
    for _ in range(prof.n_layers):
        wq.append(mat(d, d))
        wk.append(mat(d, d))
        wv.append(mat(d, d))
        wo.append(mat(d, d, 0.25))
        w1.append(mat(d, prof.ffn_dim))
        w2.append(mat(prof.ffn_dim, d, 0.25))
    w_audio = mat(prof.audio_dim, d)
    w_prompt = mat(prof.prompt_dim, d)
    w_time = mat(TIME_FEATURES, d)
    out_dim = prof.patch_dim if prof.patched else d
    w_vel = mat(d, out_dim, 0.5)
    w = Weights(wq, wk, wv, wo, w1, w2, w_audio, w_prompt, w_time, w_vel)
    if prof.patched or prof.adaln or prof.qk_norm:
        e = philox(seed, STREAM_WAN_EXTRA)

        def emat(rows, cols, gain):
            return e.standard_normal((rows, cols), dtype=F32) * F32(gain / np.sqrt(rows))

        w.w_emb = emat(prof.patch_dim, d, 1.0)
        w.b_emb = e.standard_normal(d, dtype=F32) * F32(0.02)
        w.w_mod = emat(d, 6 * d, 0.1)
        w.mod = e.standard_normal((prof.n_layers, 6, d), dtype=F32) * F32(0.1)
        w.g_q = F32(1.0) + e.standard_normal((prof.n_layers, d), dtype=F32) * F32(0.05)
        w.g_k = F32(1.0) + e.standard_normal((prof.n_layers, d), dtype=F32) * F32(0.05)
        w.mod_head = e.standard_normal((2, d), dtype=F32) * F32(0.1)
    return w


# ---------------------------------------------------------------------------
# geometry: patchify / positions
# ---------------------------------------------------------------------------

def patchify(prof: Profile, frames: np.ndarray) -> np.ndarray:
    """(F, C*H*W) latent frames -> (F*Hp*Wp, C*ph*pw) tokens, frame-major then
    row-major over the patch grid; within a token the order is (c, py, px)."""
    if not prof.patched:
        return np.asarray(frames, F32)
    f = frames.shape[0]
    c, (ph, pw), (hp, wp) = prof.channels, prof.patch, prof.grid
    x = np.asarray(frames, F32).reshape(f, c, hp, ph, wp, pw)
    return np.ascontiguousarray(x.transpose(0, 2, 4, 1, 3, 5)).reshape(f * hp * wp, c * ph * pw)


def unpatchify(prof: Profile, tokens: np.ndarray, frames: int) -> np.ndarray:
    if not prof.patched:
        return np.asarray(tokens, F32)
    c, (ph, pw), (hp, wp) = prof.channels, prof.patch, prof.grid
    x = np.asarray(tokens, F32).reshape(frames, hp, wp, c, ph, pw)
    return np.ascontiguousarray(x.transpose(0, 3, 1, 4, 2, 5)).reshape(frames, c * hp * ph * wp * pw)


def token_positions(prof: Profile, n_tokens: int, t_pos: int) -> np.ndarray:
    """(n, 3) integer (t, h, w) rotary positions.  Every token of a block sits
    at temporal position = block index (denoiser.py:237); h/w are patch-grid
    coordinates and are never shifted."""
    hp, wp = prof.grid
    s = hp * wp
    idx = np.arange(n_tokens) % s
    pos = np.empty((n_tokens, 3), dtype=np.int64)
    pos[:, 0] = t_pos
    pos[:, 1] = idx // wp
    pos[:, 2] = idx % wp
    return pos


def rope_tokens(prof: Profile, x: np.ndarray, pos: np.ndarray) -> np.ndarray:
    """Per-head rotation of (n, d) rows.  With the toy profile this is
    rope_rotate_rows(rows, block_index) on every head (denoiser.py:192-197)."""
    n = x.shape[0]
    hd = prof.head_dim
    heads = np.asarray(x, F32).reshape(n, prof.n_heads, hd)
    cos_parts, sin_parts = [], []
    for ax, dim in enumerate(prof.axes):
        if dim == 0:
            continue
        c, s = rope_cos_sin(pos[:, ax], dim, prof.rope_base)  # (n, dim/2)
        cos_parts.append(c)
        sin_parts.append(s)
    cos = np.concatenate(cos_parts, axis=1)[:, None, :]
    sin = np.concatenate(sin_parts, axis=1)[:, None, :]
    return rotate_pairs(heads, cos, sin).reshape(n, -1)


# ---------------------------------------------------------------------------
# normalisation / activation (wan extensions)
# ---------------------------------------------------------------------------

def layer_norm(x: np.ndarray, eps: float) -> np.ndarray:
    x64 = np.asarray(x, np.float64)
    mu = x64.mean(axis=-1, keepdims=True)
    var = ((x64 - mu) ** 2).mean(axis=-1, keepdims=True)
    return ((x64 - mu) / np.sqrt(var + eps)).astype(F32)


def head_rms_norm(prof: Profile, x: np.ndarray, g: np.ndarray) -> np.ndarray:
    n = x.shape[0]
    h = np.asarray(x, np.float64).reshape(n, prof.n_heads, prof.head_dim)
    r = h / np.sqrt((h * h).mean(axis=-1, keepdims=True) + prof.eps)
    return (r.reshape(n, -1) * g.astype(np.float64)).astype(F32)


def gelu_tanh(x: np.ndarray) -> np.ndarray:
    x64 = np.asarray(x, np.float64)
    return (0.5 * x64 * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x64 + 0.044715 * x64 ** 3)))).astype(F32)


def silu(x: np.ndarray) -> np.ndarray:
    x64 = np.asarray(x, np.float64)
    return (x64 / (1.0 + np.exp(-x64))).astype(F32)


# ---------------------------------------------------------------------------
# the forward (denoiser.py:201-276 + wan extensions)
# ---------------------------------------------------------------------------

@dataclass
class Entry:
    """KvEntry restated (denoiser.py:45-57): per-layer rotated keys, values."""

    keys: list
    values: list
    block_index: int
    timestep_index: int
    rope_index: int


class TimestepForcing(ValueError):
    pass


def check_view(view, t_index, max_entries, require_same_timestep=True):
    """Metadata rules of denoiser.py:219-234 (same level, == t_index,
    capacity, strictly increasing blocks)."""
    seen = {e.timestep_index for e in view}
    if len(seen) > 1:
        raise TimestepForcing(f"cache view mixes timestep indices {sorted(seen)}")
    if require_same_timestep and seen and seen != {t_index}:
        raise TimestepForcing(f"cache holds timestep {next(iter(seen))} but denoising at {t_index}")
    if max_entries is not None and len(view) > max_entries:
        raise ValueError(f"cache view exceeds capacity {max_entries}")
    for a, b in zip(view, view[1:]):
        if b.block_index <= a.block_index:
            raise ValueError("cache entries out of block order")


def cond_row(prof: Profile, w: Weights, steps: int, t_index: int, audio, prompt, mm) -> np.ndarray:
    """a*W_audio + p*W_prompt + tau(s)*W_time, three products summed in that
    order; empty audio means zeros (denoiser.py:178-185)."""
    audio = np.asarray(audio, F32)
    if audio.size == 0:
        audio = np.zeros(w.w_audio.shape[0], dtype=F32)
    s = level(steps, t_index)
    c = mm(audio[None, :], w.w_audio)
    c += mm(np.asarray(prompt, F32)[None, :], w.w_prompt)
    c += mm(time_features(s)[None, :], w.w_time)
    return c  # (1, d)


def modulation(prof, w, c, mm):
    """AdaLN vectors: e = silu(c) @ W_mod reshaped (6, d), per layer + mod[l]."""
    d = prof.model_dim
    return mm(silu(c), w.w_mod).reshape(6, d)


def embed_tokens(prof, w, frames, mm):
    tok = patchify(prof, frames)
    if not prof.patched:
        return tok
    return mm(tok, w.w_emb) + w.b_emb[None, :]


def sink_kv(prof, w, sink_frame, sink_pos, layer, mm):
    """Sink key/value rows for one layer: projections of the raw sink latent
    (no conditioning, no residual stream), key rotated at i + delta
    (denoiser.py:187-190, :246-249)."""
    sh = embed_tokens(prof, w, np.asarray(sink_frame, F32)[None, :], mm)
    if prof.pre_ln:
        sh = layer_norm(sh, prof.eps)
    sk = mm(sh, w.wk[layer])
    sv = mm(sh, w.wv[layer])
    if prof.qk_norm:
        sk = head_rms_norm(prof, sk, w.g_k[layer])
    pos = token_positions(prof, sh.shape[0], sink_pos)
    return rope_tokens(prof, sk, pos), sv


def attend(prof, q, keys, values, mm, mask=None):
    """Per-head softmax(q K^T * scale) V, no mask inside the visible set
    (denoiser.py:152-158, :255-264)."""
    hd = prof.head_dim
    scale = attn_scale(hd)
    outs = []
    for h in range(prof.n_heads):
        sl = slice(h * hd, (h + 1) * hd)
        logits = mm(q[:, sl], np.ascontiguousarray(keys[:, sl].T)) * scale
        if mask is not None:
            logits = logits + mask
        outs.append(mm(softmax_rows(logits), values[:, sl]))
    return np.concatenate(outs, axis=1)


def dit_forward(prof: Profile, w: Weights, steps: int, x_frames: np.ndarray, block_index: int,
                t_index: int, view, audio, prompt, sink_frame, sink_pos: int, mm=mm_pinned,
                require_same_timestep=True, max_entries=None):
    """One velocity prediction + this block's cache entry (denoiser.py:201-276)."""
    view = list(view)
    check_view(view, t_index, max_entries, require_same_timestep)
    x_frames = np.asarray(x_frames, F32)
    n_frames = x_frames.shape[0]
    c = cond_row(prof, w, steps, t_index, audio, prompt, mm)
    h = embed_tokens(prof, w, x_frames, mm) + c  # denoiser.py:236
    pos = token_positions(prof, h.shape[0], block_index)  # denoiser.py:237
    e = modulation(prof, w, c, mm) if prof.adaln else None
    out_k, out_v = [], []
    for l in range(prof.n_layers):
        if prof.adaln:
            m = w.mod[l] + e
            xa = layer_norm(h, prof.eps) * (F32(1) + m[1]) + m[0]
        elif prof.pre_ln:
            xa = layer_norm(h, prof.eps)
        else:
            xa = h
        q = mm(xa, w.wq[l])
        k = mm(xa, w.wk[l])
        v = mm(xa, w.wv[l])
        if prof.qk_norm:
            q = head_rms_norm(prof, q, w.g_q[l])
            k = head_rms_norm(prof, k, w.g_k[l])
        q = rope_tokens(prof, q, pos)
        k = rope_tokens(prof, k, pos)
        out_k.append(k)
        out_v.append(v)
        sk, sv = sink_kv(prof, w, sink_frame, sink_pos, l, mm)
        keys = np.vstack([sk] + [en.keys[l] for en in view] + [k])  # denoiser.py:248-252
        vals = np.vstack([sv] + [en.values[l] for en in view] + [v])  # denoiser.py:253
        attn = attend(prof, q, keys, vals, mm)
        o = mm(attn, w.wo[l])
        h = h + (m[2] * o if prof.adaln else o)  # denoiser.py:265
        if prof.adaln:
            xf = layer_norm(h, prof.eps) * (F32(1) + m[4]) + m[3]
        elif prof.pre_ln:
            xf = layer_norm(h, prof.eps)
        else:
            xf = h
        a = mm(xf, w.w1[l])
        a = gelu_tanh(a) if prof.act == "gelu_tanh" else np.maximum(a, F32(0.0))
        f = mm(a, w.w2[l])
        h = h + (m[5] * f if prof.adaln else f)  # denoiser.py:266
    if prof.adaln:
        xo = layer_norm(h, prof.eps) * (F32(1) + w.mod_head[1] + e[1]) + (w.mod_head[0] + e[0])
    elif prof.pre_ln:
        xo = layer_norm(h, prof.eps)
    else:
        xo = h
    vel = unpatchify(prof, mm(xo, w.w_vel), n_frames)  # denoiser.py:268
    entry = Entry(out_k, out_v, block_index, t_index, block_index)  # denoiser.py:269-275
    return vel, entry


def visible_mask(n: int, window: int) -> list:
    """Block visibility of attention_bruteforce (denoiser.py:396-407): block m
    is visible from block n iff m == n or n - window <= m <= n - 1."""
    return [(m == n) or (n - window <= m <= n - 1) for m in range(n + 1)]


# ---------------------------------------------------------------------------
# cache + RSFM (kvcache.py)
# ---------------------------------------------------------------------------

def push(cache: list, entry: Entry, capacity: int) -> None:
    """FIFO push with eviction of the oldest entry when full (kvcache.py:41-52)."""
    if cache and entry.block_index <= cache[-1].block_index:
        raise ValueError("block indices must be strictly increasing")
    if len(cache) == capacity:
        cache.pop(0)
    cache.append(entry)


def corrupt(cache: list, sigma: float, seed: int, block_index: int, t_index: int) -> list:
    """Perturbed copy of the view: per entry, keys of every layer then values
    of every layer get sigma*N(0,1) from stream 2^45 + 4096 i + j
    (kvcache.py:121-143)."""
    if sigma == 0.0:
        return list(cache)
    g = philox(seed, STREAM_CORRUPT + block_index * 4096 + t_index)
    out = []
    for en in cache:
        ks = [k + g.standard_normal(k.shape, dtype=F32) * F32(sigma) for k in en.keys]
        vs = [v + g.standard_normal(v.shape, dtype=F32) * F32(sigma) for v in en.values]
        out.append(Entry(ks, vs, en.block_index, en.timestep_index, en.rope_index))
    return out


class Codec:
    """Seeded linear decoder + pinv encoder (latent.py:150-193)."""

    def __init__(self, seed: int, latent_dim: int, pixel_dim: int, upsample: int):
        g = philox(seed, STREAM_CODEC)
        sc = F32(1.0 / np.sqrt(latent_dim))
        self.dec = [g.standard_normal((pixel_dim, latent_dim), dtype=F32) * sc for _ in range(upsample)]
        self.enc = np.linalg.pinv(self.dec[0].astype(np.float64)).astype(F32)

    def encode(self, frame):
        return mm_pinned(self.enc, np.asarray(frame, F32)[:, None])[:, 0]

    def decode(self, block_values):
        return np.concatenate([
            np.stack([mm_pinned(m, f[:, None])[:, 0] for m in self.dec]) for f in block_values
        ])


class PatchCodec:
    """Builder-defined stand-in for the video VAE on patched profiles (no
    reference counterpart): the Codec contract above
    (latent.py:150-193 -- r maps N(0,1)/sqrt(C) from the codec stream, encoder
    = float64 pinv of map 0) applied per latent location.  Latent frame
    (C, H, W); pixel frame (pc, H*s, W*s); map rows q = (ch*s + dy)*s + dx.
    Sums are pinned (ascending c for decode, ascending q for encode)."""

    def __init__(self, seed, channels, height, width, pixel_channels=3, scale=8, upsample=4):
        g = philox(seed, STREAM_CODEC)
        sc = F32(1.0 / np.sqrt(channels))
        q = pixel_channels * scale * scale
        self.C, self.H, self.W, self.pc, self.s, self.r = channels, height, width, pixel_channels, scale, upsample
        self.maps = np.stack([g.standard_normal((q, channels), dtype=F32) * sc for _ in range(upsample)])
        self.enc = np.linalg.pinv(self.maps[0].astype(np.float64)).astype(F32)

    def decode(self, block_values):
        C, H, W, pc, s, r = self.C, self.H, self.W, self.pc, self.s, self.r
        lat = np.asarray(block_values, F32).reshape(-1, C, H * W)
        out = []
        for f in range(lat.shape[0]):
            for u in range(r):
                acc = np.zeros((pc * s * s, H * W), F32)
                for c in range(C):
                    acc += np.multiply.outer(self.maps[u][:, c], lat[f, c])
                # (ch, dy, dx, h, w) -> (ch, h, dy, w, dx)
                img = acc.reshape(pc, s, s, H, W).transpose(0, 3, 1, 4, 2).reshape(-1)
                out.append(img)
        return np.stack(out)

    def encode(self, frame):
        C, H, W, pc, s = self.C, self.H, self.W, self.pc, self.s
        pix = np.asarray(frame, F32).reshape(pc, H, s, W, s).transpose(0, 2, 4, 1, 3).reshape(pc * s * s, H * W)
        acc = np.zeros((C, H * W), F32)
        for q in range(pc * s * s):
            acc += np.multiply.outer(self.enc[:, q], pix[q])
        return acc.reshape(-1)


# ---------------------------------------------------------------------------
# rollouts (engine.py:204-285, Algorithm 3 / 4)
# ---------------------------------------------------------------------------

@dataclass
class RolloutCfg:
    """EngineConfig fields that shape the math (engine.py:73-106)."""

    steps: int = 4
    cache_capacity: int = 4
    frames_per_block: int = 3
    pixel_dim: int = 32
    upsample: int = 4
    sink_delta: int = 1
    blocks: int = 8
    weight_seed: int = 7
    noise_seed: int = 11
    history_sigma: float = 0.0
    history_mode: str = "fixed"
    profile: Profile = field(default_factory=Profile)


def noise_block(cfg: RolloutCfg, i: int) -> np.ndarray:
    """N(0,1) from Philox(noise_seed, stream=i) (engine.py:204-210)."""
    return normal(cfg.noise_seed, i, (cfg.frames_per_block, cfg.profile.latent_dim))


def conditions(cfg: RolloutCfg):
    """Per-block audio (2^41+i), prompt (2^42), reference sink (2^43) (latent.py:104-117)."""
    p = cfg.profile
    audio = np.stack([normal(cfg.noise_seed, STREAM_AUDIO + i, p.audio_dim) for i in range(cfg.blocks)])
    prompt = normal(cfg.noise_seed, STREAM_PROMPT, p.prompt_dim)
    ref = normal(cfg.noise_seed, STREAM_REFERENCE, p.latent_dim)
    return audio, prompt, ref


def run_sequential(cfg: RolloutCfg, weights: Weights | None = None, mm=mm_pinned, codec=True):
    """Algorithm 3: per block, T steps against per-timestep rolling caches;
    decode; one-shot AAS after block 0 (engine.py:255-285).  Returns
    (final latents per block, decoded frames or None, final sink)."""
    p = cfg.profile
    w = weights if weights is not None else build_weights(cfg.weight_seed, p)
    audio, prompt, ref = conditions(cfg)
    cd = codec if hasattr(codec, "decode") else (Codec(cfg.weight_seed, p.latent_dim, cfg.pixel_dim, cfg.upsample)
                                                    if codec else None)
    dt = -1.0 / cfg.steps
    caches = {j: [] for j in range(1, cfg.steps + 1)}
    sink = ref.copy()
    blocks, frames = [], []
    for i in range(cfg.blocks):
        x = noise_block(cfg, i)
        for j in range(cfg.steps, 0, -1):
            sigma = cfg.history_sigma
            if cfg.history_mode == "scaled" and j >= 1:
                sigma = sigma * level(cfg.steps, j)
            view = corrupt(caches[j], sigma, cfg.noise_seed, i, j)
            vel, entry = dit_forward(p, w, cfg.steps, x, i, j, view, audio[i], prompt, sink,
                                     i + cfg.sink_delta, mm=mm, max_entries=cfg.cache_capacity)
            x = euler(x, vel, dt)
            push(caches[j], entry, cfg.cache_capacity)
        blocks.append(x)
        if cd is not None:
            frames.append(cd.decode(x))
            if i == 0:
                sink = cd.encode(cd.decode(x)[0])  # kvcache.py:93-109
        elif i == 0:
            sink = x[0].copy()
    return blocks, (np.concatenate(frames) if frames else None), sink


def run_clean_kv(cfg: RolloutCfg, weights: Weights | None = None, mm=mm_pinned, codec=True):
    """Clean-cache baseline (engine.py:292-331): one unified cache (timestep
    0) fed by an extra full-stack pass on each block's final latent at level
    0 (cache_entry, denoiser.py:278-291); every step attends to it with the
    level check lifted.  Returns (blocks, frames or None, nfe)."""
    p = cfg.profile
    w = weights if weights is not None else build_weights(cfg.weight_seed, p)
    audio, prompt, ref = conditions(cfg)
    cd = codec if hasattr(codec, "decode") else (Codec(cfg.weight_seed, p.latent_dim, cfg.pixel_dim, cfg.upsample)
                                                    if codec else None)
    dt = -1.0 / cfg.steps
    unified = []
    sink = ref.copy()
    blocks, frames, nfe = [], [], 0
    for i in range(cfg.blocks):
        x = noise_block(cfg, i)
        for j in range(cfg.steps, 0, -1):
            sigma = cfg.history_sigma
            if cfg.history_mode == "scaled" and j >= 1:
                sigma = sigma * level(cfg.steps, j)
            view = corrupt(unified, sigma, cfg.noise_seed, i, j)
            vel, _ = dit_forward(p, w, cfg.steps, x, i, j, view, audio[i], prompt, sink, i + cfg.sink_delta, mm=mm,
                                 require_same_timestep=False, max_entries=cfg.cache_capacity)
            nfe += 1
            x = euler(x, vel, dt)
        _, entry = dit_forward(p, w, cfg.steps, x, i, 0, list(unified), audio[i], prompt, sink, i + cfg.sink_delta,
                               mm=mm, require_same_timestep=False)
        nfe += 1
        push(unified, entry, cfg.cache_capacity)
        blocks.append(x)
        if cd is not None:
            frames.append(cd.decode(x))
            if i == 0:
                sink = cd.encode(cd.decode(x)[0])
        elif i == 0:
            sink = x[0].copy()
    return blocks, (np.concatenate(frames) if frames else None), nfe


def latents_bytes(blocks) -> bytes:
    """LPD1 dump: magic + (D, F, M) as little-endian u32, then the blocks'
    fp32 frames row-major, block-ascending (harness.py:254-264)."""
    import struct

    arr = np.stack([np.asarray(b, F32) for b in blocks])
    head = b"LPD1" + struct.pack("<III", arr.shape[2], arr.shape[1], arr.shape[0])
    return head + arr.astype("<f4").tobytes()


def visible_schedule(blocks: int, capacity: int) -> list:
    """Integer replay of the rolling cache: for each block i, the ordered list
    of block indices visible at every timestep (kvcache.py:41-56)."""
    cache, out = [], []
    for i in range(blocks):
        out.append(list(cache))
        cache.append(i)
        if len(cache) > capacity:
            cache.pop(0)
    return out
