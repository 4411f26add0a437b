"""Model profile, seeded host weights and their device layouts.

The reference model is ``ToyDenoiser`` (denoiser.py:161-276): one token per
latent frame, additive conditioning, block-index RoPE, ReLU FFN, no norms.
``ModelProfile`` keeps those semantics as the all-flags-off case and adds the
Wan-shaped extensions the north star asks for (patch embed, pre-LN + AdaLN
shift/scale/gate, per-head q/k RMSNorm, 3-axis RoPE, GELU-tanh FFN,
modulated output head).  With every flag off the forward takes exactly the
toy code path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .numerics import F32, Prng

WEIGHT_STREAM = 1 << 44  # denoiser.py:35
WAN_EXTRA_STREAM = 1 << 47  # builder-defined, collision-free with the reference streams
TIME_FEATURES = 8  # denoiser.py:38
FFN_MULT = 2  # denoiser.py:37


@dataclass(frozen=True)
class ModelProfile:
    n_layers: int = 2
    n_heads: int = 2
    head_dim: int = 8
    ffn_dim: int = 32
    audio_dim: int = 8
    prompt_dim: int = 8
    channels: int = 0  # 0 = toy: latent frame is a flat model_dim vector, 1 token per frame
    height: int = 1
    width: int = 1
    patch: tuple = (1, 1)
    pre_ln: bool = False
    adaln: bool = False
    qk_norm: bool = False
    act: str = "relu"
    rope_axes: tuple | None = None
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
        return (self.height // self.patch[0], self.width // self.patch[1]) if self.patched else (1, 1)

    @property
    def tokens_per_frame(self) -> int:
        return self.grid[0] * self.grid[1]

    @property
    def patch_dim(self) -> int:
        return self.channels * self.patch[0] * self.patch[1] if self.patched else self.model_dim

    @property
    def latent_dim(self) -> int:
        return self.channels * self.height * self.width if self.patched else self.model_dim

    @property
    def out_dim(self) -> int:
        return self.patch_dim

    @property
    def axes(self) -> tuple:
        return self.rope_axes if self.rope_axes is not None else (self.head_dim, 0, 0)

    def params(self) -> int:
        d, f = self.model_dim, self.ffn_dim
        per_layer = 4 * d * d + 2 * d * f
        extra = (self.audio_dim + self.prompt_dim + TIME_FEATURES) * d + d * self.out_dim
        if self.patched:
            extra += self.patch_dim * d
        if self.adaln:
            extra += 6 * d * d
        return self.n_layers * per_layer + extra

    def flops_per_forward(self, n_tokens: int, n_kv: int) -> float:
        """Algorithmic FLOPs of one block forward:
        L * [2 N (4 d^2 + 2 d d_ff) + 4 N N_kv d] (projections + attention)."""
        d, f = self.model_dim, self.ffn_dim
        return float(self.n_layers * (2 * n_tokens * (4 * d * d + 2 * d * f) + 4 * n_tokens * n_kv * d))


TOY = ModelProfile()


def toy_profile(n_layers=2, n_heads=2, head_dim=8, audio_dim=8, prompt_dim=8, ffn_dim=None) -> ModelProfile:
    d = n_heads * head_dim
    return ModelProfile(n_layers=n_layers, n_heads=n_heads, head_dim=head_dim,
                        ffn_dim=ffn_dim if ffn_dim is not None else FFN_MULT * d,
                        audio_dim=audio_dim, prompt_dim=prompt_dim)


def wan_profile(n_layers, n_heads, head_dim=128, ffn_dim=None, channels=16, height=60, width=104,
                audio_dim=8, prompt_dim=8) -> ModelProfile:
    third = head_dim // 6
    return ModelProfile(n_layers=n_layers, n_heads=n_heads, head_dim=head_dim,
                        ffn_dim=ffn_dim if ffn_dim is not None else 2 * n_heads * head_dim,
                        audio_dim=audio_dim, prompt_dim=prompt_dim, channels=channels, height=height,
                        width=width, patch=(2, 2), pre_ln=True, adaln=True, qk_norm=True,
                        act="gelu_tanh", rope_axes=(head_dim - 4 * third, 2 * third, 2 * third))


# Named shapes of BASELINE.json configs.
WAN_1_3B = wan_profile(n_layers=30, n_heads=12, head_dim=128, ffn_dim=8960)
WAN_14B = wan_profile(n_layers=40, n_heads=40, head_dim=128, ffn_dim=13824)


# ---------------------------------------------------------------------------
# host weights (reference-compatible containers, denoiser.py:75-97)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class LayerWeights:
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    w1: np.ndarray
    w2: np.ndarray


@dataclass
class DenoiserWeights:
    layers: tuple
    w_audio: np.ndarray
    w_prompt: np.ndarray
    w_time: np.ndarray
    w_vel: np.ndarray
    n_heads: int
    head_dim: int
    profile: ModelProfile = field(default=TOY)
    w_emb: np.ndarray | None = None
    b_emb: np.ndarray | None = None
    w_mod: np.ndarray | None = None
    mod: np.ndarray | None = None
    g_q: np.ndarray | None = None
    g_k: np.ndarray | None = None
    mod_head: np.ndarray | None = None

    @property
    def model_dim(self) -> int:
        return self.n_heads * self.head_dim


def _draw_weights(seed: int, prof: ModelProfile):
    """The seeded draw sequence of ``build_weights``, one piece at a time:
    yields each layer's ``LayerWeights``, then a dict of the head/conditioning
    matrices, then (profiles with extensions) a dict of the extension
    tensors.  Consuming it lazily keeps one layer on the host at a time."""
    gen = Prng(seed, WEIGHT_STREAM)
    d = prof.model_dim

    def mat(rows, cols, gain=1.0):
        return gen.normal((rows, cols)) * F32(gain / np.sqrt(rows))

    for _ in range(prof.n_layers):
        wq, wk, wv = mat(d, d), mat(d, d), mat(d, d)
        wo = mat(d, d, 0.25)
        w1 = mat(d, prof.ffn_dim)
        w2 = mat(prof.ffn_dim, d, 0.25)
        yield LayerWeights(wq, wk, wv, wo, w1, w2)
    yield dict(w_audio=mat(prof.audio_dim, d), w_prompt=mat(prof.prompt_dim, d), w_time=mat(TIME_FEATURES, d),
               w_vel=mat(d, prof.out_dim, 0.5))
    if prof.patched or prof.adaln or prof.qk_norm:
        ex = Prng(seed, WAN_EXTRA_STREAM)

        def emat(rows, cols, gain):
            return ex.normal((rows, cols)) * F32(gain / np.sqrt(rows))

        w_emb = emat(prof.patch_dim, d, 1.0)
        b_emb = ex.normal(d) * F32(0.02)
        w_mod = emat(d, 6 * d, 0.1)
        mod = ex.normal((prof.n_layers, 6, d)) * F32(0.1)
        g_q = F32(1.0) + ex.normal((prof.n_layers, d)) * F32(0.05)
        g_k = F32(1.0) + ex.normal((prof.n_layers, d)) * F32(0.05)
        mod_head = ex.normal((2, d)) * F32(0.1)
        yield dict(w_emb=w_emb, b_emb=b_emb, w_mod=w_mod, mod=mod, g_q=g_q, g_k=g_k, mod_head=mod_head)


def build_weights(seed: int, n_layers: int = 2, n_heads: int = 2, head_dim: int = 8, audio_dim: int = 8,
                  prompt_dim: int = 8, profile: ModelProfile | None = None) -> DenoiserWeights:
    """Seeded host weights.  Same signature and (for the toy profile) the
    same numbers as the reference ``build_weights`` (denoiser.py:100-138):
    one Philox stream (1<<44), order wq, wk, wv, wo, w1, w2 per layer, then
    w_audio, w_prompt, w_time, w_vel; N(0,1) * gain / sqrt(rows).
    Profile extension tensors are drawn from stream 1<<47."""
    prof = profile if profile is not None else toy_profile(n_layers, n_heads, head_dim, audio_dim, prompt_dim)
    draws = _draw_weights(seed, prof)
    layers = tuple(next(draws) for _ in range(prof.n_layers))
    head = next(draws)
    w = DenoiserWeights(layers, head["w_audio"], head["w_prompt"], head["w_time"], head["w_vel"], prof.n_heads,
                        prof.head_dim, prof)
    for extra in draws:
        for k, v in extra.items():
            setattr(w, k, v)
    return w


def time_features(s: float) -> np.ndarray:
    """tau(s) = [sin(2 pi s 2^k), cos(2 pi s 2^k)]_{k<4}, fp64 -> fp32 (denoiser.py:141-145)."""
    ang = 2.0 * np.pi * s * (2.0 ** np.arange(TIME_FEATURES // 2, dtype=np.float64))
    return np.concatenate([np.sin(ang), np.cos(ang)]).astype(F32)


# ---------------------------------------------------------------------------
# device weights
# ---------------------------------------------------------------------------

class DeviceWeights:
    """Weights resident in HBM in the layout the kernels consume.

    fp32 (validation) mode keeps the reference's (in, out) row-major layout
    (QKV concatenated to (d, 3d)); bf16 mode stores W^T (out, in) K-major
    for tcgen05 (QKV stacked to (3d, d)).  Layers are stacked in one tensor
    per matrix kind.  Conditioning/modulation vectors stay fp32.
    """

    def __init__(self, prof: ModelProfile, precision: str, device: torch.device):
        self.prof = prof
        self.precision = precision
        self.device = device
        self.dtype = torch.float32 if precision == "fp32" else torch.bfloat16
        self.ldt = L.LP_F32 if precision == "fp32" else L.LP_BF16

    # -- construction -------------------------------------------------------
    def _f32(self, a) -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(self.device)

    def _mm(self, a) -> torch.Tensor:
        """A (in, out) host matrix in the kernel layout: fp32 (in, out) or bf16 W^T (out, in)."""
        if self.precision == "fp32":
            return self._f32(a)
        return self._f32(np.ascontiguousarray(np.asarray(a).T)).to(torch.bfloat16)

    def _qkv(self, x: LayerWeights) -> torch.Tensor:
        if self.precision == "fp32":
            return self._f32(np.concatenate([x.wq, x.wk, x.wv], axis=1))
        return self._f32(np.concatenate([x.wq.T, x.wk.T, x.wv.T], axis=0)).to(torch.bfloat16)

    def _alloc_layers(self) -> None:
        p, nl, d, f = self.prof, self.prof.n_layers, self.prof.model_dim, self.prof.ffn_dim
        t = lambda *shape: torch.empty(shape, dtype=self.dtype, device=self.device)  # noqa: E731
        if self.precision == "fp32":
            self.wqkv, self.wo, self.w1, self.w2 = t(nl, d, 3 * d), t(nl, d, d), t(nl, d, f), t(nl, f, d)
        else:
            self.wqkv, self.wo, self.w1, self.w2 = t(nl, 3 * d, d), t(nl, d, d), t(nl, f, d), t(nl, d, f)

    def _put_layer(self, l: int, x: LayerWeights) -> None:
        self.wqkv[l].copy_(self._qkv(x))
        self.wo[l].copy_(self._mm(x.wo))
        self.w1[l].copy_(self._mm(x.w1))
        self.w2[l].copy_(self._mm(x.w2))

    def _put_rest(self, w) -> None:
        """Head, conditioning and extension tensors from an object/namespace
        with the DenoiserWeights attribute names."""
        prof, f32 = self.prof, self._f32
        self.w_vel = self._mm(w.w_vel)
        self.w_audio, self.w_prompt, self.w_time = f32(w.w_audio), f32(w.w_prompt), f32(w.w_time)
        self.w_emb = self._mm(w.w_emb) if prof.patched else None
        self.b_emb = f32(w.b_emb) if prof.patched else None
        if prof.adaln:
            self.w_mod = self._mm(w.w_mod)
            self.mod = f32(w.mod.reshape(prof.n_layers, 6 * prof.model_dim))
            self.mod_head = f32(w.mod_head.reshape(-1))
        else:
            self.w_mod = self.mod = self.mod_head = None
        self.g_q = f32(w.g_q) if prof.qk_norm else None
        self.g_k = f32(w.g_k) if prof.qk_norm else None

    @classmethod
    def from_seed(cls, seed: int, prof: ModelProfile, precision: str, devices) -> list:
        """The reference-seeded weights (``build_weights``, bitwise the same
        numbers) drawn one layer at a time and uploaded to every device in
        ``devices`` as they are drawn: host memory holds one layer, not the
        whole model (39 GB fp32 at the 14B shape)."""
        dws = [cls(prof, precision, torch.device(dv)) for dv in devices]
        for dw in dws:
            dw._alloc_layers()
        draws = _draw_weights(seed, prof)
        for l in range(prof.n_layers):
            x = next(draws)
            for dw in dws:
                dw._put_layer(l, x)
        rest = type("_Rest", (), {})()
        for part in draws:
            for k, v in part.items():
                setattr(rest, k, v)
        for dw in dws:
            dw._put_rest(rest)
        return dws

    @classmethod
    def from_host(cls, w: DenoiserWeights, prof: ModelProfile, precision: str, device) -> "DeviceWeights":
        dw = cls(prof, precision, torch.device(device))
        dw._alloc_layers()
        for l, x in enumerate(w.layers):
            dw._put_layer(l, x)
        dw._put_rest(w)
        return dw

    @classmethod
    def random(cls, prof: ModelProfile, precision: str, device, seed: int = 7) -> "DeviceWeights":
        """Random-init weights generated on the device (perf runs at 1.3B/14B
        shape): N(0,1) * gain / sqrt(fan_in) with the reference's gains,
        drawn by the library's Philox kernel straight into the kernel layout."""
        dw = cls(prof, precision, torch.device(device))
        d, f, nl = prof.model_dim, prof.ffn_dim, prof.n_layers
        stream = torch.cuda.current_stream(dw.device).cuda_stream
        counter = [0]

        def rnd(shape, fan_in, gain=1.0, dtype=None):
            dtype = dtype or dw.dtype
            t = torch.empty(shape, dtype=dtype, device=dw.device)
            counter[0] += 1
            fn = "lp_randn_bf16" if dtype == torch.bfloat16 else "lp_randn"
            L.call(fn, t.data_ptr(), t.numel(), seed, (WAN_EXTRA_STREAM << 1) + counter[0],
                   float(gain / math.sqrt(fan_in)), stream)
            return t

        if precision == "fp32":
            dw.wqkv = rnd((nl, d, 3 * d), d)
            dw.wo, dw.w1, dw.w2 = rnd((nl, d, d), d, 0.25), rnd((nl, d, f), d), rnd((nl, f, d), f, 0.25)
            dw.w_vel = rnd((d, prof.out_dim), d, 0.5)
        else:
            dw.wqkv = rnd((nl, 3 * d, d), d)
            dw.wo, dw.w1, dw.w2 = rnd((nl, d, d), d, 0.25), rnd((nl, f, d), d), rnd((nl, d, f), f, 0.25)
            dw.w_vel = rnd((prof.out_dim, d), d, 0.5)
        fp = torch.float32
        dw.w_audio = rnd((prof.audio_dim, d), prof.audio_dim, dtype=fp)
        dw.w_prompt = rnd((prof.prompt_dim, d), prof.prompt_dim, dtype=fp)
        dw.w_time = rnd((TIME_FEATURES, d), TIME_FEATURES, dtype=fp)
        if prof.patched:
            dw.w_emb = rnd((prof.patch_dim, d) if precision == "fp32" else (d, prof.patch_dim), prof.patch_dim)
            dw.b_emb = rnd((d,), 1, 0.02, dtype=fp)
        else:
            dw.w_emb = dw.b_emb = None
        if prof.adaln:
            dw.w_mod = rnd((d, 6 * d) if precision == "fp32" else (6 * d, d), d, 0.1)
            dw.mod = rnd((nl, 6 * d), 1, 0.1, dtype=fp)
            dw.mod_head = rnd((2 * d,), 1, 0.1, dtype=fp)
        else:
            dw.w_mod = dw.mod = dw.mod_head = None
        if prof.qk_norm:
            dw.g_q = rnd((nl, d), 1, 0.05, dtype=fp) + 1.0
            dw.g_k = rnd((nl, d), 1, 0.05, dtype=fp) + 1.0
        else:
            dw.g_q = dw.g_k = None
        return dw

    def nbytes(self) -> int:
        tot = 0
        for v in self.__dict__.values():
            if isinstance(v, torch.Tensor):
                tot += v.numel() * v.element_size()
        return tot
