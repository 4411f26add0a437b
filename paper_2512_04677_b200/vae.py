"""Decode stage, VAE stand-in: a Wan-VAE-like causal 3-D convolutional
decoder on tcgen05 implicit-GEMM convolutions.

The reference decodes with its linear codec (latent.py:150-193) on the decode
worker (engine.py:465-480); the paper's 4+1 layout puts the Wan VAE decoder
on a fifth GPU and shows the DiT pipeline halving without it
(PAPER.md:304).  No VAE weights exist offline, so this module reproduces the
decoder's *shape and cost*: random-init weights, the Wan-2.1 decoder's stage
structure (conv_in, residual blocks of RMS-norm + SiLU + 3x3x3 causal conv,
nearest x2 upsampling in space with x2 in time twice, conv_out to RGB), so a
480p block of 3 latent frames becomes 12 frames of 3 x 480 x 832 at about
47 TFLOP.  Channel widths are multiples of 64 (the tcgen05 K chunk): 384,
384, 192, 128 where the Wan decoder uses 384, 384, 192, 96.

Layout: every activation is [T][H+2][W+2][C] rows with a one-pixel zero
border; a 3x3x3 causal conv is one lp_gemm whose K walks the 27 taps
(lp_conv_taps): with the geometry given, as halo tiles of 8 x 16 pixels whose
10 x 16 window per (dt, dx) feeds the three dy taps (conv_tc_kernel), else as
constant row shifts of the A operand -- TMA zero-fills the frames before 0
(causal temporal padding) and the border pixels supply the spatial padding.
Conv outputs on border rows are don't-care; the norm / cast kernels that
build the next conv input write the border as 0.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L

TAPS = [(dt, dy, dx) for dt in (-2, -1, 0) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]


def tap_rows(h: int, w: int) -> list:
    """Row offset of each (dt, dy, dx) tap in the bordered layout."""
    hp, wp = h + 2, w + 2
    return [dt * hp * wp + dy * wp + dx for dt, dy, dx in TAPS]


class VaeDecoder:
    """``decode_into(latent, frames, stream)``: one block's latent
    [F, C*H*W] (fp32, device) -> frames [4F, 3*8H*8W] (fp32, device)."""

    def __init__(self, channels: int, height: int, width: int, device, seed: int = 7,
                 widths: tuple = (384, 384, 192, 128), res_blocks: int = 2, out_channels: int = 3,
                 eps: float = 1e-6):
        if any(c % 64 for c in widths):
            raise ValueError("VAE stand-in widths must be multiples of 64")
        self.device = torch.device(device)
        self.c_lat, self.h, self.w = channels, height, width
        self.widths, self.res_blocks, self.c_out, self.eps = widths, res_blocks, out_channels, eps
        self.c_in_pad = max(64, (channels + 63) // 64 * 64)
        self.c_out_pad = 64
        L.init_device(self.device.index or 0)
        g = torch.Generator().manual_seed(seed)

        def conv_w(cin, cout, cin_real=None):
            w = torch.randn((cout, 27, cin), generator=g) / np.sqrt(27 * (cin_real or cin))
            if cin_real is not None:
                w[:, :, cin_real:] = 0.0
            return w.reshape(cout, 27 * cin).to(self.device, torch.bfloat16).contiguous()

        c0, c1, c2, c3 = widths
        # (name, cin, cout): the conv chain, residual blocks expanded
        self.w = {"in": conv_w(self.c_in_pad, c0, channels)}
        for s, c in enumerate(widths):
            for r in range(res_blocks):
                self.w[f"s{s}r{r}a"] = conv_w(c, c)
                self.w[f"s{s}r{r}b"] = conv_w(c, c)
        self.w["up1"] = conv_w(c0, c1)
        self.w["up2"] = conv_w(c1, c2)
        self.w["up3"] = conv_w(c2, c3)
        self.w["out"] = conv_w(c3, self.c_out_pad)
        self.gamma = {c: torch.ones(c, dtype=torch.float32, device=self.device) for c in set(widths)}
        # stage geometry: (T, H, W, C); upsampling x2 in time before stages 1, 2
        self.geom = [(3, height, width, c0), (6, 2 * height, 2 * width, c1), (12, 4 * height, 4 * width, c2),
                     (12, 8 * height, 8 * width, c3)]
        self.t_up = (2, 2, 1)
        self._bufs = {}
        self._taps = {}

    # -- buffers ----------------------------------------------------------
    @staticmethod
    def rows(t: int, h: int, w: int) -> int:
        return t * (h + 2) * (w + 2)

    def _buf(self, name: str, shape: tuple, dtype) -> torch.Tensor:
        b = self._bufs.get(name)
        if b is None or b.shape != torch.Size(shape):
            b = self._bufs[name] = torch.empty(shape, dtype=dtype, device=self.device)
        return b

    def flops_per_block(self, frames: int = 3) -> float:
        """2 * rows * K * N summed over the convs of one block."""
        tot = 0.0
        t0, h0, w0, c0 = self.geom[0]
        tot += 2 * self.rows(t0, h0, w0) * 27 * self.c_in_pad * c0
        for s, (t, h, w, c) in enumerate(self.geom):
            tot += self.res_blocks * 2 * (2 * self.rows(t, h, w) * 27 * c * c)
            if s > 0:
                tc, hc, wc, cc = self.geom[s - 1]
                tot += 2 * self.rows(t, h, w) * 27 * cc * c
        t, h, w, c = self.geom[-1]
        tot += 2 * self.rows(t, h, w) * 27 * c * self.c_out_pad
        return tot * frames / 3

    # -- launches ---------------------------------------------------------
    def _conv(self, st: int, a: torch.Tensor, t: int, h: int, w: int, cin: int, wt: torch.Tensor, cout: int,
              out: torch.Tensor, resid: bool) -> None:
        key = (t, h, w, cin)
        ct = self._taps.get(key)
        if ct is None:  # with the geometry the library runs the halo-tile conv kernel
            ct = self._taps[key] = L.ConvTaps(27, cin, (C.c_int32 * 27)(*tap_rows(h, w)), t, h, w)
        args = L.GemmArgs()
        args.in_dtype, args.out_dtype = L.LP_BF16, L.LP_F32
        args.epilogue = L.EPI_RESID if resid else L.EPI_STORE
        args.m, args.n, args.k = self.rows(t, h, w), cout, 27 * cin
        args.lda, args.ldw, args.ldc = cin, 27 * cin, cout
        args.a, args.w, args.c = a.data_ptr(), wt.data_ptr(), out.data_ptr()
        args.conv = C.pointer(ct)
        L.call("lp_gemm", C.byref(args), st)

    def _norm(self, st, hbuf, t, h, w, c, mode, out) -> None:
        g = self.gamma[c].data_ptr() if mode == 1 else None
        L.call("lp_vae_norm_silu", hbuf.data_ptr(), g, t, h, w, c, mode, self.eps, out.data_ptr(), st)

    def _resblock(self, st, s, r, hbuf, tbuf, abuf, t, h, w, c) -> None:
        self._norm(st, hbuf, t, h, w, c, 1, abuf)
        self._conv(st, abuf, t, h, w, c, self.w[f"s{s}r{r}a"], c, tbuf, False)
        self._norm(st, tbuf, t, h, w, c, 1, abuf)
        self._conv(st, abuf, t, h, w, c, self.w[f"s{s}r{r}b"], c, hbuf, True)

    def decode_into(self, latent: torch.Tensor, frames: torch.Tensor, stream=None) -> None:
        """latent: [F=3, C*H*W] fp32 device; frames: [12, 3*8H*8W] fp32 device."""
        s_obj = stream if stream is not None else torch.cuda.current_stream(self.device)
        st = s_obj.cuda_stream
        t0, h0, w0, c0 = self.geom[0]
        if latent.shape[0] != t0:
            raise ValueError(f"the VAE stand-in decodes blocks of {t0} latent frames")
        lat = self._buf("lat", (self.rows(t0, h0, w0), self.c_in_pad), torch.bfloat16)
        L.call("lp_vae_pack_latent", latent.data_ptr(), t0, self.c_lat, h0, w0, self.c_in_pad, lat.data_ptr(), st)
        hb = self._buf("h0", (self.rows(t0, h0, w0), c0), torch.float32)
        self._conv(st, lat, t0, h0, w0, self.c_in_pad, self.w["in"], c0, hb, False)
        for s, (t, h, w, c) in enumerate(self.geom):
            n = self.rows(t, h, w)
            if s > 0:  # cast, nearest upsample (x2 space, x t_up time), channel-changing conv
                tp, hp_, wp_, cp = self.geom[s - 1]
                ab_prev = self._buf(f"a{s - 1}", (self.rows(tp, hp_, wp_), cp), torch.bfloat16)
                self._norm(st, hb, tp, hp_, wp_, cp, 0, ab_prev)
                ub = self._buf(f"u{s}", (n, cp), torch.bfloat16)
                L.call("lp_vae_upsample", ab_prev.data_ptr(), tp, hp_, wp_, cp, self.t_up[s - 1], ub.data_ptr(), st)
                hb = self._buf(f"h{s}", (n, c), torch.float32)
                self._conv(st, ub, t, h, w, cp, self.w[f"up{s}"], c, hb, False)
            tb = self._buf(f"t{s}", (n, c), torch.float32)
            ab = self._buf(f"a{s}", (n, c), torch.bfloat16)
            for r in range(self.res_blocks):
                self._resblock(st, s, r, hb, tb, ab, t, h, w, c)
        t, h, w, c = self.geom[-1]
        n = self.rows(t, h, w)
        ab = self._buf(f"a{len(self.geom) - 1}", (n, c), torch.bfloat16)
        self._norm(st, hb, t, h, w, c, 1, ab)
        ob = self._buf("o", (n, self.c_out_pad), torch.float32)
        self._conv(st, ab, t, h, w, c, self.w["out"], self.c_out_pad, ob, False)
        L.call("lp_vae_frames", ob.data_ptr(), t, h, w, self.c_out_pad, self.c_out, frames.data_ptr(), st)


__all__ = ["VaeDecoder", "tap_rows", "TAPS"]
