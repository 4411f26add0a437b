"""Decode-stage VAE stand-in (paper_2512_04677_b200/vae.py): the implicit-GEMM
causal 3-D convolution (lp_gemm + lp_conv_taps) and the whole decoder
against a plain PyTorch fp32 reference of the same operations on the same
bf16 operands (F.conv3d with causal temporal / zero spatial padding, RMS
norm over channels, SiLU, nearest upsampling)."""

import ctypes as C

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2512_04677_b200 import _lib as L
from paper_2512_04677_b200.vae import TAPS, VaeDecoder, tap_rows

from gpu_helpers import rel_l2

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module", autouse=True)
def _init():
    L.init_device(0)


def _to_ncthw(rows: torch.Tensor, t, h, w, c) -> torch.Tensor:
    """Bordered rows [T*(H+2)*(W+2), C] -> interior [1, C, T, H, W]."""
    x = rows.float().reshape(t, h + 2, w + 2, c)[:, 1:h + 1, 1:w + 1, :]
    return x.permute(3, 0, 1, 2).unsqueeze(0)


def _weight(wt: torch.Tensor, cin, cout) -> torch.Tensor:
    """[cout, 27*cin] tap-major -> conv3d weight [cout, cin, 3, 3, 3]."""
    w = wt.float().reshape(cout, 27, cin)
    k = torch.zeros(cout, cin, 3, 3, 3, device=wt.device)
    for i, (dt, dy, dx) in enumerate(TAPS):
        k[:, :, dt + 2, dy + 1, dx + 1] = w[:, i, :]
    return k


def _conv_ref(x, k):
    """Causal in time (2 frames of zeros in front), zero-padded 1 in H and W."""
    return F.conv3d(F.pad(x, (1, 1, 1, 1, 2, 0)), k)


@pytest.mark.parametrize("halo", [False, True])
@pytest.mark.parametrize("t,h,w,cin,cout", [(3, 6, 9, 64, 64), (4, 10, 7, 128, 256), (2, 5, 5, 192, 128),
                                           (3, 17, 35, 64, 192), (2, 16, 32, 128, 384)])
def test_conv_taps_gemm_matches_conv3d(t, h, w, cin, cout, halo):
    # row-shifted taps (geometry 0) and halo tiles (geometry given): ragged
    # 8 x 16 tiles at the right / bottom edges, causal frames, N = 64..384
    g = torch.Generator(device=DEV).manual_seed(t * 100 + cin)
    rows = t * (h + 2) * (w + 2)
    a = torch.randn((rows, cin), generator=g, device=DEV).to(torch.bfloat16)
    a4 = a.reshape(t, h + 2, w + 2, cin)
    a4[:, 0] = 0
    a4[:, -1] = 0
    a4[:, :, 0] = 0
    a4[:, :, -1] = 0
    wt = (torch.randn((cout, 27 * cin), generator=g, device=DEV) / np.sqrt(27 * cin)).to(torch.bfloat16)
    out = torch.full((rows, cout), float("nan"), device=DEV)
    ct = L.ConvTaps(27, cin, (C.c_int32 * 27)(*tap_rows(h, w)), *((t, h, w) if halo else (0, 0, 0)))
    args = L.GemmArgs()
    args.in_dtype, args.out_dtype, args.epilogue = L.LP_BF16, L.LP_F32, L.EPI_STORE
    args.m, args.n, args.k = rows, cout, 27 * cin
    args.lda, args.ldw, args.ldc = cin, 27 * cin, cout
    args.a, args.w, args.c = a.data_ptr(), wt.data_ptr(), out.data_ptr()
    args.conv = C.pointer(ct)
    L.call("lp_gemm", C.byref(args), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = _to_ncthw(out, t, h, w, cout)
    ref = _conv_ref(_to_ncthw(a, t, h, w, cin), _weight(wt, cin, cout))
    assert rel_l2(got.cpu(), ref.cpu()) < 1e-5


def _decoder_ref(dec: VaeDecoder, latent: torch.Tensor) -> torch.Tensor:
    """The same decoder in fp32 torch ops, conv inputs rounded to bf16 where
    the device path stores bf16."""
    bf = lambda x: x.to(torch.bfloat16).float()  # noqa: E731

    def rms_silu(x, c):
        y = x * torch.rsqrt((x * x).mean(dim=1, keepdim=True) + dec.eps) * dec.gamma[c].view(1, c, 1, 1, 1)
        return bf(F.silu(y))

    t0, h0, w0, c0 = dec.geom[0]
    x = latent.reshape(t0, dec.c_lat, h0, w0).permute(1, 0, 2, 3).unsqueeze(0)
    x = F.pad(bf(x), (0, 0, 0, 0, 0, 0, 0, dec.c_in_pad - dec.c_lat))
    h = _conv_ref(x, _weight(dec.w["in"], dec.c_in_pad, c0))
    for s, (t, hh, ww, c) in enumerate(dec.geom):
        if s > 0:
            cp = dec.geom[s - 1][3]
            u = bf(h)
            u = u.repeat_interleave(dec.t_up[s - 1], dim=2).repeat_interleave(2, dim=3).repeat_interleave(2, dim=4)
            h = _conv_ref(u, _weight(dec.w[f"up{s}"], cp, c))
        for r in range(dec.res_blocks):
            tt = _conv_ref(rms_silu(h, c), _weight(dec.w[f"s{s}r{r}a"], c, c))
            h = h + _conv_ref(rms_silu(tt, c), _weight(dec.w[f"s{s}r{r}b"], c, c))
    c = dec.geom[-1][3]
    o = _conv_ref(rms_silu(h, c), _weight(dec.w["out"], c, dec.c_out_pad))[:, :dec.c_out]
    return o[0].permute(1, 0, 2, 3).reshape(o.shape[2], -1)  # [T, 3*H*W]


def test_vae_decoder_matches_torch_reference():
    c, h, w = 16, 6, 10
    dec = VaeDecoder(c, h, w, DEV, seed=3, widths=(128, 64, 64, 64), res_blocks=1)
    g = torch.Generator(device=DEV).manual_seed(5)
    latent = torch.randn((3, c * h * w), generator=g, device=DEV)
    frames = torch.full((12, 3 * 64 * h * w), float("nan"), device=DEV)
    dec.decode_into(latent, frames)
    torch.cuda.synchronize()
    ref = _decoder_ref(dec, latent)
    assert torch.isfinite(frames).all()
    assert rel_l2(frames.cpu(), ref.cpu()) < 2e-2


def test_vae_decoder_480p_block_shape_and_cost():
    # the benched geometry: 3 x 16 x 60 x 104 latent -> 12 x 3 x 480 x 832
    dec = VaeDecoder(16, 60, 104, DEV)
    latent = torch.randn((3, 16 * 60 * 104), device=DEV)
    frames = torch.empty((12, 3 * 480 * 832), device=DEV)
    dec.decode_into(latent, frames)
    dec.decode_into(latent, frames)  # repeatable, buffers reused
    torch.cuda.synchronize()
    assert torch.isfinite(frames).all()
    assert 40e12 < dec.flops_per_block() < 60e12
