"""tcgen05 GEMM (lp_gemm, LP_BF16) against a torch fp32 reference on the
same bf16 operands, for every epilogue; plus the fp32 pinned GEMM against
the reference's ascending-k order (bitwise)."""

import ctypes as C

import numpy as np
import pytest
import torch

from paper_2512_04677_b200 import _lib as L
from paper_2512_04677_b200.numerics import spatial_tables

from gpu_helpers import make_desc, rel_l2, rope_ref, upload_desc

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module", autouse=True)
def _init():
    L.init_device(0)


_FORK = []


def _fork():
    if not _FORK:
        _FORK.append(L.fork_create())
    return _FORK[0]


def _gemm(a, w_t, c, epi, out_dtype, bias=None, gate=None, qkv=None, in_dtype=L.LP_BF16, fork=False, stats=None):
    args = L.GemmArgs()
    args.row_stats = stats.data_ptr() if stats is not None else None
    args.fork = _fork() if fork else None
    args.in_dtype, args.out_dtype, args.epilogue = in_dtype, out_dtype, epi
    args.m, args.k = a.shape
    args.n = w_t.shape[0] if in_dtype == L.LP_BF16 else w_t.shape[1]
    args.lda, args.ldw = a.shape[1], w_t.shape[1]
    args.ldc = c.shape[1] if c is not None else 0
    args.a, args.w = a.data_ptr(), w_t.data_ptr()
    args.c = c.data_ptr() if c is not None else None
    args.bias = bias.data_ptr() if bias is not None else None
    args.gate = gate.data_ptr() if gate is not None else None
    args.qkv = C.pointer(qkv) if qkv is not None else None
    L.call("lp_gemm", C.byref(args), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()


def _ab(m, k, n, seed=0):
    g = torch.Generator(device=DEV).manual_seed(seed)
    a = torch.randn((m, k), generator=g, device=DEV).to(torch.bfloat16)
    w = (torch.randn((n, k), generator=g, device=DEV) / k ** 0.5).to(torch.bfloat16)
    return a, w


@pytest.mark.parametrize("m,k,n", [(128, 64, 256), (300, 256, 512), (4680 // 4, 512, 384), (77, 1024, 64),
                                   (1, 512, 768), (1000, 128, 128), (4680, 128, 13824)])
def test_store_bf16_and_f32(m, k, n):
    a, w = _ab(m, k, n)
    ref = a.float() @ w.float().T
    c32 = torch.zeros((m, n), device=DEV)
    _gemm(a, w, c32, L.EPI_STORE, L.LP_F32)
    assert rel_l2(c32.cpu(), ref.cpu()) < 1e-5
    c16 = torch.zeros((m, n), device=DEV, dtype=torch.bfloat16)
    bias = torch.randn(n, device=DEV)
    _gemm(a, w, c16, L.EPI_STORE, L.LP_BF16, bias=bias)
    assert rel_l2(c16.float().cpu(), (ref + bias).cpu()) < 5e-3


@pytest.mark.parametrize("epi", [L.EPI_RELU, L.EPI_GELU])
def test_activation_epilogues(epi):
    m, k, n = 333, 320, 768
    a, w = _ab(m, k, n, 1)
    ref = a.float() @ w.float().T
    ref = torch.relu(ref) if epi == L.EPI_RELU else torch.nn.functional.gelu(ref, approximate="tanh")
    c = torch.zeros((m, n), device=DEV, dtype=torch.bfloat16)
    _gemm(a, w, c, epi, L.LP_BF16)
    assert rel_l2(c.float().cpu(), ref.cpu()) < 5e-3


@pytest.mark.parametrize("m,k,n", [(600, 256, 512), (4680, 512, 1024), (300, 128, 15360 // 4)])
def test_pair_split_with_side_stream_tail(monkeypatch, m, k, n):
    # pair tiles on rows [0, 256 * floor(m / 256)), single-CTA tail rows on the
    # fork's side stream: same results as one launch, for STORE and RESID
    monkeypatch.setenv("LP_PAIR_SPLIT_ALL", "1")
    a, w = _ab(m, k, n, 5)
    ref = a.float() @ w.float().T
    c32 = torch.full((m, n), float("nan"), device=DEV)
    _gemm(a, w, c32, L.EPI_STORE, L.LP_F32, fork=True)
    assert rel_l2(c32.cpu(), ref.cpu()) < 1e-5
    h = torch.randn((m, n), device=DEV)
    gate = torch.randn(n, device=DEV)
    want = h + gate * ref
    _gemm(a, w, h, L.EPI_RESID, L.LP_F32, gate=gate, fork=True)
    assert rel_l2(h.cpu(), want.cpu()) < 1e-5
    # and bitwise the same as the unsplit launch (same per-tile k order)
    c_one = torch.zeros((m, n), device=DEV)
    monkeypatch.delenv("LP_PAIR_SPLIT_ALL")
    _gemm(a, w, c_one, L.EPI_STORE, L.LP_F32, fork=False)
    assert torch.equal(c_one, c32)


def test_pair_split_inside_graph_capture(monkeypatch):
    monkeypatch.setenv("LP_PAIR_SPLIT_ALL", "1")
    m, k, n = 1000, 256, 1024
    a, w = _ab(m, k, n, 6)
    c = torch.zeros((m, n), device=DEV)
    args = L.GemmArgs()
    args.in_dtype, args.out_dtype, args.epilogue = L.LP_BF16, L.LP_F32, L.EPI_STORE
    args.m, args.n, args.k = m, n, k
    args.lda, args.ldw, args.ldc = k, k, n
    args.a, args.w, args.c = a.data_ptr(), w.data_ptr(), c.data_ptr()
    args.fork = _fork()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        L.call("lp_gemm", C.byref(args), s.cuda_stream)
    c.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert rel_l2(c.cpu(), (a.float() @ w.float().T).cpu()) < 1e-5


def test_gated_residual_epilogue():
    m, k, n = 250, 448, 256
    a, w = _ab(m, k, n, 2)
    h = torch.randn((m, n), device=DEV)
    gate = torch.randn(n, device=DEV)
    ref = h + gate * (a.float() @ w.float().T)
    _gemm(a, w, h, L.EPI_RESID, L.LP_F32, gate=gate)
    assert rel_l2(h.cpu(), ref.cpu()) < 1e-5


@pytest.mark.parametrize("qk_norm,spatial,n_heads,frames,split", [(False, False, 4, 0, False),
                                                                   (True, True, 4, 3, False),
                                                                   (True, True, 8, 5, False),
                                                                   (True, True, 8, 5, True)])
def test_qkv_epilogue(monkeypatch, qk_norm, spatial, n_heads, frames, split):
    # m >= 256 takes the cluster-pair kernel (390 / 650 tokens: ragged last pair tile)
    hd = 128
    d = n_heads * hd
    n_tok = 130 * frames if spatial else 200
    a, w = _ab(n_tok, d, 3 * d, 3)
    if spatial:
        third = hd // 6
        t_dim, dh, dw = hd - 4 * third, 2 * third, 2 * third
        gh, gw = 5, 26  # 130 tokens per frame, 3 frames
        sc, ss = spatial_tables(gh, gw, dh, dw, 10000.0)
    else:
        t_dim, dh, dw, gh, gw = hd, 0, 0, 1, 1
        sc = ss = np.zeros((1, 0), np.float32)
    spc, sps = torch.from_numpy(sc).to(DEV), torch.from_numpy(ss).to(DEV)
    rows = 1000
    karena = torch.zeros((rows, d), device=DEV, dtype=torch.bfloat16)
    varena = torch.zeros_like(karena)
    q = torch.zeros((n_tok, d), device=DEV, dtype=torch.bfloat16)
    cur = 300
    desc = make_desc(7, [(0, 10), (cur, n_tok)], cur, n_tok, t_dim)
    ddev = upload_desc(desc)
    g_q = (1 + 0.1 * torch.randn(d, device=DEV)) if qk_norm else None
    g_k = (1 + 0.1 * torch.randn(d, device=DEV)) if qk_norm else None
    geom = L.RopeGeom(hd, t_dim // 2, gh * gw, (dh + dw) // 2, spc.data_ptr(), sps.data_ptr())
    epi = L.QkvEpi(d, n_heads, hd, int(qk_norm), 1e-6, g_q.data_ptr() if qk_norm else 0,
                   g_k.data_ptr() if qk_norm else 0, q.data_ptr(), karena.data_ptr(), varena.data_ptr(),
                   ddev.data_ptr(), geom)
    if split:
        monkeypatch.setenv("LP_PAIR_SPLIT_ALL", "1")
    _gemm(a, w, None, L.EPI_QKV, L.LP_BF16, qkv=epi, fork=split)
    y = a.float() @ w.float().T
    qr, kr, vr = y[:, :d], y[:, d:2 * d], y[:, 2 * d:]

    def norm(x, g):
        if not qk_norm:
            return x
        xh = x.reshape(n_tok, n_heads, hd)
        xh = xh * torch.rsqrt((xh * xh).mean(-1, keepdim=True) + 1e-6)
        return xh.reshape(n_tok, d) * g

    tc = np.array(desc.rope_cos[: t_dim // 2], np.float32)
    ts = np.array(desc.rope_sin[: t_dim // 2], np.float32)
    qref = rope_ref(norm(qr, g_q), n_heads, hd, tc, ts, spc, sps, gh * gw)
    kref = rope_ref(norm(kr, g_k), n_heads, hd, tc, ts, spc, sps, gh * gw)
    assert rel_l2(q.float().cpu(), qref.cpu()) < 5e-3
    assert rel_l2(karena[cur:cur + n_tok].float().cpu(), kref.cpu()) < 5e-3
    assert rel_l2(varena[cur:cur + n_tok].float().cpu(), vr.cpu()) < 5e-3
    assert karena[:cur].abs().sum().item() == 0 and karena[cur + n_tok:].abs().sum().item() == 0


def test_f32_pinned_gemm_is_bitwise_reference_order():
    rng = np.random.default_rng(0)
    a = rng.standard_normal((37, 70)).astype(np.float32)
    b = rng.standard_normal((70, 45)).astype(np.float32)
    ref = np.zeros((37, 45), np.float32)
    for kk in range(70):
        ref += np.multiply.outer(a[:, kk], b[kk])
    ta, tb = torch.from_numpy(a).to(DEV), torch.from_numpy(b).to(DEV)
    c = torch.zeros((37, 45), device=DEV)
    _gemm(ta, tb, c, L.EPI_STORE, L.LP_F32, in_dtype=L.LP_F32)
    assert c.cpu().numpy().tobytes() == ref.tobytes()


@pytest.mark.parametrize("patched", [True, False])
def test_euler_epilogue(patched):
    # velocity head + flow step fused (K6): x_out = x_in + unpatchify(a . W^T) * dt
    frames, C_, H, W, ph, pw = 3, 16, 8, 12, 2, 2
    if patched:
        tpf, pd = (H // ph) * (W // pw), C_ * ph * pw
        m, n = frames * tpf, pd
    else:
        m, n = 96, 128
    k = 256
    a, w = _ab(m, k, n, 5)
    v = a.float() @ w.float().T
    dt = -0.25
    desc = upload_desc(make_desc(3, [(0, 1), (0, m)], 0, m, 128, dt=dt))
    lat = C_ * H * W
    if patched:
        x_in = torch.randn((frames, lat), device=DEV)
        vu = v.reshape(frames, H // ph, W // pw, C_, ph, pw).permute(0, 3, 1, 4, 2, 5).reshape(frames, lat)
    else:
        x_in = torch.randn((m, n), device=DEV)
        vu = v
    x_out = torch.zeros_like(x_in)
    ep = L.EulerEpi(x_in.data_ptr(), x_out.data_ptr(), C_ if patched else 0, H, W, ph if patched else 0,
                    pw if patched else 0, desc.data_ptr())
    args = L.GemmArgs()
    args.in_dtype, args.out_dtype, args.epilogue = L.LP_BF16, L.LP_F32, L.EPI_EULER
    args.m, args.n, args.k = m, n, k
    args.lda, args.ldw, args.ldc = k, k, n
    args.a, args.w, args.c = a.data_ptr(), w.data_ptr(), None
    args.euler = C.pointer(ep)
    L.call("lp_gemm", C.byref(args), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = x_in + vu * dt
    assert rel_l2(x_out.cpu(), ref.cpu()) < 1e-5


@pytest.mark.parametrize("d", [256, 1536, 5120, 6144])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_norm_mod_rows(d, mode):
    # pre-LN + AdaLN row kernel at the 1.3B / 14B widths and a wider
    # re-read one: out = LN(h) * (1 + scale) + shift (mode 2), LN(h) (1), copy (0)
    rows = 37
    g = torch.Generator(device=DEV).manual_seed(d + mode)
    h = torch.randn((rows, d), generator=g, device=DEV) * 3 + 0.5
    sh, sc = torch.randn(d, generator=g, device=DEV), torch.randn(d, generator=g, device=DEV)
    if mode == 0:
        ref = h
    else:
        ref = torch.nn.functional.layer_norm(h.double(), (d,), eps=1e-6).float()
        if mode == 2:
            ref = ref * (1 + sc) + sh
    st = torch.cuda.current_stream().cuda_stream
    for dt, tol in ((torch.float32, 1e-5), (torch.bfloat16, 5e-3)):
        out = torch.empty((rows, d), device=DEV, dtype=dt)
        L.call("lp_norm_mod", h.data_ptr(), rows, d, mode, 1e-6, sh.data_ptr(), sc.data_ptr(), out.data_ptr(),
               L.LP_F32 if dt == torch.float32 else L.LP_BF16, st)
        torch.cuda.synchronize()
        assert rel_l2(out.float().cpu(), ref.cpu()) < tol, (d, mode, dt)


def test_argument_errors_are_reported_not_launched():
    # the C ABI validates before launching and returns LP_EINVAL with a message
    a, w = _ab(128, 100, 256)  # k not a multiple of 64 (bf16 tcgen05 path)
    c = torch.zeros((128, 256), device=DEV)
    with pytest.raises(L.LivepipeError, match="multiple of 64"):
        _gemm(a, w, c, L.EPI_STORE, L.LP_F32)
    a, w = _ab(128, 128, 100)  # n not a multiple of 64
    c = torch.zeros((128, 100), device=DEV)
    with pytest.raises(L.LivepipeError, match="multiple of 64"):
        _gemm(a, w, c, L.EPI_STORE, L.LP_F32)
    with pytest.raises(L.LivepipeError, match="null"):
        L.call("lp_codec_patch_decode", None, 1, 16, 2, 2, None, 1, 3, 8, None, None)
    with pytest.raises(L.LivepipeError, match="channels"):
        x = torch.zeros(64, device=DEV)
        L.call("lp_codec_patch_decode", x.data_ptr(), 1, 64, 1, 1, x.data_ptr(), 1, 3, 8, x.data_ptr(), None)


# ---- the exact benched 14B shapes: M = 4680 tokens, the
# pair + side-stream tail split the engines use (default policy, fork on)

def _qkv_14b_case(seed=11):
    n_heads, hd, frames, gh, gw = 40, 128, 3, 30, 52
    d, n_tok = n_heads * hd, 3 * 30 * 52
    a, w = _ab(n_tok, d, 3 * d, seed)
    third = hd // 6
    t_dim, dh, dw = hd - 4 * third, 2 * third, 2 * third
    sc, ss = spatial_tables(gh, gw, dh, dw, 10000.0)
    return n_heads, hd, d, n_tok, a, w, t_dim, gh, gw, torch.from_numpy(sc).to(DEV), torch.from_numpy(ss).to(DEV)


def test_qkv_epilogue_at_benched_14b_shape():
    # 4680 x 5120 -> 15360 with 40-head RMSNorm + 3-axis RoPE + ring scatter
    n_heads, hd, d, n_tok, a, w, t_dim, gh, gw, spc, sps = _qkv_14b_case()
    s_tok = gh * gw
    rows = s_tok + 5 * n_tok
    karena = torch.zeros((rows, d), device=DEV, dtype=torch.bfloat16)
    varena = torch.zeros_like(karena)
    q = torch.zeros((n_tok, d), device=DEV, dtype=torch.bfloat16)
    cur = s_tok + 3 * n_tok
    desc = make_desc(836, [(0, s_tok), (cur, n_tok)], cur, n_tok, t_dim)
    ddev = upload_desc(desc)
    g_q = 1 + 0.05 * torch.randn(d, device=DEV)
    g_k = 1 + 0.05 * torch.randn(d, device=DEV)
    geom = L.RopeGeom(hd, t_dim // 2, s_tok, (hd - t_dim) // 2, spc.data_ptr(), sps.data_ptr())
    epi = L.QkvEpi(d, n_heads, hd, 1, 1e-6, g_q.data_ptr(), g_k.data_ptr(), q.data_ptr(), karena.data_ptr(),
                   varena.data_ptr(), ddev.data_ptr(), geom)
    _gemm(a, w, None, L.EPI_QKV, L.LP_BF16, qkv=epi, fork=True)
    y = a.float() @ w.float().T
    qr, kr, vr = y[:, :d], y[:, d:2 * d], y[:, 2 * d:]

    def norm(x, g):
        xh = x.reshape(n_tok, n_heads, hd)
        return (xh * torch.rsqrt((xh * xh).mean(-1, keepdim=True) + 1e-6)).reshape(n_tok, d) * g

    tc = np.array(desc.rope_cos[: t_dim // 2], np.float32)
    ts = np.array(desc.rope_sin[: t_dim // 2], np.float32)
    qref = rope_ref(norm(qr, g_q), n_heads, hd, tc, ts, spc, sps, s_tok)
    kref = rope_ref(norm(kr, g_k), n_heads, hd, tc, ts, spc, sps, s_tok)
    assert rel_l2(q.float().cpu(), qref.cpu()) < 5e-3
    assert rel_l2(karena[cur:cur + n_tok].float().cpu(), kref.cpu()) < 5e-3
    assert rel_l2(varena[cur:cur + n_tok].float().cpu(), vr.cpu()) < 5e-3
    # nothing outside the current block's rows is touched
    assert karena[:cur].abs().sum().item() == 0 and karena[cur + n_tok:].abs().sum().item() == 0


@pytest.mark.parametrize("k,n", [(5120, 5120), (13824, 5120)])
def test_resid_at_benched_14b_shapes(k, n):
    # O-proj (K = 5120) and FFN-down (K = 13824): gated residual into fp32 h
    m = 4680
    a, w = _ab(m, k, n, 12)
    h = torch.randn((m, n), device=DEV)
    gate = torch.randn(n, device=DEV) * 0.1
    want = h + gate * (a.float() @ w.float().T)
    _gemm(a, w, h, L.EPI_RESID, L.LP_F32, gate=gate, fork=True)
    assert rel_l2(h.cpu(), want.cpu()) < 1e-5


def test_ffn_up_gelu_at_benched_14b_shape():
    m, k, n = 4680, 5120, 13824
    a, w = _ab(m, k, n, 13)
    ref = torch.nn.functional.gelu(a.float() @ w.float().T, approximate="tanh")
    c = torch.zeros((m, n), device=DEV, dtype=torch.bfloat16)
    _gemm(a, w, c, L.EPI_GELU, L.LP_BF16, fork=True)
    assert rel_l2(c.float().cpu(), ref.cpu()) < 5e-3


@pytest.mark.parametrize("m,k,n,fork", [(300, 256, 512, False), (4680, 5120, 5120, True), (4680, 13824, 5120, True)])
def test_resid_row_stats_feed_the_norm_apply_pass(m, k, n, fork):
    # AdaLN with its reduction fused into the producing RESID GEMM: the
    # epilogue's (mean, M2) per 32-column chunk of the new h, merged by
    # lp_norm_mod_stats, gives the same modulated norm as the full-row
    # lp_norm_mod (K7: pre-LN + AdaLN of the Wan profile); 14B O-proj and
    # FFN-down shapes run through the pair + side-stream tail split
    a, w = _ab(m, k, n, 7)
    g = torch.Generator(device=DEV).manual_seed(8)
    h0 = torch.randn((m, n), generator=g, device=DEV) * 3.0 + 0.5
    gate = torch.rand(n, generator=g, device=DEV) + 0.5
    h = h0.clone()
    stats = torch.full((m, n // 32, 2), float("nan"), device=DEV)
    _gemm(a, w, h, L.EPI_RESID, L.LP_F32, gate=gate, fork=fork, stats=stats)
    ref_h = h0 + gate * (a.float() @ w.float().T)
    assert rel_l2(h.cpu(), ref_h.cpu()) < 1e-5
    chunks = h.reshape(m, n // 32, 32)
    torch.testing.assert_close(stats[..., 0], chunks.mean(-1), rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(stats[..., 1], ((chunks - chunks.mean(-1, keepdim=True)) ** 2).sum(-1),
                               rtol=1e-4, atol=1e-4)
    shift = torch.randn(n, generator=g, device=DEV) * 0.1
    scale = torch.randn(n, generator=g, device=DEV) * 0.1
    st = torch.cuda.current_stream().cuda_stream
    for mode in (1, 2):
        want = torch.empty((m, n), dtype=torch.bfloat16, device=DEV)
        got = torch.empty_like(want)
        sh, sc = (shift.data_ptr(), scale.data_ptr()) if mode == 2 else (None, None)
        L.call("lp_norm_mod", h.data_ptr(), m, n, mode, 1e-6, sh, sc, want.data_ptr(), L.LP_BF16, st)
        L.call("lp_norm_mod_stats", h.data_ptr(), stats.data_ptr(), m, n, mode, 1e-6, sh, sc, got.data_ptr(),
               L.LP_BF16, st)
        torch.cuda.synchronize()
        ln = torch.nn.functional.layer_norm(h, (n,), eps=1e-6)
        ref = ln * (1 + scale) + shift if mode == 2 else ln
        assert rel_l2(got.float().cpu(), ref.cpu()) < 4e-3
        # the two kernels differ only in fp32 rounding of the moments: at most one bf16 ulp apart
        diff = (got.float() - want.float()).abs()
        assert float((diff > 0).float().mean()) < 0.01
        assert bool(torch.all(diff <= want.float().abs() * 2 ** -7 + 1e-6))


@pytest.mark.parametrize("rows,d", [(1, 5120), (4680, 5120), (1001, 1536), (37, 2048), (300, 4096)])
def test_norm_mod_matches_torch_layer_norm(rows, d):
    # pre-LN + AdaLN (K7): the software-pipelined resident-grid kernel walks
    # rows beyond the grid (4680 > 4 x 148) and handles partial float4 tails
    g = torch.Generator(device=DEV).manual_seed(rows + d)
    h = torch.randn((rows, d), generator=g, device=DEV) * 2.0 + 0.3
    shift = torch.randn(d, generator=g, device=DEV) * 0.1
    scale = torch.randn(d, generator=g, device=DEV) * 0.1
    st = torch.cuda.current_stream().cuda_stream
    ln = torch.nn.functional.layer_norm(h.double(), (d,), eps=1e-6)
    for mode in (1, 2):
        ref = (ln * (1 + scale.double()) + shift.double() if mode == 2 else ln).float()
        out = torch.empty((rows, d), device=DEV)
        sh, sc = (shift.data_ptr(), scale.data_ptr()) if mode == 2 else (None, None)
        L.call("lp_norm_mod", h.data_ptr(), rows, d, mode, 1e-6, sh, sc, out.data_ptr(), L.LP_F32, st)
        o16 = torch.empty((rows, d), device=DEV, dtype=torch.bfloat16)
        L.call("lp_norm_mod", h.data_ptr(), rows, d, mode, 1e-6, sh, sc, o16.data_ptr(), L.LP_BF16, st)
        torch.cuda.synchronize()
        assert rel_l2(out.cpu(), ref.cpu()) < 1e-6
        assert torch.equal(o16, out.to(torch.bfloat16))
