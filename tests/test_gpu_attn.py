"""tcgen05 flash attention (lp_attention, LP_BF16) vs a torch fp32 reference
on the same bf16 inputs and vs the SIMT kernel; visible-set / ordering of the
descriptor segments (sink, wrapped ring slots, current) bit-exact by
construction of the reference."""

import ctypes as C

import numpy as np
import pytest
import torch

from paper_2512_04677_b200 import _lib as L

from gpu_helpers import make_desc, rel_l2, upload_desc

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module", autouse=True)
def _init():
    L.init_device(0)


def _workspace(n_q, n_heads):
    nb = C.c_int64(0)
    L.call("lp_attention_workspace", n_q, n_heads, 128, C.byref(nb))
    return torch.empty(max(int(nb.value), 16) // 4, dtype=torch.float32, device=DEV), int(nb.value)


def _run(fn, q, karena, varena, desc, n_heads, scale, n_kv_max, split=True):
    out = torch.zeros_like(q)
    ddev = upload_desc(desc)
    ws, nb = _workspace(q.shape[0], n_heads) if split else (None, 0)
    args = L.AttnArgs(L.LP_BF16, q.shape[0], n_heads, 128, scale, q.data_ptr(), karena.data_ptr(),
                      varena.data_ptr(), out.data_ptr(), ddev.data_ptr(), karena.shape[0], n_kv_max,
                      ws.data_ptr() if ws is not None else None, nb)
    L.call(fn, C.byref(args), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out


def _ref(q, karena, varena, segs, n_heads, scale):
    rows = torch.cat([torch.arange(r, r + n, device=DEV) for r, n in segs])
    k = karena[rows].float()
    v = varena[rows].float()
    qf = q.float()
    outs = []
    for h in range(n_heads):
        sl = slice(h * 128, (h + 1) * 128)
        s = (qf[:, sl] @ k[:, sl].T) * scale
        outs.append(torch.softmax(s, dim=-1) @ v[:, sl])
    return torch.cat(outs, dim=1)


CASES = [
    # (n_q, sink, [history (row, len)], heads)
    (390, 130, [], 2),
    (390, 130, [(520, 390), (130, 390)], 3),          # wrapped ring: newer slot at a lower row
    (200, 1, [(700, 200), (300, 200), (900, 200)], 1),  # toy-like single-token sink, ragged tiles
    (4680 // 10, 156, [(156 + 468 * s, 468) for s in (2, 0, 1)], 4),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_flash_attention_matches_reference(case):
    n_q, s_tok, hist, heads = CASES[case]
    d = heads * 128
    rows = 2400
    g = torch.Generator(device=DEV).manual_seed(case)
    karena = torch.randn((rows, d), generator=g, device=DEV).to(torch.bfloat16)
    varena = torch.randn((rows, d), generator=g, device=DEV).to(torch.bfloat16)
    q = (torch.randn((n_q, d), generator=g, device=DEV) * 2).to(torch.bfloat16)
    cur = rows - n_q - 7
    segs = [(0, s_tok)] + hist + [(cur, n_q)]
    desc = make_desc(5, segs, cur, n_q, 128)
    scale = float(np.float32(1.0) / np.float32(np.sqrt(128)))
    n_kv = sum(n for _, n in segs)
    ref = _ref(q, karena, varena, segs, heads, scale)
    tc = _run("lp_attention", q, karena, varena, desc, heads, scale, n_kv)
    assert rel_l2(tc.float().cpu(), ref.cpu()) < 1e-2
    simt = _run("lp_attention_simt", q, karena, varena, desc, heads, scale, n_kv)
    assert rel_l2(simt.float().cpu(), ref.cpu()) < 5e-3
    # deterministic: bitwise repeatable
    tc2 = _run("lp_attention", q, karena, varena, desc, heads, scale, n_kv)
    assert torch.equal(tc, tc2)


def test_segment_order_modes():
    # softmax(QK^T)V does not depend on key order.  arena_order = 1 (the
    # engines): segments walked in arena-row order, adjacent ones merged, so
    # the descriptor's logical order changes nothing (bitwise) and a merged
    # range equals its parts.  arena_order = 0 (the drop-in): logical order,
    # so moving the same keys to other rows changes nothing (bitwise).
    heads, n_q, d = 2, 256, 256
    g = torch.Generator(device=DEV).manual_seed(9)
    ka = torch.randn((1500, d), generator=g, device=DEV).to(torch.bfloat16)
    va = torch.randn((1500, d), generator=g, device=DEV).to(torch.bfloat16)
    q = torch.randn((n_q, d), generator=g, device=DEV).to(torch.bfloat16)
    scale = 0.0883883461356163
    sa = [(0, 64), (300, 256), (556, 144), (700, 256), (1200, n_q)]
    sb = [(0, 64), (700, 256), (556, 144), (300, 256), (1200, n_q)]
    sc = [(0, 64), (300, 656), (1200, n_q)]

    def run(ka_, va_, segs, order):
        return _run("lp_attention", q, ka_, va_, make_desc(3, segs, 1200, n_q, 128, arena_order=order), heads,
                    scale, 976)

    a = run(ka, va, sa, 1)
    assert torch.equal(a, run(ka, va, sb, 1))
    assert torch.equal(a, run(ka, va, sc, 1))
    # logical order: swap which rows hold blocks 1 and 3 and list them so the
    # logical key order is unchanged -> bitwise equal
    kb, vb = ka.clone(), va.clone()
    kb[300:556], kb[700:956] = ka[700:956], ka[300:556]
    vb[300:556], vb[700:956] = va[700:956], va[300:556]
    l0 = run(ka, va, sa, 0)
    assert torch.equal(l0, run(kb, vb, sb, 0))
    # the two modes differ only by rounding
    assert rel_l2(l0.float().cpu(), a.float().cpu()) < 1e-2


@pytest.mark.parametrize("heads,arena_order", [(40, 0), (12, 0), (40, 1), (12, 1)])
def test_full_shape_tail_split_matches_reference(heads, arena_order):
    # 480p block: 4680 queries over [sink 1560 | 4 ring slots | current]; at
    # 40 heads the grid tail (ragged query pairs + the last units) is split
    # into KV pieces merged by the combine kernel; must agree with the
    # unsplit kernel and with fp32 torch per head
    n_q, s_tok, d = 4680, 1560, heads * 128
    rows = s_tok + 5 * n_q
    g = torch.Generator(device=DEV).manual_seed(heads)
    karena = torch.randn((rows, d), generator=g, device=DEV).to(torch.bfloat16)
    varena = torch.randn((rows, d), generator=g, device=DEV).to(torch.bfloat16)
    q = (torch.randn((n_q, d), generator=g, device=DEV) * 2).to(torch.bfloat16)
    order = [3, 4, 0, 1]  # ring slots oldest -> newest, wrapped
    segs = [(0, s_tok)] + [(s_tok + n_q * s, n_q) for s in order] + [(s_tok + 2 * n_q, n_q)]
    cur = s_tok + 2 * n_q
    # arena_order = 1 is the engines' benched path: the wrapped ring plus sink
    # and current block are walked as ONE merged 24,960-row range
    desc = make_desc(7, segs, cur, n_q, 128, arena_order=arena_order)
    scale = float(np.float32(1.0) / np.float32(np.sqrt(128)))
    n_kv = sum(n for _, n in segs)
    ws, nb = _workspace(n_q, heads)
    tc = _run("lp_attention", q, karena, varena, desc, heads, scale, n_kv)
    whole = _run("lp_attention", q, karena, varena, desc, heads, scale, n_kv, split=False)
    assert rel_l2(tc.float().cpu(), whole.float().cpu()) < 5e-3
    for h in range(0, heads, max(1, heads // 6)):
        ref = _ref(q[:, h * 128:(h + 1) * 128].contiguous(), karena[:, h * 128:(h + 1) * 128].contiguous(),
                   varena[:, h * 128:(h + 1) * 128].contiguous(), segs, 1, scale)
        assert rel_l2(tc[:, h * 128:(h + 1) * 128].float().cpu(), ref.cpu()) < 1e-2, h
    tc2 = _run("lp_attention", q, karena, varena, desc, heads, scale, n_kv)
    assert torch.equal(tc, tc2)


def test_exponent_window_fallback(monkeypatch):
    # The bounded-exponent kernel fixes each row's exponent offset at the max
    # of its first KV tile.  Head 0 gets a block of "hot" keys in a later
    # tile whose scores sit ~98 log2 units above it (outside the 2^64
    # window): those work units must be flagged and recomputed by the exact
    # online-max kernel, while head 1 (ordinary scores) stays on the bounded
    # kernel.  Both match fp32 torch.
    heads, n_q, d, rows = 2, 300, 256, 2000
    g = torch.Generator(device=DEV).manual_seed(21)
    ka = torch.randn((rows, d), generator=g, device=DEV)
    va = torch.randn((rows, d), generator=g, device=DEV).to(torch.bfloat16)
    q = torch.randn((n_q, d), generator=g, device=DEV) * 0.5
    q[:, :128] += 1.0
    ka[1500:1510, :128] = 6.0  # s ~ 128*6/sqrt(128) = 68 nats above the sink tile's max
    ka, q = ka.to(torch.bfloat16), q.to(torch.bfloat16)
    segs = [(0, 130), (1400, 300), (1700, n_q)]
    scale = float(np.float32(1.0) / np.float32(np.sqrt(128)))
    desc = make_desc(5, segs, 1700, n_q, 128, arena_order=1)
    n_kv = sum(n for _, n in segs)
    ref = _ref(q, ka, va, segs, heads, scale)
    fast = _run("lp_attention", q, ka, va, desc, heads, scale, n_kv)
    monkeypatch.setenv("LP_ATTN_EXACT", "1")
    exact = _run("lp_attention", q, ka, va, desc, heads, scale, n_kv)
    monkeypatch.delenv("LP_ATTN_EXACT")
    for h in range(heads):
        sl = slice(h * 128, (h + 1) * 128)
        assert rel_l2(fast[:, sl].float().cpu(), ref[:, sl].cpu()) < 1e-2, h
        assert rel_l2(exact[:, sl].float().cpu(), ref[:, sl].cpu()) < 1e-2, h
    # without the rerun, head 0's hot keys would be weighted by the clamped
    # exponentials (2^65 on the polynomial pairs vs 2^94 on MUFU ones) and
    # miss the reference by O(1); head 1 ran the bounded kernel itself
    assert not torch.equal(fast[:, 128:], exact[:, 128:])


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_device_history_noise_moments(dtype):
    # kvcache.py:121-137 with the device Philox stream (perf runs): the
    # corrupted view = ring + sigma * N(0,1) in the scratch rows, ring
    # untouched; moments as the reference checks them (tests/test_kvcache.py:178-194)
    d, n_tok, rows = 512, 300, 2400
    sigma = 0.3
    arena = torch.zeros((rows, d), dtype=dtype, device=DEV)
    arena[0:n_tok] = 1.0  # ring slot contents
    desc = make_desc(4, [(2000, 8), (1200, n_tok), (2100, 8)], 2100, 8, 128)
    desc.src_row[1] = 0  # corrupted copy of ring rows [0, n_tok) into scratch rows [1200, +n_tok)
    desc.sigma = sigma
    desc.noise_key = 12345
    ddev = upload_desc(desc)
    ldt = L.LP_F32 if dtype == torch.float32 else L.LP_BF16
    L.call("lp_history_noise", arena.data_ptr(), ldt, d, None, 1, 0, 0, ddev.data_ptr(), n_tok,
           torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    z = (arena[1200:1200 + n_tok].float() - 1.0) / sigma
    assert abs(float(z.mean())) < 0.02
    assert abs(float(z.std()) - 1.0) < 0.05
    kurt = float(((z - z.mean()) ** 4).mean() / z.var() ** 2)
    assert abs(kurt - 3.0) < 0.1, kurt
    assert abs(float((z.abs() > 2.0).float().mean()) - 0.0455) < 0.003  # two-sided 2-sigma tail
    assert torch.all(arena[0:n_tok] == 1.0)  # stored ring untouched


def test_device_history_noise_streams_independent():
    # perf-run noise: every (layer, K/V, entry) stream and every (block, step)
    # key draws its own N(0,1) sequence -- no two streams may repeat or
    # correlate (the reference draws each corrupted view from its own Prng,
    # engine.py:217-224 / kvcache.py:121-137)
    d, n_tok, rows = 512, 256, 4096
    sigma = 1.0
    ldt = L.LP_BF16
    outs = []
    for key, layer, kv in [(7, 0, 0), (7, 0, 1), (7, 1, 0), (8, 0, 0)]:
        arena = torch.zeros((rows, d), dtype=torch.bfloat16, device=DEV)
        desc = make_desc(4, [(3000, 8), (1000, n_tok), (2000, n_tok), (3100, 8)], 3100, 8, 128)
        desc.src_row[1] = 0
        desc.src_row[2] = 0
        desc.sigma = sigma
        desc.noise_key = key
        ddev = upload_desc(desc)
        L.call("lp_history_noise", arena.data_ptr(), ldt, d, None, 2, layer, kv, ddev.data_ptr(), 2 * n_tok,
               torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        outs.append(arena[1000:1000 + n_tok].float().flatten())
        outs.append(arena[2000:2000 + n_tok].float().flatten())  # second history entry
        assert torch.all(arena[0:n_tok] == 0)
    for i in range(len(outs)):
        z = outs[i]
        assert abs(float(z.mean())) < 0.01 and abs(float(z.std()) - 1.0) < 0.02
        for j in range(i):
            c = float(torch.corrcoef(torch.stack([outs[i], outs[j]]))[0, 1])
            assert abs(c) < 0.015, (i, j, c)
            assert not torch.equal(outs[i], outs[j])


def test_dynamic_item_queue_stress_bitwise_repeatable():
    # the persistent kernel's items are claimed dynamically (global counter +
    # a cluster-scope shared-memory ring per cluster pair): which cluster runs
    # which item changes from launch to launch, the output must not.  30
    # back-to-back launches on one stream (counter re-zeroed by the init
    # kernel each time) and 10 more interleaved with a second workspace on a
    # second stream, at the full 14B shape, all bitwise equal.
    n_q, s_tok, heads = 4680, 1560, 40
    d, rows = heads * 128, s_tok + 5 * n_q
    g = torch.Generator(device=DEV).manual_seed(77)
    karena = torch.randn((rows, d), generator=g, device=DEV).to(torch.bfloat16)
    varena = torch.randn((rows, d), generator=g, device=DEV).to(torch.bfloat16)
    q = torch.randn((n_q, d), generator=g, device=DEV).to(torch.bfloat16)
    segs = [(0, s_tok)] + [(s_tok + n_q * s, n_q) for s in (3, 4, 0, 1)] + [(s_tok + 2 * n_q, n_q)]
    desc = make_desc(9, segs, s_tok + 2 * n_q, n_q, 128, arena_order=1)
    ddev = upload_desc(desc)
    scale = float(np.float32(1.0) / np.float32(np.sqrt(128)))
    n_kv = sum(n for _, n in segs)
    streams = [torch.cuda.current_stream(), torch.cuda.Stream()]
    wss = [_workspace(n_q, heads) for _ in streams]
    outs = []

    def launch(i, si):
        out = torch.empty_like(q)
        ws, nb = wss[si]
        args = L.AttnArgs(L.LP_BF16, n_q, heads, 128, scale, q.data_ptr(), karena.data_ptr(), varena.data_ptr(),
                          out.data_ptr(), ddev.data_ptr(), rows, n_kv, ws.data_ptr(), nb)
        L.call("lp_attention", C.byref(args), streams[si].cuda_stream)
        return out

    for i in range(30):
        outs.append(launch(i, 0))
    streams[1].wait_stream(streams[0])
    for i in range(10):
        outs.append(launch(i, i % 2))
    torch.cuda.synchronize()
    ref = outs[0]
    assert bool(torch.isfinite(ref.float()).all())
    for o in outs[1:]:
        assert torch.equal(o, ref)
