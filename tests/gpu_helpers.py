"""Helpers shared by the GPU tests (device descriptors, reference math in torch fp32)."""

import ctypes as C

import numpy as np
import torch

from paper_2512_04677_b200 import _lib as L
from paper_2512_04677_b200.numerics import rope_table


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def upload_desc(desc: L.BlockDesc, device="cuda:0") -> torch.Tensor:
    raw = bytes(C.string_at(C.addressof(desc), C.sizeof(desc)))
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(device)


def make_desc(block_index, segs, cur_row, n_tokens, t_dim, sink_pos=None, base=10000.0, dt=-0.25, arena_order=0):
    d = L.BlockDesc()
    d.arena_order = arena_order
    d.block_index = block_index
    d.sink_pos = block_index + 1 if sink_pos is None else sink_pos
    d.n_seg = len(segs)
    d.cur_row = cur_row
    d.n_tokens = n_tokens
    for s, (r, n) in enumerate(segs):
        d.seg_row[s], d.seg_len[s], d.src_row[s] = r, n, r
    d.dt = dt
    c, s_ = rope_table(block_index, t_dim, base)
    cs, ss = rope_table(d.sink_pos, t_dim, base)
    for p in range(t_dim // 2):
        d.rope_cos[p], d.rope_sin[p] = float(c[p]), float(s_[p])
        d.sink_cos[p], d.sink_sin[p] = float(cs[p]), float(ss[p])
    return d


def rope_ref(x: torch.Tensor, n_heads: int, hd: int, t_cos, t_sin, sp_cos=None, sp_sin=None, tokens_per_frame=1):
    """Interleaved-pair rotation per head; temporal pairs first, then spatial."""
    n = x.shape[0]
    xh = x.reshape(n, n_heads, hd // 2, 2)
    tp = len(t_cos)
    cos = torch.empty((n, hd // 2), dtype=torch.float32, device=x.device)
    sin = torch.empty_like(cos)
    cos[:, :tp] = torch.as_tensor(t_cos, device=x.device)
    sin[:, :tp] = torch.as_tensor(t_sin, device=x.device)
    if tp < hd // 2:
        idx = torch.arange(n, device=x.device) % tokens_per_frame
        cos[:, tp:] = torch.as_tensor(sp_cos, device=x.device)[idx]
        sin[:, tp:] = torch.as_tensor(sp_sin, device=x.device)[idx]
    cos, sin = cos[:, None, :], sin[:, None, :]
    e, o = xh[..., 0], xh[..., 1]
    out = torch.stack([e * cos - o * sin, e * sin + o * cos], dim=-1)
    return out.reshape(n, n_heads * hd)
