"""Run one lp_attention case (debug harness; used under `timeout`)."""
import ctypes as C
import sys
import os

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import numpy as np
import torch

from paper_2512_04677_b200 import _lib as L
from gpu_helpers import make_desc, upload_desc, rel_l2

n_q, heads, split, hist = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
L.init_device(0)
DEV = "cuda:0"
d = heads * 128
s_tok = 130
rows = s_tok + (hist + 1) * n_q + 64
g = torch.Generator(device=DEV).manual_seed(0)
ka = torch.randn((rows, d), generator=g, device=DEV).to(torch.bfloat16)
va = torch.randn((rows, d), generator=g, device=DEV).to(torch.bfloat16)
q = torch.randn((n_q, d), generator=g, device=DEV).to(torch.bfloat16)
segs = [(0, s_tok)] + [(s_tok + n_q * (h + 1), n_q) for h in range(hist)] + [(s_tok, n_q)]
desc = upload_desc(make_desc(3, segs, s_tok, n_q, 128))
nb = C.c_int64(0)
L.call("lp_attention_workspace", n_q, heads, 128, C.byref(nb))
ws = torch.empty(max(nb.value, 16), dtype=torch.uint8, device=DEV)
out = torch.zeros_like(q)
scale = 0.08838834764831845
args = L.AttnArgs(L.LP_BF16, n_q, heads, 128, scale, q.data_ptr(), ka.data_ptr(), va.data_ptr(), out.data_ptr(),
                  desc.data_ptr(), rows, sum(n for _, n in segs), ws.data_ptr() if split else None,
                  nb.value if split else 0)
print("workspace", nb.value, flush=True)
L.call("lp_attention", C.byref(args), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
rr = torch.cat([torch.arange(r, r + n, device=DEV) for r, n in segs])
ref = []
for h in range(heads):
    sl = slice(h * 128, (h + 1) * 128)
    s = (q[:, sl].float() @ ka[rr][:, sl].float().T) * scale
    ref.append(torch.softmax(s, -1) @ va[rr][:, sl].float())
ref = torch.cat(ref, 1)
print("OK rel", rel_l2(out.float().cpu(), ref.cpu()), flush=True)
