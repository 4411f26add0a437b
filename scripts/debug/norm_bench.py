"""norm_mod (14B row: 4680 x 5120, fp32 in, bf16 out, AdaLN modulation) timed
with CUDA events; LP_NORM_VARIANT picks the launch shape."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2512_04677_b200 import _lib as L  # noqa: E402

L.init_device(0)
rows, d = 4680, 5120
h = torch.randn((rows, d), device="cuda:0")
sh, sc = torch.randn(d, device="cuda:0"), torch.randn(d, device="cuda:0")
out = torch.empty((rows, d), device="cuda:0", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")


def once():
    L.call("lp_norm_mod", h.data_ptr(), rows, d, 2, 1e-6, sh.data_ptr(), sc.data_ptr(), out.data_ptr(), L.LP_BF16, st)


for _ in range(3):
    once()
ts = []
for _ in range(20):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    once()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
ms = ts[len(ts) // 2]
ref = torch.nn.functional.layer_norm(h, (d,), eps=1e-6) * (1 + sc) + sh
err = float((out.float() - ref).norm() / ref.norm())
print(f"variant {os.environ.get('LP_NORM_VARIANT', '0')}: {ms * 1e3:.1f} us, {rows * d * 6 / ms / 1e6:.0f} GB/s, rel {err:.2e}")
