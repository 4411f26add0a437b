"""A/B timing of the pair + side-stream-tail split for the 14B GEMM shapes
(CUDA events, 20 reps after warm-up)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2512_04677_b200 import _lib as L  # noqa: E402

L.init_device(0)
DEV = "cuda:0"
fork = L.fork_create()


def run(m, n, k, mode, reps=20):
    a = torch.randn((m, k), device=DEV).to(torch.bfloat16)
    w = (torch.randn((n, k), device=DEV) / k ** 0.5).to(torch.bfloat16)
    h = torch.zeros((m, n), device=DEV)
    args = L.GemmArgs()
    args.in_dtype, args.out_dtype, args.epilogue = L.LP_BF16, L.LP_F32, L.EPI_RESID
    args.m, args.n, args.k = m, n, k
    args.lda, args.ldw, args.ldc = k, k, n
    args.a, args.w, args.c = a.data_ptr(), w.data_ptr(), h.data_ptr()
    args.fork = fork if mode == "split" else None
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        L.call("lp_gemm", C.byref(args), st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        L.call("lp_gemm", C.byref(args), st)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for (m, n, k, name) in [(4680, 5120, 5120, "o_proj"), (4680, 5120, 13824, "ffn_down"), (4608, 5120, 5120, "o_pair_only"),
                        (72, 5120, 5120, "o_tail_only")]:
    r = {mode: run(m, n, k, mode) for mode in ("plain", "split")}
    print(f"{name:12s} m={m} n={n} k={k}: plain {r['plain']:.1f} us, split {r['split']:.1f} us", flush=True)
