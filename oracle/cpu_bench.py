"""CPU-reference timing for bench.py (TEST/BENCH INFRASTRUCTURE ONLY).

Times the reference algorithm's dominant operation -- numerics.matmul's
pinned ascending-k rank-1 accumulation (numerics.py:50-64), 99.4% of
denoise_block time at 14B dims -- on a bounded
K-slice of a projection at the benchmark's token count, split over host
cores by row blocks (the per-element order is unchanged), and extrapolates
linearly in FLOPs to whole blocks.  Reported as an extrapolated baseline,
never as a target.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from .livepipe_oracle import mm_pinned


def _work(args):
    rows, k_slice, n_cols, seed, reps = args
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((rows, k_slice)).astype(np.float32)
    b = rng.standard_normal((k_slice, n_cols)).astype(np.float32)
    t0 = time.perf_counter()
    for _ in range(reps):
        mm_pinned(a, b)
    return time.perf_counter() - t0


def pinned_matmul_rate(n_tokens: int, d_model: int, k_slice: int = 64, target_s: float = 12.0,
                       cores: int | None = None) -> dict:
    """FLOP/s of the reference's pinned-order matmul on an (n_tokens x k_slice)
    . (k_slice x d_model) slice, rows split over ``cores`` processes."""
    cores = cores or os.cpu_count() or 1
    rows = max(1, n_tokens // cores)
    # calibrate one rep on one core
    t1 = _work((rows, k_slice, d_model, 0, 1))
    reps = max(1, int(target_s / max(t1, 1e-3)))
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        times = pool.map(_work, [(rows, k_slice, d_model, s, reps) for s in range(cores)])
    wall = time.perf_counter() - t0
    flops = 2.0 * rows * cores * k_slice * d_model * reps
    return {"flops_per_s": flops / max(times), "wall_s": wall, "cores": cores, "reps": reps,
            "sample": f"pinned-order matmul ({rows * cores}x{k_slice})x({k_slice}x{d_model}) x{reps}, "
                      f"rows split over {cores} processes"}
