"""Cache slow oracle rollouts at the BENCHMARKED Wan geometry as fixtures.

TEST INFRASTRUCTURE ONLY.  The oracle (oracle/livepipe_oracle.py, a NumPy
restatement of denoiser.py:201-276 plus the wan-profile extensions) runs
here on the CPU -- hours of BLAS time would not fit in a GPU test -- and the
final latents of every block are committed under tests/golden/ for
tests/test_gpu_wan_shapes.py to compare the B200 path against.

Cases (VERDICT r1 "next round" item 1):

* ``w14_l2`` -- the 14B width and 480p geometry exactly (d 5120 = 40 heads x
  128, d_ff 13824, latent 16x60x104 -> 1,560 tokens per frame, 4,680 per
  block, one sink frame, L = 4 so block >= 4 attends over
  N_kv = 1,560 + 4*4,680 + 4,680 = 24,960 keys), 2 layers, 4 steps,
  6 blocks, AAS after block 0.  fp64 BLAS products (``mm_f64``).
* ``w14_d40`` -- the full 14B depth and width (40 layers, d 5120, d_ff
  13824) at a reduced patch grid (latent 16x16x24 -> 8x12 patches, 96
  tokens per frame, 288 per block), 4 steps, 6 blocks, L = 4.  fp64 BLAS.

Weights, noise, conditioning and the sink come from the seeded generators
both sides share (weight_seed 7, noise_seed 11), so the GPU test rebuilds
the identical inputs.  Run:

    python tests/golden/make_wan_fixtures.py [case ...]
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import livepipe_oracle as O  # noqa: E402

CASES = {
    "w14_l2": dict(profile=dict(n_layers=2, n_heads=40, head_dim=128, ffn_dim=13824, channels=16, height=60,
                                width=104),
                   rollout=dict(steps=4, blocks=6, cache_capacity=4, sink_delta=1)),
    "w14_d40": dict(profile=dict(n_layers=40, n_heads=40, head_dim=128, ffn_dim=13824, channels=16, height=16,
                                 width=24),
                    rollout=dict(steps=4, blocks=6, cache_capacity=4, sink_delta=1)),
}


def fixture_path(name: str) -> str:
    return os.path.join(HERE, f"wan_{name}.npz")


def run_case(name: str) -> dict:
    spec = CASES[name]
    prof = O.wan_profile(**spec["profile"])
    cfg = O.RolloutCfg(profile=prof, **spec["rollout"])
    t0 = time.time()
    w = O.build_weights(cfg.weight_seed, prof)
    t1 = time.time()
    blocks, _, sink = O.run_sequential(cfg, weights=w, mm=O.mm_f64, codec=False)
    t2 = time.time()
    np.savez(fixture_path(name), blocks=np.stack(blocks).astype(np.float32), sink=np.asarray(sink, np.float32))
    meta = {"case": name, **spec, "weights_s": round(t1 - t0, 1), "oracle_s": round(t2 - t1, 1),
            "mm": "mm_f64", "numpy": np.__version__}
    print(json.dumps(meta), flush=True)
    return meta


def main(argv) -> None:
    names = argv or list(CASES)
    meta_path = os.path.join(HERE, "wan_fixtures.json")
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {}
    for n in names:
        meta[n] = run_case(n)
        with open(meta_path, "w") as f:
            json.dump(meta, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
