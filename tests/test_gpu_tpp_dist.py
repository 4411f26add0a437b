"""One-process-per-GPU TPP on the device: ranks exchange CUDA IPC handles
(gloo), latents cross ranks through IpcLink (device-initiated copies +
release/acquire flags), the sink is broadcast once after block 0.  The box
has one GPU, so the ranks share cuda:0 (same IPC + flag protocol as across
NVLink peers).  Results must equal the single-process sequential run
bitwise (reference tests/test_acceptance.py:60-83)."""

import json

import numpy as np
import pytest

import paper_2512_04677_b200 as lp

from test_tpp_dist_cpu import META, launch
from dist_worker import wan_small

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nproc,name,fused", [(2, "c1", 1), (4, "c1_sigma", 1), (2, "c1_L1", 0)])
def test_ipc_tpp_fp32_equals_sequential(tmp_path, nproc, name, fused):
    # fused: x' stored into the peer slot by the last step's Euler epilogue;
    # 0: side-stream copy kernel (lp_link_send)
    kw = dict(META[name]["kw"])
    out = tmp_path / "res"
    launch(nproc, "gpu", out, dict(kw, link_timeout_s=60.0, fused=fused), timeout=600)
    got = np.load(f"{out}.0.npy")
    seq = lp.run_sequential(lp.EngineConfig(mode="sequential", **kw))
    assert got.tobytes() == np.stack([b.values for b in seq.blocks]).tobytes()
    rec = json.load(open(f"{out}.0"))
    assert rec["nfe"] == META[name]["nfe"]


def test_ipc_tpp_bf16_wan_equals_sequential(tmp_path):
    kw = dict(steps=4, blocks=4, cache_capacity=2)
    out = tmp_path / "res"
    launch(2, "gpu", out, dict(kw, precision="bf16", profile="wan_small", link_timeout_s=60.0), timeout=600)
    got = np.load(f"{out}.0.npy")
    seq = lp.run_sequential(lp.EngineConfig(mode="sequential", precision="bf16", profile=wan_small(), **kw))
    assert got.tobytes() == np.stack([b.values for b in seq.blocks]).tobytes()


def test_ipc_tpp_with_decode_rank(tmp_path):
    # the paper's DiT ranks + 1 decode rank layout (here 2 + 1 sharing one GPU)
    kw = dict(META["c1"]["kw"])
    out = tmp_path / "res"
    launch(3, "gpu", out, dict(kw, link_timeout_s=60.0, decode_gpu=1), timeout=600)
    got = np.load(f"{out}.0.npy")
    seq = lp.run_sequential(lp.EngineConfig(mode="sequential", **kw))
    assert got.tobytes() == np.stack([b.values for b in seq.blocks]).tobytes()


def test_ipc_tpp_bf16_wan_history_noise_equals_sequential(tmp_path):
    # corrupted views with the reference's host draws across ranks (parity
    # noise uploads into fixed buffers while peer link kernels spin)
    kw = dict(steps=4, blocks=4, cache_capacity=2, history_sigma=0.2, history_mode="scaled")
    out = tmp_path / "res"
    launch(4, "gpu", out, dict(kw, precision="bf16", profile="wan_small", link_timeout_s=60.0), timeout=600)
    got = np.load(f"{out}.0.npy")
    seq = lp.run_sequential(lp.EngineConfig(mode="sequential", precision="bf16", profile=wan_small(), **kw))
    assert got.tobytes() == np.stack([b.values for b in seq.blocks]).tobytes()


def test_ipc_tpp_decode_rank_runs_patch_codec(tmp_path):
    # 2 DiT ranks + 1 decode rank on the Wan profile with the patch codec: the
    # decode rank decodes every block on its GPU and runs the AAS round trip;
    # latents and frames equal the single-process sequential run bitwise
    import hashlib

    kw = dict(steps=4, blocks=3, cache_capacity=2, patch_codec=1, pixel_scale=4, upsample=2)
    out = tmp_path / "res"
    launch(3, "gpu", out, dict(kw, precision="bf16", profile="wan_small", link_timeout_s=60.0, decode_gpu=1),
           timeout=600)
    got = np.load(f"{out}.0.npy")
    rec = json.load(open(f"{out}.0"))
    seq = lp.run_sequential(lp.EngineConfig(mode="sequential", precision="bf16", profile=wan_small(),
                                            **dict(kw, patch_codec=True)))
    assert got.tobytes() == np.stack([b.values for b in seq.blocks]).tobytes()
    assert rec["frames_sha256"] == hashlib.sha256(seq.frames.astype("<f4").tobytes()).hexdigest()


def test_ipc_4_plus_1_layout_with_vae_decode_rank(tmp_path):
    # the paper's 4 DiT + 1 VAE GPU layout (4 stage ranks + the decode rank
    # running the VAE stand-in on every received block), 5 ranks sharing one
    # GPU: the latents equal the single-process sequential run bitwise
    kw = dict(steps=4, blocks=3, cache_capacity=2, vae_decode=1)
    out = tmp_path / "res"
    launch(5, "gpu", out, dict(kw, precision="bf16", profile="wan_small", link_timeout_s=90.0, decode_gpu=1),
           timeout=900)
    got = np.load(f"{out}.0.npy")
    seq = lp.run_sequential(lp.EngineConfig(mode="sequential", precision="bf16", profile=wan_small(),
                                            **dict(kw, vae_decode=False)))
    assert got.tobytes() == np.stack([b.values for b in seq.blocks]).tobytes()


def test_ipc_two_pipelines_of_four_ranks(tmp_path):
    # the 8-GPU layout (two independent 4-stage pipelines, different noise
    # seeds) with 8 ranks sharing one GPU: each pipeline equals the
    # sequential run with its own seed, bitwise
    import dataclasses

    from paper_2512_04677_b200 import tpp_dist

    kw = dict(steps=4, blocks=3, cache_capacity=2)
    out = tmp_path / "res"
    launch(8, "gpu", out, dict(kw, precision="bf16", profile="wan_small", link_timeout_s=90.0), timeout=900)
    for pipe in (0, 1):
        got = np.load(f"{out}.{pipe}.npy")
        cfg = lp.EngineConfig(mode="sequential", precision="bf16", profile=wan_small(), **kw)
        cfg = dataclasses.replace(cfg, noise_seed=tpp_dist.pipe_noise_seed(cfg, pipe))
        seq = lp.run_sequential(cfg)
        assert got.tobytes() == np.stack([b.values for b in seq.blocks]).tobytes(), pipe


def test_ipc_tpp_stalled_consumer_raises_and_keeps_unconsumed_slot(tmp_path):
    # injected failure (engine.py:425-429 abort propagation): rank 1 (the
    # consumer) stops consuming for 6 s before block 2 with a 2 s link
    # timeout.  Rank 0's fused send for block 3 times out on the slot's free
    # counter: the sticky status gates its Euler-epilogue store and ready
    # publish, so block 2's latent -- sent but not yet consumed -- is NOT
    # overwritten; rank 1 then receives block 2 intact and fails on block 3.
    # Both ranks raise PipelineInvariantError.
    kw = dict(steps=4, blocks=6, cache_capacity=2)
    out = tmp_path / "res"
    launch(2, "gpu", out, dict(kw, precision="bf16", profile="wan_small", link_timeout_s=2.0, fused=1,
                               stall_rank=1, stall_block=2, stall_s=6.0), timeout=600)
    r0 = json.load(open(f"{out}.rank0"))
    r1 = json.load(open(f"{out}.rank1"))
    assert r0["error"] and "status" in r0["error"], r0
    assert r1["error"], r1
    assert r1["blocks_done"] == 3, r1  # blocks 0, 1 and the unconsumed block 2
    got = np.load(f"{out}.rank1.npy")
    seq = lp.run_sequential(lp.EngineConfig(mode="sequential", precision="bf16", profile=wan_small(), **kw))
    assert got.tobytes() == np.stack([b.values for b in seq.blocks[:3]]).tobytes()
