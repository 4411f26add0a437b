"""The drop-in inside the UNMODIFIED reference engine.

The reference package is staged (unmodified) into the git-ignored
``baseline/_ref`` by ``scripts/stage_reference.sh``; that directory travels
to the GPU box with the repo snapshot.  These tests rebind the reference's
``build_runtime`` (engine.py:177-201) with ``integration.install`` -- the
recipe INTEGRATION.md section 1 gives -- and run the reference's OWN
``run_sequential`` / ``run_tpp`` / ``run_clean_kv`` (engine.py:255-496),
``RollingKvCache``, ``corrupt_history`` (its ``dataclasses.replace`` on the
B200 entries, kvcache.py:121-137), AAS and codec around the B200 denoiser:
latents match the goldens the reference produced to the fp32 bar, TPP ==
sequential bitwise, and the reference's ``except`` clauses catch the B200
path's errors."""

import json
import os
import sys

import numpy as np
import pytest

import paper_2512_04677_b200 as lp
from paper_2512_04677_b200 import integration

from gpu_helpers import rel_l2

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(os.path.dirname(HERE), "baseline", "_ref")
G = np.load(os.path.join(HERE, "golden", "golden.npz"))
META = json.load(open(os.path.join(HERE, "golden", "golden.json")))
TOL_FP32 = 1e-5


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "livepipe")):
        pytest.skip("reference not staged in baseline/_ref (scripts/stage_reference.sh)")
    sys.path.insert(0, REF)
    import livepipe  # noqa: F401  (the unmodified reference)
    import livepipe.engine as E

    yield E


@pytest.fixture()
def installed(ref):
    h = integration.install(ref, precision="fp32")
    yield h
    h.uninstall()


@pytest.mark.parametrize("name", ["c1", "c1_sigma", "c1_scaled", "c1_delta3"])
def test_reference_run_sequential_with_b200_denoiser(ref, installed, name):
    kw = META[name]["kw"]
    res = ref.run_sequential(ref.EngineConfig(mode="sequential", **kw))
    assert installed.denoisers and isinstance(installed.denoisers[-1], lp.B200Denoiser)
    got = np.stack([b.values for b in res.blocks])
    assert rel_l2(got, G[f"{name}_latents"]) < TOL_FP32
    assert rel_l2(res.frames, G[f"{name}_frames"]) < TOL_FP32
    assert res.nfe == META[name]["nfe"]


@pytest.mark.parametrize("name", ["c1", "c1_sigma"])
def test_reference_run_tpp_bitwise_equals_its_sequential(ref, installed, name):
    kw = META[name]["kw"]
    seq = ref.run_sequential(ref.EngineConfig(mode="sequential", **kw))
    tpp = ref.run_tpp(ref.EngineConfig(mode="tpp", **kw))
    assert all(a.values.tobytes() == b.values.tobytes() for a, b in zip(seq.blocks, tpp.blocks))
    assert rel_l2(np.stack([b.values for b in tpp.blocks]), G[f"{name}_latents"]) < TOL_FP32


def test_reference_run_clean_kv_with_b200_denoiser(ref, installed):
    kw = META["c1_clean"]["kw"]
    res = ref.run_clean_kv(ref.EngineConfig(mode="clean_kv", **kw))
    assert rel_l2(np.stack([b.values for b in res.blocks]), G["c1_clean_latents"]) < TOL_FP32
    assert res.nfe == META["c1_clean"]["nfe"]


def test_reference_exceptions_catch_b200_errors(ref):
    import livepipe.denoiser as RD

    dn = lp.B200Denoiser(lp.build_weights(7), lp.TimestepSchedule.uniform(4), precision="fp32")
    x = lp.LatentBlock(G["call_x"][0], 0)
    cond = lp.BlockCond(audio=G["call_audio"][0], prompt=G["call_prompt"])
    out = dn.denoise_block(x, 3, (), cond, G["call_sink"], 1)
    with pytest.raises(RD.TimestepForcingError, match="but denoising at 2"):
        dn.denoise_block(lp.LatentBlock(G["call_x"][1], 1), 2, (out.kv,), cond, G["call_sink"], 2)
    with pytest.raises(lp.TimestepForcingError):
        dn.denoise_block(lp.LatentBlock(G["call_x"][1], 1), 2, (out.kv,), cond, G["call_sink"], 2)


def test_reference_typed_entries_and_pool_growth(ref):
    # the reference's own KvEntry objects (host tuples) in the view, and a
    # pool started at ONE slot so every call grows it while entries live
    import livepipe.denoiser as RD
    import livepipe.latent as RL

    w = RD.build_weights(7)
    sched = RL.TimestepSchedule.uniform(4)
    toy = RD.ToyDenoiser(w, sched)
    dn = lp.B200Denoiser(w, sched, precision="fp32", max_live_entries=1)
    cache_ref, cache_b = [], []
    for i in range(6):
        x = lp.LatentBlock(G["call_x"][i], i)
        cond = RD.BlockCond(audio=G["call_audio"][i], prompt=G["call_prompt"])
        want = toy.denoise_block(x, 3, tuple(cache_ref), cond, G["call_sink"], i + 1, max_entries=4)
        # mixed view: reference-typed host entries for even blocks, device entries for odd ones
        view = tuple(r if (e.block_index % 2 == 0) else b for e, r, b in
                     zip(cache_ref, cache_ref, cache_b))
        got = dn.denoise_block(x, 3, view, cond, G["call_sink"], i + 1, max_entries=4)
        assert rel_l2(got.velocity, want.velocity) < TOL_FP32
        assert rel_l2(np.stack(got.kv.keys), np.stack(want.kv.keys)) < TOL_FP32
        cache_ref = (cache_ref + [want.kv])[-4:]
        cache_b = (cache_b + [got.kv])[-4:]
    assert dn._pool.n_slots > 1  # grew on demand


def test_dataclasses_replace_yields_host_entry():
    import dataclasses

    dn = lp.B200Denoiser(lp.build_weights(7), lp.TimestepSchedule.uniform(4), precision="fp32")
    x = lp.LatentBlock(G["call_x"][0], 0)
    cond = lp.BlockCond(audio=G["call_audio"][0], prompt=G["call_prompt"])
    e = dn.denoise_block(x, 3, (), cond, G["call_sink"], 1).kv
    assert e.on_device
    keys = tuple(k + 1.0 for k in e.keys)
    h = dataclasses.replace(e, keys=keys)
    assert not h.on_device and h.block_index == 0 and h.timestep_index == 3
    assert np.array_equal(h.keys[0], e.keys[0] + 1.0) and np.array_equal(h.values[1], e.values[1])


def test_dropin_14b_shape_fits_in_hbm():
    # the drop-in at the 14B shape (40 layers, d 5120, 4,680 tokens per block):
    # the reference engine's window of L=4 device entries plus the in-flight
    # one through denoise_block; the VMM slot pool maps only what is alive,
    # so device memory stays far below the 180 GB of HBM (the round-1 pool
    # reserved ~385 GB up front)
    import torch

    from paper_2512_04677_b200.model import DeviceWeights

    prof = lp.WAN_14B
    dw = DeviceWeights.random(prof, "bf16", "cuda:0", 7)
    sched = lp.TimestepSchedule.uniform(4)
    dn = lp.B200Denoiser(None, sched, precision="bf16", device_weights=dw)
    conds = lp.synthetic_conditions(11, 6, prof.audio_dim, prof.prompt_dim, prof.latent_dim)
    cache = lp.RollingKvCache(4, 4)
    rng = np.random.default_rng(0)
    for i in range(6):
        x = lp.LatentBlock(rng.standard_normal((3, prof.latent_dim), dtype=np.float32), i)
        out = dn.denoise_block(x, 4, cache.view(), lp.BlockCond(conds.audio_for(i), conds.prompt),
                               conds.reference, i + 1, max_entries=4)
        assert np.isfinite(out.velocity).all()
        cache.push(out.kv)
    torch.cuda.empty_cache()  # allocator cache of earlier tests in this process
    free, total = torch.cuda.mem_get_info(0)
    used_gb = (total - free) / 1e9
    assert used_gb < 120.0, used_gb
