"""Pin the CPU oracle (oracle/livepipe_oracle.py) against golden vectors
produced by the reference itself (tests/golden/make_golden.py)."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import livepipe_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))
META = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def _cfg(kw):
    return O.RolloutCfg(**kw)


@pytest.mark.parametrize("name", ["c1", "c1_sigma", "c1_scaled", "c1_L1", "c1_delta3"])
def test_rollout_digests_match_reference(name):
    m = META[name]
    blocks, frames, _ = O.run_sequential(_cfg(m["kw"]))
    assert hashlib.sha256(O.latents_bytes(blocks)).hexdigest() == m["latents_sha256"]
    assert hashlib.sha256(frames.astype("<f4").tobytes()).hexdigest() == m["frames_sha256"]
    np.testing.assert_array_equal(np.stack(blocks), G[f"{name}_latents"])


def test_single_calls_bitwise():
    w = O.build_weights(7, O.TOY)
    cache = []
    for i in range(6):
        vel, e = O.dit_forward(O.TOY, w, 4, G["call_x"][i], i, 3, cache, G["call_audio"][i],
                               G["call_prompt"], G["call_sink"], i + 1, max_entries=4)
        assert vel.tobytes() == G[f"call{i}_velocity"].tobytes()
        assert e.keys[0].tobytes() == G[f"call{i}_k0"].tobytes()
        assert e.values[1].tobytes() == G[f"call{i}_v1"].tobytes()
        O.push(cache, e, 4)
    view = O.corrupt(cache, 0.25, 11, 9, 3)
    assert np.stack([e.keys[0] for e in view]).tobytes() == G["corrupt_k0"].tobytes()
    assert np.stack([e.values[1] for e in view]).tobytes() == G["corrupt_v1"].tobytes()


def test_window_matches_bruteforce_golden():
    # rolling cache with L=2 reproduces the reference's mask-based oracle
    w = O.build_weights(7, O.TOY)
    cache = []
    for i in range(6):
        vel, e = O.dit_forward(O.TOY, w, 4, G["call_x"][i], i, 3, cache, G["call_audio"][i],
                               G["call_prompt"], G["call_sink"], i + 1, max_entries=2)
        np.testing.assert_allclose(vel, G["brute_w2"][i], atol=1e-5)
        O.push(cache, e, 2)


def test_numerics_golden():
    np.testing.assert_array_equal(O.softmax_rows(np.array([1.0, 2.0, 3.0], np.float32)),
                                  G["softmax_123"])
    c, s = O.rope_cos_sin(40_000, 8, 10000.0)
    v = O.normal(3, 0, 8)
    assert O.rotate_pairs(v, c, s).tobytes() == G["rope_40000"].tobytes()
    w = O.build_weights(7, O.TOY)
    assert w.w2[1].tobytes() == G["w_l1_w2"].tobytes()
    assert w.w_vel.tobytes() == G["w_vel"].tobytes()
    assert O.noise_block(O.RolloutCfg(), 5).tobytes() == G["noise_b5"].tobytes()


def test_visible_schedule_matches_window_rule():
    for cap in (1, 2, 4):
        sched = O.visible_schedule(20, cap)
        for i, vis in enumerate(sched):
            mask = O.visible_mask(i, cap)
            assert vis == [m for m in range(i) if mask[m]]


@pytest.mark.parametrize("name", ["c1_clean", "c1_clean_sigma"])
def test_clean_kv_digests_match_reference(name):
    m = META[name]
    blocks, frames, nfe = O.run_clean_kv(_cfg(m["kw"]))
    assert hashlib.sha256(O.latents_bytes(blocks)).hexdigest() == m["latents_sha256"]
    assert hashlib.sha256(frames.astype("<f4").tobytes()).hexdigest() == m["frames_sha256"]
    assert nfe == m["nfe"]
