"""Generate golden vectors by importing the REFERENCE implementation.

Run in the build container (needs /root/reference, read-only):

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz and tests/golden/golden.json.  These pin the
oracle (tests/test_oracle_golden.py) and, through it, the CUDA path.  The
reference is imported read-only from /root/reference/pkg/src; nothing is
copied from it.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    import livepipe as lp  # noqa: E402  (reference, read-only)
    from livepipe.denoiser import attention_bruteforce, build_weights, ToyDenoiser  # noqa: E402
    from livepipe.kvcache import RollingKvCache, corrupt_history, corruption_prng  # noqa: E402

    arrays: dict = {}
    meta: dict = {"numpy": np.__version__, "python": sys.version.split()[0]}

    # 1. config #1 rollouts (EngineConfig defaults with blocks=3, T=4): digests
    for name, kw in {
        "c1": dict(steps=4, blocks=3),
        "c1_sigma": dict(steps=4, blocks=3, history_sigma=0.3),
        "c1_scaled": dict(steps=4, blocks=5, history_sigma=0.2, history_mode="scaled"),
        "c1_L1": dict(steps=2, blocks=6, cache_capacity=1),
        "c1_delta3": dict(steps=3, blocks=4, sink_delta=3),
        "c1_oracle": dict(steps=4, blocks=3, denoiser_kind="oracle"),
    }.items():
        seq = lp.run_sequential(lp.EngineConfig(mode="sequential", **kw))
        tpp = lp.run_tpp(lp.EngineConfig(mode="tpp", **kw))
        assert lp.latents_digest(seq.blocks) == lp.latents_digest(tpp.blocks)
        meta[name] = {
            "kw": kw,
            "latents_sha256": lp.latents_digest(seq.blocks),
            "frames_sha256": lp.frames_digest(seq.frames),
            "nfe": seq.nfe,
        }
        arrays[f"{name}_latents"] = np.stack([b.values for b in seq.blocks])
        arrays[f"{name}_frames"] = seq.frames

    # 1b. clean-KV baseline rollouts (engine.py:292-331): unified cache fed by the
    # extra cache_entry pass, NFE = (T+1) per block
    for name, kw in {
        "c1_clean": dict(steps=4, blocks=3),
        "c1_clean_sigma": dict(steps=3, blocks=4, cache_capacity=2, history_sigma=0.2),
    }.items():
        res = lp.run_clean_kv(lp.EngineConfig(mode="clean_kv", **kw))
        meta[name] = {"kw": kw, "latents_sha256": lp.latents_digest(res.blocks),
                      "frames_sha256": lp.frames_digest(res.frames), "nfe": res.nfe}
        arrays[f"{name}_latents"] = np.stack([b.values for b in res.blocks])
        arrays[f"{name}_frames"] = res.frames

    # 2. single denoise_block calls with a history view (velocity + kv)
    w = build_weights(7)
    sched = lp.TimestepSchedule.uniform(4)
    toy = ToyDenoiser(w, sched)
    cache = RollingKvCache(3, 4)
    xs, conds = [], []
    for i in range(6):
        x = lp.LatentBlock(lp.Prng(20, i).normal((3, 16)), i)
        cond = lp.BlockCond(audio=lp.Prng(8, i).gaussian(8), prompt=lp.Prng(9, 0).gaussian(8))
        xs.append(x.values)
        conds.append(cond.audio)
        out = toy.denoise_block(x, 3, cache.view(), cond, lp.Prng(5, 0).gaussian(16), i + 1,
                                max_entries=4)
        arrays[f"call{i}_velocity"] = out.velocity
        arrays[f"call{i}_k0"] = out.kv.keys[0]
        arrays[f"call{i}_v1"] = out.kv.values[1]
        cache.push(out.kv)
    arrays["call_x"] = np.stack(xs)
    arrays["call_audio"] = np.stack(conds)
    arrays["call_prompt"] = lp.Prng(9, 0).gaussian(8)
    arrays["call_sink"] = lp.Prng(5, 0).gaussian(16)

    # 3. brute-force (mask-based) velocities for window 2 over 6 blocks
    bl = [lp.LatentBlock(a, i) for i, a in enumerate(xs)]
    cn = [lp.BlockCond(audio=a, prompt=arrays["call_prompt"]) for a in conds]
    brute = attention_bruteforce(bl, 3, cn, arrays["call_sink"], 1, 2, w, sched)
    arrays["brute_w2"] = np.stack(brute)

    # 4. corrupted view of the call cache at (block 9, step 3), sigma 0.25
    view = corrupt_history(cache, 0.25, corruption_prng(11, 9, 3))
    arrays["corrupt_k0"] = np.stack([e.keys[0] for e in view])
    arrays["corrupt_v1"] = np.stack([e.values[1] for e in view])

    # 5. numerics: softmax frozen values, rope rows at a long position, weights
    arrays["softmax_123"] = lp.softmax(np.array([1.0, 2.0, 3.0], dtype=np.float32))
    arrays["rope_40000"] = lp.rope_rotate(lp.Prng(3, 0).gaussian(8), 40_000)
    arrays["w_l1_w2"] = w.layers[1].w2
    arrays["w_vel"] = w.w_vel
    arrays["noise_b5"] = lp.noise_block(lp.EngineConfig(), 5).values

    # 6. simulate() fit and speed-up law (virtual clock, for the timeline tests)
    sim = lp.simulate([0.574] * 5, "tpp", blocks=32, frames_per_block=12)
    meta["table3_fps_steady"] = lp.compute_fps(sim.timeline, sim.total_frames).steady
    meta["table3_ttff"] = lp.compute_ttff(0.0, sim.timeline)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    blob = json.dumps(meta, indent=1, sort_keys=True)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        fh.write(blob + "\n")
    print("wrote", len(arrays), "arrays;", hashlib.sha256(blob.encode()).hexdigest()[:12])


if __name__ == "__main__":
    main()
