"""Worker for the multi-process TPP tests (launched by torch.distributed.run).

    python -m torch.distributed.run --nproc-per-node N tests/dist_worker.py <mode> <out.json> [k=v ...]

mode ``cpu``: gloo process group, the TPP host runtime (tpp_dist.DistTPP)
driving an ORACLE backend over torch.distributed send/recv -- checks the
layout / sequencing / sink-broadcast logic on a CPU box.  The oracle here is
the checker's compute, never the product path.
mode ``gpu``: gloo process group for the handle exchange + IPC links on the
GPU(s) (several ranks may share cuda:0), the real device backend.
The last rank of every pipeline writes its latents digest to <out.json>.<pipe>.
"""

import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402


class OracleBackend:
    """CPU compute for the owned steps of one rank (test infrastructure)."""

    def __init__(self, cfg, role):
        from oracle import livepipe_oracle as O

        self.O = O
        self.role = role
        self.rc = O.RolloutCfg(steps=cfg.steps, cache_capacity=cfg.cache_capacity,
                               frames_per_block=cfg.frames_per_block, pixel_dim=cfg.pixel_dim,
                               upsample=cfg.upsample, sink_delta=cfg.sink_delta, blocks=cfg.blocks,
                               weight_seed=cfg.weight_seed, noise_seed=cfg.noise_seed,
                               history_sigma=cfg.history_sigma, history_mode=cfg.history_mode)
        self.w = O.build_weights(cfg.weight_seed, self.rc.profile)
        self.audio, self.prompt, self.ref = O.conditions(self.rc)
        self.codec = O.Codec(cfg.weight_seed, self.rc.profile.latent_dim, cfg.pixel_dim, cfg.upsample)
        self.caches = {j: [] for j in role.steps}
        self.shape = (cfg.frames_per_block, self.rc.profile.latent_dim)
        self.sink = None
        self.x = None
        self._nfe = 0

    def reference_sink(self):
        return self.ref.copy()

    def set_sink(self, content):
        self.sink = np.asarray(content, np.float32).copy()

    def load_host(self, x):
        self.x = np.asarray(x, np.float32).copy()

    def denoise(self, i):
        O, rc = self.O, self.rc
        for j in self.role.steps:
            sigma = rc.history_sigma
            if rc.history_mode == "scaled":
                sigma = sigma * O.level(rc.steps, j)
            view = O.corrupt(self.caches[j], sigma, rc.noise_seed, i, j)
            vel, e = O.dit_forward(rc.profile, self.w, rc.steps, self.x, i, j, view, self.audio[i], self.prompt,
                                   self.sink, i + rc.sink_delta, max_entries=rc.cache_capacity)
            self.x = O.euler(self.x, vel, -1.0 / rc.steps)
            O.push(self.caches[j], e, rc.cache_capacity)
            self._nfe += 1

    def read_output(self):
        return self.x.copy()

    def nfe(self):
        return self._nfe

    def aas(self, sink, xb):
        from paper_2512_04677_b200.kvcache import SinkLockedError

        if sink.locked:
            raise SinkLockedError("sink already replaced once this rollout")
        sink.content = self.codec.encode(self.codec.decode(xb.values)[0])
        sink.locked = True

    def decode(self, xb):
        return self.codec.decode(xb.values)


def wan_small():
    """The small Wan-shaped profile of tests/test_gpu_wan.py."""
    import paper_2512_04677_b200 as lp

    return lp.wan_profile(n_layers=2, n_heads=2, head_dim=128, ffn_dim=384, channels=16, height=8, width=12)


def main():
    mode, out = sys.argv[1], sys.argv[2]
    kw = {}
    for a in sys.argv[3:]:
        k, v = a.split("=")
        kw[k] = float(v) if "." in v else (int(v) if v.lstrip("-").isdigit() else v)
    dist.init_process_group("gloo")
    import paper_2512_04677_b200 as lp
    from paper_2512_04677_b200 import tpp_dist
    from oracle import livepipe_oracle as O

    rank, world = dist.get_rank(), dist.get_world_size()
    decode_gpu = bool(kw.pop("decode_gpu", 0))
    if mode == "cpu":
        cfg = lp.EngineConfig(mode="tpp", **kw)
        role = tpp_dist.pipeline_layout(world, cfg.steps, decode_gpu)[rank]
        seed = tpp_dist.pipe_noise_seed(cfg, role.pipe)
        import dataclasses

        be = OracleBackend(dataclasses.replace(cfg, noise_seed=seed), role)
        res = tpp_dist.run_tpp_dist(cfg, backend=be, transport="dist", decode_gpu=decode_gpu)
    else:
        import torch

        dev = int(os.environ.get("LP_TEST_DEVICE", "0"))
        torch.cuda.set_device(dev)
        prec = kw.pop("precision", "fp32")
        fused = bool(kw.pop("fused", 1))
        if kw.pop("profile", None) == "wan_small":
            kw["profile"] = wan_small()
        stall = (int(kw.pop("stall_rank", -1)), int(kw.pop("stall_block", -1)), float(kw.pop("stall_s", 0.0)))
        cfg = lp.EngineConfig(mode="tpp", precision=prec, devices=(dev,), **kw)
        role = tpp_dist.pipeline_layout(world, cfg.steps, decode_gpu)[rank]
        if stall[0] < 0:
            res = tpp_dist.run_tpp_dist(cfg, transport="ipc", device=dev, fused_send=fused, decode_gpu=decode_gpu)
        else:
            # injected failure: rank stall[0] stops consuming for stall[2] s
            # before block stall[1] (longer than link_timeout_s); every rank
            # records what it raised and the blocks it completed
            import time

            res = None
            runner = tpp_dist.DistTPP(cfg, transport="ipc", device=dev, fused_send=fused)
            done, err = [], None
            try:
                for i in range(cfg.blocks):
                    if rank == stall[0] and i == stall[1]:
                        time.sleep(stall[2])
                    xb = runner.step(i)
                    if xb is not None:
                        done.append(np.asarray(xb.values, np.float32))
                runner.finish()
            except lp.PipelineInvariantError as e:
                err = str(e)
                runner.abort_peers()
            torch.cuda.synchronize(dev)
            with open(f"{out}.rank{rank}", "w") as f:
                json.dump({"rank": rank, "error": err, "blocks_done": len(done)}, f)
            if done:
                np.save(f"{out}.rank{rank}.npy", np.stack(done))
            runner.close()
    if res is not None:
        lat = np.stack([np.asarray(b.values, np.float32) for b in res.blocks])
        rec = {"latents_sha256": hashlib.sha256(O.latents_bytes(list(lat))).hexdigest(), "nfe": res.nfe,
               "frames_sha256": (hashlib.sha256(res.frames.astype("<f4").tobytes()).hexdigest()
                                 if res.frames is not None else None), "rank": rank}
        np.save(f"{out}.{role.pipe}.npy", lat)
        with open(f"{out}.{role.pipe}", "w") as f:
            json.dump(rec, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
