"""Decode stage on the GPU: the reference codec through
lp_gemm's pinned fp32 path and the patch codec (VAE stand-in) through
lp_codec_patch_decode/_encode, bit-identical to the CPU restatements; the
engines decode and run the AAS round trip with them."""

import dataclasses
import hashlib
import json
import os

import numpy as np
import pytest
import torch

import paper_2512_04677_b200 as lp
from oracle import livepipe_oracle as O

from gpu_helpers import rel_l2

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
META = json.load(open(os.path.join(HERE, "golden", "golden.json")))


@pytest.mark.parametrize("dims", [(16, 32, 4), (64, 300, 3), (128, 1000, 1)])
def test_dense_codec_bitwise(dims):
    D, P, r = dims
    host = lp.ToyVideoCodec(7, D, P, r)
    dc = lp.DeviceCodec(host, 0)
    x = np.random.default_rng(D).standard_normal((3, D)).astype(np.float32)
    fr = dc.decode(lp.LatentBlock(x, 0))
    assert fr.tobytes() == host.decode(lp.LatentBlock(x, 0)).tobytes()
    assert dc.encode(fr[0]).tobytes() == host.encode(fr[0]).tobytes()
    assert dc.decode_frame(x[1]).tobytes() == host.decode_frame(x[1]).tobytes()


def test_dense_codec_reproduces_golden_frames():
    # c1 latents from the (golden-pinned) oracle decoded on the GPU -> the reference's frame digest
    blocks, frames, _ = O.run_sequential(O.RolloutCfg(**META["c1"]["kw"]))
    dc = lp.DeviceCodec(lp.ToyVideoCodec(7, 16, 32, 4), 0)
    out = np.concatenate([dc.decode(lp.LatentBlock(b, i)) for i, b in enumerate(blocks)])
    assert hashlib.sha256(out.astype("<f4").tobytes()).hexdigest() == META["c1"]["frames_sha256"]


@pytest.mark.parametrize("geom", [(16, 6, 10, 3, 8, 4), (5, 3, 7, 2, 3, 2), (20, 2, 5, 3, 4, 1),
                                  (16, 1, 1, 32, 1, 4), (16, 4, 130, 3, 8, 2)])
def test_patch_codec_bitwise(geom):
    C, H, W, pc, s, r = geom
    o = O.PatchCodec(7, C, H, W, pc, s, r)
    dc = lp.DeviceCodec(lp.PatchVideoCodec(7, C, H, W, pc, s, r), 0)
    x = np.random.default_rng(2).standard_normal((3, C * H * W)).astype(np.float32)
    fr = dc.decode(lp.LatentBlock(x, 0))
    assert fr.tobytes() == o.decode(x).tobytes()
    assert dc.encode(fr[0]).tobytes() == o.encode(fr[0]).tobytes()


def test_patch_codec_480p_bitwise_and_bandwidth():
    # the 14B/480p decode: latent (3, 16, 60, 104) -> 12 frames of 3 x 480 x 832
    C, H, W, pc, s, r = 16, 60, 104, 3, 8, 4
    o = O.PatchCodec(7, C, H, W, pc, s, r)
    dc = lp.DeviceCodec(lp.PatchVideoCodec(7, C, H, W, pc, s, r), 0)
    x = torch.randn((3, C * H * W), device="cuda:0")
    out = torch.empty((3 * r, dc.pixel_dim), device="cuda:0")
    dc.decode_into(x, out)
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == o.decode(x.cpu().numpy()).tobytes()
    z = dc.aas_sink_device(x)
    assert z.cpu().numpy().tobytes() == o.encode(o.decode(x.cpu().numpy()[:1])[0]).tobytes()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        dc.decode_into(x, out)
    e0.record()
    n = 20
    for _ in range(n):
        dc.decode_into(x, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    gbs = (x.numel() + out.numel()) * 4 / (ms * 1e-3) / 1e9
    print(f"patch decode 480p: {ms * 1e3:.1f} us/block, {gbs:.0f} GB/s")
    assert ms < 1.0  # HBM-bound: ~60 MB per block


def _wan(layers=2, heads=2, ffn=384, h=8, w=12):
    po = O.wan_profile(n_layers=layers, n_heads=heads, head_dim=128, ffn_dim=ffn, channels=16, height=h, width=w)
    return po, lp.ModelProfile(**dataclasses.asdict(po))


@pytest.mark.parametrize("mode", ["sequential", "tpp"])
def test_wan_rollout_with_patch_codec_matches_oracle(mode):
    po, pp = _wan()
    kw = dict(steps=3, blocks=4, cache_capacity=2, upsample=2)
    oc = O.PatchCodec(7, 16, 8, 12, 3, 4, 2)
    blocks, frames, sink = O.run_sequential(O.RolloutCfg(profile=po, **kw), mm=O.mm_f64, codec=oc)
    cfg = lp.EngineConfig(mode=mode, profile=pp, precision="fp32", patch_codec=True, pixel_scale=4, **kw)
    res = lp.run(cfg)
    assert max(rel_l2(b.values, r) for b, r in zip(res.blocks, blocks)) < 1e-5
    assert res.frames.shape == frames.shape
    assert rel_l2(res.frames, frames) < 1e-5


def test_aas_round_trip_on_device_is_bitwise():
    _, pp = _wan()
    cfg = lp.EngineConfig(mode="sequential", profile=pp, precision="bf16", patch_codec=True, steps=2, blocks=2,
                          cache_capacity=2)
    rt = lp.build_runtime(cfg)
    pipe = lp.StreamingPipeline(cfg, rt)
    noise = torch.from_numpy(lp.noise_block(cfg, 0).values).cuda()
    x = pipe.submit(0, noise)
    torch.cuda.synchronize()
    pipe.aas(x)
    o = O.PatchCodec(7, 16, 8, 12, 3, 8, cfg.upsample)
    xh = x.float().cpu().numpy()
    want = o.encode(o.decode(xh)[0])
    assert pipe.sink.content.tobytes() == want.tobytes()
    assert pipe.sink.locked
