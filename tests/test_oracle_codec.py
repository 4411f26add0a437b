"""The decode-stage codec restatements, CPU only.

The reference codec (latent.py:150-193) is pinned through the golden frame
digests (test_oracle_golden.py).  The patch codec that stands in for the VAE
on patched profiles is builder-defined; it is pinned here by reducing it to
the reference codec (H = W = 1, s = 1, pc = pixel_dim draws the same maps in
the same order and sums in the same order) and by its round trip."""

import numpy as np
import pytest

from oracle import livepipe_oracle as O
from paper_2512_04677_b200.latent import PatchVideoCodec, ToyVideoCodec


def _golden_c1_block0():
    blocks, frames, _ = O.run_sequential(O.RolloutCfg(steps=4, blocks=1))
    return blocks[0], frames


def test_patch_codec_reduces_to_reference_codec():
    x, frames = _golden_c1_block0()  # golden-pinned latents and frames (digest c1)
    cfg = O.RolloutCfg()
    dense = O.Codec(cfg.weight_seed, 16, cfg.pixel_dim, cfg.upsample)
    patch = O.PatchCodec(cfg.weight_seed, 16, 1, 1, pixel_channels=cfg.pixel_dim, scale=1, upsample=cfg.upsample)
    np.testing.assert_array_equal(patch.maps, np.stack(dense.dec))
    np.testing.assert_array_equal(patch.enc, dense.enc)
    np.testing.assert_array_equal(patch.decode(x), frames)
    np.testing.assert_array_equal(patch.encode(frames[0]), dense.encode(frames[0]))


@pytest.mark.parametrize("geom", [(16, 6, 10, 3, 8, 4), (5, 3, 7, 2, 3, 2), (20, 2, 5, 3, 4, 1)])
def test_patch_codec_round_trip_and_parameters(geom):
    C, H, W, pc, s, r = geom
    o = O.PatchCodec(7, C, H, W, pc, s, r)
    p = PatchVideoCodec(7, C, H, W, pc, s, r)
    assert o.maps.tobytes() == p.maps.tobytes() and o.enc.tobytes() == p.enc.tobytes()
    assert p.latent_dim == C * H * W and p.pixel_dim == pc * H * s * W * s
    x = np.random.default_rng(1).standard_normal((3, C * H * W)).astype(np.float32)
    fr = o.decode(x)
    assert fr.shape == (3 * r, p.pixel_dim)
    # frame u of latent frame f is the per-location map applied at every location
    f, u, h, w = 1, r - 1, H - 1, W // 2
    img = fr[f * r + u].reshape(pc, H * s, W * s)
    patch = img[:, h * s:(h + 1) * s, w * s:(w + 1) * s].reshape(-1)
    lat = x[f].reshape(C, H, W)[:, h, w]
    np.testing.assert_allclose(patch, o.maps[u].astype(np.float64) @ lat, rtol=1e-5, atol=1e-5)
    z = o.encode(fr[0])
    assert np.abs(z - x[0]).max() < 1e-4 * max(1.0, np.abs(x[0]).max())


def test_patch_codec_geometry_errors():
    with pytest.raises(ValueError):
        PatchVideoCodec(7, 16, 4, 4, pixel_channels=1, scale=2)  # 4 pixels < 16 channels: no left inverse
    with pytest.raises(ValueError):
        PatchVideoCodec(7, 16, 4, 4, upsample=0)
    with pytest.raises(ValueError):
        ToyVideoCodec(7, 16, 8, 4)


def test_engine_config_codec_fields():
    import paper_2512_04677_b200 as lp

    for bad in (dict(pixel_scale=0), dict(pixel_channels=0), dict(upsample=0)):
        with pytest.raises(lp.EngineConfigError):
            lp.EngineConfig(**bad)
    cfg = lp.EngineConfig(patch_codec=True, pixel_channels=3, pixel_scale=8)
    assert cfg.patch_codec and cfg.pixel_scale == 8
