"""LPD1 dumps and timeline files (reference harness.py:194-292 formats):
byte-identical to the reference's on the golden rollouts, round trips."""

import json
import os

import numpy as np
import pytest

from oracle import livepipe_oracle as O
from paper_2512_04677_b200 import artifacts as A
from paper_2512_04677_b200.metrics import TimelineEvent, metrics_from_timeline

HERE = os.path.dirname(os.path.abspath(__file__))
META = json.load(open(os.path.join(HERE, "golden", "golden.json")))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))


@pytest.mark.parametrize("name", ["c1", "c1_sigma", "c1_L1"])
def test_lpd1_digest_matches_reference(name, tmp_path):
    blocks = list(G[f"{name}_latents"])
    assert A.latents_digest(blocks) == META[name]["latents_sha256"]
    assert A.latents_bytes(blocks) == O.latents_bytes(blocks)
    assert A.frames_digest(G[f"{name}_frames"]) == META[name]["frames_sha256"]
    p = A.write_latents(str(tmp_path / "x.lpd"), blocks)
    np.testing.assert_array_equal(A.read_latents(p), np.stack(blocks))


def test_lpd1_rejects_bad_files(tmp_path):
    p = tmp_path / "bad"
    p.write_bytes(b"XXXX" + bytes(12))
    with pytest.raises(A.ArtifactError):
        A.read_latents(str(p))
    p.write_bytes(A.latents_bytes([np.zeros((3, 16), np.float32)])[:-4])
    with pytest.raises(A.ArtifactError, match="truncated"):
        A.read_latents(str(p))


def test_timeline_roundtrip_exact(tmp_path):
    tl = [TimelineEvent(1, 0, 0.0, 0.1234567891234, "denoise"), TimelineEvent(2, 0, 0.2, 0.3, "denoise"),
          TimelineEvent(3, 0, 0.3, 0.35, "decode"), TimelineEvent(1, 1, 0.1234567891234, 0.24, "denoise"),
          TimelineEvent(2, 1, 0.3, 0.4, "denoise"), TimelineEvent(3, 1, 0.4, 0.45, "decode")]
    m = metrics_from_timeline(tl, 24, 0.0, 4)
    p = A.export_timeline(tl, str(tmp_path / "t.csv"), m)
    ev, rec = A.parse_timeline(p)
    assert ev == tl
    assert rec["nfe"] == 4 and rec["fps_steady"] == m.fps_steady
    with open(p) as fh:
        assert fh.readline().rstrip() == "stage,block,start,end,kind"


def _random_timeline(rng, stages, blocks):
    tl, t = [], 0.0
    for b in range(blocks):
        for s in range(1, stages + 1):
            t0 = t + float(rng.uniform(0, 0.01))
            tl.append(TimelineEvent(s, b, t0, t0 + float(rng.uniform(0.001, 0.05)), "denoise"))
            t = t0
        t0 = tl[-1].end
        tl.append(TimelineEvent(stages + 1, b, t0, t0 + float(rng.uniform(0.001, 0.01)), "decode"))
        if rng.uniform() < 0.3:
            tl.append(TimelineEvent(1, b, t0, t0 + 0.002, "idle"))
    rng.shuffle(tl)
    return tl


def test_metrics_match_reference_definitions():
    # the columnar metrics against the reference module (when importable
    # here; /root/reference does not exist on the GPU box) on random timelines
    pytest.importorskip("numpy")
    import sys

    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present")
    sys.path.insert(0, ref)
    try:
        from livepipe import metrics as R
    finally:
        sys.path.remove(ref)
    from paper_2512_04677_b200 import metrics as M

    rng = np.random.default_rng(3)
    for trial in range(20):
        tl = _random_timeline(rng, 1 + trial % 5, 1 + trial % 7)
        rtl = [R.TimelineEvent(e.stage, e.block, e.start, e.end, e.kind) for e in tl]
        assert M.compute_fps(tl, 48) == tuple(R.compute_fps(rtl, 48))
        assert M.compute_ttff(0.25, tl) == R.compute_ttff(0.25, rtl)
        assert M.stage_utilization(tl) == R.stage_utilization(rtl)
        f, r = rng.standard_normal((12, 40)), rng.standard_normal(40)
        np.testing.assert_allclose(M.drift_metric(f, r), R.drift_metric(f, r), rtol=1e-14)
    for bad in ([], [TimelineEvent(1, 0, 0.0, 1.0, "denoise")]):
        with pytest.raises(ValueError) as a:
            M.compute_fps(bad, 12)
        with pytest.raises(ValueError) as b:
            R.compute_fps([R.TimelineEvent(e.stage, e.block, e.start, e.end, e.kind) for e in bad], 12)
        assert str(a.value) == str(b.value)
