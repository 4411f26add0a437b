"""Multi-process TPP host logic on CPU (gloo, world size 2 and 4): the
one-process-per-GPU runtime's layout, FIFO sequencing and one-shot sink
broadcast reproduce the reference rollout digests bit for bit when each
rank's compute is the oracle (reference tests/test_acceptance.py:60-83:
TPP == sequential, bitwise)."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2512_04677_b200 import tpp_dist
from paper_2512_04677_b200.engine import EngineConfigError

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
META = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch(nproc, mode, out, kw, timeout=240, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(HERE, "dist_worker.py"), mode,
           str(out)] + [f"{k}={v}" for k, v in kw.items()]
    e = dict(os.environ, OMP_NUM_THREADS="1", PYTHONPATH=ROOT)
    e.update(env or {})
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=e, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_layouts():
    r2 = tpp_dist.pipeline_layout(2, 4)
    assert [r.steps for r in r2] == [(4, 3), (2, 1)]
    r4 = tpp_dist.pipeline_layout(4, 4)
    assert [r.steps for r in r4] == [(4,), (3,), (2,), (1,)]
    r8 = tpp_dist.pipeline_layout(8, 4)
    assert [r.pipe for r in r8] == [0, 0, 0, 0, 1, 1, 1, 1]
    assert r8[5].prev_rank == 4 and r8[7].last and r8[4].first
    r1 = tpp_dist.pipeline_layout(1, 4)
    assert r1[0].steps == (4, 3, 2, 1) and r1[0].first and r1[0].last
    r3 = tpp_dist.pipeline_layout(3, 4)
    assert [r.steps for r in r3] == [(4, 3), (2,), (1,)]
    with pytest.raises(EngineConfigError):
        tpp_dist.pipeline_layout(6, 4)
    # the paper's 4 DiT + 1 decode GPU layout, and two of them
    r5 = tpp_dist.pipeline_layout(5, 4, decode_gpu=True)
    assert [r.steps for r in r5] == [(4,), (3,), (2,), (1,), ()]
    assert r5[4].decode and r5[4].last and r5[3].next_rank == 4 and not r5[3].last
    r10 = tpp_dist.pipeline_layout(10, 4, decode_gpu=True)
    assert [r.pipe for r in r10] == [0] * 5 + [1] * 5 and r10[9].decode
    r3 = tpp_dist.pipeline_layout(3, 4, decode_gpu=True)
    assert [r.steps for r in r3] == [(4, 3), (2, 1), ()]
    with pytest.raises(EngineConfigError):
        tpp_dist.pipeline_layout(7, 4, decode_gpu=True)
    # every step owned exactly once per pipeline
    for w in (1, 2, 3, 4, 8):
        for p in range(w // min(w, 4)):
            steps = sorted(j for r in tpp_dist.pipeline_layout(w, 4) if r.pipe == p for j in r.steps)
            assert steps == [1, 2, 3, 4]


@pytest.mark.parametrize("nproc,name", [(2, "c1"), (4, "c1_sigma"), (2, "c1_delta3")])
def test_dist_tpp_matches_reference_digest(tmp_path, nproc, name):
    m = META[name]
    out = tmp_path / "res"
    launch(nproc, "cpu", out, m["kw"])
    rec = json.load(open(f"{out}.0"))
    assert rec["latents_sha256"] == m["latents_sha256"]
    assert rec["frames_sha256"] == m["frames_sha256"]
    assert rec["nfe"] == m["nfe"]


def test_two_pipelines_stream_independent_content(tmp_path):
    # world 4 with T=2: two 2-stage pipelines; pipeline 0 reproduces the
    # single-pipeline rollout, pipeline 1 streams a different noise seed
    out = tmp_path / "res"
    launch(4, "cpu", out, {"steps": 2, "blocks": 3})
    a = np.load(f"{out}.0.npy")
    b = np.load(f"{out}.1.npy")
    assert a.shape == b.shape and not np.array_equal(a, b)
    from oracle import livepipe_oracle as O

    ref, _, _ = O.run_sequential(O.RolloutCfg(steps=2, blocks=3))
    np.testing.assert_array_equal(a, np.stack(ref))
    ref1, _, _ = O.run_sequential(O.RolloutCfg(steps=2, blocks=3, noise_seed=tpp_dist.pipe_noise_seed(
        tpp_dist.EngineConfig(), 1)))
    np.testing.assert_array_equal(b, np.stack(ref1))


@pytest.mark.parametrize("nproc,name", [(3, "c1"), (5, "c1_sigma")])
def test_dedicated_decode_rank_matches_reference(tmp_path, nproc, name):
    # DiT ranks + one decode rank that decodes, runs the one-shot AAS and
    # broadcasts the sink; same rollout digests as the reference
    m = META[name]
    out = tmp_path / "res"
    launch(nproc, "cpu", out, dict(m["kw"], decode_gpu=1))
    rec = json.load(open(f"{out}.0"))
    assert rec["latents_sha256"] == m["latents_sha256"]
    assert rec["frames_sha256"] == m["frames_sha256"]
    assert rec["nfe"] == m["nfe"]
