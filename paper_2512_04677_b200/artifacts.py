"""Run artifacts: measured timelines and LPD1 latent dumps (SURVEY.md 8f rows
2 and 4).

* Timeline files keep the reference's delimited format (harness.py:194-249):
  header ``stage,block,start,end,kind``, one event per line with floats in
  shortest round-trip repr, optional ``# metrics: {json}`` trailer.  Here the
  events are MEASURED (CUDA events + host clocks of a real run) instead of the
  reference's virtual clock, so the reference's own parser and
  ``compute_fps`` / ``compute_ttff`` / ``stage_utilization`` consume them.
* LPD1 dumps (harness.py:254-284): magic ``LPD1``, then D, F, M as
  little-endian u32, then the blocks' fp32 frames row-major, block-ascending;
  their sha256 is the cross-implementation digest (harness.py:287-292).
"""

from __future__ import annotations

import hashlib
import json

import numpy as np

from .metrics import MetricsBundle, TimelineEvent

TIMELINE_HEADER = "stage,block,start,end,kind"
LATENT_MAGIC = b"LPD1"


class ArtifactError(ValueError):
    """Malformed timeline or latent dump (the reference raises ConfigError, exit code 2)."""


def metrics_record(bundle: MetricsBundle) -> dict:
    rec = {"fps": float(bundle.fps), "fps_steady": float(bundle.fps_steady), "ttff": float(bundle.ttff),
           "nfe": int(bundle.nfe), "utilization": [float(u) for u in bundle.utilization]}
    if bundle.drift is not None and len(bundle.drift):
        d = np.asarray(bundle.drift, dtype=np.float64)
        fin = d[np.isfinite(d)]
        rec["drift_min"] = float(fin.min()) if len(fin) else None
        rec["drift_mean"] = float(fin.mean()) if len(fin) else None
    return rec


def format_timeline(timeline, metrics: MetricsBundle | None = None) -> str:
    out = [TIMELINE_HEADER]
    out += [f"{e.stage},{e.block},{float(e.start)!r},{float(e.end)!r},{e.kind}" for e in timeline]
    if metrics is not None:
        out.append("# metrics: " + json.dumps(metrics_record(metrics), sort_keys=True))
    return "\n".join(out) + "\n"


def export_timeline(timeline, path: str, metrics: MetricsBundle | None = None) -> str:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(format_timeline(timeline, metrics))
    return path


def parse_timeline(path: str):
    """Inverse of export_timeline: (events, metrics dict or None)."""
    events, metrics = [], None
    with open(path, encoding="utf-8") as fh:
        head = fh.readline().rstrip("\n")
        if head != TIMELINE_HEADER:
            raise ArtifactError(f"{path}: not a timeline file (header {head!r})")
        for line in fh:
            line = line.rstrip("\n")
            if not line:
                continue
            if line.startswith("# metrics: "):
                metrics = json.loads(line[len("# metrics: "):])
                continue
            st, blk, s, e, kind = line.split(",")
            events.append(TimelineEvent(int(st), int(blk), float(s), float(e), kind))
    return events, metrics


def latents_bytes(blocks) -> bytes:
    if not blocks:
        raise ValueError("no blocks to serialize")
    vals = [np.asarray(b.values if hasattr(b, "values") else b, dtype=np.float32) for b in blocks]
    f, d = vals[0].shape
    head = LATENT_MAGIC + np.array([d, f, len(vals)], dtype="<u4").tobytes()
    return head + b"".join(v.astype("<f4").tobytes() for v in vals)


def write_latents(path: str, blocks) -> str:
    with open(path, "wb") as fh:
        fh.write(latents_bytes(blocks))
    return path


def read_latents(path: str) -> np.ndarray:
    """(M, F, D) float32 array of a dump."""
    raw = open(path, "rb").read()
    if raw[:4] != LATENT_MAGIC:
        raise ArtifactError(f"{path}: bad magic {raw[:4]!r}")
    d, f, m = (int(x) for x in np.frombuffer(raw[4:16], dtype="<u4"))
    body = np.frombuffer(raw[16:], dtype="<f4")
    if body.size != m * f * d:
        raise ArtifactError(f"{path}: truncated latent dump")
    return body.reshape(m, f, d).astype(np.float32)


def latents_digest(blocks) -> str:
    return hashlib.sha256(latents_bytes(blocks)).hexdigest()


def frames_digest(frames: np.ndarray) -> str:
    return hashlib.sha256(np.asarray(frames).astype("<f4").tobytes()).hexdigest()
