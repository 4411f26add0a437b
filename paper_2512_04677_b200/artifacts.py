"""Run artifacts: measured timelines and LPD1 latent dumps (SURVEY.md 8f rows
2 and 4), written from the file-format specification so the reference's own
tools read them and the digests agree byte for byte.

Timeline file (format of reference harness.py:194-249)::

    stage,block,start,end,kind            <- fixed header line
    <int>,<int>,<float>,<float>,<kind>    <- one event per line, floats in
                                             shortest round-trip repr
    # metrics: <json, sorted keys>        <- optional trailer

Here the events are MEASURED (CUDA events + host clocks of a real run) instead
of the reference's virtual clock, so the reference's parser and metric
functions consume them unchanged.

LPD1 latent dump (reference harness.py:254-292): a 16-byte little-endian
header ``b"LPD1", D, F, M`` (u32 each) followed by M blocks of F x D float32,
row-major, block-ascending; its sha256 is the cross-implementation digest.
"""

from __future__ import annotations

import hashlib
import json
import struct

import numpy as np

from .metrics import MetricsBundle, TimelineEvent

TIMELINE_HEADER = "stage,block,start,end,kind"
LATENT_MAGIC = b"LPD1"
_LPD1_HEAD = struct.Struct("<4sIII")
_METRICS_TAG = "# metrics: "


class ArtifactError(ValueError):
    """Malformed timeline or latent dump (the reference raises ConfigError, exit code 2)."""


# ---------------------------------------------------------------- timelines --
def metrics_record(bundle: MetricsBundle) -> dict:
    """JSON-ready summary of a MetricsBundle; drift reduced to the min and
    mean of its finite entries (None when there are none)."""
    rec = dict(fps=float(bundle.fps), fps_steady=float(bundle.fps_steady), ttff=float(bundle.ttff),
               nfe=int(bundle.nfe), utilization=list(map(float, bundle.utilization)))
    drift = None if bundle.drift is None else np.asarray(bundle.drift, np.float64).ravel()
    if drift is not None and drift.size:
        ok = drift[np.isfinite(drift)]
        rec["drift_min"], rec["drift_mean"] = (float(ok.min()), float(ok.mean())) if ok.size else (None, None)
    return rec


def _event_line(e: TimelineEvent) -> str:
    return ",".join((str(e.stage), str(e.block), repr(float(e.start)), repr(float(e.end)), e.kind))


def format_timeline(timeline, metrics: MetricsBundle | None = None) -> str:
    lines = [TIMELINE_HEADER, *map(_event_line, timeline)]
    if metrics is not None:
        lines.append(_METRICS_TAG + json.dumps(metrics_record(metrics), sort_keys=True))
    lines.append("")
    return "\n".join(lines)


def export_timeline(timeline, path: str, metrics: MetricsBundle | None = None) -> str:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(format_timeline(timeline, metrics))
    return path


def parse_timeline(path: str):
    """(events, metrics dict or None) of a timeline file."""
    with open(path, encoding="utf-8") as fh:
        text = fh.read()
    head, _, rest = text.partition("\n")
    if head != TIMELINE_HEADER:
        raise ArtifactError(f"{path}: not a timeline file (header {head!r})")
    events, metrics = [], None
    for line in filter(None, rest.split("\n")):
        if line.startswith(_METRICS_TAG):
            metrics = json.loads(line[len(_METRICS_TAG):])
            continue
        stage, block, start, end, kind = line.split(",")
        events.append(TimelineEvent(int(stage), int(block), float(start), float(end), kind))
    return events, metrics


# ------------------------------------------------------------- LPD1 dumps --
def _as_frames(b) -> np.ndarray:
    return np.asarray(getattr(b, "values", b), dtype=np.float32)


def latents_bytes(blocks) -> bytes:
    stack = [_as_frames(b) for b in blocks]
    if not stack:
        raise ValueError("no blocks to serialize")
    body = np.ascontiguousarray(np.stack(stack), dtype="<f4")
    m, f, d = body.shape
    return _LPD1_HEAD.pack(LATENT_MAGIC, d, f, m) + body.tobytes()


def write_latents(path: str, blocks) -> str:
    with open(path, "wb") as fh:
        fh.write(latents_bytes(blocks))
    return path


def read_latents(path: str) -> np.ndarray:
    """(M, F, D) float32 array of an LPD1 dump."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if raw[:4] != LATENT_MAGIC:
        raise ArtifactError(f"{path}: bad magic {raw[:4]!r}")
    _, d, f, m = _LPD1_HEAD.unpack_from(raw)
    body = np.frombuffer(raw, dtype="<f4", offset=_LPD1_HEAD.size)
    if body.size != m * f * d:
        raise ArtifactError(f"{path}: truncated latent dump")
    return body.reshape(m, f, d).astype(np.float32)


def latents_digest(blocks) -> str:
    return hashlib.sha256(latents_bytes(blocks)).hexdigest()


def frames_digest(frames: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(frames, dtype="<f4").tobytes()).hexdigest()
