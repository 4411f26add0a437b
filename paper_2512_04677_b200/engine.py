"""Execution engines on the GPU: sequential (Algorithm 3) and TPP (Algorithm 4).

Same configuration object and result type as the reference engine
(engine.py:73-158), extended with the B200 fields (model profile, precision,
devices, graphs).  The fast path does not go through KvEntry objects: each
timestep j owns a ``Stage`` = one device KV ring of L+1 slots (slot = block
mod (L+1), so the block being written never aliases a visible entry and
eviction is free) plus a ``Forward`` workspace whose launch sequence is
captured once in a CUDA graph and replayed for every block.

* ``run_sequential`` -- one stream runs the T steps of every block, then the
  host decode; one-shot AAS after block 0 (engine.py:255-285).
* ``run_tpp`` -- stage k owns step j = T-k+1, its own stream (and device when
  several are given) and ring; latents cross stages through device links
  (lp_link_send/recv: device-initiated copies + release/acquire flags), the
  decoder thread does decode + AAS and broadcasts the sink once
  (engine.py:406-496).  Bit-identical to run_sequential (deterministic
  kernels, same math per (block, step)).
* ``run_clean_kv`` -- the clean-cache baseline through the drop-in
  B200Denoiser (engine.py:292-331).
"""

from __future__ import annotations

import os
import queue
import threading
import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _lib as L
from .denoiser import B200Denoiser, BlockCond
from .kvcache import RingIndex, RollingKvCache, SinkSlot, aas_update, corrupt_history, corruption_prng, receive_sink, \
    rolling_rope_index
from .codec import DeviceCodec
from .latent import (Conditions, LatentBlock, PatchVideoCodec, TimestepSchedule, ToyVideoCodec, flow_step,
                     synthetic_conditions)
from .metrics import MetricsBundle, TimelineEvent, drift_metric, metrics_from_timeline
from .model import DenoiserWeights, DeviceWeights, ModelProfile, build_weights, toy_profile
from .numerics import F32, Prng
from .runtime import Forward, KvArena, compute_stream, h2d, prewarm_torch, wait_event
from .errors import SinkLockedError, raise_compat

THREADS_ENV = "LIVE_PIPE_THREADS"
ORACLE_TARGET_STREAM = 1 << 46
MODES = ("sequential", "clean_kv", "tpp", "simulate")
DENOISER_KINDS = ("toy", "oracle")
ORACLE_TARGET_STREAM = 1 << 46  # Philox stream of the oracle denoiser's target (reference engine.py:59)
PRECISIONS = ("fp32", "bf16")


from .errors import EngineConfigError, PipelineInvariantError  # noqa: E402  (engine.py:65-70)


@dataclass(frozen=True)
class EngineConfig:
    """The reference fields (engine.py:82-106) plus the B200 ones."""

    mode: str = "sequential"
    steps: int = 4
    cache_capacity: int = 4
    frames_per_block: int = 3
    latent_dim: int = 16
    pixel_dim: int = 32
    upsample: int = 4
    sink_delta: int = 1
    blocks: int = 8
    weight_seed: int = 7
    noise_seed: int = 11
    denoiser_kind: str = "toy"
    oracle_target_seed: int = 99
    history_sigma: float = 0.0
    history_mode: str = "fixed"
    n_layers: int = 2
    n_heads: int = 2
    head_dim: int = 8
    rope_base: float = 10000.0
    audio_dim: int = 8
    prompt_dim: int = 8
    denoise_latency: float = 1.0
    decode_latency: float = 1.0
    arrival_offset: float = 0.0
    link_capacity: int = 1
    # ---- B200 extensions ----
    precision: str = "fp32"
    profile: ModelProfile | None = None  # None: toy profile from the fields above
    devices: tuple = (0,)  # TPP: stage k runs on devices[(k-1) * len(devices) // steps]
    use_graphs: bool = True
    device_inputs: bool = False  # perf runs: weights / noise from the device RNG
    link_timeout_s: float = 60.0
    # patched profiles: decode through the per-location patch codec (the VAE
    # stand-in, latent.PatchVideoCodec) with pixel_channels x pixel_scale^2
    # pixels per latent location; off = no frames, sink = block 0's frame 0
    patch_codec: bool = False
    pixel_channels: int = 3
    pixel_scale: int = 8
    # the dedicated decode rank (tpp_dist, decode_gpu) also runs the VAE
    # stand-in (vae.VaeDecoder) on every received block -- the decode GPU's
    # realistic cost; frames stay in its HBM
    vae_decode: bool = False

    def __post_init__(self):
        if self.mode not in MODES:
            raise EngineConfigError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.denoiser_kind not in DENOISER_KINDS:
            raise EngineConfigError(f"denoiser must be one of {DENOISER_KINDS}")
        if self.denoiser_kind == "oracle" and self.profile is not None and self.profile.patched:
            # the reference's analytic test denoiser (denoiser.py:294-343) is
            # defined over the toy model's per-frame K/V projections
            raise EngineConfigError("denoiser_kind='oracle' needs the toy profile (the reference's analytic "
                                    "test denoiser projects K/V per latent frame)")
        if (self.profile is not None and self.rope_base != 10000.0
                and self.rope_base != self.profile.rope_base):
            raise EngineConfigError(f"rope_base {self.rope_base} disagrees with the profile's "
                                    f"{self.profile.rope_base}")
        for name in ("steps", "cache_capacity", "frames_per_block", "blocks", "upsample", "sink_delta",
                     "n_layers", "n_heads", "head_dim", "link_capacity", "pixel_channels", "pixel_scale"):
            if getattr(self, name) < 1:
                raise EngineConfigError(f"{name} must be >= 1")
        if self.history_sigma < 0.0:
            raise EngineConfigError("history_sigma must be >= 0")
        if self.history_mode not in ("fixed", "scaled"):
            raise EngineConfigError("history_mode must be 'fixed' or 'scaled'")
        if self.profile is None and self.latent_dim != self.n_heads * self.head_dim:
            raise EngineConfigError(f"latent_dim ({self.latent_dim}) must equal "
                                    f"n_heads*head_dim ({self.n_heads * self.head_dim})")
        if self.pixel_dim < self.latent_dim and self.profile is None:
            raise EngineConfigError("pixel_dim must be >= latent_dim")
        if self.denoise_latency <= 0.0 or self.decode_latency <= 0.0:
            raise EngineConfigError("latencies must be positive")
        if self.precision not in PRECISIONS:
            raise EngineConfigError(f"precision must be one of {PRECISIONS}")
        if self.cache_capacity > L.MAX_SEG - 2:
            raise EngineConfigError(f"cache_capacity must be <= {L.MAX_SEG - 2}")

    @property
    def model_profile(self) -> ModelProfile:
        if self.profile is not None:
            return self.profile
        prof = toy_profile(self.n_layers, self.n_heads, self.head_dim, self.audio_dim, self.prompt_dim)
        return prof if self.rope_base == prof.rope_base else replace(prof, rope_base=self.rope_base)

    @property
    def stage_latencies(self) -> list:
        return [self.denoise_latency] * self.steps + [self.decode_latency]

    @property
    def total_frames(self) -> int:
        return self.blocks * self.frames_per_block * self.upsample


@dataclass(frozen=True)
class StageMessage:
    """What crosses a stage boundary: a latent block + bookkeeping (engine.py:141-149)."""

    block: LatentBlock
    block_index: int
    producer: int
    sequence: int


@dataclass(frozen=True)
class RolloutResult:
    blocks: tuple
    frames: np.ndarray | None
    nfe: int
    timeline: tuple
    metrics: MetricsBundle | None


def count_nfe(result) -> int:
    return result.nfe


@dataclass
class Runtime:
    schedule: TimestepSchedule
    host_weights: DenoiserWeights | None
    device_weights: dict  # device index -> DeviceWeights
    codec: ToyVideoCodec | PatchVideoCodec | None
    conditions: Conditions
    device_codecs: dict = field(default_factory=dict)  # device index -> codec.DeviceCodec
    weight_seed: int | None = None  # host weights rebuilt on demand from (seed, profile)
    profile: ModelProfile | None = None
    # denoiser_kind='oracle': the analytic velocity's target block
    # (engine.py:191-197, Philox(oracle_target_seed, 1<<46))
    oracle_target: np.ndarray | None = None

    @property
    def weights(self) -> DenoiserWeights | None:
        """Host weights (the reference container, denoiser.py:75-138).  The
        fast path streams them to the device layer by layer and keeps no host
        copy (9.9 B parameters at the 14B shape); they are redrawn from the
        seed -- identical numbers -- only when a host consumer asks."""
        if self.host_weights is None and self.weight_seed is not None:
            self.host_weights = build_weights(self.weight_seed, profile=self.profile)
        return self.host_weights


def build_runtime(cfg: EngineConfig) -> Runtime:
    """Seeded runtime (engine.py:177-201): schedule, weights, codec, conditions."""
    prof = cfg.model_profile
    schedule = TimestepSchedule.uniform(cfg.steps)
    dev_ids = sorted(set(cfg.devices))
    for d in dev_ids:
        L.init_device(d)
    seed = None
    if cfg.device_inputs:
        dws = {d: DeviceWeights.random(prof, cfg.precision, f"cuda:{d}", cfg.weight_seed) for d in dev_ids}
    else:
        # the reference's seeded weights (build_weights, denoiser.py:100-138),
        # drawn and uploaded one layer at a time
        seed = cfg.weight_seed
        dws = DeviceWeights.from_seed(seed, prof, cfg.precision, [f"cuda:{d}" for d in dev_ids])
        dws = dict(zip(dev_ids, dws))
    codec = None
    if not prof.patched:
        codec = ToyVideoCodec(cfg.weight_seed, prof.latent_dim, cfg.pixel_dim, cfg.upsample)
    elif cfg.patch_codec:
        codec = PatchVideoCodec(cfg.weight_seed, prof.channels, prof.height, prof.width, cfg.pixel_channels,
                                cfg.pixel_scale, cfg.upsample)
    conds = synthetic_conditions(cfg.noise_seed, cfg.blocks, prof.audio_dim, prof.prompt_dim, prof.latent_dim)
    target = None
    if cfg.denoiser_kind == "oracle":
        target = Prng(cfg.oracle_target_seed, ORACLE_TARGET_STREAM).normal((cfg.frames_per_block, prof.latent_dim))
    return Runtime(schedule, None, dws, codec, conds, weight_seed=seed, profile=prof, oracle_target=target)


def noise_block(cfg: EngineConfig, block_index: int) -> LatentBlock:
    """N(0,1) from Philox(noise_seed, stream=i) (engine.py:204-210)."""
    vals = Prng(cfg.noise_seed, block_index).normal((cfg.frames_per_block, cfg.model_profile.latent_dim))
    return LatentBlock(vals, block_index)


def _sigma(cfg: EngineConfig, rt: Runtime, j: int) -> float:
    s = cfg.history_sigma
    if cfg.history_mode == "scaled" and j >= 1:
        s = s * rt.schedule.level(j)
    return s


class Stage:
    """Timestep j's device state: ring of L+1 slots + forward workspace."""

    def __init__(self, cfg: EngineConfig, rt: Runtime, j: int, device: int, stream: torch.cuda.Stream):
        self.cfg, self.rt, self.j = cfg, rt, j
        self.device = device
        self.stream = stream
        dw = rt.device_weights[device]
        prof = cfg.model_profile
        n_tok = cfg.frames_per_block * prof.tokens_per_frame
        self.L = cfg.cache_capacity
        self.sigma_on = cfg.history_sigma > 0.0
        with torch.cuda.device(device):
            self.arena = KvArena(prof, n_tok, self.L + 1, self.L if self.sigma_on else 0, dw.dtype,
                                 f"cuda:{device}")
            self.fw = Forward(dw, cfg.frames_per_block, self.arena)
            self.fw.sink_v_static = True  # sink rows fixed at [0, S) (write_inputs sink_row=0)
            if rt.oracle_target is not None:  # analytic velocity + the per-frame K/V projections
                self.fw.set_oracle(rt.oracle_target, rt.schedule.level(j), rt.schedule.dt)
        self.fw.set_history_noise(self.sigma_on, None)
        self._noise_host = self._noise_dev = self._noise_ev = None
        if self.sigma_on and not cfg.device_inputs:
            # parity runs upload the reference's host draws every call: fixed
            # pinned + device buffers, so no allocation (which may synchronise
            # the device) happens while another stage's link kernel spins
            shape = (self.L, 2, prof.n_layers, n_tok, prof.model_dim)
            self._noise_host = torch.empty(shape, dtype=torch.float32).pin_memory()
            with torch.cuda.device(device):
                self._noise_dev = torch.empty(shape, dtype=torch.float32, device=f"cuda:{device}")
        self.ring = RingIndex(self.L)  # RollingKvCache replay on ring slots (kvcache.py:41-56)
        self.graph = None
        self.nfe = 0
        self.ev = []  # (block, start event, end event)

    def set_sink(self, sink: np.ndarray) -> None:
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            self.fw.set_sink(torch.from_numpy(np.asarray(sink, F32).copy()), stream=self.stream)

    def visible(self) -> list:
        return list(self.ring.blocks)

    def prepare(self, i: int) -> None:
        """Stage the descriptor for block i (cache view = current ring)."""
        cfg, ar, fw = self.cfg, self.arena, self.fw
        segs = []
        noise = None
        sigma = _sigma(self.cfg, self.rt, self.j) if self.sigma_on else 0.0
        for e, (b, slot) in enumerate(self.ring.view()):
            row = ar.slot_row(slot)
            segs.append((ar.scratch_row(e) if self.sigma_on else row, ar.n_tokens, row))
        if self.sigma_on and not cfg.device_inputs and len(self.ring):
            # reference draw order (kvcache.py:121-137): per entry keys of all layers, then values
            g = corruption_prng(cfg.noise_seed, i, self.j)
            prof = cfg.model_profile
            shape = (ar.n_tokens, prof.model_dim)
            n = len(self.ring)
            if self._noise_ev is not None:
                self._noise_ev.synchronize()  # the previous upload has left the pinned buffer
            host = self._noise_host[:n].numpy()
            for e in range(n):
                for kv in range(2):
                    for layer in range(prof.n_layers):
                        host[e, kv, layer] = g.normal(shape)
            with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
                self._noise_dev[:n].copy_(self._noise_host[:n], non_blocking=True)
                self._noise_ev = torch.cuda.Event()
                self._noise_ev.record(self.stream)
            noise = self._noise_dev[:n]
        if self.sigma_on:
            self._noise_keep = noise
            fw.noise = noise
        key = (cfg.noise_seed * 0x9E3779B97F4A7C15 + i * 4096 + self.j) & ((1 << 64) - 1)
        fw.write_inputs(i, self.j, cfg.steps, segs, ar.slot_row(self.ring.write_slot(i)),
                        rolling_rope_index(i, cfg.sink_delta), self.rt.schedule.dt,
                        self.rt.conditions.audio_for(i), self.rt.conditions.prompt, sigma=sigma, noise_key=key,
                        stream=self.stream, arena_order=True)

    eager = False  # force eager launches (per-kernel timing passes)

    @property
    def use_graph(self) -> bool:
        # host-drawn parity noise changes the noise tensor per call: eager then
        return (self.cfg.use_graphs and not self.eager
                and not (self.sigma_on and not self.cfg.device_inputs))

    def ensure_graph(self) -> None:
        """Capture the forward's launch sequence once (torch.cuda.graph
        synchronises the device on entry, so multi-stage runners capture
        every stage up front, before any link kernel is in flight)."""
        if not self.use_graph or self.graph is not None:
            return
        with torch.cuda.device(self.device):
            g = torch.cuda.CUDAGraph(keep_graph=True)
            with torch.cuda.graph(g, stream=self.stream, capture_error_mode="thread_local"):
                self.fw.launch(stream=self.stream)
            self.fw.graph_kernels = L.graph_kernel_count(g)
            g.instantiate()
            self.graph = g

    def ensure_out_graphs(self, out_ptrs) -> None:
        """Capture one forward graph per destination address of x' (TPP: the
        peer-mapped receive slots of the next stage, so the velocity-head /
        Euler epilogue stores straight over NVLink)."""
        self.out_graphs = getattr(self, "out_graphs", {})
        for ptr in out_ptrs:
            if ptr in self.out_graphs:
                continue
            with torch.cuda.device(self.device):
                g = torch.cuda.CUDAGraph(keep_graph=True)
                with torch.cuda.graph(g, stream=self.stream, capture_error_mode="thread_local"):
                    self.fw.launch(stream=self.stream, x_out=int(ptr))
                self.fw.graph_kernels = L.graph_kernel_count(g)
                g.instantiate()
                self.out_graphs[ptr] = g

    def forward(self, i: int, timed: bool = True, out_ptr: int | None = None) -> None:
        """Enqueue the forward of block i (descriptor already staged); with
        ``out_ptr`` the final latent goes to that device address instead of
        ``fw.x_out``."""
        fw = self.fw
        if out_ptr is not None:
            with torch.cuda.device(self.device):
                e0 = torch.cuda.Event(enable_timing=True) if timed else None
                e1 = torch.cuda.Event(enable_timing=True) if timed else None
                if timed:
                    e0.record(self.stream)
                g = getattr(self, "out_graphs", {}).get(out_ptr)
                if self.use_graph and g is not None:
                    with torch.cuda.stream(self.stream):
                        g.replay()
                else:
                    fw.launch(stream=self.stream, x_out=int(out_ptr))
                if timed:
                    e1.record(self.stream)
                    self.ev.append((i, e0, e1))
            self.nfe += 1
            self.ring.push(i)
            return
        with torch.cuda.device(self.device):
            e0 = torch.cuda.Event(enable_timing=True) if timed else None
            e1 = torch.cuda.Event(enable_timing=True) if timed else None
            if timed:
                e0.record(self.stream)
            if self.use_graph and self.graph is None and self.nfe >= 1:
                self.ensure_graph()
            if self.use_graph and self.graph is not None:
                with torch.cuda.stream(self.stream):
                    self.graph.replay()
            else:
                fw.launch(stream=self.stream)
            if timed:
                e1.record(self.stream)
                self.ev.append((i, e0, e1))
        self.nfe += 1
        self.ring.push(i)


def _events_to_timeline(stages, t0_event, decode_times, k_of_j):
    tl = []
    for st in stages:
        for (i, e0, e1) in st.ev:
            s = t0_event.elapsed_time(e0) / 1e3
            e = t0_event.elapsed_time(e1) / 1e3
            tl.append(TimelineEvent(k_of_j(st.j), i, s, max(s, e), "denoise"))
    for (i, s, e) in decode_times:
        tl.append(TimelineEvent(len(stages) + 1, i, s, max(s, e), "decode"))
    tl.sort(key=lambda ev: (ev.start, ev.stage, ev.block))
    return tuple(tl)


def _finish(cfg, rt, blocks, chunks, nfe, sink_content, timeline) -> RolloutResult:
    frames = np.concatenate(chunks) if chunks else None
    metrics = None
    if timeline:
        drift = drift_metric(frames, _dcodec(rt).decode_frame(sink_content)[0]) if (frames is not None) else None
        try:
            metrics = metrics_from_timeline(timeline, cfg.total_frames, cfg.arrival_offset, nfe, drift)
        except ValueError:
            metrics = None
    return RolloutResult(tuple(blocks), frames, nfe, timeline, metrics)


def _dcodec(rt: Runtime, dev: int | None = None) -> DeviceCodec | None:
    """The decode stage's codec on device `dev`."""
    if rt.codec is None:
        return None
    if dev is None:
        dev = min(rt.device_weights) if rt.device_weights else 0
    dc = rt.device_codecs.get(dev)
    if dc is None:
        dc = rt.device_codecs.setdefault(dev, DeviceCodec(rt.codec, dev))
    return dc


def _decode(rt: Runtime, x: LatentBlock, dev: int | None = None):
    """decode(block) on the GPU (engine.py:279 / :460 -> latent.py:189-193)."""
    dc = _dcodec(rt, dev)
    return dc.decode(x) if dc is not None else None


def _aas(rt: Runtime, sink: SinkSlot, x: LatentBlock, dev: int | None = None) -> None:
    if rt.codec is not None:
        aas_update(sink, x, _dcodec(rt, dev))
    else:
        # patched profiles: the decode stage is "next"; the
        # sink takes block 0's first latent frame (the round trip's fixed point)
        if sink.locked:
            raise_compat(SinkLockedError, "the sink was already replaced in this rollout")
        sink.content = np.asarray(x.values[0], F32).copy()
        sink.locked = True


# ---------------------------------------------------------------------------
# sequential (Algorithm 3)
# ---------------------------------------------------------------------------

def run_sequential(cfg: EngineConfig, rt: Runtime | None = None) -> RolloutResult:
    if cfg.mode != "sequential":
        raise EngineConfigError(f"run_sequential called with mode {cfg.mode!r}")
    rt = rt or build_runtime(cfg)
    dev = cfg.devices[0]
    with torch.cuda.device(dev):
        stream = compute_stream(dev)
        stages = {j: Stage(cfg, rt, j, dev, stream) for j in range(1, cfg.steps + 1)}
        sink = SinkSlot(rt.conditions.reference.copy(), cfg.sink_delta)
        for st in stages.values():
            st.set_sink(sink.content)
        blocks, chunks, dec_t = [], [], []
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        t0_host = None
        for i in range(cfg.blocks):
            x = noise_block(cfg, i)
            first = stages[cfg.steps]
            with torch.cuda.stream(stream):
                first.fw.x_in.copy_(torch.from_numpy(x.values), non_blocking=False)
            prev = None
            for j in range(cfg.steps, 0, -1):
                st = stages[j]
                if prev is not None:
                    with torch.cuda.stream(stream):
                        st.fw.x_in.copy_(prev.fw.x_out)
                st.prepare(i)
                st.forward(i)
                prev = st
            with torch.cuda.stream(stream):
                out = prev.fw.x_out.cpu()
            stream.synchronize()
            if t0_host is None:
                t0_host = time.perf_counter() - t0.elapsed_time(prev.ev[-1][2]) / 1e3
            xb = LatentBlock(out.numpy(), i)
            blocks.append(xb)
            ds = time.perf_counter() - t0_host
            fr = _decode(rt, xb, dev)
            if fr is not None:
                chunks.append(fr)
            if i == 0:
                _aas(rt, sink, xb, dev)
                for st in stages.values():
                    st.set_sink(sink.content)
            dec_t.append((i, ds, time.perf_counter() - t0_host))
        torch.cuda.synchronize(dev)
        nfe = sum(st.nfe for st in stages.values())
        tl = _events_to_timeline(list(stages.values()), t0, dec_t, lambda j: cfg.steps - j + 1)
    return _finish(cfg, rt, blocks, chunks, nfe, sink.content, tl)


# ---------------------------------------------------------------------------
# TPP (Algorithm 4), one process, one stream (and optionally device) per stage
# ---------------------------------------------------------------------------

class DeviceLink:
    """Bounded FIFO between adjacent stages: ``capacity`` latent slots in the
    consumer's memory + monotone ready/free counters (engine.py:342-388).
    The producer's stream copies into the slot and publishes; the consumer's
    stream waits (bounded spin, abort-aware) and releases the slot."""

    def __init__(self, nbytes: int, capacity: int, consumer_device: int, abort_word: torch.Tensor,
                 timeout_s: float):
        self.capacity = capacity
        self.nbytes = nbytes
        with torch.cuda.device(consumer_device):
            self.slots = torch.zeros((capacity, nbytes // 4), dtype=torch.float32, device=f"cuda:{consumer_device}")
            self.flags = torch.zeros(4, dtype=torch.int32, device=f"cuda:{consumer_device}")  # ready, free
        self.abort = abort_word
        self.timeout_ns = int(timeout_s * 1e9)
        self.next_send = 0
        self.next_recv = 0

    def send(self, src: torch.Tensor, stream: torch.cuda.Stream, seq: int, status: torch.Tensor) -> None:
        if seq != self.next_send:
            raise PipelineInvariantError(f"out-of-order send: expected seq {self.next_send}, got {seq}")
        self.next_send += 1
        slot = self.slots[seq % self.capacity]
        L.call("lp_link_send", src.data_ptr(), slot.data_ptr(), self.nbytes, self.flags.data_ptr(),
               self.flags.data_ptr() + 4, seq, self.capacity, self.abort.data_ptr(), self.timeout_ns,
               status.data_ptr(), stream.cuda_stream)

    def recv(self, dst: torch.Tensor, stream: torch.cuda.Stream, seq: int, status: torch.Tensor) -> None:
        if seq != self.next_recv:
            raise PipelineInvariantError(f"FIFO violated: expected seq {self.next_recv}, got {seq}")
        self.next_recv += 1
        slot = self.slots[seq % self.capacity]
        L.call("lp_link_recv", slot.data_ptr(), dst.data_ptr(), self.nbytes, self.flags.data_ptr(),
               self.flags.data_ptr() + 4, seq, self.abort.data_ptr(), self.timeout_ns, status.data_ptr(),
               stream.cuda_stream)


def _check_thread_budget(cfg: EngineConfig) -> None:
    raw = os.environ.get(THREADS_ENV)
    if raw is None:
        return
    try:
        cap = int(raw)
    except ValueError:
        raise EngineConfigError(f"{THREADS_ENV}={raw!r} is not an integer") from None
    if cap < cfg.steps + 1:
        raise EngineConfigError(f"{THREADS_ENV}={cap} but pipelined mode needs T+1={cfg.steps + 1} workers")


def stage_devices(cfg: EngineConfig) -> list:
    """Device of stage k = 1..T: contiguous step groups over cfg.devices."""
    n = len(cfg.devices)
    return [cfg.devices[min(n - 1, (k - 1) * n // cfg.steps)] for k in range(1, cfg.steps + 1)]


def run_tpp(cfg: EngineConfig, rt: Runtime | None = None) -> RolloutResult:
    if cfg.mode != "tpp":
        raise EngineConfigError(f"run_tpp called with mode {cfg.mode!r}")
    _check_thread_budget(cfg)
    rt = rt or build_runtime(cfg)
    prof = cfg.model_profile
    T = cfg.steps
    devs = stage_devices(cfg)
    last_dev = devs[-1]
    nbytes = cfg.frames_per_block * prof.latent_dim * 4
    for d in sorted(set(devs)):
        prewarm_torch(f"cuda:{d}")
    # stage k's link kernel (on its device) stores into stage k+1's slots and
    # every stage polls the abort word on the last device: peer access
    for a in sorted(set(devs)):
        for b in sorted(set(devs)):
            if a != b:
                L.init_device(a)
                L.call("lp_peer_enable", a, b)
    abort = torch.zeros(4, dtype=torch.int32, device=f"cuda:{last_dev}")
    streams = [compute_stream(d) for d in devs]
    stages = [Stage(cfg, rt, T - k + 1, devs[k - 1], streams[k - 1]) for k in range(1, T + 1)]
    # link k-1: stage k -> stage k+1 (k = 1..T-1); link T-1: stage T -> decoder
    links = [DeviceLink(nbytes, cfg.link_capacity, devs[k] if k < T else last_dev, abort, cfg.link_timeout_s)
             for k in range(1, T + 1)]
    sink_feeds = [queue.Queue(maxsize=1) for _ in range(T)]
    for st in stages:  # capture before any link kernel can be in flight
        st.ensure_graph()
    errors, err_lock = [], threading.Lock()
    abort_evt = threading.Event()
    out_blocks = [None] * cfg.blocks
    out_chunks = [None] * cfg.blocks
    decoder_sink = SinkSlot(rt.conditions.reference.copy(), cfg.sink_delta)
    dec_t = []
    t0_events = {}
    for d in sorted(set(devs)):
        with torch.cuda.device(d):
            torch.cuda.synchronize(d)
            e = torch.cuda.Event(enable_timing=True)
            e.record(torch.cuda.current_stream(d))
            t0_events[d] = e
    t0_host = time.perf_counter()

    def fail(exc):
        with err_lock:
            errors.append(exc)
        abort_evt.set()
        abort.fill_(1)

    # every device buffer the workers touch exists before the first thread
    # starts: an allocation while another stage's link kernel spins may wait
    # on the device
    # one sticky link status word per stage (recv and send of that stage) in
    # pinned, device-mapped host memory: the link kernels write a failure
    # straight into it and the worker polls it once per block.  No
    # device->host copy is enqueued on the stage streams -- such copies share
    # the copy engine's queue across streams, and a copy queued behind a
    # spinning link kernel can block the very stage that kernel waits for.
    statuses = [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in stages]
    dec_buf = torch.zeros((cfg.frames_per_block, prof.latent_dim), dtype=torch.float32, device=f"cuda:{last_dev}")
    dec_status = torch.zeros(1, dtype=torch.int32).pin_memory()
    dec_stream = torch.cuda.Stream(last_dev)
    for st in stages:  # the reference sink (its projection scratch is allocated here, not mid-stream)
        st.set_sink(rt.conditions.reference.copy())
    dc = _dcodec(rt, last_dev)  # the decode stage's device codec (map uploads) likewise
    if dc is not None:  # and one decode + AAS encode, so their buffers come from the allocator's cache later
        dc.encode(dc.decode(LatentBlock(np.zeros((cfg.frames_per_block, dc.latent_dim), F32), 0))[0])
    for d in sorted(set(devs)):
        torch.cuda.synchronize(d)

    def stage_worker(k: int) -> None:
        st = stages[k - 1]
        sink = SinkSlot(rt.conditions.reference.copy(), cfg.sink_delta)
        status = statuses[k - 1]
        try:
            for i in range(cfg.blocks):
                if int(status[0]) != 0:
                    raise PipelineInvariantError(f"stage {k} link wait failed with status {int(status[0])} "
                                                 f"(seen before block {i})")
                if i == 1:
                    while True:
                        if abort_evt.is_set():
                            return
                        try:
                            content = sink_feeds[k - 1].get(timeout=0.05)
                            break
                        except queue.Empty:
                            continue
                    receive_sink(sink, content)
                    st.set_sink(sink.content)
                with torch.cuda.device(st.device), torch.cuda.stream(st.stream):
                    if k == 1:
                        x = noise_block(cfg, i)
                        keep = h2d(st.fw.x_in, x.values, st.stream)
                    else:
                        links[k - 2].recv(st.fw.x_in, st.stream, i, status)
                    st.prepare(i)
                    st.forward(i)
                    links[k - 1].send(st.fw.x_out, st.stream, i, status)
        except BaseException as exc:  # noqa: BLE001 - worker boundary
            fail(exc)

    def decode_worker() -> None:
        dev = last_dev
        stream, buf, status = dec_stream, dec_buf, dec_status
        try:
            for i in range(cfg.blocks):
                with torch.cuda.device(dev), torch.cuda.stream(stream):
                    links[T - 1].recv(buf, stream, i, status)
                    ev = torch.cuda.Event()
                    ev.record(stream)
                wait_event(ev)
                host = buf.cpu()
                if int(status[0]) != 0:
                    raise PipelineInvariantError(f"decoder link wait failed with status {int(status[0])}")
                ds = time.perf_counter() - t0_host
                xb = LatentBlock(host.numpy(), i)
                out_blocks[i] = xb
                out_chunks[i] = _decode(rt, xb, dev)
                if i == 0:
                    _aas(rt, decoder_sink, xb, dev)
                    for feed in sink_feeds:
                        feed.put(decoder_sink.content)
                dec_t.append((i, ds, time.perf_counter() - t0_host))
        except BaseException as exc:  # noqa: BLE001
            fail(exc)

    workers = [threading.Thread(target=stage_worker, args=(k,), name=f"stage-{k}") for k in range(1, T + 1)]
    workers.append(threading.Thread(target=decode_worker, name="decoder"))
    for w in workers:
        w.start()
    for w in workers:
        w.join()
    for d in sorted(set(devs)):
        torch.cuda.synchronize(d)
    if errors:
        raise errors[0]
    bad = [(k + 1, int(s[0])) for k, s in enumerate(statuses) if int(s[0]) != 0]
    if bad:
        raise PipelineInvariantError(f"stage link waits failed (stage, status): {bad}")
    nfe = sum(st.nfe for st in stages)
    dev0 = devs[0]
    tl = ()
    if len(set(devs)) == 1:
        tl = _events_to_timeline(stages, t0_events[dev0], dec_t, lambda j: T - j + 1)
    chunks = [c for c in out_chunks if c is not None]
    return _finish(cfg, rt, out_blocks, chunks, nfe, decoder_sink.content, tl)


# ---------------------------------------------------------------------------
# clean-cache baseline (engine.py:292-331) through the drop-in denoiser
# ---------------------------------------------------------------------------

def run_clean_kv(cfg: EngineConfig, rt: Runtime | None = None) -> RolloutResult:
    if cfg.mode != "clean_kv":
        raise EngineConfigError(f"run_clean_kv called with mode {cfg.mode!r}")
    if cfg.denoiser_kind != "toy":
        raise EngineConfigError("clean_kv runs the toy denoiser through the drop-in; the oracle kind's clean-KV "
                                "baseline runs on the reference engine")
    rt = rt or build_runtime(cfg)
    if rt.weights is None:
        raise EngineConfigError("clean_kv needs host weights (device_inputs=False)")
    dn = B200Denoiser(rt.weights, rt.schedule, cfg.model_profile.rope_base, precision=cfg.precision,
                      device=f"cuda:{cfg.devices[0]}", profile=cfg.model_profile)
    unified = RollingKvCache(0, cfg.cache_capacity)
    sink = SinkSlot(rt.conditions.reference.copy(), cfg.sink_delta)
    blocks, chunks, nfe = [], [], 0
    for i in range(cfg.blocks):
        x = noise_block(cfg, i)
        cond = BlockCond(audio=rt.conditions.audio_for(i), prompt=rt.conditions.prompt)
        for j in range(cfg.steps, 0, -1):
            view = unified.view()
            s = _sigma(cfg, rt, j)
            if s > 0.0:
                view = corrupt_history(unified, s, corruption_prng(cfg.noise_seed, i, j))
            out = dn.denoise_block(x, j, view, cond, sink.content, rolling_rope_index(i, cfg.sink_delta),
                                   require_same_timestep=False, max_entries=cfg.cache_capacity)
            nfe += 1
            x = flow_step(x, out.velocity, rt.schedule.dt)
        entry = dn.cache_entry(x, unified.view(), cond, sink.content, rolling_rope_index(i, cfg.sink_delta))
        nfe += 1
        unified.push(entry)
        blocks.append(x)
        fr = _decode(rt, x, cfg.devices[0])
        if fr is not None:
            chunks.append(fr)
        if i == 0:
            _aas(rt, sink, x, cfg.devices[0])
    return _finish(cfg, rt, blocks, chunks, nfe, sink.content, ())


_RUNNERS = {"sequential": run_sequential, "clean_kv": run_clean_kv, "tpp": run_tpp}


def run(cfg: EngineConfig) -> RolloutResult:
    if cfg.mode == "simulate":
        raise EngineConfigError("mode 'simulate' has no math to run")
    return _RUNNERS[cfg.mode](cfg)


# ---------------------------------------------------------------------------
# streaming session (the call a serving loop makes per block)
# ---------------------------------------------------------------------------

class StreamingPipeline:
    """Block-at-a-time streaming API over the sequential fast path on one
    device: ``submit(i, noise, out)`` denoises block i through all T steps
    (the ring caches, sink and AAS state live on the device) and writes the
    final latent to ``out``.  ``noise``/``out`` may be device tensors or
    pinned host tensors (the copies are enqueued on the pipeline stream).
    Matches run_sequential's math per block; decode is the next stage."""

    def __init__(self, cfg: EngineConfig, rt: Runtime | None = None):
        self.cfg = cfg
        self.rt = rt or build_runtime(cfg)
        self.dev = cfg.devices[0]
        self.stream = compute_stream(self.dev)
        self.stages = {j: Stage(cfg, self.rt, j, self.dev, self.stream) for j in range(1, cfg.steps + 1)}
        self.sink = SinkSlot(self.rt.conditions.reference.copy(), cfg.sink_delta)
        for st in self.stages.values():
            st.set_sink(self.sink.content)
        self.blocks_done = 0

    def capture(self) -> None:
        for st in self.stages.values():
            st.ensure_graph()

    def kernels_per_block(self) -> int:
        return sum(st.fw.kernels_per_forward() for st in self.stages.values())

    def submit(self, i: int, noise: torch.Tensor, out: torch.Tensor | None = None, timed: bool = False):
        T = self.cfg.steps
        s = self.stream
        first = self.stages[T]
        with torch.cuda.device(self.dev), torch.cuda.stream(s):
            first.fw.x_in.copy_(noise.reshape(first.fw.x_in.shape), non_blocking=True)
            prev = None
            for j in range(T, 0, -1):
                st = self.stages[j]
                if prev is not None:
                    st.fw.x_in.copy_(prev.fw.x_out)
                st.prepare(i)
                st.forward(i, timed=timed)
                prev = st
            if out is not None:
                out.copy_(prev.fw.x_out.reshape(out.shape), non_blocking=True)
        self.blocks_done += 1
        return prev.fw.x_out

    def aas(self, block0: torch.Tensor) -> None:
        """One-shot sink swap after block 0 (kvcache.py:93-109)."""
        self.stream.synchronize()  # block0 is written on the pipeline stream
        xb = LatentBlock(block0.detach().float().cpu().numpy().reshape(self.cfg.frames_per_block, -1), 0)
        _aas(self.rt, self.sink, xb, self.dev)
        for st in self.stages.values():
            st.set_sink(self.sink.content)
