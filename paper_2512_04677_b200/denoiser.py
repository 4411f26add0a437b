"""B200Denoiser: the drop-in for the reference's denoiser plug-in point.

The reference engine calls one duck-typed object, ``Runtime.denoiser``
(engine.py:166-174, chosen in build_runtime :191-200).  ``B200Denoiser`` has
the same constructor and methods as ``ToyDenoiser`` (denoiser.py:161-291):

    denoise_block(x, t_index, cache_view, cond, sink, sink_rope_index,
                  require_same_timestep=True, max_entries=None) -> DenoiseOutput
    cache_entry(x, cache_view, cond, sink, sink_rope_index) -> KvEntry

with the same validation and exception types (TimestepForcingError,
ValueError "capacity" / "order", denoiser.py:219-234) raised BEFORE any
launch, and the same purity contract.  The math runs on the GPU through
liblivepipe_b200 (no CPU fallback).  Returned ``KvEntry`` objects keep their
keys/values in a device slot pool; ``.keys`` / ``.values`` materialise host
copies on first access, and the slot is recycled when the entry is dropped
(the reference's RollingKvCache eviction, kvcache.py:41-52).  Reentrant: each
t_index gets its own workspace and CUDA stream, as the reference's TPP engine
calls one denoiser from T threads (engine.py:431-463).
"""

from __future__ import annotations

import threading
import weakref
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .latent import LatentBlock, TimestepSchedule
from .model import DenoiserWeights, DeviceWeights, ModelProfile, build_weights, toy_profile
from .numerics import F32
from .runtime import Forward, GrowableArena, compute_stream


from .errors import TimestepForcingError, raise_compat


@dataclass(frozen=True)
class BlockCond:
    """This block's audio embedding and the shared prompt (denoiser.py:66-72)."""

    audio: np.ndarray
    prompt: np.ndarray


class _Slot:
    """One ring slot of the device pool; returns itself to the pool when the
    last object referencing it (an entry's layers, a temp list) is collected."""

    __slots__ = ("pool", "index", "__weakref__")

    def __init__(self, pool: "_SlotPool", index: int):
        self.pool = pool
        self.index = index
        weakref.finalize(self, pool.release, index)


class DeviceLayers(Sequence):
    """The per-layer keys (kv=0) or values (kv=1) of a device-resident entry:
    a read-only sequence of (F*S, d) float32 arrays materialised from the
    ring slot on first access (one D2H copy of all layers), so reference code
    that iterates ``entry.keys`` (corrupt_history kvcache.py:133-135,
    attention_bruteforce denoiser.py:346-422) keeps working.  Holds the slot
    alive; ``noise = (sigma, z)`` marks a corrupted view, whose host form is
    ring + sigma * z (kvcache.py:121-137)."""

    __slots__ = ("slot", "kv", "noise", "_host")

    def __init__(self, slot: _Slot, kv: int, noise=None):
        self.slot = slot
        self.kv = kv
        self.noise = noise
        self._host = None

    def _get(self) -> tuple:
        if self._host is None:
            layers = self.slot.pool.read(self.slot.index, self.kv)
            if self.noise is not None:
                sigma, z = self.noise
                layers = tuple(a + b * F32(sigma) for a, b in zip(layers, z))
            self._host = layers
        return self._host

    def __len__(self) -> int:
        return self.slot.pool.dw.prof.n_layers

    def __getitem__(self, i):
        return self._get()[i]

    def __iter__(self):
        return iter(self._get())


@dataclass(frozen=True, eq=False)
class KvEntry:
    """Cached keys/values of one block at one noise level (denoiser.py:45-57).

    ``keys[l]`` is rotated at ``rope_index``; ``values[l]`` is not.  Field
    for field the reference's frozen dataclass, so ``dataclasses.replace``
    (the reference's corrupt_history, kvcache.py:136) works and yields a
    host entry.  Entries the GPU denoiser returns keep K/V in a device slot
    (``keys``/``values`` are ``DeviceLayers``); host entries hold tuples of
    arrays and are uploaded when a view containing them is denoised."""

    keys: Sequence = ()
    values: Sequence = ()
    block_index: int = 0
    timestep_index: int = 0
    rope_index: int = 0

    def __post_init__(self):
        if not isinstance(self.keys, DeviceLayers):
            object.__setattr__(self, "keys", tuple(np.asarray(k, F32) for k in self.keys))
        if not isinstance(self.values, DeviceLayers):
            object.__setattr__(self, "values", tuple(np.asarray(v, F32) for v in self.values))

    @classmethod
    def on_slot(cls, slot: _Slot, block_index: int, timestep_index: int, rope_index: int,
                noise=None) -> "KvEntry":
        """A device entry; ``noise = (sigma, keys_z, values_z)`` makes it a
        corrupted view of the slot (the perturbation is applied on the
        device when denoised, on the host when materialised)."""
        nk = nv = None
        if noise is not None:
            sigma, zk, zv = noise
            nk, nv = (sigma, zk), (sigma, zv)
        return cls(DeviceLayers(slot, 0, nk), DeviceLayers(slot, 1, nv), block_index, timestep_index, rope_index)

    @property
    def _slot(self):
        return self.keys.slot if isinstance(self.keys, DeviceLayers) else None

    @property
    def _noise(self):
        if isinstance(self.keys, DeviceLayers) and self.keys.noise is not None:
            return (self.keys.noise[0], self.keys.noise[1], self.values.noise[1])
        return None

    @property
    def on_device(self) -> bool:
        return self._slot is not None


@dataclass(frozen=True)
class DenoiseOutput:
    velocity: np.ndarray  # (F, D) float32
    kv: KvEntry


class _SlotPool:
    """Device KV slots shared by all timesteps of one denoiser, plus one sink
    region per workspace, in one ``GrowableArena`` (one base per layer, so
    any view is addressable as row segments of it).  Slots are backed on
    demand: the caller (the reference engine's caches, TPP threads, views
    with host-typed or corrupted entries) decides how many stay alive, and
    growth never moves the base, so in-flight launches are unaffected."""

    def __init__(self, dw: DeviceWeights, n_tokens: int, n_workspaces: int, initial_slots: int):
        self.dw = dw
        self.n_tokens = n_tokens
        self.n_workspaces = n_workspaces
        self.lock = threading.Lock()
        s = dw.prof.tokens_per_frame
        self.arena = GrowableArena(dw.prof, n_tokens, n_workspaces * s, dw.dtype, dw.device)
        self.slot_bytes = 2 * dw.prof.n_layers * n_tokens * dw.prof.model_dim * self.arena.k.element_size()
        self.free: list = []
        self._grow_to(max(1, initial_slots))

    @property
    def n_slots(self) -> int:
        return self.arena.n_slots

    def _grow_to(self, n: int) -> None:
        old = self.arena.n_slots
        n = min(n, self.arena.max_slots)
        if n <= old:
            raise RuntimeError(f"KV slot pool exhausted: all {old} slots the device can hold at this shape are "
                               "live (the caller keeps more cache entries alive than fit in HBM)")
        self.arena.ensure_slots(n)
        torch.cuda.synchronize(self.dw.device)  # zero fill of the new pages
        self.free.extend(range(n - 1, old - 1, -1))

    def slot_row(self, i: int) -> int:
        return self.arena.slot_row(i)

    def sink_row(self, w: int) -> int:
        return w * self.dw.prof.tokens_per_frame

    def acquire(self) -> _Slot:
        with self.lock:
            if not self.free:
                n = self.arena.n_slots
                # big slots (1.9 GB per K/V at the 14B shape) grow one at a time
                step = 1 if self.slot_bytes > (1 << 30) else max(4, n // 2)
                self._grow_to(n + step)
            return _Slot(self, self.free.pop())

    def release(self, index: int) -> None:
        with self.lock:
            self.free.append(index)

    def read(self, index: int, kv: int) -> tuple:
        r = self.slot_row(index)
        t = self.arena.k if kv == 0 else self.arena.v
        a = t[:, r:r + self.n_tokens].float().cpu().numpy()
        return tuple(a[l] for l in range(a.shape[0]))

    def write(self, index: int, keys, values, stream) -> None:
        """Upload a host entry into slot ``index`` on ``stream``."""
        r = self.slot_row(index)
        N = self.n_tokens
        for t, layers in ((self.arena.k, keys), (self.arena.v, values)):
            host = torch.from_numpy(np.ascontiguousarray(np.stack([np.asarray(x, F32) for x in layers])))
            with torch.cuda.stream(stream):
                t[:, r:r + N].copy_(host.to(t.device, non_blocking=False))


def check_view(entries, t_index: int, require_same_timestep: bool, max_entries) -> None:
    """Metadata rules of denoise_block (denoiser.py:219-234), bit-exact messages."""
    seen = {e.timestep_index for e in entries}
    if len(seen) > 1:
        raise_compat(TimestepForcingError, f"cache view mixes timestep indices {sorted(seen)}")
    if require_same_timestep and seen and seen != {t_index}:
        raise_compat(TimestepForcingError, f"cache holds timestep {seen.pop()} but denoising at {t_index}")
    if max_entries is not None and len(entries) > max_entries:
        raise ValueError(f"cache view exceeds capacity {max_entries}")
    for prev, nxt in zip(entries, entries[1:]):
        if nxt.block_index <= prev.block_index:
            raise ValueError("cache entries out of block order")


class B200Denoiser:
    """GPU replacement of ToyDenoiser with the identical call contract."""

    def __init__(self, weights: DenoiserWeights, schedule: TimestepSchedule, rope_base: float = 10000.0, *,
                 precision: str = "fp32", device=None, profile: ModelProfile | None = None,
                 max_live_entries: int | None = None, device_weights: DeviceWeights | None = None):
        if precision not in ("fp32", "bf16"):
            raise ValueError("precision must be 'fp32' or 'bf16'")
        self.weights = weights
        self.schedule = schedule
        self.rope_base = rope_base
        if device_weights is not None:  # weights already resident (e.g. drawn on the device)
            if device_weights.precision != precision:
                raise ValueError(f"device_weights are {device_weights.precision}, precision is {precision}")
            profile = profile or device_weights.prof
            device = device if device is not None else device_weights.device
        prof = profile or getattr(weights, "profile", None)
        if prof is None or (not prof.patched and prof.model_dim != weights.model_dim):
            prof = toy_profile(len(weights.layers), weights.n_heads, weights.head_dim,
                               weights.w_audio.shape[0], weights.w_prompt.shape[0],
                               ffn_dim=weights.layers[0].w1.shape[1])
        if prof.rope_base != rope_base:
            from dataclasses import replace

            prof = replace(prof, rope_base=rope_base)
        self.profile = prof
        self.precision = precision
        self.device = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        L.init_device(self.device.index or 0)
        self.dw = (device_weights if device_weights is not None
                   else DeviceWeights.from_host(weights, prof, precision, self.device))
        self._lock = threading.Lock()
        self._pool = None
        self._ws = {}
        self._max_live = max_live_entries

    # -- internals ------------------------------------------------------------
    def _workspace(self, t_index: int, n_frames: int, max_entries):
        with self._lock:
            if self._pool is None:
                self._frames = n_frames
                n_tok = n_frames * self.profile.tokens_per_frame
                steps = self.schedule.steps
                n_ws = steps + 1  # t_index 0 (clean-cache pass) .. T
                # first guess at the live set: T caches of L entries + one
                # in-flight entry per stage; the pool grows on demand
                window = max_entries if max_entries is not None else 4
                initial = self._max_live or steps * (window + 1)
                self._pool = _SlotPool(self.dw, n_tok, n_ws, initial)
            if n_frames != self._frames:
                raise ValueError(f"block has {n_frames} frames; this denoiser was set up for {self._frames}")
            ws = self._ws.get(t_index)
            if ws is None:
                fw = Forward(self.dw, n_frames, self._pool.arena)
                fw.fuse_euler = False  # denoise_block returns the velocity itself
                stream = compute_stream(self.device)
                ws = self._ws[t_index] = (fw, stream, min(t_index, self._pool.n_workspaces - 1))
            return ws

    def _set_sink(self, fw: Forward, sink: np.ndarray, stream) -> None:
        sink = np.asarray(sink, F32).reshape(-1)
        key = sink.tobytes()
        if fw.sink_key != key:
            fw.set_sink(torch.from_numpy(sink.copy()), stream=stream)
            fw.sink_key = key

    # -- the plug-in API --------------------------------------------------------
    def denoise_block(self, x: LatentBlock, t_index: int, cache_view, cond: BlockCond, sink: np.ndarray,
                      sink_rope_index: int, require_same_timestep: bool = True,
                      max_entries: int | None = None) -> DenoiseOutput:
        """Velocity for ``x`` at step ``t_index`` plus this block's KvEntry
        (denoiser.py:201-276).  Pure: mutates nothing it is given.  Entries
        may be this denoiser's device entries, corrupted views of them, or
        any duck-typed host entry with keys/values/block_index/
        timestep_index (the reference's KvEntry); host ones are uploaded."""
        entries = list(cache_view)
        check_view(entries, t_index, require_same_timestep, max_entries)
        prof = self.profile
        if x.values.shape[1] != prof.latent_dim:
            raise ValueError(f"latent dim {x.values.shape[1]} != model latent dim {prof.latent_dim}")
        if len(entries) > L.MAX_SEG - 2:
            raise ValueError(f"cache view of {len(entries)} entries exceeds the device bound {L.MAX_SEG - 2}")
        fw, stream, w = self._workspace(t_index, x.values.shape[0], max_entries)
        with fw.lock:
            return self._run(fw, stream, w, x, t_index, entries, cond, sink, sink_rope_index)

    def _run(self, fw, stream, w, x, t_index, entries, cond, sink, sink_rope_index):
        pool = self._pool
        N = pool.n_tokens

        def own(en):
            slot = getattr(en, "_slot", None)
            return slot if (slot is not None and slot.pool is pool) else None

        noisy = [en._noise for en in entries if own(en) is not None and en._noise is not None]
        if noisy and len(noisy) != len(entries):
            raise ValueError("a corrupted view must perturb every entry with one sigma")
        sigma = 0.0
        if noisy:
            sig = {n[0] for n in noisy}
            if len(sig) != 1:
                raise ValueError("a corrupted view must perturb every entry with one sigma")
            sigma = sig.pop()
        # acquire EVERY slot this call writes (uploads, corrupted copies, the
        # new entry) before any launch is bound to the arena
        temps = []
        segs = []
        for en in entries:
            slot = own(en)
            if slot is None:  # host-resident (or another pool's) entry: upload
                t = pool.acquire()
                temps.append(t)
                pool.write(t.index, en.keys, en.values, stream)
                row = pool.slot_row(t.index)
                segs.append((row, N, row))
            elif noisy:  # corrupted view: ring + sigma*z written into a temp slot on the device
                t = pool.acquire()
                temps.append(t)
                segs.append((pool.slot_row(t.index), N, pool.slot_row(slot.index)))
            else:
                row = pool.slot_row(slot.index)
                segs.append((row, N, row))
        cur = pool.acquire()
        if noisy:
            # reference draw order: per entry, keys of every layer, then values
            arr = np.stack([np.stack([np.stack(nk), np.stack(nv)]) for _, nk, nv in noisy])
            fw.set_history_noise(True, torch.from_numpy(np.ascontiguousarray(arr)).to(self.device))
        else:
            fw.set_history_noise(False)
        fw.kv_bound = self.profile.tokens_per_frame + (len(entries) + 1) * N
        fw.hist_rows = max(1, len(entries)) * N
        with torch.cuda.stream(stream):
            self._set_sink(fw, sink, stream)
            fw.write_inputs(x.block_index, t_index, self.schedule.steps, segs, pool.slot_row(cur.index),
                            sink_rope_index, self.schedule.dt, cond.audio, cond.prompt, sigma=sigma,
                            stream=stream, sink_row=pool.sink_row(w))
            fw.x_in.copy_(torch.from_numpy(np.ascontiguousarray(x.values)), non_blocking=False)
            fw.launch(stream=stream)
        stream.synchronize()
        vel = fw.velocity_host()
        del temps
        kv = KvEntry.on_slot(cur, x.block_index, t_index, x.block_index)
        return DenoiseOutput(velocity=vel, kv=kv)

    def cache_entry(self, x: LatentBlock, cache_view, cond: BlockCond, sink: np.ndarray,
                    sink_rope_index: int) -> KvEntry:
        """Clean-cache baseline's extra pass: full stack at level 0 with the
        timestep check lifted (denoiser.py:278-291)."""
        return self.denoise_block(x, 0, cache_view, cond, sink, sink_rope_index,
                                  require_same_timestep=False).kv


__all__ = ["B200Denoiser", "BlockCond", "DenoiseOutput", "KvEntry", "TimestepForcingError", "build_weights",
           "DenoiserWeights", "check_view"]
