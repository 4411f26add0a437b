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
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .latent import LatentBlock, TimestepSchedule
from .model import DenoiserWeights, DeviceWeights, ModelProfile, build_weights, toy_profile
from .numerics import F32
from .runtime import Forward, KvArena


class TimestepForcingError(ValueError):
    """A cache view mixed entries from different noise levels (denoiser.py:41-42)."""


@dataclass(frozen=True)
class BlockCond:
    """This block's audio embedding and the shared prompt (denoiser.py:66-72)."""

    audio: np.ndarray
    prompt: np.ndarray


class _Slot:
    """One ring slot of the device pool; returns itself to the pool when the
    last KvEntry referencing it is collected."""

    __slots__ = ("pool", "index", "__weakref__")

    def __init__(self, pool: "_SlotPool", index: int):
        self.pool = pool
        self.index = index
        weakref.finalize(self, pool.release, index)


class KvEntry:
    """Cached keys/values of one block at one noise level (denoiser.py:45-57).

    ``keys[l]`` is rotated at ``rope_index``; ``values[l]`` is not.  Device
    resident; host tuples are materialised lazily."""

    __slots__ = ("_keys", "_values", "block_index", "timestep_index", "rope_index", "_slot", "_noise")

    def __init__(self, keys=None, values=None, block_index: int = 0, timestep_index: int = 0,
                 rope_index: int = 0, _slot: _Slot | None = None, _noise=None):
        self._keys = None if keys is None else tuple(np.asarray(k, F32) for k in keys)
        self._values = None if values is None else tuple(np.asarray(v, F32) for v in values)
        self.block_index = block_index
        self.timestep_index = timestep_index
        self.rope_index = rope_index
        self._slot = _slot
        self._noise = _noise  # (sigma, keys_noise, values_noise) for a corrupted view entry

    def _materialise(self):
        if self._keys is None:
            k, v = self._slot.pool.read(self._slot.index)
            self._keys, self._values = k, v
            if self._noise is not None:
                sigma, nk, nv = self._noise
                self._keys = tuple(a + b * F32(sigma) for a, b in zip(self._keys, nk))
                self._values = tuple(a + b * F32(sigma) for a, b in zip(self._values, nv))

    @property
    def keys(self) -> tuple:
        self._materialise()
        return self._keys

    @property
    def values(self) -> tuple:
        self._materialise()
        return self._values

    @property
    def on_device(self) -> bool:
        return self._slot is not None


@dataclass(frozen=True)
class DenoiseOutput:
    velocity: np.ndarray  # (F, D) float32
    kv: KvEntry


class _SlotPool:
    """Device KV slots shared by all timesteps of one denoiser, plus per
    workspace sink rows and corrupted-view scratch (one arena, so any view
    is addressable as row segments of a single base)."""

    def __init__(self, dw: DeviceWeights, n_tokens: int, n_slots: int, n_workspaces: int, hist_max: int):
        self.dw = dw
        self.n_tokens = n_tokens
        self.n_workspaces = n_workspaces
        self.hist_max = hist_max
        self.lock = threading.Lock()
        self.active = 0
        self._alloc(n_slots)

    def _alloc(self, n_slots: int) -> None:
        prof = self.dw.prof
        s = prof.tokens_per_frame
        # rows: [sink region per workspace | slots | scratch per workspace]
        extra_sink_rows = (self.n_workspaces - 1) * s
        hist_rows = self.n_workspaces * self.hist_max
        arena = KvArena(prof, self.n_tokens, n_slots + (extra_sink_rows + self.n_tokens - 1) // self.n_tokens,
                        hist_rows, self.dw.dtype, self.dw.device)
        self.arena = arena
        self.n_slots = n_slots
        self.slot_base = self.n_workspaces * s
        self.free = list(range(n_slots - 1, -1, -1))

    def slot_row(self, i: int) -> int:
        return self.slot_base + i * self.n_tokens

    def sink_row(self, w: int) -> int:
        return w * self.dw.prof.tokens_per_frame

    def scratch_row(self, w: int, e: int) -> int:
        return self.arena.scratch_row(w * self.hist_max + e)

    def acquire(self) -> _Slot:
        with self.lock:
            if not self.free:
                self._grow()
            return _Slot(self, self.free.pop())

    def release(self, index: int) -> None:
        with self.lock:
            if index < self.n_slots:
                self.free.append(index)

    def _grow(self) -> None:
        if self.active > 1:
            raise RuntimeError("KV slot pool exhausted while other calls are in flight; "
                               "construct B200Denoiser with a larger max_live_entries")
        old = self.arena
        torch.cuda.synchronize(self.dw.device)
        n_old = self.n_slots
        free_old = list(self.free)
        self._alloc(2 * n_old)
        # sink regions and live slots keep their row offsets
        a = self.slot_base + n_old * self.n_tokens
        self.arena.k[:, :a].copy_(old.k[:, :a])
        self.arena.v[:, :a].copy_(old.v[:, :a])
        self.free = list(range(2 * n_old - 1, n_old - 1, -1)) + free_old

    def read(self, index: int):
        r = self.slot_row(index)
        N = self.n_tokens
        k = self.arena.k[:, r:r + N].float().cpu().numpy()
        v = self.arena.v[:, r:r + N].float().cpu().numpy()
        return tuple(k), tuple(v)

    def write(self, index: int, keys, values) -> None:
        r = self.slot_row(index)
        N = self.n_tokens
        kt = torch.from_numpy(np.stack([np.asarray(x, F32) for x in keys])).to(self.arena.k.device)
        vt = torch.from_numpy(np.stack([np.asarray(x, F32) for x in values])).to(self.arena.v.device)
        self.arena.k[:, r:r + N].copy_(kt)
        self.arena.v[:, r:r + N].copy_(vt)


def check_view(entries, t_index: int, require_same_timestep: bool, max_entries) -> None:
    """Metadata rules of denoise_block (denoiser.py:219-234), bit-exact messages."""
    seen = {e.timestep_index for e in entries}
    if len(seen) > 1:
        raise TimestepForcingError(f"cache view mixes timestep indices {sorted(seen)}")
    if require_same_timestep and seen and seen != {t_index}:
        raise TimestepForcingError(f"cache holds timestep {seen.pop()} but denoising at {t_index}")
    if max_entries is not None and len(entries) > max_entries:
        raise ValueError(f"cache view exceeds capacity {max_entries}")
    for prev, nxt in zip(entries, entries[1:]):
        if nxt.block_index <= prev.block_index:
            raise ValueError("cache entries out of block order")


class B200Denoiser:
    """GPU replacement of ToyDenoiser with the identical call contract."""

    def __init__(self, weights: DenoiserWeights, schedule: TimestepSchedule, rope_base: float = 10000.0, *,
                 precision: str = "fp32", device=None, profile: ModelProfile | None = None,
                 max_live_entries: int | None = None):
        if precision not in ("fp32", "bf16"):
            raise ValueError("precision must be 'fp32' or 'bf16'")
        self.weights = weights
        self.schedule = schedule
        self.rope_base = rope_base
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
        self.dw = DeviceWeights.from_host(weights, prof, precision, self.device)
        self._lock = threading.Lock()
        self._pool = None
        self._ws = {}
        self._max_live = max_live_entries
        self._hist_max = 8

    # -- internals ------------------------------------------------------------
    def _workspace(self, t_index: int, n_frames: int):
        with self._lock:
            if self._pool is None:
                self._frames = n_frames
                n_tok = n_frames * self.profile.tokens_per_frame
                steps = self.schedule.steps
                n_ws = steps + 1  # t_index 0 (clean-cache pass) .. T
                live = self._max_live or (steps + 1) * (self._hist_max + 2) + 8
                self._pool = _SlotPool(self.dw, n_tok, live, n_ws, self._hist_max)
            if n_frames != self._frames:
                raise ValueError(f"block has {n_frames} frames; this denoiser was set up for {self._frames}")
            ws = self._ws.get(t_index)
            if ws is None:
                fw = Forward(self.dw, n_frames, self._pool.arena)
                fw.fuse_euler = False  # denoise_block returns the velocity itself
                stream = torch.cuda.Stream(self.device)
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
        (denoiser.py:201-276).  Pure: mutates nothing it is given."""
        entries = list(cache_view)
        check_view(entries, t_index, require_same_timestep, max_entries)
        prof = self.profile
        if x.values.shape[1] != prof.latent_dim:
            raise ValueError(f"latent dim {x.values.shape[1]} != model latent dim {prof.latent_dim}")
        fw, stream, w = self._workspace(t_index, x.values.shape[0])
        pool = self._pool
        with fw.lock:
            pool.active += 1
            try:
                return self._run(fw, stream, w, x, t_index, entries, cond, sink, sink_rope_index)
            finally:
                pool.active -= 1

    def _run(self, fw, stream, w, x, t_index, entries, cond, sink, sink_rope_index):
        pool = self._pool
        if len(entries) > L.MAX_SEG - 2:
            raise ValueError(f"cache view of {len(entries)} entries exceeds the device bound {L.MAX_SEG - 2}")
        if any(en._noise is not None for en in entries) and len(entries) > pool.hist_max:
            raise ValueError(f"corrupted view of {len(entries)} entries exceeds the scratch bound "
                             f"{pool.hist_max}")
        fw.arena = pool.arena
        temps = []
        segs = []
        noise_parts = []
        for e, en in enumerate(entries):
            slot = en._slot if (en._slot is not None and en._slot.pool is pool) else None
            if slot is None:  # host-resident entry: upload to a temporary slot
                slot = pool.acquire()
                temps.append(slot)
                pool.write(slot.index, en.keys, en.values)
                if en._noise is not None:
                    pass  # keys/values above already include the perturbation
            row = pool.slot_row(slot.index)
            if en._noise is not None and en._slot is not None and en._slot.pool is pool:
                sigma, nk, nv = en._noise
                segs.append((pool.scratch_row(w, e), pool.n_tokens, row))
                noise_parts.append((sigma, nk, nv))
            else:
                segs.append((row, pool.n_tokens, row))
        sigma = 0.0
        if noise_parts:
            sig = {s for s, _, _ in noise_parts}
            if len(sig) != 1 or len(noise_parts) != len(entries):
                raise ValueError("a corrupted view must perturb every entry with one sigma")
            sigma = sig.pop()
            # reference draw order: per entry, keys of every layer, then values
            arr = np.stack([np.stack([np.stack(nk), np.stack(nv)]) for _, nk, nv in noise_parts])
            fw.set_history_noise(True, torch.from_numpy(np.ascontiguousarray(arr)).to(self.device))
        else:
            fw.set_history_noise(False)
        cur = pool.acquire()
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
        kv = KvEntry(None, None, x.block_index, t_index, x.block_index, _slot=cur)
        return DenoiseOutput(velocity=vel, kv=kv)

    def cache_entry(self, x: LatentBlock, cache_view, cond: BlockCond, sink: np.ndarray,
                    sink_rope_index: int) -> KvEntry:
        """Clean-cache baseline's extra pass: full stack at level 0 with the
        timestep check lifted (denoiser.py:278-291)."""
        return self.denoise_block(x, 0, cache_view, cond, sink, sink_rope_index,
                                  require_same_timestep=False).kv


__all__ = ["B200Denoiser", "BlockCond", "DenoiseOutput", "KvEntry", "TimestepForcingError", "build_weights",
           "DenoiserWeights", "check_view"]
