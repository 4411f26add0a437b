"""One-process-per-GPU TPP runtime: Algorithm 4 (reference engine.py:406-496)
with each pipeline stage group on its own GPU and latents crossing GPUs over
NVLink peer memory.

Reference -> B200 mapping:

* stage thread k (engine.py:431-463), owning step j = T-k+1 and a private
  ``RollingKvCache`` -> a rank owning a contiguous group of steps, each an
  ``engine.Stage`` (device ring of L+1 slots + captured forward graph);
* ``_Link`` (engine.py:342-388), a bounded ``queue.Queue`` carrying only the
  ``LatentBlock`` -> ``IpcLink``: ``capacity`` latent slots + ready/free
  counters in the CONSUMER's HBM, mapped into the producer's process with
  CUDA IPC.  Default (fused) send: the producer's last step writes x'
  straight into the consumer's slot from the velocity-head GEMM's Euler
  epilogue (NVLink stores), after a device wait on the slot's ``free``
  counter, then publishes ``ready`` with a system-scope release; fallback:
  a side-stream copy kernel (lp_link_send) overlapped with the next block.
  The consumer's stream waits on ``ready`` on the device (lp_link_recv) --
  no host round trip per block, and sequence numbers keep the FIFO
  invariant (engine.py:360-363, :383-387);
* decoder thread (engine.py:465-480) -> the last rank of a pipeline, which
  reads each final latent back, decodes, and after block 0 performs the
  one-shot AAS and broadcasts the sink to the pipeline's ranks
  (engine.py:417, :438-439, :475-478) -- the "secondary warm-up" bubble;
* ``fail()`` / abort Event (engine.py:425-429) -> an abort word in every
  rank's HBM, peer-mapped, polled by every device-side wait.

Layouts: P = min(world, T) ranks per pipeline; stage k runs on
pipeline rank (k-1)*P // T (2 GPUs: steps {4,3} | {2,1}; 4 GPUs: one step
each); world / P independent pipelines (8 GPUs: two 4-stage pipelines with
different noise seeds).  There is no collective in the data path.

The host logic (layout, sequencing, sink broadcast, result assembly) is
independent of the compute: ``DistTPP`` drives a ``backend`` (the device
``DeviceBackend`` in production) over a ``transport`` (``IpcLink`` pairs on
GPUs; ``DistTransport`` = torch.distributed send/recv of host tensors, used
by the CPU/gloo tests of this logic).
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from .engine import (EngineConfig, EngineConfigError, PipelineInvariantError, RolloutResult, Stage, _aas, _decode,
                     _finish, build_runtime, noise_block)
from .kvcache import SinkSlot, receive_sink
from .latent import LatentBlock
from .metrics import TimelineEvent
from .runtime import compute_stream, prewarm_torch
from .numerics import F32

# ---------------------------------------------------------------------------
# layout
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class RankRole:
    """What one rank does in the TPP layout."""

    rank: int
    world: int
    pipe: int            # pipeline index (0 .. n_pipes-1)
    n_pipes: int
    pos: int             # position in the pipeline (0 = first stage group)
    ranks: tuple         # global ranks of this pipeline, stage order
    steps: tuple         # owned t_index values, descending (denoising order)
    stages: tuple        # owned stage numbers k (1-based, reference numbering)
    decode: bool = False  # dedicated decode rank (the paper's "+1" VAE GPU): no steps

    @property
    def first(self) -> bool:
        return self.pos == 0

    @property
    def last(self) -> bool:
        return self.pos == len(self.ranks) - 1

    @property
    def prev_rank(self):
        return None if self.first else self.ranks[self.pos - 1]

    @property
    def next_rank(self):
        return None if self.last else self.ranks[self.pos + 1]


def pipeline_layout(world: int, steps: int, decode_gpu: bool = False) -> list:
    """RankRole for every rank.  P = min(world, T) DiT ranks per pipeline,
    stage k on pipeline position (k-1)*P // T, world // P pipelines.  With
    ``decode_gpu`` every pipeline has one more rank that only decodes, runs
    the one-shot AAS and broadcasts the sink (the paper's 4 DiT + 1 VAE
    layout); world must then be a multiple of P + 1."""
    if world < 1 or steps < 1:
        raise EngineConfigError("world and steps must be >= 1")
    extra = 1 if decode_gpu else 0
    if world < 1 + extra:
        raise EngineConfigError(f"world size {world} too small for a pipeline with a decode rank")
    p = min(world - extra, steps)
    width = p + extra
    if world % width:
        raise EngineConfigError(f"world size {world} is not a multiple of the pipeline width {width} "
                                f"({p} DiT ranks{' + 1 decode rank' if extra else ''}, T={steps})")
    n_pipes = world // width
    roles = []
    for r in range(world):
        pipe, pos = divmod(r, width)
        ranks = tuple(range(pipe * width, pipe * width + width))
        if pos == p:  # the decode rank
            roles.append(RankRole(r, world, pipe, n_pipes, pos, ranks, (), (), True))
            continue
        ks = tuple(k for k in range(1, steps + 1) if (k - 1) * p // steps == pos)
        if not ks:
            raise EngineConfigError(f"pipeline position {pos} owns no step (world {world}, T={steps})")
        roles.append(RankRole(r, world, pipe, n_pipes, pos, ranks, tuple(steps - k + 1 for k in ks), ks))
    return roles


def pipe_noise_seed(cfg: EngineConfig, pipe: int) -> int:
    """Independent pipelines stream different content;
    pipeline 0 keeps cfg.noise_seed so it reproduces the 1-pipeline run."""
    return cfg.noise_seed + 1000003 * pipe


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------


def _ipc_export(t: torch.Tensor) -> tuple:
    h = (C.c_uint8 * 64)()
    off = C.c_int64(0)
    L.call("lp_ipc_handle", t.data_ptr(), h, C.byref(off))
    return bytes(h), int(off.value)


_IPC_MAPPED: dict = {}  # handle bytes -> [mapped base, refcount]; a handle maps once per process


def _ipc_open(handle: bytes, offset: int) -> int:
    """Map a peer allocation (once per handle; several exported tensors can
    live in one caching-allocator segment) and return base + offset."""
    ent = _IPC_MAPPED.get(handle)
    if ent is None:
        h = (C.c_uint8 * 64).from_buffer_copy(handle)
        p = C.c_void_p(0)
        L.call("lp_ipc_open", h, 0, C.byref(p))
        ent = _IPC_MAPPED[handle] = [int(p.value), 0]
    ent[1] += 1
    return ent[0] + int(offset)


def _ipc_release(handle: bytes) -> None:
    ent = _IPC_MAPPED.get(handle)
    if ent is None:
        return
    ent[1] -= 1
    if ent[1] <= 0:
        del _IPC_MAPPED[handle]
        try:
            L.call("lp_ipc_close", ent[0])
        except L.LivepipeError:
            pass


class IpcLink:
    """Consumer-owned bounded FIFO of latent slots (engine.py:342-388 _Link).

    The consumer allocates ``capacity`` slots + [ready, free] counters in its
    HBM and exports them; the producer maps them (CUDA IPC, NVLink peer
    access).  send/recv are stream-ordered device operations."""

    def __init__(self, nbytes: int, capacity: int, device: int, abort_ptr: int, timeout_s: float):
        self.nbytes, self.capacity = nbytes, capacity
        self.device = device
        self.abort_ptr = abort_ptr
        self.timeout_ns = int(timeout_s * 1e9)
        self.slots = None
        self.flags = None
        self.peer = None  # producer side: (slots_ptr, flags_ptr, mapped bases)
        self.next_seq = 0

    # consumer side
    def create(self) -> dict:
        with torch.cuda.device(self.device):
            self.slots = torch.zeros((self.capacity, self.nbytes // 4), dtype=torch.float32,
                                     device=f"cuda:{self.device}")
            self.flags = torch.zeros(4, dtype=torch.int32, device=f"cuda:{self.device}")
            torch.cuda.synchronize(self.device)
        return {"slots": _ipc_export(self.slots), "flags": _ipc_export(self.flags)}

    # producer side
    def attach(self, exported: dict) -> None:
        s = _ipc_open(*exported["slots"])
        f = _ipc_open(*exported["flags"])
        self.peer = (s, f, exported["slots"][0], exported["flags"][0])

    def _check(self, seq: int) -> None:
        if seq != self.next_seq:
            raise PipelineInvariantError(f"FIFO violated: expected sequence {self.next_seq}, got {seq}")
        self.next_seq += 1

    def send(self, src: torch.Tensor, stream: torch.cuda.Stream, seq: int, status: torch.Tensor) -> None:
        self._check(seq)
        slots, flags = self.peer[0], self.peer[1]
        dst = slots + (seq % self.capacity) * self.nbytes
        L.call("lp_link_send", src.data_ptr(), dst, self.nbytes, flags, flags + 4, seq, self.capacity,
               self.abort_ptr, self.timeout_ns, status.data_ptr(), stream.cuda_stream)

    def recv(self, dst: torch.Tensor, stream: torch.cuda.Stream, seq: int, status: torch.Tensor) -> None:
        self._check(seq)
        slot = self.slots[seq % self.capacity]
        L.call("lp_link_recv", slot.data_ptr(), dst.data_ptr(), self.nbytes, self.flags.data_ptr(),
               self.flags.data_ptr() + 4, seq, self.abort_ptr, self.timeout_ns, status.data_ptr(),
               stream.cuda_stream)

    def close(self) -> None:
        if self.peer is not None:
            for handle in self.peer[2:]:
                _ipc_release(handle)
            self.peer = None


class DistTransport:
    """Latent FIFO over torch.distributed point-to-point (host tensors).
    Used to exercise the TPP host logic on CPU (gloo); same sequencing rules
    as IpcLink."""

    def __init__(self, role: RankRole, shape):
        self.role = role
        self.shape = shape
        self.next_send = 0
        self.next_recv = 0

    def send(self, x: np.ndarray, seq: int) -> None:
        if seq != self.next_send:
            raise PipelineInvariantError(f"out-of-order send: expected {self.next_send}, got {seq}")
        self.next_send += 1
        dist.send(torch.tensor([seq], dtype=torch.int64), self.role.next_rank)
        dist.send(torch.from_numpy(np.ascontiguousarray(x, F32)), self.role.next_rank)

    def recv(self, seq: int) -> np.ndarray:
        if seq != self.next_recv:
            raise PipelineInvariantError(f"FIFO violated: expected {self.next_recv}, got {seq}")
        self.next_recv += 1
        hdr = torch.zeros(1, dtype=torch.int64)
        dist.recv(hdr, self.role.prev_rank)
        if int(hdr.item()) != seq:  # engine.py:383-387
            raise PipelineInvariantError(f"link delivered sequence {int(hdr.item())}, expected {seq}")
        buf = torch.zeros(self.shape, dtype=torch.float32)
        dist.recv(buf, self.role.prev_rank)
        return buf.numpy()


# ---------------------------------------------------------------------------
# the device backend: this rank's stages on its GPU
# ---------------------------------------------------------------------------


class DecodeBackend:
    """The dedicated decode rank: receives each final latent over the link
    into HBM and reads it back for the (host) decode; no denoising steps."""

    def __init__(self, cfg: EngineConfig, device: int):
        prof = cfg.model_profile
        self.device = device
        self.stream = torch.cuda.Stream(device)
        self.shape = (cfg.frames_per_block, prof.latent_dim)
        self.buf = torch.zeros(self.shape, dtype=torch.float32, device=f"cuda:{device}")
        self.status = _status_word()
        self.stages = []
        self.fused = None
        self.vae = self.frames = None
        if cfg.vae_decode and prof.patched:  # buffers allocated now, not while a link kernel spins
            from .vae import VaeDecoder

            self.vae = VaeDecoder(prof.channels, prof.height, prof.width, f"cuda:{device}")
            self.frames = torch.empty((4 * cfg.frames_per_block, 3 * 64 * prof.height * prof.width),
                                      device=f"cuda:{device}")
            with torch.cuda.stream(self.stream):
                self.vae.decode_into(self.buf, self.frames, self.stream)
            self.stream.synchronize()

    def _vae_decode(self) -> None:
        if self.vae is not None:
            self.vae.decode_into(self.buf, self.frames, self.stream)

    def capture(self) -> None:
        pass

    def set_sink(self, content: np.ndarray) -> None:
        pass

    def denoise(self, i: int, timed: bool = True) -> None:
        pass

    def recv(self, link: "IpcLink", i: int) -> None:
        link.recv(self.buf, self.stream, i, self.status)

    def read_output(self, out: torch.Tensor | None = None) -> np.ndarray | None:
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            self._vae_decode()
            if out is not None:
                out.copy_(self.buf.reshape(out.shape), non_blocking=True)
                return None
            host = self.buf.cpu()
        st = int(self.status.item())
        if st != 0:
            raise PipelineInvariantError(f"decode link wait failed with status {st}")
        return host.numpy().copy()

    def nfe(self) -> int:
        return 0

    def sync(self) -> None:
        torch.cuda.synchronize(self.device)


class DeviceBackend:
    """The owned steps of one rank: one ``Stage`` per step on one stream,
    chained on the device (x_out of step j -> x_in of step j-1)."""

    def __init__(self, cfg: EngineConfig, rt, role: RankRole, device: int):
        self.cfg, self.rt, self.role, self.device = cfg, rt, role, device
        self.stream = compute_stream(device)
        self.side = torch.cuda.Stream(device)  # link sends overlap the next block
        self.stages = [Stage(cfg, rt, j, device, self.stream) for j in role.steps]
        prof = cfg.model_profile
        self.shape = (cfg.frames_per_block, prof.latent_dim)
        # sticky link status (lp_link_*): written by failed device waits,
        # gates every later send / fused store / ready publish of this rank;
        # lives in pinned host memory, so the host polls it with no copy
        self.status = _status_word()
        # double-buffered send staging: block i's x' leaves from sendbuf[i % 2]
        self.sendbuf = torch.zeros((2,) + self.shape, dtype=torch.float32, device=f"cuda:{device}")
        self.sent = [None, None]
        self._keep = None
        self.fused = None  # (link, slot addresses): x' stored by the Euler epilogue into the peer's slots

    @property
    def x_in(self) -> torch.Tensor:
        return self.stages[0].fw.x_in

    @property
    def x_out(self) -> torch.Tensor:
        return self.stages[-1].fw.x_out

    def capture(self) -> None:
        for st in self.stages:
            st.ensure_graph()

    def set_sink(self, content: np.ndarray) -> None:
        for st in self.stages:
            st.set_sink(content)

    def load_host(self, x: np.ndarray) -> None:
        from .runtime import h2d

        self._keep = h2d(self.x_in, np.asarray(x, F32), self.stream)

    def load_device(self, x: torch.Tensor) -> None:
        with torch.cuda.stream(self.stream):
            self.x_in.copy_(x.reshape(self.x_in.shape), non_blocking=True)

    def setup_fused_send(self, link: "IpcLink") -> None:
        """Fuse the stage-boundary transfer into the last owned step: its
        velocity-head GEMM's Euler epilogue stores x' straight into the
        consumer's peer-mapped receive slot over NVLink (one captured graph
        per slot); a device wait on the slot's ``free`` counter precedes the
        forward and a system-scope release of ``ready`` follows it."""
        slots = [link.peer[0] + s * link.nbytes for s in range(link.capacity)]
        self.stages[-1].fw.euler_gate = self.status.data_ptr()  # baked into the captured epilogue args
        self.stages[-1].ensure_out_graphs(slots)
        self.fused = (link, slots)

    def denoise(self, i: int, timed: bool = True) -> None:
        prev = None
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            for n, st in enumerate(self.stages):
                if prev is not None:
                    st.fw.x_in.copy_(prev.fw.x_out)
                st.prepare(i)
                if self.fused is not None and n == len(self.stages) - 1:
                    link, slots = self.fused
                    link._check(i)
                    flags = link.peer[1]
                    need = i + 1 - link.capacity
                    if need > 0:  # slot i % capacity consumed by block i - capacity
                        L.call("lp_wait", flags + 4, need, link.abort_ptr, link.timeout_ns, self.status.data_ptr(),
                               self.stream.cuda_stream)
                    st.forward(i, timed=timed, out_ptr=slots[i % link.capacity])
                    L.call("lp_signal", flags, i + 1, self.status.data_ptr(), self.stream.cuda_stream)
                else:
                    st.forward(i, timed=timed)
                prev = st

    def send(self, link: IpcLink, i: int) -> None:
        """Stage x' into sendbuf[i % 2] on the main stream, then ship it on the
        side stream so the next block's forward starts immediately."""
        b = i % 2
        with torch.cuda.device(self.device):
            if self.sent[b] is not None:
                self.stream.wait_event(self.sent[b])
            with torch.cuda.stream(self.stream):
                self.sendbuf[b].copy_(self.x_out)
                ready = torch.cuda.Event()
                ready.record(self.stream)
            self.side.wait_event(ready)
            link.send(self.sendbuf[b], self.side, i, self.status)
            done = torch.cuda.Event()
            done.record(self.side)
            self.sent[b] = done

    def recv(self, link: IpcLink, i: int) -> None:
        link.recv(self.x_in, self.stream, i, self.status)

    def read_output(self, out: torch.Tensor | None = None) -> np.ndarray | None:
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            if out is not None:
                out.copy_(self.x_out.reshape(out.shape), non_blocking=True)
                return None
            host = self.x_out.cpu()
        st = int(self.status.item())
        if st != 0:
            raise PipelineInvariantError(f"stage link wait failed with status {st}")
        return host.numpy().copy()

    def nfe(self) -> int:
        return sum(st.nfe for st in self.stages)

    def sync(self) -> None:
        torch.cuda.synchronize(self.device)


# ---------------------------------------------------------------------------
# the rank driver
# ---------------------------------------------------------------------------


class DistTPP:
    """One rank of the multi-process TPP runtime.

    ``run()`` executes a whole rollout (cfg.blocks blocks) with the
    reference's semantics and returns the ``RolloutResult`` on the last rank
    of each pipeline (None elsewhere).  ``submit``/``finish`` give the
    streaming form used by bench.py."""

    def __init__(self, cfg: EngineConfig, rt=None, backend=None, transport: str = "ipc", device: int | None = None,
                 rank: int | None = None, world: int | None = None, fused_send: bool = True,
                 decode_gpu: bool = False):
        if cfg.mode != "tpp":
            raise EngineConfigError(f"DistTPP needs mode 'tpp', got {cfg.mode!r}")
        self.rank = dist.get_rank() if rank is None else rank
        self.world = dist.get_world_size() if world is None else world
        self.roles = pipeline_layout(self.world, cfg.steps, decode_gpu)
        self.role = self.roles[self.rank]
        self.seed = pipe_noise_seed(cfg, self.role.pipe)
        cfg = _with_seed(cfg, self.seed)
        self.cfg = cfg
        self.pipe_group = None
        if self.role.n_pipes > 1:  # every rank creates every group, same order
            groups = [dist.new_group(list(r.ranks)) for r in self.roles if r.pos == 0]
            self.pipe_group = groups[self.role.pipe]
        self.transport = transport
        self.fused_send = fused_send and transport == "ipc"
        if transport == "ipc":
            self.device = torch.cuda.current_device() if device is None else device
            L.init_device(self.device)
            self.rt = rt or build_runtime(_with_devices(cfg, (self.device,)))
            if backend is None:
                dcfg = _with_devices(cfg, (self.device,))
                backend = (DecodeBackend(dcfg, self.device) if self.role.decode
                           else DeviceBackend(dcfg, self.rt, self.role, self.device))
            self.backend = backend
            self._setup_ipc()
        else:
            self.device = None
            self.rt = rt
            self.backend = backend
            self.link_in = DistTransport(self.role, self.backend.shape) if not self.role.first else None
            self.link_out = DistTransport(self.role, self.backend.shape) if not self.role.last else None
        self.sink = SinkSlot(self._reference_sink(), cfg.sink_delta)
        self.backend.set_sink(self.sink.content)
        self.blocks_in = 0

    def _reference_sink(self) -> np.ndarray:
        if self.rt is not None:
            return self.rt.conditions.reference.copy()
        return self.backend.reference_sink()

    # -- IPC wiring ------------------------------------------------------
    def _setup_ipc(self) -> None:
        cfg = self.cfg
        dev = self.device
        nbytes = int(np.prod(self.backend.shape)) * 4
        prewarm_torch(f"cuda:{dev}")
        self.abort = torch.zeros(4, dtype=torch.int32, device=f"cuda:{dev}")
        torch.cuda.synchronize(dev)
        self.link_in = None
        self.link_out = None
        exported = None
        if not self.role.first:
            self.link_in = IpcLink(nbytes, cfg.link_capacity, dev, self.abort.data_ptr(), cfg.link_timeout_s)
            exported = self.link_in.create()
        mine = {"link": exported, "abort": _ipc_export(self.abort), "pid": os.getpid()}
        every = [None] * self.world
        dist.all_gather_object(every, mine)
        if not self.role.last:
            self.link_out = IpcLink(nbytes, cfg.link_capacity, dev, self.abort.data_ptr(), cfg.link_timeout_s)
            self.link_out.attach(every[self.role.next_rank]["link"])
        # peers' abort words (fail() raises them so every device wait unwinds)
        self.peer_aborts = []
        self._abort_handles = []
        for r in self.role.ranks:
            if r != self.rank:
                self.peer_aborts.append(_ipc_open(*every[r]["abort"]))
                self._abort_handles.append(every[r]["abort"][0])
        self.backend.capture()  # graphs before any link kernel is in flight
        if self.fused_send and self.link_out is not None:
            self.backend.setup_fused_send(self.link_out)
        torch.cuda.synchronize(dev)
        dist.barrier()

    def abort_peers(self) -> None:
        """Raise the abort word of every rank of this pipeline (engine.py:425-429)."""
        if self.transport != "ipc":
            return
        s = torch.cuda.Stream(self.device)
        for p in self.peer_aborts + [self.abort.data_ptr()]:
            try:
                L.call("lp_signal", p, 1, None, s.cuda_stream)
            except L.LivepipeError:
                pass

    # -- per block ---------------------------------------------------------
    def _recv(self, i: int) -> None:
        if self.transport == "ipc":
            self.backend.recv(self.link_in, i)
        else:
            self.backend.load_host(self.link_in.recv(i))

    def _send(self, i: int) -> None:
        if self.transport == "ipc":
            self.backend.send(self.link_out, i)
        else:
            self.link_out.send(self.backend.read_output(), i)

    def _sink_broadcast(self, content) -> np.ndarray:
        """One-shot fan-out of the AAS sink from the pipeline's last rank
        (engine.py:417, :438-439, :477-478)."""
        obj = [None if content is None else np.asarray(content, F32)]
        src = self.role.ranks[-1]
        dist.broadcast_object_list(obj, src=src, group=self.pipe_group)
        return obj[0]

    def _maybe_receive_sink(self, i: int) -> None:
        if i == 1 and not self.role.last:
            content = self._sink_broadcast(None)
            receive_sink(self.sink, content)
            self.backend.set_sink(self.sink.content)

    def _aas_last(self, xb: LatentBlock) -> None:
        if self.rt is not None:
            _aas(self.rt, self.sink, xb, self.device)
        else:
            self.backend.aas(self.sink, xb)
        self._sink_broadcast(self.sink.content)
        self.backend.set_sink(self.sink.content)

    def step(self, i: int, noise=None, out: torch.Tensor | None = None, decode: bool = True):
        """Process block i on this rank: receive (or draw) the input, run the
        owned steps, ship x' to the next rank (or, on the last rank, read it
        back; block 0 triggers the one-shot AAS + sink broadcast).  Returns
        the final LatentBlock on the last rank when it is read to the host."""
        if i != self.blocks_in:
            raise PipelineInvariantError(f"blocks must be submitted in order: expected {self.blocks_in}, got {i}")
        self._poll_status(i)
        self.blocks_in += 1
        self._maybe_receive_sink(i)
        if self.role.first:
            if noise is None:
                vals = noise_block(self.cfg, i).values
                self.backend.load_host(vals)
            elif isinstance(noise, torch.Tensor) and self.transport == "ipc":
                self.backend.load_device(noise)
            else:
                self.backend.load_host(np.asarray(noise, F32))
        else:
            self._recv(i)
        self.backend.denoise(i)
        if not self.role.last:
            if not (self.fused_send and self.backend.fused is not None):
                self._send(i)
            return None
        if out is not None and i != 0:
            self.backend.read_output(out)
            return None
        host = self.backend.read_output()
        xb = LatentBlock(host, i)
        if out is not None:
            out.copy_(torch.from_numpy(host).reshape(out.shape))
        if i == 0:
            self._aas_last(xb)
        return xb

    def _poll_status(self, i: int) -> None:
        """Per-block host check of the sticky link status, as of the last
        device write that has landed (no device synchronisation): a failed
        wait on this rank surfaces at the next block instead of at finish()."""
        if self.transport != "ipc":
            return
        st = int(self.backend.status[0])
        if st != 0:
            raise PipelineInvariantError(f"rank {self.rank}: stage link wait failed with status {st} "
                                         f"(seen before block {i})")

    # -- whole rollout -------------------------------------------------------
    def run(self) -> RolloutResult | None:
        cfg = self.cfg
        blocks, chunks, dec_t = [], [], []
        t0 = time.perf_counter()
        try:
            for i in range(cfg.blocks):
                s = time.perf_counter() - t0
                xb = self.step(i)
                if xb is not None:
                    blocks.append(xb)
                    fr = _decode(self.rt, xb, self.device) if self.rt is not None else self.backend.decode(xb)
                    if fr is not None:
                        chunks.append(fr)
                    dec_t.append(TimelineEvent(len(self.roles[0].ranks) + 1, i, s, time.perf_counter() - t0,
                                               "decode"))
        except BaseException:
            self.abort_peers()
            raise
        self.finish()
        nfe_local = self.backend.nfe()
        nfe = self._sum_over_pipe(nfe_local)
        if not self.role.last:
            return None
        if self.rt is None:
            return RolloutResult(tuple(blocks), np.concatenate(chunks) if chunks else None, nfe, (), None)
        return _finish(cfg, self.rt, blocks, chunks, nfe, self.sink.content, ())

    def _sum_over_pipe(self, v: int) -> int:
        t = torch.tensor([v], dtype=torch.int64)
        if dist.get_backend() == "nccl":
            t = t.to(f"cuda:{self.device}")
        dist.all_reduce(t, group=self.pipe_group)
        return int(t.item())

    def finish(self) -> None:
        if self.transport == "ipc":
            self.backend.sync()
            st = int(self.backend.status.item())
            if st != 0:
                raise PipelineInvariantError(f"stage link wait failed with status {st}")

    def close(self) -> None:
        for lk in (self.link_in, self.link_out):
            if isinstance(lk, IpcLink):
                lk.close()
        for h in getattr(self, "_abort_handles", []):
            _ipc_release(h)
        self._abort_handles = []


def _status_word() -> torch.Tensor:
    """A sticky link status word in pinned host memory.  Pinned memory is
    device-mapped at the same address (UVA), so the link kernels write a
    failure code straight into it and the host polls it without enqueueing a
    device->host copy: such a copy shares the copy engine's queue with other
    streams and, queued behind a spinning link kernel, can stall the stage
    that kernel is waiting for."""
    return torch.zeros(1, dtype=torch.int32).pin_memory()


def _with_devices(cfg: EngineConfig, devices: tuple) -> EngineConfig:
    import dataclasses

    return dataclasses.replace(cfg, devices=devices)


def _with_seed(cfg: EngineConfig, seed: int) -> EngineConfig:
    import dataclasses

    return cfg if seed == cfg.noise_seed else dataclasses.replace(cfg, noise_seed=seed)


def run_tpp_dist(cfg: EngineConfig, **kw) -> RolloutResult | None:
    """Whole-rollout entry point for one rank (call under torchrun / spawn
    with the process group initialised)."""
    runner = DistTPP(cfg, **kw)
    try:
        return runner.run()
    finally:
        runner.close()
