"""The decode stage on the GPU: codec decode of every
final latent block and the one-shot AAS encode (kvcache.py:93-109), run on
the decode device instead of the host.

``DeviceCodec`` wraps either codec:

* ``ToyVideoCodec`` (latent.py:150-193): decode_frame = r dense matvecs and
  encode = one, all in the reference's pinned matmul order
  (numerics.py:50-64), through lp_gemm's fp32 path.  One launch per map
  decodes the whole block: y_u = X (F, D) . M_u^T written to rows f*r + u.
* ``PatchVideoCodec`` (this package): lp_codec_patch_decode / _encode.

Both are bit-identical to the host restatements (tests/test_gpu_codec.py).
The numpy-facing methods keep the reference codec's API (``decode``,
``decode_frame``, ``encode``, ``latent_dim``, ``pixel_dim``, ``upsample``)
so ``kvcache.aas_update`` accepts a DeviceCodec unchanged; the device-facing
``decode_into`` / ``encode_into`` are what the engines call on their own
streams."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L
from .latent import LatentBlock, PatchVideoCodec, ToyVideoCodec
from .numerics import F32


class DeviceCodec:
    def __init__(self, codec, device: int | str = 0):
        self.codec = codec
        self.device = torch.device(device if isinstance(device, str) else f"cuda:{device}")
        L.init_device(self.device.index or 0)
        self.latent_dim, self.pixel_dim, self.upsample = codec.latent_dim, codec.pixel_dim, codec.upsample
        dev = self.device
        if isinstance(codec, ToyVideoCodec):
            self.kind = "dense"
            # fp32 lp_gemm takes W as (k, n) row-major: the transposed maps
            self.maps_t = [torch.from_numpy(np.ascontiguousarray(m.T)).to(dev) for m in codec.decode_maps]
            self.enc_t = torch.from_numpy(np.ascontiguousarray(codec.encode_map.T)).to(dev)
        elif isinstance(codec, PatchVideoCodec):
            self.kind = "patch"
            self.maps = torch.from_numpy(np.ascontiguousarray(codec.maps)).to(dev)
            self.enc = torch.from_numpy(np.ascontiguousarray(codec.enc)).to(dev)
        else:
            raise TypeError(f"unsupported codec {type(codec).__name__}")
        self.stream = torch.cuda.Stream(dev)

    # ---------------------------------------------------------------- device
    def _gemm(self, a_ptr: int, m: int, k: int, w: torch.Tensor, n: int, c_ptr: int, ldc: int, st: int) -> None:
        args = L.GemmArgs()
        args.in_dtype, args.out_dtype, args.epilogue = L.LP_F32, L.LP_F32, L.EPI_STORE
        args.m, args.n, args.k = m, n, k
        args.lda, args.ldw, args.ldc = k, n, ldc
        args.a, args.w, args.c = a_ptr, w.data_ptr(), c_ptr
        args.bias, args.gate, args.qkv, args.euler = 0, 0, None, None
        L.call("lp_gemm", C.byref(args), st)

    def decode_into(self, x: torch.Tensor, out: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
        """x (F, latent_dim) fp32 on the device -> out (F*r, pixel_dim) fp32."""
        frames = x.shape[0]
        if x.dtype != torch.float32 or out.dtype != torch.float32:
            raise ValueError("codec tensors must be fp32")
        if x.numel() != frames * self.latent_dim or out.numel() != frames * self.upsample * self.pixel_dim:
            raise ValueError("codec: bad decode shapes")
        if not (x.is_contiguous() and out.is_contiguous()):
            raise ValueError("codec tensors must be contiguous")
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        r, P = self.upsample, self.pixel_dim
        if self.kind == "dense":
            for u in range(r):
                self._gemm(x.data_ptr(), frames, self.latent_dim, self.maps_t[u], P,
                           out.data_ptr() + 4 * u * P, r * P, st)
        else:
            c = self.codec
            L.call("lp_codec_patch_decode", x.data_ptr(), frames, c.channels, c.height, c.width,
                   self.maps.data_ptr(), r, c.pixel_channels, c.scale, out.data_ptr(), st)

    def encode_into(self, frame: torch.Tensor, out: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
        """frame (pixel_dim,) fp32 -> out (latent_dim,) fp32."""
        if frame.numel() != self.pixel_dim or out.numel() != self.latent_dim:
            raise ValueError("codec: bad encode shapes")
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        if self.kind == "dense":
            self._gemm(frame.data_ptr(), 1, self.pixel_dim, self.enc_t, self.latent_dim, out.data_ptr(),
                       self.latent_dim, st)
        else:
            c = self.codec
            L.call("lp_codec_patch_encode", frame.data_ptr(), c.channels, c.height, c.width, self.enc.data_ptr(),
                   c.pixel_channels, c.scale, out.data_ptr(), st)

    def decode_device(self, x: torch.Tensor, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        out = torch.empty((x.shape[0] * self.upsample, self.pixel_dim), dtype=torch.float32, device=self.device)
        self.decode_into(x.contiguous(), out, stream)
        return out

    def aas_sink_device(self, x: torch.Tensor, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """encode(decode(block)[0]) (kvcache.py:107) without leaving the device:
        only frame 0 of latent frame 0 is decoded."""
        st = stream or torch.cuda.current_stream(self.device)
        fr = torch.empty((self.upsample, self.pixel_dim), dtype=torch.float32, device=self.device)
        self.decode_into(x[:1].contiguous(), fr, st)
        z = torch.empty(self.latent_dim, dtype=torch.float32, device=self.device)
        self.encode_into(fr[0], z, st)
        return z

    # ------------------------------------------------- reference codec API
    def _up(self, a: np.ndarray) -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(a, dtype=F32)).to(self.device, non_blocking=False)

    def decode(self, block: LatentBlock) -> np.ndarray:
        """Latent block -> (F*r, P) pixel frames in temporal order (latent.py:189-193)."""
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            out = self.decode_device(self._up(block.values), self.stream).cpu()
        return out.numpy()

    def decode_frame(self, latent: np.ndarray) -> np.ndarray:
        latent = np.asarray(latent, dtype=F32)
        if latent.shape != (self.latent_dim,):
            raise ValueError(f"expected latent ({self.latent_dim},), got {latent.shape}")
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            out = self.decode_device(self._up(latent[None]), self.stream).cpu()
        return out.numpy()

    def encode(self, frame: np.ndarray) -> np.ndarray:
        frame = np.asarray(frame, dtype=F32)
        if frame.shape != (self.pixel_dim,):
            raise ValueError(f"expected pixel frame ({self.pixel_dim},), got {frame.shape}")
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            z = torch.empty(self.latent_dim, dtype=torch.float32, device=self.device)
            self.encode_into(self._up(frame), z, self.stream)
            out = z.cpu()
        return out.numpy()
