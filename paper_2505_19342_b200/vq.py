"""Grouped vector quantization — drop-in for seqvq.vq (vq.py:24-233, inference subset).

Same names, argument meaning and error behaviour as the reference:
``index_bits``, ``Codebook``, ``QuantizedTokens``, ``quantize`` (-> (QuantizedTokens,
x_hat)), ``dequantize``; ties go to the lowest index and indices are bit-identical to
the reference's fp64 search.  The arithmetic runs in the native library
(astra_vq_encode / astra_vq_decode, include/astra_b200.h); NumPy in, NumPy out,
torch CUDA tensors in, torch CUDA tensors out.
"""

from __future__ import annotations

import ctypes
import math
import zlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .errors import IndexCorruptionError, ShapeError


def index_bits(codebook_size: int) -> int:
    """Bits to name one centroid: ceil(log2 K); 0 for K=1 (vq.py:24-28)."""
    if codebook_size < 1:
        raise ValueError("codebook size must be >= 1")
    return max(0, math.ceil(math.log2(codebook_size)))


class _CB(ctypes.Structure):
    _fields_ = [("groups", ctypes.c_int), ("size", ctypes.c_int), ("group_dim", ctypes.c_int),
                ("padded_dim", ctypes.c_int), ("centroids", ctypes.c_void_p),
                ("c_hi", ctypes.c_void_p), ("c_lo", ctypes.c_void_p), ("c_sq", ctypes.c_void_p),
                ("c_sq64", ctypes.c_void_p), ("c_norm_max", ctypes.c_void_p),
                ("c_win", ctypes.c_void_p)]


class DeviceCodebook:
    """A codebook resident in HBM with its derived encode tables (astra_vq_prepare)."""

    def __init__(self, centroids: torch.Tensor, layer_id: int = 0):
        if centroids.dim() != 3:
            raise ShapeError("centroids must be [G, K, D/G]")
        self.layer_id = layer_id
        self.centroids = centroids.contiguous().float()
        g, k, gd = self.centroids.shape
        self.groups, self.size, self.group_dim = g, k, gd
        self.padded_dim = ((gd + 63) // 64) * 64
        dev = self.centroids.device
        self.c_hi = torch.empty(g, k, self.padded_dim, dtype=torch.bfloat16, device=dev)
        self.c_lo = torch.empty_like(self.c_hi)
        self.c_sq = torch.empty(g, k, dtype=torch.float32, device=dev)
        self.c_sq64 = torch.empty(g, k, dtype=torch.float64, device=dev)
        self.c_norm_max = torch.empty(g, dtype=torch.float32, device=dev)
        self.c_win = torch.empty(g, k, 4, dtype=torch.float32, device=dev)
        self.struct = _CB(g, k, gd, self.padded_dim, self.centroids.data_ptr(), self.c_hi.data_ptr(),
                          self.c_lo.data_ptr(), self.c_sq.data_ptr(), self.c_sq64.data_ptr(),
                          self.c_norm_max.data_ptr(), self.c_win.data_ptr())
        _native.call("astra_vq_prepare", ctypes.byref(self.struct), _stream())

    @property
    def dim(self) -> int:
        return self.groups * self.group_dim

    @property
    def bits_per_token(self) -> int:
        return self.groups * index_bits(self.size)

    def workspace_bytes(self, m: int) -> int:
        return int(_native.load().astra_vq_encode_workspace(m, self.groups, self.size,
                                                            self.padded_dim))

    def encode(self, x: torch.Tensor, out: torch.Tensor | None = None, rows: torch.Tensor | None = None,
               workspace: torch.Tensor | None = None, stats: torch.Tensor | None = None) -> torch.Tensor:
        """Nearest-code indices int32 [M, G] of rows (x[rows] if given) of fp32 x."""
        m = rows.shape[0] if rows is not None else x.shape[0]
        if x.dim() != 2 or x.shape[1] < self.dim or x.stride(1) != 1 or x.dtype != torch.float32:
            raise ShapeError(f"quantize expects fp32 [T, {self.dim}], got {tuple(x.shape)}")
        if out is None:
            out = torch.empty(m, self.groups, dtype=torch.int32, device=x.device)
        need = self.workspace_bytes(m)
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=x.device)
        _native.call("astra_vq_encode", ctypes.byref(self.struct), x.data_ptr(), m, x.stride(0),
                     rows.data_ptr() if rows is not None else None, out.data_ptr(),
                     stats.data_ptr() if stats is not None else None, workspace.data_ptr(),
                     workspace.numel(), _stream())
        return out

    def decode(self, idx: torch.Tensor, out: torch.Tensor | None = None,
               err: torch.Tensor | None = None) -> torch.Tensor:
        if idx.dim() != 2 or idx.shape[1] != self.groups:
            raise ShapeError("index width does not match the codebook's groups")
        idx = idx.to(torch.int32).contiguous()
        if out is None:
            out = torch.empty(idx.shape[0], self.dim, dtype=torch.float32, device=idx.device)
        check = err is None
        if err is None:
            err = torch.zeros(1, dtype=torch.int32, device=idx.device)
        _native.call("astra_vq_decode", ctypes.byref(self.struct), idx.data_ptr(), idx.shape[0],
                     out.data_ptr(), out.stride(0), err.data_ptr(), _stream())
        if check and int(err.item()) != 0:
            raise IndexCorruptionError(f"index outside [0, {self.size}) in layer {self.layer_id}")
        return out


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("astra VQ runs on the GPU only (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class Codebook:
    """Per-layer grouped codebook (vq.py:31-76).  ``centroids[g]`` is [K, D/G]."""

    layer_id: int
    groups: int
    centroids: list
    ema_counts: np.ndarray | None = None
    ema_sums: list | None = None
    decay: float = 0.99
    smoothing: float = 1e-5
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        if self.groups < 1 or len(self.centroids) != self.groups:
            raise ShapeError("codebook needs one centroid table per group")
        k, gd = np.asarray(self.centroids[0]).shape
        for c in self.centroids:
            if np.asarray(c).ndim != 2 or np.asarray(c).shape != (k, gd):
                raise ShapeError("all groups must share a [K, D/G] shape")
        if not (0.0 < self.decay < 1.0):
            raise ValueError("EMA decay must lie strictly inside (0, 1)")
        if self.smoothing <= 0.0:
            raise ValueError("Laplace smoothing must be positive")

    @property
    def size(self) -> int:
        return np.asarray(self.centroids[0]).shape[0]

    @property
    def group_dim(self) -> int:
        return np.asarray(self.centroids[0]).shape[1]

    @property
    def dim(self) -> int:
        return self.groups * self.group_dim

    @property
    def bits_per_token(self) -> int:
        return self.groups * index_bits(self.size)

    def on_device(self, device: torch.device | None = None) -> DeviceCodebook:
        """HBM copy (cached per device; codebooks are read-only at inference)."""
        device = device or _device()
        # identity AND content: ema_update swaps the tables, a caller may edit them in place
        crc = 0
        for c in self.centroids:
            crc = zlib.crc32(np.ascontiguousarray(c).view(np.uint8), crc)
        key = (str(device), tuple(id(c) for c in self.centroids), crc)
        dc = self._dev.get(key)
        if dc is None:
            tables = np.stack([np.asarray(c, dtype=np.float32) for c in self.centroids])
            dc = DeviceCodebook(torch.from_numpy(tables).to(device), self.layer_id)
            self._dev.clear()
            self._dev[key] = dc
        return dc


@dataclass(frozen=True)
class QuantizedTokens:
    """Indices for a batch of tokens under one codebook (vq.py:79-94)."""

    layer_id: int
    token_count: int
    indices: np.ndarray  # [T, G] int32
    bits_per_token: int

    def __post_init__(self):
        if self.indices.shape[0] != self.token_count:
            raise ShapeError("token_count does not match index rows")

    @property
    def payload_bits(self) -> int:
        return self.token_count * self.bits_per_token


def _nearest_f64(x: torch.Tensor, c: torch.Tensor, rows: int = 4096) -> torch.Tensor:
    """fp64 nearest centroid on the GPU for fp64 models (vq.py:126-131): the reference's
    expression ``(|p|^2 - 2 p.c) + |c|^2`` in fp64 via cuBLAS DGEMM, argmin with the first
    index on ties (torch.argmin's contract, like np.argmin)."""
    cc = (c * c).sum(1)
    out = torch.empty(x.shape[0], dtype=torch.int64, device=x.device)
    for r0 in range(0, x.shape[0], rows):
        p = x[r0:r0 + rows]
        d2 = (p * p).sum(1, keepdim=True) - 2.0 * (p @ c.T) + cc[None, :]
        out[r0:r0 + rows] = d2.argmin(1)
    return out


def _quantize_f64(codebook: Codebook, xa, is_torch: bool):
    dev = xa.device if is_torch and xa.is_cuda else _device()
    xt = (xa if is_torch else torch.from_numpy(np.ascontiguousarray(xa))).to(dev, torch.float64)
    gd = codebook.group_dim
    idx = torch.empty(xt.shape[0], codebook.groups, dtype=torch.int32, device=dev)
    tables = []
    for g in range(codebook.groups):
        c = np.asarray(codebook.centroids[g])
        ct = torch.from_numpy(np.ascontiguousarray(c, dtype=np.float64)).to(dev)
        tables.append(torch.from_numpy(np.ascontiguousarray(c)).to(dev))
        idx[:, g] = _nearest_f64(xt[:, g * gd:(g + 1) * gd].contiguous(), ct).to(torch.int32)
    # x_hat in the centroids' dtype, groups concatenated in order (vq.py:225-233)
    xhat = torch.cat([tables[g][idx[:, g].long()] for g in range(codebook.groups)], dim=1)
    q = QuantizedTokens(codebook.layer_id, xt.shape[0], idx if is_torch else idx.cpu().numpy(),
                        codebook.bits_per_token)
    return q, (xhat if is_torch else xhat.cpu().numpy())


def quantize(codebook: Codebook, x):
    """Encode tokens to per-group nearest-centroid indices (vq.py:207-222).

    Returns (QuantizedTokens, x_hat); x_hat equals dequantize(codebook, indices)
    bitwise.  Accepts NumPy (returns NumPy) or a CUDA tensor (returns tensors).
    fp32 inputs and centroids take the tcgen05 encode (indices bit-identical to the fp64
    reference); fp64 inputs or centroids take an fp64 GPU search so the reference's fp64
    semantics are kept, and x_hat comes back in the centroids' dtype."""
    is_torch = isinstance(x, torch.Tensor)
    xa = x if is_torch else np.asarray(x)
    if xa.ndim != 2 or xa.shape[1] != codebook.dim:
        raise ShapeError(f"quantize expects [T, {codebook.dim}], got {tuple(xa.shape)}")
    c_dtype = np.asarray(codebook.centroids[0]).dtype
    x_f64 = (xa.dtype == torch.float64) if is_torch else (xa.dtype == np.float64)
    if x_f64 or c_dtype == np.float64:
        return _quantize_f64(codebook, xa, is_torch)
    dc = codebook.on_device()
    xt = (xa if is_torch else torch.from_numpy(np.ascontiguousarray(xa, dtype=np.float32)))
    xt = xt.to(dc.centroids.device, torch.float32).contiguous()
    idx = dc.encode(xt)
    xhat = dc.decode(idx)
    if is_torch:
        return QuantizedTokens(codebook.layer_id, xt.shape[0], idx, codebook.bits_per_token), xhat
    q = QuantizedTokens(codebook.layer_id, xt.shape[0], idx.cpu().numpy(), codebook.bits_per_token)
    return q, xhat.cpu().numpy()


def dequantize(codebook: Codebook, q: QuantizedTokens):
    """Reconstruct embeddings by centroid lookup, groups concatenated in order (vq.py:225-233)."""
    idx = q.indices
    if idx.shape[1] != codebook.groups:
        raise ShapeError("index width does not match the codebook's groups")
    if np.asarray(codebook.centroids[0]).dtype != np.float32:
        # non-fp32 tables (fp64 models): gather in their own dtype, same range check
        it = idx if isinstance(idx, torch.Tensor) else torch.from_numpy(np.asarray(idx))
        if it.numel() and (int(it.min()) < 0 or int(it.max()) >= codebook.size):
            raise IndexCorruptionError(f"index outside [0, {codebook.size}) in layer {q.layer_id}")
        dev = it.device if it.is_cuda else _device()
        it = it.to(dev).long()
        out = torch.cat([torch.from_numpy(np.ascontiguousarray(codebook.centroids[g])).to(dev)[it[:, g]]
                         for g in range(codebook.groups)], dim=1)
        return out if isinstance(idx, torch.Tensor) else out.cpu().numpy()
    if isinstance(idx, torch.Tensor):
        return codebook.on_device(idx.device).decode(idx)
    idx = np.asarray(idx)
    if idx.size and (idx.min() < 0 or idx.max() >= codebook.size):
        raise IndexCorruptionError(f"index outside [0, {codebook.size}) in layer {q.layer_id}")
    dc = codebook.on_device()
    out = dc.decode(torch.from_numpy(np.ascontiguousarray(idx, dtype=np.int32)).to(
        dc.centroids.device))
    return out.cpu().numpy()


MAGIC = b"AVQ1"


def save_codebook(codebook: Codebook) -> bytes:
    """AVQ1 blob (vq.py:328-339): magic, (layer, G, K, D/G) LE u32, fp32 centroids
    group-major, then fp64 EMA counts and sums."""
    import struct
    g, k, gd = codebook.groups, codebook.size, codebook.group_dim
    counts = codebook.ema_counts if codebook.ema_counts is not None else np.zeros((g, k))
    sums = codebook.ema_sums if codebook.ema_sums is not None else [np.zeros((k, gd))] * g
    head = MAGIC + struct.pack("<4I", codebook.layer_id, g, k, gd)
    body = b"".join(np.ascontiguousarray(c, dtype="<f4").tobytes() for c in codebook.centroids)
    ema = np.ascontiguousarray(counts, dtype="<f8").tobytes()
    ema += b"".join(np.ascontiguousarray(s, dtype="<f8").tobytes() for s in sums)
    return head + body + ema


def load_codebook(blob: bytes) -> Codebook:
    """Inverse of save_codebook (vq.py:342-361), same validation."""
    import struct
    if len(blob) < 20 or blob[:4] != MAGIC:
        raise ValueError("not a codebook blob (bad magic)")
    layer_id, groups, k, gd = struct.unpack("<4I", blob[4:20])
    expect = 20 + 4 * groups * k * gd + 8 * groups * k + 8 * groups * k * gd
    if len(blob) != expect:
        raise ValueError(f"codebook blob length {len(blob)} != expected {expect}")
    flat = np.frombuffer(blob, dtype="<f4", offset=20, count=groups * k * gd)
    tables = [flat[g * k * gd:(g + 1) * k * gd].reshape(k, gd).copy() for g in range(groups)]
    off = 20 + 4 * groups * k * gd
    counts = np.frombuffer(blob, dtype="<f8", offset=off, count=groups * k).reshape(groups, k).copy()
    off += 8 * groups * k
    sums_flat = np.frombuffer(blob, dtype="<f8", offset=off)
    sums = [sums_flat[g * k * gd:(g + 1) * k * gd].reshape(k, gd).copy() for g in range(groups)]
    return Codebook(layer_id=layer_id, groups=groups, centroids=tables, ema_counts=counts,
                    ema_sums=sums)
