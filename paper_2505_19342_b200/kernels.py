"""Torch-facing wrappers over the C-ABI kernels (device memory and streams come
from PyTorch; all arithmetic happens in the native library).

Every function here requires CUDA tensors and raises if the native library
is missing; there is no CPU or eager-PyTorch fallback on the hot path.
"""

from __future__ import annotations

import torch

from . import _native
from .errors import ShapeError

BF16 = torch.bfloat16


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise RuntimeError("astra kernels run on CUDA tensors only (no CPU fallback)")


def split_bf16(x: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """fp32 -> (hi, lo) bf16 pair with x ~= hi + lo (setup-time helper for weights)."""
    hi = x.to(BF16)
    lo = (x - hi.float()).to(BF16)
    return hi, lo


def gemm(a_hi: torch.Tensor, b_hi: torch.Tensor, *, a_lo: torch.Tensor | None = None,
         b_lo: torch.Tensor | None = None, bias: torch.Tensor | None = None,
         residual: torch.Tensor | None = None, gelu: bool = False,
         out_f32: torch.Tensor | None = None, out_hi: torch.Tensor | None = None,
         out_lo: torch.Tensor | None = None) -> None:
    """out = epilogue(A @ B^T).  A: [M, K] bf16, B: [N, K] bf16 (weight transposed).

    passes = 3 (split-precision) when both lo operands are given.
    """
    _require_cuda(a_hi, b_hi, a_lo, b_lo, bias, residual, out_f32, out_hi, out_lo)
    M, K = a_hi.shape
    N, K2 = b_hi.shape
    if K != K2:
        raise ShapeError(f"gemm: inner dims {tuple(a_hi.shape)} x {tuple(b_hi.shape)}")
    passes = 3 if (a_lo is not None and b_lo is not None) else 1
    for t in (a_hi, b_hi, a_lo, b_lo):
        if t is not None and (t.dtype != BF16 or t.stride(1) != 1):
            raise ShapeError("gemm operands must be row-major bf16")
    if a_lo is not None and a_lo.stride(0) != a_hi.stride(0):
        raise ShapeError("gemm: A hi/lo must share a row pitch")
    if b_lo is not None and b_lo.stride(0) != b_hi.stride(0):
        raise ShapeError("gemm: B hi/lo must share a row pitch")
    ld_res = residual.stride(0) if residual is not None else 0
    ld_f32 = out_f32.stride(0) if out_f32 is not None else 0
    ld_bf = out_hi.stride(0) if out_hi is not None else 0
    if out_lo is not None and out_lo.stride(0) != ld_bf:
        raise ShapeError("gemm: out hi/lo must share a row pitch")
    _native.call("astra_gemm", _ptr(a_hi), _ptr(a_lo), a_hi.stride(0), _ptr(b_hi), _ptr(b_lo),
                 b_hi.stride(0), M, N, K, passes, _ptr(bias), _ptr(residual), ld_res,
                 _ptr(out_f32), ld_f32, _ptr(out_hi), _ptr(out_lo), ld_bf, int(gelu), _stream())


def pack_indices(idx: torch.Tensor, bits: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """int32 codes -> LSB-first ``bits``-bit stream in uint32 words (astra_pack_indices)."""
    _require_cuda(idx)
    idx = idx.contiguous()
    n = idx.numel()
    nwords = (n * bits + 31) // 32
    if out is None:
        out = torch.empty(nwords, dtype=torch.int32, device=idx.device)
    _native.call("astra_pack_indices", idx.data_ptr(), n, bits, out.data_ptr(), _stream())
    return out


def unpack_indices(words: torch.Tensor, count: int, bits: int, size: int,
                   out: torch.Tensor | None = None, err: torch.Tensor | None = None) -> torch.Tensor:
    """Inverse of pack_indices; codes >= size set *err (IndexCorruptionError upstream)."""
    _require_cuda(words)
    if out is None:
        out = torch.empty(count, dtype=torch.int32, device=words.device)
    if err is None:
        err = torch.zeros(1, dtype=torch.int32, device=words.device)
    _native.call("astra_unpack_indices", words.data_ptr(), count, bits, size, out.data_ptr(),
                 err.data_ptr(), _stream())
    return out
