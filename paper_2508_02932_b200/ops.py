"""Torch-tensor front end of the C-ABI: packed-LoRA linear forward/backward,
plain bf16 GEMM and the fused per-adapter AdamW.

Every function takes caller-owned CUDA tensors, validates them, and enqueues the
sm_100a kernels on torch's current stream through libplora.  No CPU fallback
exists: non-CUDA tensors are rejected.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .meta import PackMeta


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _need(t: torch.Tensor | None, name: str, dtype=torch.bfloat16, allow_none=False) -> int | None:
    if t is None:
        if allow_none:
            return None
        raise ValueError(f"{name} is required")
    if not t.is_cuda:
        raise _lib.PloraError(f"{name} must be a CUDA tensor (libplora has no CPU path)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def gemm(a: torch.Tensor, w: torch.Tensor, w_kmajor: bool = True, out: torch.Tensor | None = None,
         residual: torch.Tensor | None = None) -> torch.Tensor:
    """out[M][N] = a[M][K] @ (w.T if w_kmajor else w) (+ residual), bf16, tcgen05."""
    M, K = a.shape
    N = w.shape[0] if w_kmajor else w.shape[1]
    if (w.shape[1] if w_kmajor else w.shape[0]) != K:
        raise ValueError(f"gemm: weight {tuple(w.shape)} does not match K={K}")
    if out is None:
        out = torch.empty((M, N), dtype=torch.bfloat16, device=a.device)
    _lib.check(_lib.lib().plora_gemm_bf16(
        _stream(), M, N, K, _need(a, "a"), _need(w, "w"), int(w_kmajor), _need(out, "out"),
        out.stride(0), _need(residual, "residual", allow_none=True)), "plora_gemm_bf16")
    return out


def linear_fwd(meta: PackMeta, x: torch.Tensor, w: torch.Tensor, w_kmajor: bool,
               a_sh: torch.Tensor, bt_sh: torch.Tensor, hs_out: torch.Tensor | None = None,
               y_out: torch.Tensor | None = None, residual: torch.Tensor | None = None):
    """Packed LoRA linear forward.  Returns (y [T][k] bf16, hs [T][64nb] bf16)."""
    T, d = x.shape
    k = w.shape[0] if w_kmajor else w.shape[1]
    if T != meta.total_tokens:
        raise ValueError(f"x has {T} rows but the pack has {meta.total_tokens} tokens")
    if hs_out is None:
        hs_out = torch.empty((T, meta.rpad64), dtype=torch.bfloat16, device=x.device)
    if y_out is None:
        y_out = torch.empty((T, k), dtype=torch.bfloat16, device=x.device)
    s = meta.struct
    _lib.check(_lib.lib().plora_linear_fwd(
        _stream(), ctypes.byref(s), _need(x, "x"), d, k, _need(w, "w"), int(w_kmajor),
        _need(a_sh, "a_sh"), _need(bt_sh, "bt_sh"), _need(hs_out, "hs_out"), _need(y_out, "y"),
        y_out.stride(0), _need(residual, "residual", allow_none=True)), "plora_linear_fwd")
    return y_out, hs_out


def linear_expand(meta: PackMeta, x: torch.Tensor, w: torch.Tensor, w_kmajor: bool,
                  bt_sh: torch.Tensor, hs: torch.Tensor, y_out: torch.Tensor | None = None,
                  residual: torch.Tensor | None = None) -> torch.Tensor:
    """K1 + K2b with a caller-provided Hs: y = x op(W) + Hs_i B_i (+ residual)."""
    T, d = x.shape
    k = w.shape[0] if w_kmajor else w.shape[1]
    if y_out is None:
        y_out = torch.empty((T, k), dtype=torch.bfloat16, device=x.device)
    s = meta.struct
    _lib.check(_lib.lib().plora_linear_expand(
        _stream(), ctypes.byref(s), _need(x, "x"), d, k, _need(w, "w"), int(w_kmajor),
        _need(bt_sh, "bt_sh"), _need(hs, "hs"), _need(y_out, "y"), y_out.stride(0),
        _need(residual, "residual", allow_none=True)), "plora_linear_expand")
    return y_out


def linear_bwd(meta: PackMeta, x: torch.Tensor, w: torch.Tensor, w_kmajor: bool,
               a_sh: torch.Tensor, bt_sh: torch.Tensor, hs: torch.Tensor, dy: torch.Tensor,
               grad_a: torch.Tensor | None, grad_b: torch.Tensor | None,
               dx_out: torch.Tensor | None = None, need_dx: bool = True,
               dh_ws: torch.Tensor | None = None):
    """Packed LoRA linear backward (Cases 1-4).  Writes fp32 grads into grad_a /
    grad_b (adapter-major regions) and returns dx (or None)."""
    T, d = x.shape
    k = w.shape[0] if w_kmajor else w.shape[1]
    if dh_ws is None:
        dh_ws = torch.empty((T, meta.rpad64), dtype=torch.bfloat16, device=x.device)
    if need_dx and dx_out is None:
        dx_out = torch.empty((T, d), dtype=torch.bfloat16, device=x.device)
    s = meta.struct
    _lib.check(_lib.lib().plora_linear_bwd(
        _stream(), ctypes.byref(s), _need(x, "x"), d, k, _need(w, "w"), int(w_kmajor),
        _need(a_sh, "a_sh"), _need(bt_sh, "bt_sh"), _need(hs, "hs"), _need(dy, "dy"),
        _need(dh_ws, "dh_ws"), _need(dx_out, "dx", allow_none=True) if need_dx else None,
        dx_out.stride(0) if (need_dx and dx_out is not None) else 0,
        _need(grad_a, "grad_a", torch.float32, allow_none=True),
        _need(grad_b, "grad_b", torch.float32, allow_none=True)), "plora_linear_bwd")
    return dx_out if need_dx else None


def adamw(chunks: torch.Tensor, param: torch.Tensor, grad: torch.Tensor, exp_avg: torch.Tensor,
          exp_avg_sq: torch.Tensor, shadow: torch.Tensor, hp: torch.Tensor, step: int,
          beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8) -> None:
    """Fused per-adapter AdamW over the chunk table (see include/plora.h)."""
    _lib.check(_lib.lib().plora_adamw(
        _stream(), chunks.shape[0], _need(chunks, "chunks", torch.int64),
        _need(param, "param", torch.float32), _need(grad, "grad", torch.float32),
        _need(exp_avg, "exp_avg", torch.float32), _need(exp_avg_sq, "exp_avg_sq", torch.float32),
        _need(shadow, "shadow"), _need(hp, "hp", torch.float32), beta1, beta2, eps, int(step)),
        "plora_adamw")
