"""Non-GEMM ops of the decoder step (off the packed-LoRA hot path).

RMSNorm, RoPE, SwiGLU and the chunked cross-entropy are small HBM-bound passes
run by fused sm_100a kernels in libplora (csrc/elementwise.cu).  The ``ref_*``
functions are plain-torch fp32 restatements used only by the tests as the
reference for those kernels; the model never calls them.
"""

from __future__ import annotations

import torch

from . import _lib
from .ops import _LAUNCHES, _need, _stream

bf16 = torch.bfloat16


def rmsnorm_fwd(x: torch.Tensor, w: torch.Tensor, eps: float):
    rows, d = x.shape
    y = torch.empty_like(x)
    rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
    _lib.check(_lib.lib().plora_rmsnorm_fwd(_stream(), rows, d, _need(x, "x"), _need(w, "w"), eps,
                                            _need(y, "y"), _need(rstd, "rstd", torch.float32), 0), "rmsnorm_fwd")
    _LAUNCHES[0] += 1
    return y, rstd


def add_rmsnorm_fwd(a: torch.Tensor, b: torch.Tensor, w: torch.Tensor, eps: float):
    """(sum = a + b, rmsnorm(sum) * w, rstd): the residual add fused into the norm."""
    rows, d = a.shape
    s_ = torch.empty_like(a)
    y = torch.empty_like(a)
    rstd = torch.empty(rows, dtype=torch.float32, device=a.device)
    _lib.check(_lib.lib().plora_add_rmsnorm_fwd(_stream(), rows, d, _need(a, "a"), _need(b, "b"), _need(w, "w"), eps,
                                                _need(s_, "sum"), _need(y, "y"), _need(rstd, "rstd", torch.float32)),
               "add_rmsnorm_fwd")
    _LAUNCHES[0] += 1
    return s_, y, rstd


def rmsnorm_apply(x: torch.Tensor, rstd: torch.Tensor, w: torch.Tensor, out: torch.Tensor | None = None):
    rows, d = x.shape
    y = torch.empty_like(x) if out is None else out
    _lib.check(_lib.lib().plora_rmsnorm_fwd(_stream(), rows, d, _need(x, "x"), _need(w, "w"), 0.0,
                                            _need(y, "y"), _need(rstd, "rstd", torch.float32), 1), "rmsnorm_apply")
    _LAUNCHES[0] += 1
    return y


def rmsnorm_bwd(dy: torch.Tensor, x: torch.Tensor, rstd: torch.Tensor, w: torch.Tensor,
                residual_grad: torch.Tensor | None = None, out: torch.Tensor | None = None):
    rows, d = x.shape
    dx = torch.empty_like(x) if out is None else out
    _lib.check(_lib.lib().plora_rmsnorm_bwd(_stream(), rows, d, _need(dy, "dy"), _need(x, "x"),
                                            _need(rstd, "rstd", torch.float32), _need(w, "w"),
                                            _need(residual_grad, "residual_grad", allow_none=True),
                                            _need(dx, "dx")), "rmsnorm_bwd")
    _LAUNCHES[0] += 1
    return dx


def swiglu_fwd(g: torch.Tensor, u: torch.Tensor, out: torch.Tensor | None = None):
    a = torch.empty_like(g) if out is None else out
    _lib.check(_lib.lib().plora_swiglu_fwd(_stream(), g.numel(), _need(g, "g"), _need(u, "u"), _need(a, "a")),
               "swiglu_fwd")
    _LAUNCHES[0] += 1
    return a


def swiglu_bwd(da: torch.Tensor, g: torch.Tensor, u: torch.Tensor, out_g=None, out_u=None,
               act_out: torch.Tensor | None = None):
    """(dg, du) from da; dg/du may alias g/u.  act_out (optional) receives silu(g) * u,
    bit-identical to swiglu_fwd, from the same pass."""
    dg = torch.empty_like(g) if out_g is None else out_g
    du = torch.empty_like(u) if out_u is None else out_u
    _lib.check(_lib.lib().plora_swiglu_bwd(_stream(), g.numel(), _need(da, "da"), _need(g, "g"), _need(u, "u"),
                                           _need(dg, "dg"), _need(du, "du"),
                                           _need(act_out, "act_out", allow_none=True)), "swiglu_bwd")
    _LAUNCHES[0] += 1
    return dg, du


def rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor, seq_len: int, out: torch.Tensor | None = None,
         inverse: bool = False, rotate: bool = True) -> torch.Tensor:
    """x is a [B, s, H, hd] or [B, H, s, hd]-strided view (given as [B, s, H, hd] dims order
    via ``bshd``); returns a contiguous [B*s, H*hd] tensor (may be x itself if in place)."""
    B, s, H, hd = x.shape
    if x.stride(-1) != 1:
        raise ValueError("rope: last dim must be contiguous")
    T = B * s
    if out is None:
        out = torch.empty((T, H * hd), dtype=x.dtype, device=x.device)
    _lib.check(_lib.lib().plora_rope(_stream(), x.data_ptr(), _need(out, "out"),
                                     _need(cos, "cos", torch.float32), _need(sin, "sin", torch.float32),
                                     T, s, H, hd, x.stride(0), x.stride(1), x.stride(2), int(rotate),
                                     int(inverse)), "rope")
    _LAUNCHES[0] += 1
    return out


def cross_entropy(logits: torch.Tensor, labels: torch.Tensor, weight: torch.Tensor, tok_loss: torch.Tensor):
    """Overwrites bf16 logits [Tc][V] with weight_t (softmax_t - onehot_t); tok_loss[t] = weight_t CE_t."""
    rows, V = logits.shape
    _lib.check(_lib.lib().plora_cross_entropy(_stream(), rows, V, _need(logits, "logits"),
                                              _need(labels, "labels", torch.int64),
                                              _need(weight, "weight", torch.float32),
                                              _need(tok_loss, "tok_loss", torch.float32)), "cross_entropy")
    _LAUNCHES[0] += 1


def ce_stats(logits: torch.Tensor, labels: torch.Tensor, v0: int, stats: torch.Tensor | None = None):
    """Vocabulary-parallel CE pass 1: stats [rows][3] f32 = (max, sum exp(x - max), x[label] or 0)
    over this rank's vocabulary slice [v0, v0 + V)."""
    rows, V = logits.shape
    if stats is None:
        stats = torch.empty((rows, 3), dtype=torch.float32, device=logits.device)
    _lib.check(_lib.lib().plora_ce_stats(_stream(), rows, V, _need(logits, "logits"),
                                         _need(labels, "labels", torch.int64), int(v0),
                                         _need(stats, "stats", torch.float32)), "ce_stats")
    _LAUNCHES[0] += 1
    return stats


def ce_apply(logits: torch.Tensor, labels: torch.Tensor, v0: int, lse: torch.Tensor, weight: torch.Tensor):
    """Vocabulary-parallel CE pass 2: logits <- weight_t (exp(x - lse_t) - onehot_t) on the slice."""
    rows, V = logits.shape
    _lib.check(_lib.lib().plora_ce_apply(_stream(), rows, V, _need(logits, "logits"),
                                         _need(labels, "labels", torch.int64), int(v0),
                                         _need(lse, "lse", torch.float32), _need(weight, "weight", torch.float32)),
               "ce_apply")
    _LAUNCHES[0] += 1


# ---------------------------------------------------------------------------- torch references
def ref_rmsnorm_fwd(x, w, eps):
    xf = x.float()
    rstd = torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)
    return (xf * rstd * w.float()).to(bf16), rstd.squeeze(-1)


def ref_rmsnorm_bwd(dy, x, rstd, w, residual_grad=None):
    r = rstd.unsqueeze(-1)
    xhat = x.float() * r
    g = dy.float() * w.float()
    dx = r * (g - xhat * (g * xhat).mean(-1, keepdim=True))
    if residual_grad is not None:
        dx = dx + residual_grad.float()
    return dx.to(bf16)


def ref_rope(x, cos, sin, inverse=False):
    """x [B, s, H, hd] -> [B, s, H, hd] rotated (half-rotation)."""
    h = x.shape[-1] // 2
    c = cos[None, :, None, :]
    s = -sin[None, :, None, :] if inverse else sin[None, :, None, :]
    x1, x2 = x[..., :h].float(), x[..., h:].float()
    return torch.cat((x1 * c - x2 * s, x2 * c + x1 * s), dim=-1).to(bf16)


def ref_swiglu_fwd(g, u):
    return (torch.nn.functional.silu(g.float()) * u.float()).to(bf16)


def ref_swiglu_bwd(da, g, u):
    gf, uf, daf = g.float(), u.float(), da.float()
    sg = torch.sigmoid(gf)
    return (daf * uf * sg * (1 + gf * (1 - sg))).to(bf16), (daf * gf * sg).to(bf16)


def ref_cross_entropy(logits, labels, weight):
    lf = logits.float()
    lse = torch.logsumexp(lf, dim=-1)
    tok = (lse - lf.gather(1, labels.view(-1, 1)).squeeze(1)) * weight
    p = torch.softmax(lf, dim=-1)
    p.scatter_add_(1, labels.view(-1, 1), -torch.ones_like(lse).view(-1, 1))
    return (p * weight.unsqueeze(1)).to(bf16), tok
