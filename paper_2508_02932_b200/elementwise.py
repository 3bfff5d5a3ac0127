"""Non-GEMM ops of the decoder step (off the packed-LoRA hot path).

RMSNorm, RoPE, SwiGLU and the chunked cross-entropy are small HBM-bound passes.
They dispatch to fused sm_100a kernels in libplora when available (``fused``)
and are otherwise written in plain torch (which also serves as the fp32
reference for the fused kernels' tests).
"""

from __future__ import annotations

import torch

bf16 = torch.bfloat16


def rmsnorm_fwd(x: torch.Tensor, w: torch.Tensor, eps: float):
    xf = x.float()
    rstd = torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)
    return (xf * rstd * w.float()).to(bf16), rstd.squeeze(-1)


def rmsnorm_apply(x: torch.Tensor, rstd: torch.Tensor, w: torch.Tensor):
    return (x.float() * rstd.unsqueeze(-1) * w.float()).to(bf16)


def rmsnorm_bwd(dy: torch.Tensor, x: torch.Tensor, rstd: torch.Tensor, w: torch.Tensor,
                residual_grad: torch.Tensor | None = None):
    r = rstd.unsqueeze(-1)
    xhat = x.float() * r
    g = dy.float() * w.float()
    dx = r * (g - xhat * (g * xhat).mean(-1, keepdim=True))
    if residual_grad is not None:
        dx = dx + residual_grad.float()
    return dx.to(bf16)


def rope_fwd(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor):
    """x [B, s, H, hd] (half-rotation convention); cos/sin [s, hd/2]."""
    h = x.shape[-1] // 2
    c = cos[None, :, None, :]
    s = sin[None, :, None, :]
    x1, x2 = x[..., :h].float(), x[..., h:].float()
    return torch.cat((x1 * c - x2 * s, x2 * c + x1 * s), dim=-1).to(bf16)


def rope_bwd(dy: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor):
    h = dy.shape[-1] // 2
    c = cos[None, :, None, :]
    s = sin[None, :, None, :]
    d1, d2 = dy[..., :h].float(), dy[..., h:].float()
    return torch.cat((d1 * c + d2 * s, d2 * c - d1 * s), dim=-1).to(bf16).contiguous()


def swiglu_fwd(g: torch.Tensor, u: torch.Tensor):
    return (torch.nn.functional.silu(g.float()) * u.float()).to(bf16)


def swiglu_bwd(da: torch.Tensor, g: torch.Tensor, u: torch.Tensor):
    gf, uf, daf = g.float(), u.float(), da.float()
    sg = torch.sigmoid(gf)
    du = daf * gf * sg
    dg = daf * uf * sg * (1 + gf * (1 - sg))
    return dg.to(bf16), du.to(bf16)


def cross_entropy_fwd_bwd(logits: torch.Tensor, labels: torch.Tensor, weight: torch.Tensor,
                          token_adapter: torch.Tensor, losses: torch.Tensor) -> None:
    """Weighted CE over a token chunk.  Overwrites ``logits`` (bf16 [Tc][V]) with
    d loss / d logits = weight_t * (softmax_t - onehot_t) and adds
    sum_t weight_t * CE_t into losses[adapter(t)]."""
    lf = logits.float()
    lse = torch.logsumexp(lf, dim=-1)
    tgt = lf.gather(1, labels.view(-1, 1)).squeeze(1)
    losses.index_add_(0, token_adapter, (lse - tgt) * weight)
    p = torch.exp(lf - lse.unsqueeze(1))
    p.scatter_add_(1, labels.view(-1, 1), -torch.ones_like(tgt).view(-1, 1))
    p.mul_(weight.unsqueeze(1))
    logits.copy_(p.to(bf16))
