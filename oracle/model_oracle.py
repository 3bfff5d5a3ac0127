"""ORACLE -- test infrastructure only.  Not part of the product path.

Float64 CPU decoder for model-level parity (logits / per-adapter losses /
per-adapter LoRA gradients).  The reference has no model, so this is a plain
restatement of the same architecture, except that EVERY LoRA linear's arithmetic
is the oracle restatement of lorasweep.packed_forward / packed_backward
(oracle/lorapack_oracle.py, pinned to the real reference by golden vectors):
reference-in-the-loop.  Everything else (RMSNorm, RoPE, attention, SwiGLU,
cross-entropy) is torch float64 autograd.

Used by tests/test_gpu_model.py at config C1 (tiny, d=256) and by
__graft_entry__.smoke().
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from oracle import lorapack_oracle as O


class _OracleLoraLinear(torch.autograd.Function):
    """y = packed_forward(pack(x, A_i, B_i), W); grads via packed_backward (fp64 numpy)."""

    @staticmethod
    def forward(ctx, x, w, meta, *ab):
        n = len(meta["alphas"])
        downs = [a.detach().numpy() for a in ab[:n]]
        ups = [b.detach().numpy() for b in ab[n:]]
        so = meta["row_offsets"]
        xs = [x.detach().numpy()[so[i]:so[i + 1]] for i in range(n)]
        p = O.pack(downs, ups, meta["alphas"], xs)
        ctx.p, ctx.w, ctx.n = p, w.detach().numpy(), n
        ys = O.packed_forward(p, ctx.w)
        return torch.from_numpy(np.concatenate(ys, axis=0))

    @staticmethod
    def backward(ctx, dy):
        so = ctx.p["row_offsets"]
        d = dy.detach().numpy()
        dys = [d[so[i]:so[i + 1]] for i in range(ctx.n)]
        dd, du, dx = O.packed_backward(ctx.p, ctx.w, dys)
        grads = [torch.from_numpy(np.ascontiguousarray(g)) for g in dd + du]
        return (torch.from_numpy(np.concatenate(dx, axis=0)), None, None, *grads)


def _rms(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def _rope(x, cos, sin):
    h = x.shape[-1] // 2
    c, s = cos[None, :, None, :], sin[None, :, None, :]
    x1, x2 = x[..., :h], x[..., h:]
    return torch.cat((x1 * c - x2 * s, x2 * c + x1 * s), dim=-1)


def oracle_step(cfg, base, adapters, alphas, row_offsets, tokens, seq_len, cos, sin, n_lab):
    """fp64 forward + backward.

    base: dict of fp64 CPU tensors (nn.Linear layout [h_out][h_in] per target, per layer list)
    adapters: {(layer, target): (downs[list d x r], ups[list r x k])} fp64
    Returns (per-adapter losses [n], grads {(layer, target): (d_downs, d_ups)}, logits [T][V])."""
    n = len(alphas)
    meta = {"alphas": tuple(alphas), "row_offsets": tuple(row_offsets)}
    leaves = {}
    for key, (downs, ups) in adapters.items():
        leaves[key] = ([d.clone().requires_grad_() for d in downs], [u.clone().requires_grad_() for u in ups])
    T = int(row_offsets[-1])
    B = T // seq_len
    H, KV, hd = cfg.n_heads, cfg.n_kv, cfg.head_dim

    def lin(layer, tname, x):
        downs, ups = leaves[(layer, tname)]
        w = base["layers"][layer][tname].t().contiguous()   # reference layout d x k
        return _OracleLoraLinear.apply(x, w, meta, *downs, *ups)

    h = base["embed"][tokens]
    for layer in range(cfg.n_layers):
        lw = base["layers"][layer]
        x1 = _rms(h, lw["attn_norm"], cfg.norm_eps)
        q, k, v = lin(layer, "q", x1), lin(layer, "k", x1), lin(layer, "v", x1)
        if cfg.qkv_bias:
            q, k, v = q + lw["q_bias"], k + lw["k_bias"], v + lw["v_bias"]
        q = _rope(q.view(B, seq_len, H, hd), cos, sin).transpose(1, 2)
        k = _rope(k.view(B, seq_len, KV, hd), cos, sin).transpose(1, 2)
        v = v.view(B, seq_len, KV, hd).transpose(1, 2)
        if KV != H:
            k = k.repeat_interleave(H // KV, dim=1)
            v = v.repeat_interleave(H // KV, dim=1)
        o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        h = h + lin(layer, "o", o.transpose(1, 2).reshape(T, H * hd))
        x2 = _rms(h, lw["mlp_norm"], cfg.norm_eps)
        a = F.silu(lin(layer, "gate", x2)) * lin(layer, "up", x2)
        h = h + lin(layer, "down", a)
    xf = _rms(h, base["final_norm"], cfg.norm_eps)
    logits = xf @ base["lm_head"].t()
    labels = torch.roll(tokens, -1)
    pos = torch.arange(T) % seq_len
    ce = F.cross_entropy(logits, labels, reduction="none")
    ce = torch.where(pos != seq_len - 1, ce, torch.zeros_like(ce))
    losses = torch.stack([ce[row_offsets[i]:row_offsets[i + 1]].sum() / n_lab[i] for i in range(n)])
    losses.sum().backward()
    grads = {key: ([d.grad for d in downs], [u.grad for u in ups]) for key, (downs, ups) in leaves.items()}
    return losses.detach(), grads, logits.detach()


def from_trainer(trainer):
    """fp64 CPU copies of a PackedLoraTrainer's base weights and adapter masters."""
    cfg = trainer.cfg
    b = trainer.base

    def f64(t):
        return t.detach().to("cpu", torch.float64)

    base = {"embed": f64(b.embed), "final_norm": f64(b.final_norm), "lm_head": f64(b.lm_head),
            "layers": [{k: f64(v) for k, v in lw.items()} for lw in b.layers]}
    adapters = {}
    n = trainer.meta.n_adapters
    for layer in range(cfg.n_layers):
        for t in cfg.targets():
            downs = [f64(trainer.bank.down(layer, t.name, i)) for i in range(n)]
            ups = [f64(trainer.bank.up(layer, t.name, i)) for i in range(n)]
            adapters[(layer, t.name)] = (downs, ups)
    return base, adapters
