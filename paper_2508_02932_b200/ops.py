"""Torch-tensor front end of the C-ABI: packed-LoRA linear forward/backward,
plain bf16 GEMM and the fused per-adapter AdamW.

Every function takes caller-owned CUDA tensors, validates them, and enqueues the
sm_100a kernels on torch's current stream through libplora.  No CPU fallback
exists: non-CUDA tensors are rejected.
"""

from __future__ import annotations

import ctypes

import numpy as np

import torch

from . import _lib
from .meta import PackMeta


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


class KernelTimer:
    """Per-kernel-class CUDA-event timing inside a timed region (bench.py roofline).

    While active, packed linears are issued as their component launches
    (shrink / segment reductions / GEMM) with events recorded on the launching
    stream around each, together with that launch's ALGORITHMIC flops and HBM bytes
    (``nbytes``: the roofline bytes of the HBM-bound kernels; ``algo_bytes``: operand +
    output bytes of every launch, the denominator of ncu's DRAM-traffic ratio)."""

    def __init__(self, external: bool = False):
        # external=True: the events become event-record nodes when the timed step is captured
        # into a CUDA graph, so every replay re-times each launch on the device without the
        # eager step's host enqueue gaps (bench.py's kernel-stats pass)
        self.records: list = []
        self.external = external

    def start(self):
        e = torch.cuda.Event(enable_timing=True, external=self.external)
        e.record()
        return e

    def stop(self, kind: str, e0, flops: float = 0.0, nbytes: float = 0.0, detail: str | None = None,
             algo_bytes: float | None = None):
        e1 = torch.cuda.Event(enable_timing=True, external=self.external)
        e1.record()
        self.records.append((kind, e0, e1, flops, nbytes, detail, nbytes if algo_bytes is None else algo_bytes))

    def summary(self) -> dict:
        """Per kernel class (and per GEMM shape, keys 'gemm[N..K..]'): launches, ms, flops, bytes."""
        torch.cuda.synchronize()
        out: dict = {}
        for kind, e0, e1, fl, nb, detail, _ in self.records:
            ms = e0.elapsed_time(e1)
            keys = [kind] + ([f"{kind}[{detail}]"] if detail is not None else [])
            for key in keys:
                d = out.setdefault(key, {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0})
                d["launches"] += 1
                d["ms"] += ms
                d["flops"] += fl
                d["bytes"] += nb
        return out

    def dump(self) -> list:
        """One entry per timed libplora launch, in issue order (for matching an ncu launch list)."""
        torch.cuda.synchronize()
        return [{"kind": k, "detail": d, "ms": round(e0.elapsed_time(e1), 4), "flops": fl, "hbm_bytes": nb,
                 "algo_bytes": ab} for k, e0, e1, fl, nb, d, ab in self.records]


_TIMER: KernelTimer | None = None
_LAUNCHES = [0]


def set_timer(t: KernelTimer | None) -> None:
    global _TIMER
    _TIMER = t


def launch_count() -> int:
    """Number of libplora kernel launches issued by this process so far."""
    return _LAUNCHES[0]


def count_launches(n: int) -> None:
    """Account for ``n`` libplora kernels launched from a replayed CUDA graph."""
    _LAUNCHES[0] += n


_WS: dict = {}


def _workspace() -> torch.Tensor:
    """The pack workspace of the stream-K shrink / segment-reduction kernels for the
    current (device, stream): zero-filled once, left zeroed by the kernels, so launches
    on one stream share it (include/plora.h, plora_pack_t.d_ws).  Created under CUDA-graph
    capture it comes from the graph's pool and its zero-fill is part of the graph."""
    dev = torch.cuda.current_device()
    key = (dev, torch.cuda.current_stream().cuda_stream)
    ws = _WS.get(key)
    if ws is None:
        ws = torch.zeros(int(_lib.lib().plora_lora_workspace_bytes()), dtype=torch.uint8, device=f"cuda:{dev}")
        _WS[key] = ws
    return ws


def _pack(meta: PackMeta):
    """meta's plora_pack_t with the current stream's workspace attached."""
    s = meta.struct
    ws = _workspace()
    s.d_ws = ws.data_ptr()
    s.ws_bytes = ws.numel()
    return s


def _lora_work(meta: PackMeta) -> tuple[int, int]:
    """(sum_i T_i r_i, R = sum_i r_i) for the algorithmic-work formulas."""
    if not hasattr(meta, "_work"):
        meta._work = (sum(t * r for t, r in zip(meta.tokens, meta.ranks)), sum(meta.ranks))
    return meta._work


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


def _on_current_device(t: torch.Tensor, name: str) -> None:
    """libplora launches on the current device's stream: operands of another device would
    be dereferenced on the wrong GPU."""
    if t.is_cuda and t.device.index != torch.cuda.current_device():
        raise ValueError(f"{name} is on {t.device} but the current device is cuda:{torch.cuda.current_device()} "
                         f"(run the op under torch.cuda.device({t.device.index}))")


def _size(t: torch.Tensor | None, name: str, numel: int) -> None:
    """Kernels write through raw pointers: a buffer smaller than the pack needs would be an
    out-of-bounds device write, so sizes are checked against the pack metadata here."""
    if t is not None and t.numel() < numel:
        raise ValueError(f"{name} has {t.numel()} elements, the pack needs {numel}")


def _lora_shapes(meta: PackMeta, K: int, l_sh: torch.Tensor, out: torch.Tensor, T: int) -> None:
    _size(l_sh, "lora operand", meta.n_adapters * K * meta.rpad64)
    _size(out, "low-rank output", T * meta.rpad64)


def gemm(a: torch.Tensor, w: torch.Tensor, w_kmajor: bool = True, out: torch.Tensor | None = None,
         residual: torch.Tensor | None = None) -> torch.Tensor:
    """out[M][N] = a[M][K] @ (w.T if w_kmajor else w) (+ residual), bf16, tcgen05."""
    M, K = a.shape
    N = w.shape[0] if w_kmajor else w.shape[1]
    if (w.shape[1] if w_kmajor else w.shape[0]) != K:
        raise ValueError(f"gemm: weight {tuple(w.shape)} does not match K={K}")
    _on_current_device(a, "a")
    if out is None:
        out = torch.empty((M, N), dtype=torch.bfloat16, device=a.device)
    _size(out, "out", M * N)
    t = _TIMER.start() if _TIMER else None
    _lib.check(_lib.lib().plora_gemm_bf16(
        _stream(), M, N, K, _need(a, "a"), _need(w, "w"), int(w_kmajor), _need(out, "out"),
        out.stride(0), _need(residual, "residual", allow_none=True)), "plora_gemm_bf16")
    _LAUNCHES[0] += 1
    if t is not None:
        _TIMER.stop("gemm", t, flops=2.0 * M * N * K, detail=f"N{N}K{K}{'k' if w_kmajor else 'mn'}",
                    algo_bytes=2.0 * (M * K + N * K + M * N))
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
    _on_current_device(x, "x")
    _lora_shapes(meta, d, a_sh, hs_out, T)
    _size(bt_sh, "bt_sh", meta.n_adapters * k * meta.rpad64)
    s = _pack(meta)
    if _TIMER is not None:
        shrink(meta, x, a_sh, hs_out)
        linear_expand(meta, x, w, w_kmajor, bt_sh, hs_out, y_out, residual)
        return y_out, hs_out
    _lib.check(_lib.lib().plora_linear_fwd(
        _stream(), ctypes.byref(s), _need(x, "x"), d, k, _need(w, "w"), int(w_kmajor),
        _need(a_sh, "a_sh"), _need(bt_sh, "bt_sh"), _need(hs_out, "hs_out"), _need(y_out, "y"),
        y_out.stride(0), _need(residual, "residual", allow_none=True)), "plora_linear_fwd")
    _LAUNCHES[0] += 2
    return y_out, hs_out


def shrink(meta: PackMeta, p: torch.Tensor, l_sh: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """K2a / K4: out = alpha_i * p_i @ L_i  (L_sh [n][K][rpad64])."""
    T, K = p.shape
    _on_current_device(p, "p")
    _lora_shapes(meta, K, l_sh, out, meta.total_tokens)
    t = _TIMER.start() if _TIMER else None
    _lib.check(_lib.lib().plora_lora_shrink(_stream(), ctypes.byref(_pack(meta)), K, _need(p, "p"),
                                            _need(l_sh, "l_sh"), _need(out, "out")), "plora_lora_shrink")
    _LAUNCHES[0] += 1
    if t is not None:
        tr, R = _lora_work(meta)
        _TIMER.stop("shrink", t, flops=2.0 * K * tr, nbytes=2.0 * T * K + 2.0 * K * R + 2.0 * tr, detail=f"K{K}")
    return out


def segred(meta: PackMeta, p: torch.Tensor, q: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    """K3 / K5: G_i = p_i^T q_i per token segment, fp32 into the adapter-major region g."""
    T, Mdim = p.shape
    _on_current_device(p, "p")
    _size(q, "q", meta.total_tokens * meta.rpad64)
    _size(g, "g", Mdim * meta.rpad16_total)
    t = _TIMER.start() if _TIMER else None
    _lib.check(_lib.lib().plora_lora_segred(_stream(), ctypes.byref(_pack(meta)), Mdim, _need(p, "p"),
                                            _need(q, "q"), _need(g, "g", torch.float32)), "plora_lora_segred")
    _LAUNCHES[0] += 1
    if t is not None:
        tr, R = _lora_work(meta)
        _TIMER.stop("segred", t, flops=2.0 * Mdim * tr, nbytes=2.0 * T * Mdim + 2.0 * tr + 4.0 * Mdim * R,
                    detail=f"M{Mdim}")
    return g


_DUAL_WS: dict = {}


def _dual_workspace(nbytes: int) -> torch.Tensor:
    """Partials workspace of the fused K3 + K4 pass for the current (device, stream), grown
    to the largest request (no zero-fill needed; launches on one stream are ordered)."""
    dev = torch.cuda.current_device()
    key = (dev, torch.cuda.current_stream().cuda_stream)
    ws = _DUAL_WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=f"cuda:{dev}")
        _DUAL_WS[key] = ws
    return ws


def _h_rpad(meta: PackMeta):
    if not hasattr(meta, "_h_rpad_c"):
        meta._h_rpad_c = np.ascontiguousarray(meta.rpad_off, dtype=np.int32)
    return meta._h_rpad_c.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def lora_dual(meta: PackMeta, dy, bt_sh, hs, dh_out, g):
    """K4 + K3 in one pass over dY (reference lorapack.py:224-225) for one target or a list of
    up to 3 targets of the pack (one launch): dh_out[t] = alpha_i dY[t]_i B[t]_i^T (bf16
    [T][rpad64]) and, where g[t] is given, the dB_i^T grad region = Hs[t]_i^T dY[t]_i (fp32).
    Packs a time model expects to run faster as separate passes run the separate K4 / K3
    kernels (plora_lora_dual)."""
    multi = isinstance(dy, (list, tuple))
    dys, bts, hss, dhs, gs = ([x] for x in (dy, bt_sh, hs, dh_out, g)) if not multi else \
        (list(dy), list(bt_sh), list(hs), list(dh_out), list(g))
    n_t = len(dys)
    if not 1 <= n_t <= 3 or not all(len(x) == n_t for x in (bts, hss, dhs, gs)):
        raise ValueError("lora_dual: 1..3 targets with one dy, bt_sh, hs, dh_out, g each")
    T = dys[0].shape[0]
    ks = []
    for dy_t, bt_t, hs_t, dh_t, g_t in zip(dys, bts, hss, dhs, gs):
        k = dy_t.shape[1]
        ks.append(k)
        _on_current_device(dy_t, "dy")
        _lora_shapes(meta, k, bt_t, dh_t, meta.total_tokens)
        if g_t is not None:
            _size(hs_t, "hs", meta.total_tokens * meta.rpad64)
            _size(g_t, "g", k * meta.rpad16_total)
    s = _pack(meta)
    rp = _h_rpad(meta)
    karr = (ctypes.c_int64 * n_t)(*ks)
    need = int(_lib.lib().plora_lora_dual_workspace_bytes(ctypes.byref(s), n_t, karr, rp))
    ws = _dual_workspace(need) if need > 0 else None
    yp, _k1 = _ptr_array(dys, "dy")
    bp, _k2 = _ptr_array(bts, "bt_sh")
    hp = (ctypes.c_void_p * n_t)(*[_need(h, "hs", allow_none=gt is None) for h, gt in zip(hss, gs)])
    op, _k3 = _ptr_array(dhs, "dh_out")
    gp = (ctypes.c_void_p * n_t)(*[_need(gt, "g", torch.float32, allow_none=True) for gt in gs])
    t = _TIMER.start() if _TIMER else None
    _lib.check(_lib.lib().plora_lora_dual(_stream(), ctypes.byref(s), n_t, karr, rp, yp, bp,
                                          ctypes.cast(hp, ctypes.POINTER(ctypes.c_void_p)), op,
                                          ctypes.cast(gp, ctypes.POINTER(ctypes.c_void_p)),
                                          ws.data_ptr() if ws is not None else None, need),
               "plora_lora_dual")
    _LAUNCHES[0] += 2 if need > 0 else sum(1 + (gt is not None) for gt in gs)
    if t is not None:
        tr, R = _lora_work(meta)
        ksum = float(sum(ks))
        if need > 0:
            _TIMER.stop("dual", t, flops=4.0 * ksum * tr, nbytes=2.0 * T * ksum + n_t * 4.0 * tr + 6.0 * ksum * R,
                        detail="K" + "+".join(str(k) for k in ks))
        else:   # separate K4 + K3 launches: both passes' algorithmic bytes
            _TIMER.stop("dual", t, flops=4.0 * ksum * tr, nbytes=4.0 * T * ksum + n_t * 6.0 * tr + 6.0 * ksum * R,
                        detail="K" + "+".join(str(k) for k in ks) + "sep")
    return dh_out


def swiglu_bwd_segred(meta: PackMeta, d_act: torch.Tensor, g: torch.Tensor, u: torch.Tensor, dh: torch.Tensor,
                      grad_a: torch.Tensor, out_g: torch.Tensor | None = None,
                      out_u: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """SwiGLU backward fused with the down projection's dA (K5, reference lorapack.py:226 on
    act = silu(g) u): returns (dg, du) (may alias g / u) and writes dA_i = act_i^T dH_i into
    grad_a; act is formed on chip and never stored (plora_swiglu_bwd_segred)."""
    T, ffn = g.shape
    _on_current_device(g, "g")
    for t_, nm in ((d_act, "d_act"), (u, "u")):
        if t_.shape != g.shape:
            raise ValueError(f"{nm} must have the shape of g {tuple(g.shape)}")
    _size(dh, "dh", meta.total_tokens * meta.rpad64)
    _size(grad_a, "grad_a", ffn * meta.rpad16_total)
    dg = torch.empty_like(g) if out_g is None else out_g
    du = torch.empty_like(u) if out_u is None else out_u
    t = _TIMER.start() if _TIMER else None
    _lib.check(_lib.lib().plora_swiglu_bwd_segred(
        _stream(), ctypes.byref(_pack(meta)), ffn, _need(d_act, "d_act"), _need(g, "g"), _need(u, "u"),
        _need(dh, "dh"), _need(dg, "dg"), _need(du, "du"), _need(grad_a, "grad_a", torch.float32)),
        "plora_swiglu_bwd_segred")
    _LAUNCHES[0] += 1
    if t is not None:
        tr, R = _lora_work(meta)
        _TIMER.stop("swiglu_segred", t, flops=2.0 * ffn * tr, nbytes=10.0 * T * ffn + 2.0 * tr + 4.0 * ffn * R,
                    detail=f"M{ffn}")
    return dg, du


def _ptr_array(ts, name, dtype=torch.bfloat16):
    arr = (ctypes.c_void_p * len(ts))(*[_need(t, f"{name}[{j}]", dtype) for j, t in enumerate(ts)])
    return ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p)), arr


def shrink_multi(meta: PackMeta, p: torch.Tensor, l_shs, outs) -> list:
    """K2a for targets sharing the input p (q/k/v or gate/up): outs[j] = alpha_i p_i L_j,i,
    p read once (one launch when every rank <= 64)."""
    T, K = p.shape
    _on_current_device(p, "p")
    for j, (l_sh, out) in enumerate(zip(l_shs, outs)):
        _lora_shapes(meta, K, l_sh, out, meta.total_tokens)
    t = _TIMER.start() if _TIMER else None
    lp, _k1 = _ptr_array(l_shs, "l_sh")
    op, _k2 = _ptr_array(outs, "out")
    _lib.check(_lib.lib().plora_lora_shrink_multi(_stream(), ctypes.byref(_pack(meta)), K, _need(p, "p"),
                                                  len(outs), lp, op), "plora_lora_shrink_multi")
    _LAUNCHES[0] += 1 if meta.nb == 1 else len(outs)
    if t is not None:
        tr, R = _lora_work(meta)
        m = len(outs)
        _TIMER.stop("shrink", t, flops=2.0 * K * tr * m, nbytes=2.0 * T * K + m * (2.0 * K * R + 2.0 * tr),
                    detail=f"K{K}x{m}")
    return outs


def segred_multi(meta: PackMeta, p: torch.Tensor, qs, gs) -> list:
    """K5 for targets sharing p: G_j,i = p_i^T Q_j,i (fp32, adapter-major regions), p read once."""
    T, Mdim = p.shape
    _on_current_device(p, "p")
    for q, g in zip(qs, gs):
        _size(q, "q", meta.total_tokens * meta.rpad64)
        _size(g, "g", Mdim * meta.rpad16_total)
    t = _TIMER.start() if _TIMER else None
    qp, _k1 = _ptr_array(qs, "q")
    gp, _k2 = _ptr_array(gs, "g", torch.float32)
    _lib.check(_lib.lib().plora_lora_segred_multi(_stream(), ctypes.byref(_pack(meta)), Mdim, _need(p, "p"),
                                                  len(gs), qp, gp), "plora_lora_segred_multi")
    _LAUNCHES[0] += 1 if meta.nb == 1 else len(gs)
    if t is not None:
        tr, R = _lora_work(meta)
        m = len(gs)
        _TIMER.stop("segred", t, flops=2.0 * Mdim * tr * m, nbytes=2.0 * T * Mdim + m * (2.0 * tr + 4.0 * Mdim * R),
                    detail=f"M{Mdim}x{m}")
    return gs


def linear_expand_group(meta: PackMeta, x: torch.Tensor, ws, bt_shs, hss, w_kmajor: bool = True,
                        biases=None, y_outs=None) -> list:
    """K1 + K2b for targets sharing x (q/k/v, gate/up) in ONE pair-GEMM launch:
    y_j = x op(W_j) + Hs_j,i B_j,i (+ bias_j, in the epilogue) (returns the new y_j [T][k_j])."""
    T, d = x.shape
    _on_current_device(x, "x")
    ks = [w.shape[0] if w_kmajor else w.shape[1] for w in ws]
    for k, bt, hs in zip(ks, bt_shs, hss):
        _size(bt, "bt_sh", meta.n_adapters * k * meta.rpad64)
        _size(hs, "hs", T * meta.rpad64)
    ys = list(y_outs) if y_outs is not None else [torch.empty((T, k), dtype=torch.bfloat16, device=x.device)
                                                   for k in ks]
    karr = (ctypes.c_int64 * len(ks))(*ks)
    t = _TIMER.start() if _TIMER else None
    wp, _k1 = _ptr_array(ws, "w")
    bp, _k2 = _ptr_array(bt_shs, "bt_sh")
    hp, _k3 = _ptr_array(hss, "hs")
    yp, _k4 = _ptr_array(ys, "y")
    if biases is not None:
        barr = (ctypes.c_void_p * len(ws))(*[None if b is None else _need(b, f"bias[{j}]") for j, b in
                                             enumerate(biases)])
        bip = ctypes.cast(barr, ctypes.POINTER(ctypes.c_void_p))
    else:
        bip = None
    _lib.check(_lib.lib().plora_linear_expand_group(_stream(), ctypes.byref(_pack(meta)), _need(x, "x"), d, len(ws),
                                                    karr, wp, int(w_kmajor), bp, hp, yp, bip),
               "plora_linear_expand_group")
    _LAUNCHES[0] += 1
    if t is not None:
        tr, R = _lora_work(meta)
        _TIMER.stop("gemm", t, flops=sum(2.0 * T * d * k + 2.0 * k * tr for k in ks),
                    detail="grp" + "+".join(f"N{k}" for k in ks) + f"K{d}{'k' if w_kmajor else 'mn'}",
                    algo_bytes=2.0 * (T * d + sum(k * d + T * k + T * meta.rpad64 for k in ks)))
    return ys


def linear_gate_up_swiglu(meta: PackMeta, x: torch.Tensor, w_gate: torch.Tensor, w_up: torch.Tensor,
                          bt_gate: torch.Tensor, bt_up: torch.Tensor, hs_gate: torch.Tensor, hs_up: torch.Tensor,
                          outs=None):
    """gate/up K1+K2b in one launch with the SwiGLU forward in the epilogue: returns
    (g, u, act), act = silu(g) u bit-identical to elementwise.swiglu_fwd(g, u)."""
    T, d = x.shape
    ffn = w_gate.shape[0]
    _on_current_device(x, "x")
    for nm, t_ in (("bt_gate", bt_gate), ("bt_up", bt_up)):
        _size(t_, nm, meta.n_adapters * ffn * meta.rpad64)
    for nm, t_ in (("hs_gate", hs_gate), ("hs_up", hs_up)):
        _size(t_, nm, T * meta.rpad64)
    if outs is not None:
        g, u, act = outs
    else:
        g = torch.empty((T, ffn), dtype=torch.bfloat16, device=x.device)
        u = torch.empty_like(g)
        act = torch.empty_like(g)
    t = _TIMER.start() if _TIMER else None
    _lib.check(_lib.lib().plora_linear_gate_up_swiglu(
        _stream(), ctypes.byref(_pack(meta)), _need(x, "x"), d, ffn, _need(w_gate, "w_gate"), _need(w_up, "w_up"),
        _need(bt_gate, "bt_gate"), _need(bt_up, "bt_up"), _need(hs_gate, "hs_gate"), _need(hs_up, "hs_up"),
        _need(g, "g"), _need(u, "u"), _need(act, "act")), "plora_linear_gate_up_swiglu")
    _LAUNCHES[0] += 1
    if t is not None:
        tr, R = _lora_work(meta)
        _TIMER.stop("gemm", t, flops=2 * (2.0 * T * d * ffn + 2.0 * ffn * tr), detail=f"gateup+swiglu N{ffn}K{d}k",
                    algo_bytes=2.0 * (T * d + 2 * ffn * d + 3 * T * ffn + 2 * T * meta.rpad64))
    return g, u, act


def linear_dx_group(meta: PackMeta, dys, ws, a_shs, dhs, d: int, w_kmajor: bool = True,
                    dx_out: torch.Tensor | None = None, dx_residual: torch.Tensor | None = None) -> torch.Tensor:
    """K6 for targets sharing an input: dx = sum_j dy_j op(W_j)^T + dH_j A_j^T in ONE launch
    (one fp32 accumulator over the concatenated K range)."""
    T = dys[0].shape[0]
    ks = [dy.shape[1] for dy in dys]
    _on_current_device(dys[0], "dy")
    for a_sh, dh in zip(a_shs, dhs):
        _size(a_sh, "a_sh", meta.n_adapters * d * meta.rpad64)
        _size(dh, "dh", T * meta.rpad64)
    if dx_out is None:
        dx_out = torch.empty((T, d), dtype=torch.bfloat16, device=dys[0].device)
    karr = (ctypes.c_int64 * len(ks))(*ks)
    t = _TIMER.start() if _TIMER else None
    yp, _k1 = _ptr_array(dys, "dy")
    wp, _k2 = _ptr_array(ws, "w")
    ap, _k3 = _ptr_array(a_shs, "a_sh")
    hp, _k4 = _ptr_array(dhs, "dh")
    _lib.check(_lib.lib().plora_linear_dx_group(_stream(), ctypes.byref(_pack(meta)), len(dys), yp, karr, wp,
                                                int(w_kmajor), ap, hp, d, _need(dx_out, "dx"), dx_out.stride(0),
                                                _need(dx_residual, "dx_residual", allow_none=True)),
               "plora_linear_dx_group")
    _LAUNCHES[0] += 1
    if t is not None:
        tr, R = _lora_work(meta)
        _TIMER.stop("gemm", t, flops=sum(2.0 * T * d * k + 2.0 * d * tr for k in ks),
                    detail="grp" + "+".join(f"K{k}" for k in ks) + f"N{d}{'mn' if w_kmajor else 'k'}",
                    algo_bytes=2.0 * (T * d + sum(T * k + k * d + T * meta.rpad64 for k in ks)))
    return dx_out


def linear_expand(meta: PackMeta, x: torch.Tensor, w: torch.Tensor, w_kmajor: bool,
                  bt_sh: torch.Tensor, hs: torch.Tensor, y_out: torch.Tensor | None = None,
                  residual: torch.Tensor | None = None) -> torch.Tensor:
    """K1 + K2b with a caller-provided Hs: y = x op(W) + Hs_i B_i (+ residual)."""
    T, d = x.shape
    k = w.shape[0] if w_kmajor else w.shape[1]
    if y_out is None:
        y_out = torch.empty((T, k), dtype=torch.bfloat16, device=x.device)
    _on_current_device(x, "x")
    _size(bt_sh, "bt_sh", meta.n_adapters * k * meta.rpad64)
    _size(hs, "hs", T * meta.rpad64)
    s = _pack(meta)
    t = _TIMER.start() if _TIMER else None
    _lib.check(_lib.lib().plora_linear_expand(
        _stream(), ctypes.byref(s), _need(x, "x"), d, k, _need(w, "w"), int(w_kmajor),
        _need(bt_sh, "bt_sh"), _need(hs, "hs"), _need(y_out, "y"), y_out.stride(0),
        _need(residual, "residual", allow_none=True)), "plora_linear_expand")
    _LAUNCHES[0] += 1
    if t is not None:
        tr, R = _lora_work(meta)
        _TIMER.stop("gemm", t, flops=2.0 * T * d * k + 2.0 * k * tr, detail=f"N{k}K{d}{'k' if w_kmajor else 'mn'}",
                    algo_bytes=2.0 * (T * d + k * d + T * k + T * meta.rpad64) + (2.0 * T * k if residual is not None
                                                                                 else 0.0))
    return y_out


def linear_bwd(meta: PackMeta, x: torch.Tensor, w: torch.Tensor, w_kmajor: bool,
               a_sh: torch.Tensor, bt_sh: torch.Tensor, hs: torch.Tensor, dy: torch.Tensor,
               grad_a: torch.Tensor | None, grad_b: torch.Tensor | None,
               dx_out: torch.Tensor | None = None, need_dx: bool = True,
               dh_ws: torch.Tensor | None = None, dx_residual: torch.Tensor | None = None):
    """Packed LoRA linear backward (Cases 1-4).  Writes fp32 grads into grad_a /
    grad_b (adapter-major regions) and returns dx (or None)."""
    T, d = x.shape
    k = w.shape[0] if w_kmajor else w.shape[1]
    if dh_ws is None:
        dh_ws = torch.empty((T, meta.rpad64), dtype=torch.bfloat16, device=x.device)
    if need_dx and dx_out is None:
        dx_out = torch.empty((T, d), dtype=torch.bfloat16, device=x.device)
    _on_current_device(x, "x")
    _size(a_sh, "a_sh", meta.n_adapters * d * meta.rpad64)
    _size(bt_sh, "bt_sh", meta.n_adapters * k * meta.rpad64)
    _size(hs, "hs", T * meta.rpad64)
    _size(dh_ws, "dh_ws", T * meta.rpad64)
    _size(dy, "dy", T * k)
    _size(grad_a, "grad_a", d * meta.rpad16_total)
    _size(grad_b, "grad_b", k * meta.rpad16_total)
    s = _pack(meta)
    if _TIMER is not None:
        shrink(meta, dy, bt_sh, dh_ws)                       # Case 2 (K4)
        if grad_b is not None:
            segred(meta, dy, hs, grad_b)                     # Case 1 (K3)
        if grad_a is not None:
            segred(meta, x, dh_ws, grad_a)                   # Case 3 (K5)
        if need_dx:                                          # Case 4 (K6): dX = dY op(W)^T + dH A^T
            linear_expand(meta, dy, w, not w_kmajor, a_sh, dh_ws, dx_out, dx_residual)
        return dx_out if need_dx else None
    _LAUNCHES[0] += 1 + (grad_a is not None) + (grad_b is not None) + bool(need_dx)
    _lib.check(_lib.lib().plora_linear_bwd(
        _stream(), ctypes.byref(s), _need(x, "x"), d, k, _need(w, "w"), int(w_kmajor),
        _need(a_sh, "a_sh"), _need(bt_sh, "bt_sh"), _need(hs, "hs"), _need(dy, "dy"),
        _need(dh_ws, "dh_ws"), _need(dx_out, "dx", allow_none=True) if need_dx else None,
        dx_out.stride(0) if (need_dx and dx_out is not None) else 0,
        _need(dx_residual, "dx_residual", allow_none=True) if need_dx else None,
        _need(grad_a, "grad_a", torch.float32, allow_none=True),
        _need(grad_b, "grad_b", torch.float32, allow_none=True)), "plora_linear_bwd")
    return dx_out if need_dx else None


def adamw(chunks: torch.Tensor, param: torch.Tensor, grad: torch.Tensor, exp_avg: torch.Tensor,
          exp_avg_sq: torch.Tensor, shadow: torch.Tensor, hp: torch.Tensor, step: int,
          beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, algo_params: int | None = None) -> None:
    """Fused per-adapter AdamW over the chunk table (see include/plora.h)."""
    _LAUNCHES[0] += 1
    t = _TIMER.start() if _TIMER else None
    _lib.check(_lib.lib().plora_adamw(
        _stream(), chunks.shape[0], _need(chunks, "chunks", torch.int64),
        _need(param, "param", torch.float32), _need(grad, "grad", torch.float32),
        _need(exp_avg, "exp_avg", torch.float32), _need(exp_avg_sq, "exp_avg_sq", torch.float32),
        _need(shadow, "shadow"), _need(hp, "hp", torch.float32), beta1, beta2, eps, int(step)),
        "plora_adamw")
    if t is not None:
        # 30 B per trainable parameter: read p,g,m,v (16) + write p,m,v (12) + bf16 shadow (2)
        _TIMER.stop("adamw", t, nbytes=30.0 * (algo_params if algo_params is not None else param.numel()),
                    detail="K7")


# ------------------------------------------------------------------ torch training op
class PackedLoraLinearFn(torch.autograd.Function):
    """Autograd op over plora_linear_fwd / plora_linear_bwd: the training form of the
    reference ``packed_forward`` / ``packed_backward`` (lorapack.py:183-231).

    Differentiable inputs: ``x`` [T][d] bf16 (tokens adapter-major, segments of ``meta``)
    and the fp32 LoRA masters in the region layout the kernels write gradients into
    (adapters.py): ``a_master`` = A_i [d][rpad16_i] blocks, ``b_master`` = B_i^T
    [k][rpad16_i] blocks, back to back.  The forward reads their bf16 shadows
    ``a_sh`` [n][d][64nb] / ``bt_sh`` [n][k][64nb] (kept equal to the masters by the
    caller, see PackedLoraLinear).  Saved for the backward: x and Hs = alpha_i X_i A_i
    (the reference recomputes ``hidden``, :216; here it is kept from the forward)."""

    @staticmethod
    def forward(ctx, x, a_master, b_master, meta, w, a_sh, bt_sh, w_kmajor=True):
        y, hs = linear_fwd(meta, x, w, w_kmajor, a_sh, bt_sh)
        ctx.save_for_backward(x, hs)
        ctx.meta, ctx.w, ctx.a_sh, ctx.bt_sh, ctx.w_kmajor = meta, w, a_sh, bt_sh, w_kmajor
        ctx.shapes = (a_master.shape, b_master.shape)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, hs = ctx.saved_tensors
        need_x, need_a, need_b = ctx.needs_input_grad[:3]
        dev = x.device
        ga = torch.empty(ctx.shapes[0], dtype=torch.float32, device=dev) if need_a else None
        gb = torch.empty(ctx.shapes[1], dtype=torch.float32, device=dev) if need_b else None
        dx = linear_bwd(ctx.meta, x, ctx.w, ctx.w_kmajor, ctx.a_sh, ctx.bt_sh, hs, dy.contiguous(), ga, gb,
                        need_dx=need_x)
        return dx, ga, gb, None, None, None, None, None


class PackedLoraLinear(torch.nn.Module):
    """A frozen bf16 base projection with n packed LoRA adapters (heterogeneous rank and
    alpha) over token segments: y_t = x_t W^T + alpha_i (x_t A_i) B_i for token t of
    adapter i.  Parameters ``a`` / ``b`` are the fp32 masters (region layout); any torch
    optimizer may update them -- the bf16 shadows are refreshed before the next forward
    when a parameter's version changed.  ``weight`` is nn.Linear-layout [k][d] bf16."""

    def __init__(self, meta: PackMeta, weight: torch.Tensor, init_std: float = 0.02, seed: int = 0):
        super().__init__()
        dev = weight.device
        self.meta = meta.to(dev)
        k, d = weight.shape
        self.d, self.k = d, k
        self.register_buffer("weight", weight.detach().to(torch.bfloat16).contiguous(), persistent=False)
        R16, R64, n = meta.rpad16_total, meta.rpad64, meta.n_adapters
        g = torch.Generator(device=dev).manual_seed(seed)
        a = torch.zeros(d * R16, dtype=torch.float32, device=dev)
        b = torch.zeros(k * R16, dtype=torch.float32, device=dev)
        self.a = torch.nn.Parameter(a)
        self.b = torch.nn.Parameter(b)
        for i in range(n):
            r = meta.ranks[i]
            self.block("a", i)[:, :r] = (torch.rand(d, r, generator=g, device=dev) * 2 - 1) / d ** 0.5
            self.block("b", i)[:, :r] = torch.randn(k, r, generator=g, device=dev) * init_std
        self.register_buffer("a_sh", torch.zeros((n, d, R64), dtype=torch.bfloat16, device=dev), persistent=False)
        self.register_buffer("bt_sh", torch.zeros((n, k, R64), dtype=torch.bfloat16, device=dev), persistent=False)
        self._versions = None

    def block(self, which: str, i: int) -> torch.Tensor:
        """Adapter i's fp32 block: A_i [d][rpad16_i] ("a") or B_i^T [k][rpad16_i] ("b")."""
        p, rows = (self.a, self.d) if which == "a" else (self.b, self.k)
        ro = self.meta.rpad_off
        return p.data[rows * int(ro[i]): rows * int(ro[i + 1])].view(rows, int(ro[i + 1] - ro[i]))

    def down(self, i: int) -> torch.Tensor:
        """Reference-layout A_i (d x r)."""
        return self.block("a", i)[:, : self.meta.ranks[i]]

    def up(self, i: int) -> torch.Tensor:
        """Reference-layout B_i (r x k)."""
        return self.block("b", i)[:, : self.meta.ranks[i]].t()

    @torch.no_grad()
    def refresh_shadows(self) -> None:
        for i in range(self.meta.n_adapters):
            rp = int(self.meta.rpad_off[i + 1] - self.meta.rpad_off[i])
            self.a_sh[i, :, :rp] = self.block("a", i).to(torch.bfloat16)
            self.bt_sh[i, :, :rp] = self.block("b", i).to(torch.bfloat16)
        self._versions = (self.a._version, self.b._version)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if self._versions != (self.a._version, self.b._version):
            self.refresh_shadows()
        return PackedLoraLinearFn.apply(x, self.a, self.b, self.meta, self.weight, self.a_sh, self.bt_sh, True)
