"""Drop-in for ``lorasweep.lorapack`` backed by the sm_100a kernels.

Same public names, argument order, return structure and ``ValueError`` message
substrings as the reference module (pkg/src/lorasweep/lorapack.py:31-42):

    AdapterWeights, PackedAdapters, GradCheckReport, pack_adapters,
    unpack_adapters, adapter_forward, adapter_backward, packed_forward,
    packed_backward, grad_check

Arrays go in and come out as numpy (the reference's contract); in between they
live on the current CUDA device as bf16 operands with fp32 accumulation, and
every contraction runs in libplora (tcgen05 GEMM + fused LoRA expand, segmented
shrink and token-segment reductions).  Offsets are exact Python ints produced
by the C++ segment-index builder and compare equal to the reference's.

Numerics: the reference is float64; this path computes in bf16 with fp32
accumulation, so results match the reference within the bf16 tier stated in
DESIGN.md (relative Frobenius error <= 1e-2, max-abs/max-ref <= 2e-2), not at
the reference's 1e-12.  Indexing (offsets, slices, round trips) is bit-exact.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from .meta import PackMeta, build_meta

__all__ = [
    "AdapterWeights",
    "PackedAdapters",
    "GradCheckReport",
    "pack_adapters",
    "unpack_adapters",
    "adapter_forward",
    "adapter_backward",
    "packed_forward",
    "packed_backward",
    "grad_check",
]

# bf16 tier; the reference's fp64 value is 1e-5.
GRAD_CHECK_TOLERANCE = 5e-2


@dataclass(frozen=True)
class AdapterWeights:
    """One adapter: down-projection A (d x r), up-projection B (r x k), raw alpha.
    Reference: lorapack.py:47-64."""

    down: np.ndarray
    up: np.ndarray
    alpha: float

    def __post_init__(self):
        if np.ndim(self.down) != 2 or np.ndim(self.up) != 2:
            raise ValueError("adapter projections must be matrices")
        if self.down.shape[1] != self.up.shape[0]:
            raise ValueError(f"rank mismatch: down is {self.down.shape}, up is {self.up.shape}")

    @property
    def rank(self) -> int:
        return self.down.shape[1]


@dataclass(frozen=True)
class PackedAdapters:
    """Concatenated adapter blocks plus offsets.  Reference: lorapack.py:67-125.

    ``down_block`` (d x R), ``up_block`` (R x k), ``inputs`` (T x d) as in the
    reference; ``rank_offsets`` / ``row_offsets`` are tuples of ints.
    """

    down_block: np.ndarray
    up_block: np.ndarray
    inputs: np.ndarray
    alphas: tuple
    rank_offsets: tuple
    row_offsets: tuple
    # device segment index, built once per instance (init=False: ``dataclasses.replace``
    # gives the new instance an empty cache instead of sharing a stale one)
    _meta: list = field(init=False, default_factory=list, repr=False, compare=False)
    _dev: list = field(init=False, default_factory=list, repr=False, compare=False)   # staged device operands

    def __post_init__(self):
        n = len(self.alphas)
        if len(self.rank_offsets) != n + 1 or len(self.row_offsets) != n + 1:
            raise ValueError("offset arrays must have one more entry than adapters")
        ro, so = self.rank_offsets, self.row_offsets
        if any(ro[i] >= ro[i + 1] for i in range(n)):
            raise ValueError("rank offsets must be strictly increasing")
        if any(so[i] > so[i + 1] for i in range(n)):
            raise ValueError("row offsets must be non-decreasing")
        if ro[0] != 0 or ro[-1] != self.down_block.shape[1]:
            raise ValueError("rank offsets must partition the packed rank dimension")
        if so[0] != 0 or so[-1] != self.inputs.shape[0]:
            raise ValueError("row offsets must partition the packed sequence dimension")
        if self.up_block.shape[0] != self.down_block.shape[1]:
            raise ValueError("down/up blocks disagree on the packed rank dimension")
        if self.inputs.shape[1] != self.down_block.shape[0]:
            raise ValueError("inputs and down block disagree on the hidden dimension")

    @property
    def adapter_count(self) -> int:
        return len(self.alphas)

    @property
    def d(self) -> int:
        return self.down_block.shape[0]

    @property
    def k(self) -> int:
        return self.up_block.shape[1]

    def rank_slice(self, i: int) -> slice:
        return slice(self.rank_offsets[i], self.rank_offsets[i + 1])

    def row_slice(self, i: int) -> slice:
        return slice(self.row_offsets[i], self.row_offsets[i + 1])

    def adapter(self, i: int) -> AdapterWeights:
        rs = self.rank_slice(i)
        return AdapterWeights(down=self.down_block[:, rs], up=self.up_block[rs, :], alpha=self.alphas[i])

    def input_slice(self, i: int) -> np.ndarray:
        return self.inputs[self.row_slice(i)]

    # --- device metadata (segment index built by the C++ K8 builder) -------
    def meta(self) -> PackMeta:
        if self._meta:
            m = self._meta[0]
            if (m.alphas != tuple(float(a) for a in self.alphas) or m.rank_offsets != tuple(self.rank_offsets)
                    or m.row_offsets != tuple(self.row_offsets)):
                self._meta.clear()
        if not self._meta:
            ranks = np.diff(self.rank_offsets)
            tokens = np.diff(self.row_offsets)
            m = build_meta(ranks, tokens, self.alphas)
            if m.rank_offsets != tuple(self.rank_offsets) or m.row_offsets != tuple(self.row_offsets):
                raise ValueError("segment index disagrees with the pack offsets")
            self._meta.append(m)
        return self._meta[0]


def pack_adapters(adapters: Sequence[AdapterWeights], inputs: Sequence[np.ndarray]) -> PackedAdapters:
    """Concatenate adapters and their input slices (reference lorapack.py:128-158).
    Offsets come from the C++ segment-index builder (bit-exact prefix sums)."""
    if not adapters:
        raise ValueError("nothing to pack")
    if len(adapters) != len(inputs):
        raise ValueError(f"{len(adapters)} adapters but {len(inputs)} inputs")
    d = adapters[0].down.shape[0]
    k = adapters[0].up.shape[1]
    for i, a in enumerate(adapters):
        if a.down.shape[0] != d or a.up.shape[1] != k:
            raise ValueError(f"adapter {i} has shape ({a.down.shape[0]}, {a.up.shape[1]}), expected ({d}, {k})")
    for i, x in enumerate(inputs):
        if np.ndim(x) != 2 or x.shape[1] != d:
            raise ValueError(f"input {i} must be (tokens, {d}), got {np.shape(x)}")
    meta = build_meta([a.rank for a in adapters], [x.shape[0] for x in inputs],
                      [float(a.alpha) for a in adapters])
    packed = PackedAdapters(
        down_block=np.concatenate([a.down for a in adapters], axis=1),
        up_block=np.concatenate([a.up for a in adapters], axis=0),
        inputs=np.concatenate(list(inputs), axis=0),
        alphas=meta.alphas,
        rank_offsets=meta.rank_offsets,
        row_offsets=meta.row_offsets,
    )
    packed._meta.append(meta)
    return packed


def unpack_adapters(packed: PackedAdapters) -> tuple[list[AdapterWeights], list[np.ndarray]]:
    """Inverse of pack_adapters (reference lorapack.py:161-164)."""
    adapters = [packed.adapter(i) for i in range(packed.adapter_count)]
    inputs = [packed.input_slice(i).copy() for i in range(packed.adapter_count)]
    return adapters, inputs


# ----------------------------------------------------------------- device staging
def _round_up(v: int, m: int) -> int:
    return (v + m - 1) // m * m


def _upload(a: np.ndarray, dev):
    """numpy -> device in the caller's float dtype (converted to bf16 on the device: a host
    fp64 -> fp32 pass over a 4096 x 14336 weight costs more than the PCIe copy itself),
    through a page-locked block of torch's caching host allocator (async DMA; the host
    copy of the next array overlaps it)."""
    import torch

    a = np.asarray(a)
    if a.dtype not in (np.float64, np.float32):
        a = a.astype(np.float64)
    host = torch.empty(a.shape, dtype=torch.float64 if a.dtype == np.float64 else torch.float32, pin_memory=True)
    _copy_parallel(host.numpy(), a)
    return host.to(dev, non_blocking=True)


_POOL = []


def _copy_parallel(dst: np.ndarray, src: np.ndarray, chunk_bytes: int = 8 << 20) -> None:
    """np.copyto split over host threads along the first axis (numpy releases the GIL in
    its copy loops): one thread copies ~5-10 GB/s, the staging of a 4096 x 14336 fp64
    weight into page-locked memory would otherwise cost more than its PCIe transfer."""
    if src.ndim == 0 or src.nbytes <= 2 * chunk_bytes or src.shape[0] < 2:
        np.copyto(dst, src)
        return
    if not _POOL:
        import os
        from concurrent.futures import ThreadPoolExecutor

        _POOL.append(ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 1))))
    pool = _POOL[0]
    parts = min(pool._max_workers * 2, max(1, src.nbytes // chunk_bytes), src.shape[0])
    bounds = np.linspace(0, src.shape[0], parts + 1).astype(int)
    futs = [pool.submit(np.copyto, dst[a:b], src[a:b]) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    for f in futs:
        f.result()


def _fingerprint(a: np.ndarray) -> tuple:
    """Identity of a host array for the staged-weight cache: buffer address, layout and
    a strided sample of up to 4096 values (catches re-filled buffers)."""
    flat = a.reshape(-1) if a.flags.c_contiguous else np.ascontiguousarray(a).reshape(-1)
    step = max(1, flat.size // 4096)
    return (a.__array_interface__["data"][0], a.shape, a.strides, a.dtype.str, flat[::step].tobytes())


class _WeightCache:
    """Staged bf16 base weights, reused while the caller passes the same (unchanged) array
    -- the forward and backward of one pack, or a loop over packs on one frozen base.
    At most two weights stay resident."""

    def __init__(self, size: int = 2):
        self.size = size
        self.entries: list = []   # (weakref to the array, fingerprint, device, staged tensor)

    def get(self, w: np.ndarray, dev, dp: int, kp: int):
        import weakref

        import torch

        fp = _fingerprint(w)
        for e in self.entries:
            ref, efp, edev, t = e
            if ref() is w and efp == fp and edev == dev:
                return t
        t = torch.zeros((dp, kp), dtype=torch.bfloat16, device=dev)   # reference layout [d][k]
        t[: w.shape[0], : w.shape[1]] = _upload(w, dev).to(torch.bfloat16)
        try:
            ref = weakref.ref(w)
        except TypeError:   # not weak-referenceable: never reused
            return t
        self.entries = [e for e in self.entries if e[0]() is not None][-(self.size - 1):] + [(ref, fp, dev, t)]
        return t


_W_CACHE = _WeightCache()


class _Staged:
    """bf16 device operands of one pack (padded for TMA: d, k -> multiples of 64).  Built
    once per PackedAdapters instance (the frozen dataclass's fields never change) and
    kept with it, so packed_backward reuses packed_forward's X, adapters and Hs."""

    def __init__(self, packed: PackedAdapters):
        import torch

        if not torch.cuda.is_available():
            raise _lib.PloraError("no CUDA device: the packed-LoRA operators run only on sm_100a")
        _lib.check(_lib.lib().plora_device_check(), "plora_device_check")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.torch = torch
        self.dev = dev
        self.meta = packed.meta().to(dev)
        m = self.meta
        d, k, T, n = packed.d, packed.k, packed.inputs.shape[0], packed.adapter_count
        self.d, self.k, self.T, self.n = d, k, T, n
        self.dp, self.kp = _round_up(d, 64), _round_up(k, 64)
        bf = torch.bfloat16
        self.x = torch.zeros((T, self.dp), dtype=bf, device=dev)
        if T:
            self.x[:, :d] = _upload(packed.inputs, dev).to(bf)
        R64 = m.rpad64
        self.a_sh = torch.zeros((n, self.dp, R64), dtype=bf, device=dev)
        self.bt_sh = torch.zeros((n, self.kp, R64), dtype=bf, device=dev)
        down = _upload(packed.down_block, dev).to(bf)     # one transfer per block, split on the device
        up_t = _upload(packed.up_block, dev).to(bf).t()
        for i in range(n):
            rs = packed.rank_slice(i)
            r = rs.stop - rs.start
            self.a_sh[i, :d, :r] = down[:, rs]
            self.bt_sh[i, :k, :r] = up_t[:, rs]
        self.hs = None

    @classmethod
    def of(cls, packed: PackedAdapters) -> "_Staged":
        import torch

        dev = torch.cuda.current_device() if torch.cuda.is_available() else None
        st = packed._dev[0] if packed._dev else None
        if st is None or st.dev.index != dev:
            st = cls(packed)
            packed._dev[:] = [st]
        return st

    def hidden(self):
        """Hs = alpha_i X_i A_i (K2a), computed once per pack."""
        from . import ops

        if self.hs is None:
            self.hs = self.torch.empty((self.T, self.meta.rpad64), dtype=self.torch.bfloat16, device=self.dev)
            ops.shrink(self.meta, self.x, self.a_sh, self.hs)
        return self.hs

    def forward(self, w):
        from . import ops

        y = self.torch.empty((self.T, self.kp), dtype=self.torch.bfloat16, device=self.dev)
        ops.linear_expand(self.meta, self.x, w, False, self.bt_sh, self.hidden(), y_out=y)
        return y


def _out_dtype(*arrays) -> np.dtype:
    return np.result_type(*[np.asarray(a).dtype for a in arrays], np.float32)


def _to_host(t, dtype: np.dtype) -> np.ndarray:
    """Device tensor -> numpy in the reference's output dtype: converted on the device and
    DMA'd into page-locked memory from torch's caching host allocator (a pageable D2H of
    a 2048 x 14336 float64 output runs at ~2 GB/s; pinned at PCIe speed).  The returned
    array keeps its pinned block alive; the block is recycled only after it is freed."""
    import torch

    tdt = torch.float64 if dtype == np.float64 else torch.float32
    src = t.to(tdt)
    host = torch.empty(src.shape, dtype=tdt, pin_memory=True)
    host.copy_(src)
    out = host.numpy()
    return out if out.dtype == dtype else out.astype(dtype)


def _staged_weight(packed: PackedAdapters, w_base: np.ndarray, st: _Staged):
    return _W_CACHE.get(np.asarray(w_base), st.dev, st.dp, st.kp)


def packed_forward(packed: PackedAdapters, w_base: np.ndarray) -> list[np.ndarray]:
    """Per-adapter outputs y_i = x_i W + alpha_i (x_i A_i) B_i (reference lorapack.py:183-199).

    One fused launch pair on the GPU: K2a shrink (Hs = alpha X A) then the K1
    tcgen05 base GEMM whose tiles add Hs_i B_i as extra K-steps."""
    if w_base.shape != (packed.d, packed.k):
        raise ValueError(f"base weight must be ({packed.d}, {packed.k}), got {w_base.shape}")
    st = _Staged.of(packed)
    y = st.forward(_staged_weight(packed, w_base, st))
    host = _to_host(y[:, : packed.k], _out_dtype(packed.inputs, w_base))
    return [host[packed.row_slice(i)] for i in range(packed.adapter_count)]


def packed_backward(packed: PackedAdapters, w_base: np.ndarray, upstreams: Sequence[np.ndarray]
                    ) -> tuple[list[np.ndarray], list[np.ndarray], list[np.ndarray]]:
    """Per-adapter (d_down, d_up, d_input) (reference lorapack.py:202-231).

    Hs = alpha X A comes from this pack's forward when it ran (else one K2a shrink: the
    reference recomputes ``hidden = X @ A_all``, :216), then Case 2 (K4 shrink), Case 1
    (K3), Case 3 (K5) segment reductions and Case 4 (K6 GEMM with the LoRA term as extra
    K-steps)."""
    if len(upstreams) != packed.adapter_count:
        raise ValueError(f"{packed.adapter_count} adapters but {len(upstreams)} upstream gradients")
    for i, dy in enumerate(upstreams):
        rows = packed.row_slice(i)
        expected = (rows.stop - rows.start, packed.k)
        if np.shape(dy) != expected:
            raise ValueError(f"upstream {i} must be {expected}, got {np.shape(dy)}")
    if w_base.shape != (packed.d, packed.k):
        raise ValueError(f"base weight must be ({packed.d}, {packed.k}), got {w_base.shape}")
    from . import ops

    st = _Staged.of(packed)
    torch = st.torch
    m = st.meta
    w = _staged_weight(packed, w_base, st)
    hs = st.hidden()
    dy = torch.zeros((st.T, st.kp), dtype=torch.bfloat16, device=st.dev)
    if st.T:
        ups = np.concatenate([np.asarray(u) for u in upstreams], axis=0)
        dy[:, : st.k] = _upload(ups, st.dev).to(torch.bfloat16)
    R16 = m.rpad16_total
    grad_a = torch.empty(st.dp * R16, dtype=torch.float32, device=st.dev)
    grad_b = torch.empty(st.kp * R16, dtype=torch.float32, device=st.dev)
    dx = ops.linear_bwd(m, st.x, w, False, st.a_sh, st.bt_sh, hs, dy, grad_a, grad_b)
    dt = _out_dtype(packed.inputs, w_base, *upstreams)
    ga = _to_host(grad_a, np.float32)
    gb = _to_host(grad_b, np.float32)
    dxh = _to_host(dx[:, : st.d], dt)
    d_downs, d_ups, d_inputs = [], [], []
    for i in range(packed.adapter_count):
        r = packed.rank_offsets[i + 1] - packed.rank_offsets[i]
        rp = int(m.rpad_off[i + 1] - m.rpad_off[i])
        blk_a = ga[st.dp * int(m.rpad_off[i]): st.dp * int(m.rpad_off[i + 1])].reshape(st.dp, rp)
        blk_b = gb[st.kp * int(m.rpad_off[i]): st.kp * int(m.rpad_off[i + 1])].reshape(st.kp, rp)
        d_downs.append(blk_a[: st.d, :r].astype(dt))
        d_ups.append(np.ascontiguousarray(blk_b[: st.k, :r].T).astype(dt))
        d_inputs.append(dxh[packed.row_slice(i)])
    return d_downs, d_ups, d_inputs


def adapter_forward(adapter: AdapterWeights, x: np.ndarray, w_base: np.ndarray) -> np.ndarray:
    """Single adapter y = x W + alpha (x A) B (reference lorapack.py:167-169): a pack of one."""
    return packed_forward(pack_adapters([adapter], [x]), w_base)[0]


def adapter_backward(adapter: AdapterWeights, x: np.ndarray, w_base: np.ndarray,
                     upstream: np.ndarray) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Single adapter (d_down, d_up, d_input) (reference lorapack.py:172-180): a pack of one."""
    dd, du, dx = packed_backward(pack_adapters([adapter], [x]), w_base, [upstream])
    return dd[0], du[0], dx[0]


# ----------------------------------------------------------------- gradient check
@dataclass(frozen=True)
class GradCheckReport:
    """Max relative finite-difference error per gradient case (reference lorapack.py:237-256)."""

    case_errors: dict
    tolerance: float

    @property
    def max_rel_error(self) -> float:
        return max(self.case_errors.values())

    @property
    def passed(self) -> bool:
        return self.max_rel_error < self.tolerance


def _rel_err(analytic: np.ndarray, numeric: np.ndarray) -> float:
    if analytic.size == 0:
        return 0.0
    scale = np.maximum(np.maximum(np.abs(analytic), np.abs(numeric)), 1.0)
    return float(np.max(np.abs(analytic - numeric) / scale))


def grad_check(packed: PackedAdapters, w_base: np.ndarray, seed: int = 0, step: float = 4.0,
               tolerance: float = GRAD_CHECK_TOLERANCE) -> GradCheckReport:
    """Finite-difference check of the GPU gradients (reference lorapack.py:279-340).

    The scalar loss is sum_i <dY_i, y_i> for a seeded random upstream.  It is
    linear in each of B, A, X and H separately, so central differences are exact
    for any step; each perturbed forward runs on the device (the perturbed bf16
    operand is edited in place, the denominator uses the bf16-rounded step) and
    the default tolerance is the bf16 tier.  Cases and the relative error with an
    absolute floor of 1 follow the reference.  Desk-scale packs only."""
    from . import ops

    rng = np.random.default_rng(seed)
    n = packed.adapter_count
    ups = [rng.standard_normal((packed.row_offsets[i + 1] - packed.row_offsets[i], packed.k))
           for i in range(n)]
    d_downs, d_ups, d_inputs = packed_backward(packed, w_base, ups)

    st = _Staged(packed)          # a private copy: its operands are perturbed in place below
    torch = st.torch
    m = st.meta
    w = _staged_weight(packed, w_base, st)
    dy = torch.zeros((st.T, st.kp), dtype=torch.float64, device=st.dev)
    if st.T:
        dy[:, : st.k] = torch.from_numpy(np.concatenate(ups, axis=0)).to(st.dev)
    hs = st.hidden()
    hs_pert = torch.empty_like(hs)
    y = torch.empty((st.T, st.kp), dtype=torch.bfloat16, device=st.dev)

    def loss(hs_t) -> float:
        ops.linear_expand(m, st.x, w, False, st.bt_sh, hs_t, y_out=y)
        return float((y.double() * dy).sum().item())

    def fd(tensor, index, recompute_hs: bool) -> float:
        orig = tensor[index].clone()
        vals, pos = [], []
        for sgn in (1.0, -1.0):
            tensor[index] = (orig.double() + sgn * step).to(tensor.dtype)
            pos.append(float(tensor[index].double().item()))
            h = ops.shrink(m, st.x, st.a_sh, hs_pert) if recompute_hs else hs
            vals.append(loss(h))
        tensor[index] = orig
        if pos[0] == pos[1]:
            raise ValueError(f"grad_check step {step} vanishes in the bf16 operands (no representable "
                             f"perturbation of {float(orig.double().item())}); use a larger step")
        return (vals[0] - vals[1]) / (pos[0] - pos[1])

    errs = {}
    num_up = np.empty_like(packed.up_block, dtype=np.float64)
    num_down = np.empty_like(packed.down_block, dtype=np.float64)
    for i in range(n):
        rs = packed.rank_slice(i)
        for j in range(rs.stop - rs.start):
            for c in range(packed.k):
                num_up[rs.start + j, c] = fd(st.bt_sh, (i, c, j), False)
            for r in range(packed.d):
                num_down[r, rs.start + j] = fd(st.a_sh, (i, r, j), True)
    num_x = np.empty_like(packed.inputs, dtype=np.float64)
    for t in range(st.T):
        for c in range(packed.d):
            num_x[t, c] = fd(st.x, (t, c), True)
    errs["up_weight"] = _rel_err(np.concatenate(d_ups, axis=0), num_up)
    errs["down_weight"] = _rel_err(np.concatenate(d_downs, axis=1), num_down)
    errs["down_input"] = _rel_err(np.concatenate(d_inputs, axis=0), num_x)

    # Case 2: gradient w.r.t. the hidden activations H_i (an intermediate).  The
    # analytic value is the K4 output dH = alpha_i dY_i B_i^T; the numeric one
    # perturbs H (i.e. Hs = alpha H) and re-runs the fused expand GEMM.
    dyb = torch.zeros((st.T, st.kp), dtype=torch.bfloat16, device=st.dev)
    dyb.copy_(dy.to(torch.bfloat16))
    dh = torch.empty((st.T, m.rpad64), dtype=torch.bfloat16, device=st.dev)
    ops.linear_bwd(m, st.x, w, False, st.a_sh, st.bt_sh, hs, dyb, None, None, need_dx=False,
                   dh_ws=dh)
    an_h = dh.float().cpu().numpy()
    worst = 0.0
    for i in range(n):
        rows = packed.row_slice(i)
        r = packed.rank_offsets[i + 1] - packed.rank_offsets[i]
        alpha = packed.alphas[i]
        for t in range(rows.start, rows.stop):
            for j in range(r):
                if alpha == 0.0:
                    num = 0.0
                else:
                    orig = hs[t, j].clone()
                    vals, pos = [], []
                    for sgn in (1.0, -1.0):
                        hs[t, j] = (orig.double() + sgn * alpha * step).to(hs.dtype)
                        pos.append(float(hs[t, j].double().item()) / alpha)
                        vals.append(loss(hs))
                    hs[t, j] = orig
                    if pos[0] == pos[1]:
                        raise ValueError(f"grad_check step {step} vanishes in the bf16 hidden activations")
                    num = (vals[0] - vals[1]) / (pos[0] - pos[1])
                worst = max(worst, _rel_err(np.array([an_h[t, j]]), np.array([num])))
    errs["up_input"] = worst
    ordered = {key: errs[key] for key in ("up_weight", "up_input", "down_weight", "down_input")}
    return GradCheckReport(case_errors=ordered, tolerance=tolerance)
