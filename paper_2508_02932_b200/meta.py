"""Segment-index / adapter-metadata builder (K8) -- host side of the pack.

Mirrors the offset bookkeeping of the reference ``pack_adapters``
(pkg/src/lorasweep/lorapack.py:146-150): ``rank_offsets`` and ``row_offsets``
are exact integer prefix sums, returned as tuples of Python ints so they compare
equal (bit-exactly) to the reference's.  The arithmetic runs in the C++ builder
behind the C-ABI (``plora_meta_build``, csrc/meta.cpp); this module only
marshals arrays and uploads the device copy the kernels read.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib


@dataclass
class PackMeta:
    """Host + device description of one pack (n adapters over T packed tokens)."""

    ranks: tuple[int, ...]
    tokens: tuple[int, ...]
    alphas: tuple[float, ...]
    rank_offsets: tuple[int, ...]
    row_offsets: tuple[int, ...]
    rpad_off: np.ndarray          # int32 [n+1], prefix sums of roundup(r_i, 16)
    mtiles: np.ndarray            # int32 [n_mtiles, 4]
    ptiles: np.ndarray            # int32 [n_ptiles, 4]  (256-row CTA-pair tiles)
    token_adapter: np.ndarray     # int32 [T]
    nb: int                       # 64-column rank blocks in the bf16 shadows
    device: object = None
    _dev: dict = field(default_factory=dict, repr=False)
    _struct: _lib.PackStruct | None = field(default=None, repr=False)

    @property
    def n_adapters(self) -> int:
        return len(self.ranks)

    @property
    def total_tokens(self) -> int:
        return self.row_offsets[-1]

    @property
    def rpad64(self) -> int:
        return 64 * self.nb

    @property
    def rpad16(self) -> np.ndarray:
        return np.diff(self.rpad_off).astype(np.int64)

    @property
    def rpad16_total(self) -> int:
        return int(self.rpad_off[-1])

    def to(self, device) -> "PackMeta":
        """Upload the device copy (int tables + alphas) and build the plora_pack_t."""
        import torch

        device = torch.device(device)
        if self.device is not None and torch.device(self.device) == device and self._struct is not None:
            return self
        dev = {
            "mtiles": torch.from_numpy(np.ascontiguousarray(self.mtiles, dtype=np.int32)).to(device),
            "ptiles": torch.from_numpy(np.ascontiguousarray(self.ptiles, dtype=np.int32)).to(device),
            "row_off": torch.tensor(self.row_offsets, dtype=torch.int64, device=device),
            "ranks": torch.tensor(self.ranks, dtype=torch.int32, device=device),
            "rpad_off": torch.from_numpy(self.rpad_off.astype(np.int32)).to(device),
            "alpha": torch.tensor(self.alphas, dtype=torch.float32, device=device),
        }
        s = _lib.PackStruct()
        s.n_adapters = self.n_adapters
        s.n_mtiles = int(self.mtiles.shape[0])
        s.total_tokens = self.total_tokens
        s.nb = self.nb
        s.rpad16_total = self.rpad16_total
        s.d_mtiles = dev["mtiles"].data_ptr() if s.n_mtiles else None
        s.d_row_off = dev["row_off"].data_ptr()
        s.d_ranks = dev["ranks"].data_ptr()
        s.d_rpad_off = dev["rpad_off"].data_ptr()
        s.d_alpha = dev["alpha"].data_ptr()
        s.n_ptiles = int(self.ptiles.shape[0])
        s.d_ptiles = dev["ptiles"].data_ptr() if s.n_ptiles else None
        self._h_row_off = np.ascontiguousarray(self.row_offsets, dtype=np.int64)   # kept alive with the struct
        s.h_row_off = self._h_row_off.ctypes.data
        self._dev = dev
        self._struct = s
        self.device = device
        return self

    def tile_chunks(self, n: int) -> list:
        """Split the CTA-pair tile list into <= n contiguous token ranges at tile
        boundaries: [(sub_meta, row_lo, row_hi)].  A sub_meta is this pack restricted to
        those pair tiles -- pair-GEMM launches (N >= 256) with it write only rows
        [row_lo, row_hi) of the full-size operands (used to overlap a tensor-parallel
        all-reduce of one chunk with the GEMM of the next)."""
        self.struct   # uploaded
        key = ("chunks", n)
        if key in self._dev:
            return self._dev[key]
        pt = self.ptiles
        nt = pt.shape[0]
        out = []
        if nt == 0:
            out = [(self, 0, self.total_tokens)]
        else:
            ends = np.cumsum(pt[:, 1].astype(np.int64))
            cuts = [0]
            for c in range(1, n):
                j = int(np.searchsorted(ends, self.total_tokens * c / n))
                if cuts[-1] < j < nt:
                    cuts.append(j)
            cuts.append(nt)
            for lo, hi in zip(cuts[:-1], cuts[1:]):
                out.append((self._sub(lo, hi), int(pt[lo, 0]), int(pt[hi - 1, 0] + pt[hi - 1, 1])))
        self._dev[key] = out
        return out

    def shard_launches_rows(self, world: int, launches: int):
        """shard_launches whose sub-packs also restrict the 128-row tile list (so the
        K2a shrinks of a launch cover exactly its rows), or None."""
        out = self.shard_launches(world, launches)
        if out is None or self._shard_mtiles.get(world) is None:
            return None
        return out

    def shard_launches(self, world: int, launches: int):
        """Sequence-parallel shards grouped into <= `launches` pair-GEMM launches:
        [(sub_meta, [(owner, row_lo, row_hi), ...])] -- each launch covers consecutive
        whole shards (fewer, fuller launches than one per shard), or None when the
        shards cannot be cut at pair-tile boundaries."""
        key = ("shard_launches", world, launches)
        if key in self._dev:
            return self._dev[key]
        per = self.shard_tile_chunks(world)
        out = None
        if per is not None:
            groups = max(1, min(launches, world))
            bounds = [round(i * world / groups) for i in range(groups + 1)]
            out = []
            mt = self._shard_mtiles.get(world)
            for a, b in zip(bounds[:-1], bounds[1:]):
                if b <= a:
                    continue
                lo, hi = self._shard_tiles[world][a][0], self._shard_tiles[world][b - 1][1]
                mlo, mhi = (mt[a][0], mt[b - 1][1]) if mt is not None else (None, None)
                out.append((self._sub(lo, hi, mlo, mhi), [(r, per[r][1], per[r][2]) for r in range(a, b)]))
        self._dev[key] = out
        return out

    def shard_tile_chunks(self, world: int):
        """The pair-tile list cut exactly at the sequence-parallel shard boundaries
        (rows r * T / world): [(sub_meta, row_lo, row_hi)] per shard, or None when a
        boundary falls inside a pair tile (T not divisible, or unaligned segments)."""
        key = ("shard_chunks", world)
        if key in self._dev:
            return self._dev[key]
        T = self.total_tokens
        out = None
        if T % world == 0 and self.ptiles.shape[0] > 0:
            starts = self.ptiles[:, 0].astype(np.int64)
            cuts = [0]
            for r in range(1, world):
                j = np.flatnonzero(starts == r * (T // world))
                if j.size == 0:
                    cuts = None
                    break
                cuts.append(int(j[0]))
            if cuts is not None:
                cuts.append(self.ptiles.shape[0])
                if not hasattr(self, "_shard_tiles"):
                    self._shard_tiles = {}
                self._shard_tiles[world] = list(zip(cuts[:-1], cuts[1:]))
                mstarts = self.mtiles[:, 0].astype(np.int64)
                mcuts = [0]
                for r in range(1, world):
                    j = np.flatnonzero(mstarts == r * (T // world))
                    if j.size == 0:
                        mcuts = None
                        break
                    mcuts.append(int(j[0]))
                if not hasattr(self, "_shard_mtiles"):
                    self._shard_mtiles = {}
                self._shard_mtiles[world] = (None if mcuts is None else
                                             list(zip(mcuts, mcuts[1:] + [self.mtiles.shape[0]])))
                out = [(self._sub(lo, hi), r * (T // world), (r + 1) * (T // world))
                       for r, (lo, hi) in enumerate(zip(cuts[:-1], cuts[1:]))]
        self._dev[key] = out
        return out

    def _sub(self, lo: int, hi: int, mlo: int | None = None, mhi: int | None = None) -> "PackMeta":
        """This pack restricted to pair tiles [lo, hi) (pair-GEMM launches only) and, when
        given, to 128-row tiles [mlo, mhi) (so K2a shrinks cover the same rows)."""
        import copy

        s = self.struct
        sub = copy.copy(self)
        st = _lib.PackStruct()
        ctypes.pointer(st)[0] = s
        st.d_ptiles = s.d_ptiles + lo * 16
        st.n_ptiles = hi - lo
        if mlo is not None:
            st.d_mtiles = s.d_mtiles + mlo * 16
            st.n_mtiles = mhi - mlo
        sub._struct = st
        sub._dev = self._dev
        if hasattr(sub, "_work"):
            del sub._work
        return sub

    @property
    def struct(self) -> _lib.PackStruct:
        if self._struct is None:
            raise _lib.PloraError("PackMeta not uploaded; call .to(device) first")
        return self._struct

    def dev(self, name: str):
        return self._dev[name]


def build_meta(ranks: Sequence[int], tokens: Sequence[int], alphas: Sequence[float],
               nb: int | None = None) -> PackMeta:
    """Build the pack metadata through ``plora_meta_build`` (C++ K8)."""
    n = len(ranks)
    if n == 0:
        raise ValueError("nothing to pack")
    if len(tokens) != n or len(alphas) != n:
        raise ValueError(f"{n} adapters but {len(tokens)} inputs")
    L = _lib.lib()
    r = np.ascontiguousarray(ranks, dtype=np.int64)
    t = np.ascontiguousarray(tokens, dtype=np.int64)
    p64 = ctypes.POINTER(ctypes.c_int64)
    p32 = ctypes.POINTER(ctypes.c_int32)
    max_tiles = int(L.plora_meta_max_mtiles(n, t.ctypes.data_as(p64)))
    rank_off = np.zeros(n + 1, dtype=np.int64)
    row_off = np.zeros(n + 1, dtype=np.int64)
    rpad_off = np.zeros(n + 1, dtype=np.int32)
    mtiles = np.zeros((max(max_tiles, 1), 4), dtype=np.int32)
    n_tiles = ctypes.c_int32(0)
    n_ptiles = ctypes.c_int32(0)
    ptiles = np.zeros((max(max_tiles, 1), 4), dtype=np.int32)
    total = int(t.sum()) if n else 0
    tok_ad = np.zeros(max(total, 1), dtype=np.int32)
    rc = L.plora_meta_build(n, r.ctypes.data_as(p64), t.ctypes.data_as(p64),
                            rank_off.ctypes.data_as(p64), row_off.ctypes.data_as(p64),
                            rpad_off.ctypes.data_as(p32), mtiles.ctypes.data_as(p32),
                            max(max_tiles, 1), ctypes.byref(n_tiles), ptiles.ctypes.data_as(p32),
                            ctypes.byref(n_ptiles), tok_ad.ctypes.data_as(p32))
    if rc != 0:
        raise ValueError(L.plora_last_error().decode())
    max_rank = int(r.max())
    need_nb = (max_rank + 63) // 64
    nb = need_nb if nb is None else max(int(nb), need_nb)
    return PackMeta(
        ranks=tuple(int(x) for x in r),
        tokens=tuple(int(x) for x in t),
        alphas=tuple(float(a) for a in alphas),
        rank_offsets=tuple(int(x) for x in rank_off),
        row_offsets=tuple(int(x) for x in row_off),
        rpad_off=rpad_off,
        mtiles=mtiles[: n_tiles.value].copy(),
        ptiles=ptiles[: n_ptiles.value].copy(),
        token_adapter=tok_ad[:total].copy(),
        nb=nb,
    )
