"""Tensor-parallel packed LoRA (config C4: a base too large for one job's GPU is
Megatron-sharded over NVLink).

The reference only models TP as a memory divisor (``ShardingSpec.d_tp``,
workload.py:106-128; ``costmodel.py:120-124``) and the paper runs it through
PyTorch DTensor.  Here the packed trainer itself shards:

  column-parallel (q, k, v, gate, up): W split along h_out; LoRA A replicated,
      B split along h_out.  Forward: no collective (Hs = alpha X A is computed
      identically on every rank).  Backward: dH_s = alpha dY_s B_s^T is partial,
      so dH is all-reduced (T x 64nb bf16, small) before dA = X^T dH; the input
      gradient dX_s = dY_s W_s + dH_s A^T is partial and all-reduced once per
      shared input (q+k+v, gate+up).
  row-parallel (o, down): W split along h_in; LoRA A split along h_in, B
      replicated.  Forward: Y_s = X_s W_s^T + Hs_s B^T with the partial Hs_s, so
      one all-reduce of Y gives X W^T + (sum_s Hs_s) B^T by linearity; Hs itself
      is all-reduced (small) for dB = Hs^T dY.  Backward: no collective.
  lm_head: vocabulary-parallel with a two-pass cross entropy
      (``plora_ce_stats`` / ``plora_ce_apply``).

Sequence parallelism (default when tp divides T): the residual stream and norms
hold only the rank's T/tp token rows; the normed input is all-gathered before the
column-parallel projections and the row-parallel partial outputs are reduced onto
their owning rank (reduce-scatter), in the backward mirrored -- the same bytes as
the all-reduce formulation with 1/tp of the activation memory.

Replicated LoRA factors (column A, row B) get bit-identical gradients on every
rank (identical inputs + deterministic kernels + all-reduced dH / Hs), so their
AdamW states evolve identically without a gradient all-reduce.

Communicators: ``DistComm`` wraps a torch.distributed process group (NCCL over
NVLink/NVSwitch on the box; gloo in CPU tests); ``AbiNcclComm`` is the same NCCL
all-reduce through libplora's C-ABI (``plora_tp_*``, for hosts without torch).  ``ThreadComm`` runs a TP group
of g ranks as g threads sharing ONE GPU (each on its own stream) with a
deterministic fixed-order sum -- it is how the sharded path is parity-tested on
a single B200 (gpurun gives one GPU).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import Callable

import torch

COLUMN = ("q", "k", "v", "gate", "up")
ROW = ("o", "down")


@dataclass(frozen=True)
class TPShard:
    """Position of one rank in a tensor-parallel group of ``world`` ranks."""
    rank: int = 0
    world: int = 1

    def span(self, n: int) -> slice:
        if n % self.world:
            raise ValueError(f"dimension {n} is not divisible by tp={self.world}")
        per = n // self.world
        return slice(self.rank * per, (self.rank + 1) * per)

    def kind(self, target: str) -> str:
        return "col" if target in COLUMN else "row"

    def weight_slice(self, target: str, h_in: int, h_out: int) -> tuple[slice, slice]:
        """(rows, cols) of the nn.Linear-layout weight [h_out][h_in] this rank owns."""
        if self.kind(target) == "col":
            return self.span(h_out), slice(0, h_in)
        return slice(0, h_out), self.span(h_in)

    def lora_rows(self, target: str, kind: str, h_in: int, h_out: int) -> slice:
        """Rows of the LoRA factor this rank owns: A is [h_in][r], B^T is [h_out][r]."""
        if kind == "A":
            return self.span(h_in) if self.kind(target) == "row" else slice(0, h_in)
        return self.span(h_out) if self.kind(target) == "col" else slice(0, h_out)

    def replicated(self, target: str, kind: str) -> bool:
        return (kind == "A") == (self.kind(target) == "col")


class Comm:
    """Collective interface the TP trainer needs.  Tensors are contiguous; in place.
      all_reduce_(t)           t = sum_r t_r (or max)
      all_gather_(out, inp)    out = concat_r inp_r (rank order, along dim 0)
      reduce_scatter_(out, inp) out = sum_r inp_r[rank block]
      reduce_(t, root)         t on `root` = sum_r t_r (other ranks: unspecified)
      broadcast_(t, root)      t = t_root"""
    rank: int = 0
    world: int = 1

    def all_reduce_(self, t: torch.Tensor, op: str = "sum") -> torch.Tensor:  # pragma: no cover
        raise NotImplementedError

    def all_gather_(self, out: torch.Tensor, inp: torch.Tensor) -> torch.Tensor:  # pragma: no cover
        raise NotImplementedError

    def reduce_scatter_(self, out: torch.Tensor, inp: torch.Tensor) -> torch.Tensor:  # pragma: no cover
        raise NotImplementedError

    def reduce_(self, t: torch.Tensor, root: int) -> torch.Tensor:  # pragma: no cover
        raise NotImplementedError

    def broadcast_(self, t: torch.Tensor, root: int) -> torch.Tensor:  # pragma: no cover
        raise NotImplementedError

    # Peer memory for the fused GEMM + reduce (model.PackedLoraTrainer tp_fused): every
    # rank allocates a buffer of the same shape and gets device views of all ranks' copies.
    supports_peer_memory = False

    def peer_buffers(self, shape, dtype):  # pragma: no cover
        """(this rank's buffer, [view of rank r's buffer for r in group])."""
        raise NotImplementedError

    def barrier_(self) -> None:  # pragma: no cover
        """Stream-ordered barrier over the group (all ranks' prior work on their current
        streams is complete -- and visible -- before any rank's later work starts)."""
        raise NotImplementedError


class DistComm(Comm):
    """torch.distributed process group (backend nccl on GPU, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_reduce_(self, t, op="sum"):
        d = self._dist
        d.all_reduce(t, op=d.ReduceOp.SUM if op == "sum" else d.ReduceOp.MAX, group=self.group)
        return t

    def all_gather_(self, out, inp):
        self._dist.all_gather_into_tensor(out, inp, group=self.group)
        return out

    def reduce_scatter_(self, out, inp):
        self._dist.reduce_scatter_tensor(out, inp, group=self.group)
        return out

    def reduce_(self, t, root):
        d = self._dist
        d.reduce(t, dst=d.get_global_rank(self.group, root) if self.group is not None else root, group=self.group)
        return t

    def broadcast_(self, t, root):
        d = self._dist
        d.broadcast(t, src=d.get_global_rank(self.group, root) if self.group is not None else root, group=self.group)
        return t

    supports_peer_memory = True

    def peer_buffers(self, shape, dtype):
        """torch symmetric memory (CUDA IPC over NVLink): each rank maps every peer's copy."""
        import torch.distributed._symmetric_memory as symm_mem

        buf = symm_mem.empty(tuple(shape), dtype=dtype, device=torch.cuda.current_device())
        group = self.group if self.group is not None else self._dist.group.WORLD
        self._symm = symm_mem.rendezvous(buf, group)
        return buf, [self._symm.get_buffer(r, tuple(shape), dtype) for r in range(self.world)]

    def barrier_(self):
        self._symm.barrier(channel=0)


class AbiNcclComm(Comm):
    """The TP group's NCCL communicator created through libplora's C-ABI
    (plora_tp_comm_init / plora_tp_allreduce) -- what a non-torch host uses.  ``group``
    (a torch.distributed group) only carries the 128-byte NCCL id from rank 0; for a
    one-rank group no process group is needed."""

    _DT = {torch.bfloat16: 0, torch.float32: 1}

    def __init__(self, rank: int = 0, world: int = 1, group=None):
        import ctypes

        from . import _lib

        self._ct, self._lib = ctypes, _lib
        self.rank, self.world = rank, world
        idbuf = ctypes.create_string_buffer(128)
        if rank == 0:
            _lib.check(_lib.lib().plora_tp_get_unique_id(idbuf), "plora_tp_get_unique_id")
        if world > 1:
            import torch.distributed as dist

            obj = [idbuf.raw if rank == 0 else None]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            idbuf = ctypes.create_string_buffer(obj[0], 128)
        self._comm = ctypes.c_void_p()
        _lib.check(_lib.lib().plora_tp_comm_init(ctypes.byref(self._comm), idbuf, world, rank), "plora_tp_comm_init")

    def all_reduce_(self, t, op="sum"):
        if t.dtype not in self._DT or not t.is_cuda or not t.is_contiguous():
            raise ValueError("tp all-reduce needs a contiguous CUDA bf16 / f32 tensor")
        self._lib.check(self._lib.lib().plora_tp_allreduce(
            torch.cuda.current_stream().cuda_stream, self._comm, t.data_ptr(), t.numel(), self._DT[t.dtype],
            0 if op == "sum" else 1), "plora_tp_allreduce")
        return t

    def all_gather_(self, out, inp):
        self._check(out, inp)
        self._lib.check(self._lib.lib().plora_tp_allgather(
            torch.cuda.current_stream().cuda_stream, self._comm, inp.data_ptr(), out.data_ptr(), inp.numel(),
            self._DT[inp.dtype]), "plora_tp_allgather")
        return out

    def reduce_scatter_(self, out, inp):
        self._check(out, inp)
        self._lib.check(self._lib.lib().plora_tp_reducescatter(
            torch.cuda.current_stream().cuda_stream, self._comm, inp.data_ptr(), out.data_ptr(), out.numel(),
            self._DT[inp.dtype]), "plora_tp_reducescatter")
        return out

    def reduce_(self, t, root):
        self._check(t)
        self._lib.check(self._lib.lib().plora_tp_reduce(
            torch.cuda.current_stream().cuda_stream, self._comm, t.data_ptr(), t.numel(), self._DT[t.dtype], root),
            "plora_tp_reduce")
        return t

    def broadcast_(self, t, root):
        self._check(t)
        self._lib.check(self._lib.lib().plora_tp_broadcast(
            torch.cuda.current_stream().cuda_stream, self._comm, t.data_ptr(), t.numel(), self._DT[t.dtype], root),
            "plora_tp_broadcast")
        return t

    def _check(self, *ts):
        for t in ts:
            if t.dtype not in self._DT or not t.is_cuda or not t.is_contiguous():
                raise ValueError("tp collectives need contiguous CUDA bf16 / f32 tensors")

    def close(self):
        if self._comm:
            self._lib.check(self._lib.lib().plora_tp_comm_destroy(self._comm), "plora_tp_comm_destroy")
            self._comm = self._ct.c_void_p()


class _ThreadGroup:
    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots: list = [None] * world
        self.result = None


class ThreadComm(Comm):
    """One rank of a TP group emulated by threads on a single GPU (tests / smoke).

    all_reduce_: every rank synchronises its stream, deposits its tensor, rank 0 sums
    in fixed rank order in fp32 (deterministic) and every rank copies the result."""

    def __init__(self, group: _ThreadGroup, rank: int):
        self.g = group
        self.rank = rank
        self.world = group.world

    def _exchange(self, t, combine, deliver):
        """Every rank deposits t; rank 0 computes combine(slots) (fp32, fixed rank order);
        every rank then runs deliver(result)."""
        g = self.g
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        g.slots[self.rank] = t
        g.barrier.wait()
        if self.rank == 0:
            g.result = combine(g.slots)
            if t.is_cuda:
                torch.cuda.current_stream().synchronize()
        g.barrier.wait()
        deliver(g.result)
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        g.barrier.wait()   # everyone has read the result before any rank deposits again

    @staticmethod
    def _sum(slots, op="sum"):
        acc = slots[0].float().clone()
        for other in slots[1:]:
            o = other.float()
            acc = acc + o if op == "sum" else torch.maximum(acc, o)
        return acc

    def all_reduce_(self, t, op="sum"):
        self._exchange(t, lambda sl: self._sum(sl, op), t.copy_)
        return t

    def all_gather_(self, out, inp):
        self._exchange(inp, lambda sl: torch.cat([x.clone() for x in sl], 0), out.copy_)
        return out

    def reduce_scatter_(self, out, inp):
        n = out.shape[0]
        self._exchange(inp, self._sum, lambda r: out.copy_(r[self.rank * n:(self.rank + 1) * n]))
        return out

    def reduce_(self, t, root):
        self._exchange(t, self._sum, lambda r: t.copy_(r) if self.rank == root else None)
        return t

    def broadcast_(self, t, root):
        self._exchange(t, lambda sl: sl[root].clone(), t.copy_)
        return t

    supports_peer_memory = True

    def peer_buffers(self, shape, dtype):
        """Threads share one device: the 'peers' are the other ranks' buffers on it."""
        g = self.g
        buf = torch.empty(tuple(shape), dtype=dtype, device=torch.cuda.current_device())
        g.slots[self.rank] = buf
        g.barrier.wait()
        peers = list(g.slots)
        g.barrier.wait()
        return buf, peers

    def barrier_(self):
        torch.cuda.current_stream().synchronize()
        self.g.barrier.wait()


def run_threaded(world: int, fn: Callable[[Comm], object]) -> list:
    """Run fn(comm) for every rank of a ThreadComm group; returns per-rank results.
    Each rank gets its own CUDA stream (if CUDA is available)."""
    group = _ThreadGroup(world)
    results: list = [None] * world
    errors: list = []

    def body(r):
        comm = ThreadComm(group, r)
        try:
            if torch.cuda.is_available():
                torch.cuda.set_device(0)
                with torch.cuda.stream(torch.cuda.Stream()):
                    results[r] = fn(comm)
                    torch.cuda.current_stream().synchronize()
            else:
                results[r] = fn(comm)
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            errors.append(exc)
            group.barrier.abort()

    threads = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        real = [e for e in errors if not isinstance(e, threading.BrokenBarrierError)]
        raise (real or errors)[0]
    return results
