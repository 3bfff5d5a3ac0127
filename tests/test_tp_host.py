"""Tensor-parallel host logic on CPU under torch.distributed gloo, world size 2:
the Megatron shard rules (tp.TPShard), the sharded model / adapter construction
(BaseWeights / AdapterBank with ``shard=``) and the all-reduce placement of the
TP packed linear (tp.DistComm), with the per-rank linear arithmetic done by the
oracle restatement of lorasweep.packed_forward / packed_backward.  The GPU
kernels under the same plan are tested in tests/test_gpu_tp.py."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lorapack_oracle as O
from paper_2508_02932_b200.adapters import AdapterBank
from paper_2508_02932_b200.meta import build_meta
from paper_2508_02932_b200.model import PRESETS, BaseWeights, bench_adapters
from paper_2508_02932_b200.tp import DistComm, TPShard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bank(cfg, meta, shard, targets):
    return AdapterBank(meta, cfg.n_layers, targets, [1e-4] * meta.n_adapters, device="cpu",
                       full_targets=cfg.targets(), shard=shard)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = DistComm()
    sh = TPShard(comm.rank, comm.world)
    cfg = PRESETS["tiny-qwen"]
    specs, s = bench_adapters("tiny-qwen")
    toks = [sp.batch * 8 for sp in specs]                      # short segments: CPU-sized
    meta = build_meta([sp.rank for sp in specs], toks, [sp.alpha for sp in specs])
    local = [t.__class__(t.name, t.h_in, t.h_out // world) if sh.kind(t.name) == "col"
             else t.__class__(t.name, t.h_in // world, t.h_out) for t in cfg.targets()]
    full_b = BaseWeights(cfg, device="cpu")
    base = BaseWeights(cfg, device="cpu", shard=sh)
    full_bank = _bank(cfg, meta, None, cfg.targets())
    bank = _bank(cfg, meta, sh, local)
    errs = {}

    # 1) shards are exact slices
    ok = True
    for t in cfg.targets():
        rows, cols = sh.weight_slice(t.name, t.h_in, t.h_out)
        ok &= torch.equal(base.layers[0][t.name], full_b.layers[0][t.name][rows, cols])
        for kind in ("A", "B"):
            for i in range(meta.n_adapters):
                ok &= torch.equal(bank.block(bank.P, 0, t.name, kind, i),
                                  full_bank.block(full_bank.P, 0, t.name, kind, i)[sh.lora_rows(t.name, kind, t.h_in,
                                                                                                t.h_out)])
    errs["slices"] = bool(ok)

    rng = np.random.default_rng(7)
    n = meta.n_adapters
    T = meta.total_tokens

    def pack_for(b, tname, xs):
        downs = [b.down(0, tname, i).double().numpy() for i in range(n)]
        ups = [b.up(0, tname, i).double().numpy() for i in range(n)]
        return O.pack(downs, ups, list(meta.alphas), xs)

    def w_ref(bw, tname):                          # reference layout d x k
        return bw.layers[0][tname].double().t().contiguous().numpy()

    # 2) row-parallel forward ("o"): sum over ranks of the partial packed outputs == full
    t_o = cfg.targets()[3]
    X = rng.standard_normal((T, t_o.h_in))         # same on every rank (same seed)
    cs = sh.span(t_o.h_in)
    xs_full = [X[meta.row_offsets[i]:meta.row_offsets[i + 1]] for i in range(n)]
    xs_loc = [x[:, cs] for x in xs_full]
    y_part = torch.from_numpy(np.concatenate(O.packed_forward(pack_for(bank, "o", xs_loc), w_ref(base, "o"))))
    comm.all_reduce_(y_part)
    y_full = np.concatenate(O.packed_forward(pack_for(full_bank, "o", xs_full), w_ref(full_b, "o")))
    errs["row_fwd"] = float(np.abs(y_part.numpy() - y_full).max() / np.abs(y_full).max())

    # 3) column-parallel backward ("q"): dA and dX are sums of per-rank partials, dB_s is local
    t_q = cfg.targets()[0]
    Xq = rng.standard_normal((T, t_q.h_in))
    dY = rng.standard_normal((T, t_q.h_out))
    osl = sh.span(t_q.h_out)
    xs = [Xq[meta.row_offsets[i]:meta.row_offsets[i + 1]] for i in range(n)]
    dys_full = [dY[meta.row_offsets[i]:meta.row_offsets[i + 1]] for i in range(n)]
    dd, du, dx = O.packed_backward(pack_for(bank, "q", xs), w_ref(base, "q"), [d[:, osl] for d in dys_full])
    fd, fu, fx = O.packed_backward(pack_for(full_bank, "q", xs), w_ref(full_b, "q"), dys_full)
    dA = torch.from_numpy(np.concatenate([a.ravel() for a in dd]))
    dX = torch.from_numpy(np.concatenate(dx))
    comm.all_reduce_(dA)
    comm.all_reduce_(dX)
    errs["col_dA"] = float(np.abs(dA.numpy() - np.concatenate([a.ravel() for a in fd])).max())
    errs["col_dX"] = float(np.abs(dX.numpy() - np.concatenate(fx)).max())
    errs["col_dB"] = max(float(np.abs(u - f[:, osl]).max()) for u, f in zip(du, fu))

    # 4) max all-reduce (vocabulary-parallel CE statistics)
    m = torch.tensor([float(rank), -float(rank)])
    comm.all_reduce_(m, "max")
    errs["max"] = m.tolist()
    out[rank] = errs
    dist.destroy_process_group()


def test_tp_sharding_and_collectives_gloo():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        e = out[r]
        assert e["slices"]
        assert e["row_fwd"] < 1e-12
        assert e["col_dA"] < 1e-9 and e["col_dX"] < 1e-9 and e["col_dB"] < 1e-12
        assert e["max"] == [1.0, 0.0]


def _coll_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = DistComm()
    x = torch.arange(6, dtype=torch.float32).reshape(3, 2) + 10 * rank
    g = torch.empty(3 * world, 2)
    comm.all_gather_(g, x)
    full = torch.arange(4 * world, dtype=torch.float32).reshape(2 * world, 2) * (rank + 1)
    rs = torch.empty(2, 2)
    comm.reduce_scatter_(rs, full)
    t = torch.full((3,), float(rank + 1))
    comm.reduce_(t, 1)
    out[rank] = (g.tolist(), rs.tolist(), t.tolist())
    dist.destroy_process_group()


def test_sequence_parallel_collectives_gloo():
    """all_gather_ / reduce_scatter_ / reduce_ semantics of the TP communicator (the
    sequence-parallel pieces) under gloo, world size 2."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_coll_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    base = torch.arange(6, dtype=torch.float32).reshape(3, 2)
    want_g = torch.cat([base, base + 10]).tolist()
    full = torch.arange(8, dtype=torch.float32).reshape(4, 2)
    for r in range(2):
        g, rs, t = out[r]
        assert g == want_g
        assert rs == (full * 3)[2 * r:2 * r + 2].tolist()     # (rank 0 x1 + rank 1 x2) rows of this rank
    assert out[1][2] == [3.0, 3.0, 3.0]                        # reduce onto rank 1
