"""Packed multi-LoRA training step on a frozen Llama/Qwen2-style decoder.

Every one of the 7 LoRA targets per layer (q, k, v, o, gate, up, down)
is a packed LoRA linear executed by libplora (K2a shrink -> K1 tcgen05 GEMM with the
K2b expand fused as extra K-steps; backward K4 -> K3/K5 segment reductions -> K6
dX GEMM with the LoRA term as extra K-steps).  Token segments are adapter-major:
adapter i owns b_i whole sequences of length s, so attention never crosses
adapters.  The frozen lm_head runs on the same tcgen05 GEMM engine.  The loss is
sum_i mean_{tokens of i} CE, so every adapter's gradient equals its solo-training
gradient.

Off the hot path: RMSNorm, RoPE, SwiGLU and cross-entropy run as fused libplora
kernels (``elementwise``); attention is torch SDPA (cuDNN on B200); the embedding
gather is a torch index.

The backward is written out explicitly (no autograd tape) so that exactly the
tensors listed in ``_LayerSave`` are kept: per layer the residual input, the
post-attention residual, q/k/v (inside the attention graph), the attention output,
gate/up projections and the 7 bf16 Hs tiles; normed inputs and SwiGLU output are
recomputed.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Sequence

import torch
import torch.nn.functional as F

from . import elementwise as ew
from . import ops
from .adapters import AdapterBank, Target
from .meta import PackMeta, build_meta
from .tp import Comm, TPShard

bf16 = torch.bfloat16


@dataclass(frozen=True)
class ModelConfig:
    name: str
    d: int
    n_layers: int
    ffn: int
    n_heads: int
    n_kv: int
    vocab: int
    tied: bool = False
    rope_theta: float = 500000.0
    norm_eps: float = 1e-5
    qkv_bias: bool = False
    rope_llama3: bool = False

    @property
    def head_dim(self) -> int:
        return self.d // self.n_heads

    def targets(self) -> list[Target]:
        hd = self.head_dim
        return [Target("q", self.d, self.n_heads * hd), Target("k", self.d, self.n_kv * hd),
                Target("v", self.d, self.n_kv * hd), Target("o", self.n_heads * hd, self.d),
                Target("gate", self.d, self.ffn), Target("up", self.d, self.ffn),
                Target("down", self.ffn, self.d)]

    def base_linear_params(self) -> int:
        """Sum of h_in*h_out over the targeted projections plus the lm_head."""
        per_layer = sum(t.h_in * t.h_out for t in self.targets())
        return self.n_layers * per_layer + self.d * self.vocab

    def base_flops_per_token(self) -> float:
        """Base-GEMM roofline FLOPs/token: 4 * (sum h_in*h_out + d*V) (fwd X W + bwd dY W^T;
        the base is frozen so there is no dW).  SURVEY.md section 8(d)."""
        return 4.0 * self.base_linear_params()

    def lora_flops_per_token_per_rank(self) -> float:
        """6 * sum(h_in + h_out) * L: matches lora_flop (costmodel.py:168-178)."""
        return 6.0 * self.n_layers * sum(t.h_in + t.h_out for t in self.targets())


PRESETS = {
    # C1: tiny 2-layer transformer, runs on the CPU reference
    "tiny": ModelConfig("tiny-d256", d=256, n_layers=2, ffn=1024, n_heads=4, n_kv=4, vocab=1024,
                        rope_theta=10000.0),
    # C1 variant with the Qwen2 features C2/C4 use: GQA, q/k/v bias, tied embeddings
    "tiny-qwen": ModelConfig("tiny-qwen-d256", d=256, n_layers=2, ffn=768, n_heads=4, n_kv=2, vocab=1024,
                             tied=True, rope_theta=1000000.0, norm_eps=1e-6, qkv_bias=True),
    # C2: Qwen2.5-3B (tied embeddings, q/k/v bias)
    "qwen2.5-3b": ModelConfig("Qwen2.5-3B", d=2048, n_layers=36, ffn=11008, n_heads=16, n_kv=2,
                              vocab=151936, tied=True, rope_theta=1000000.0, norm_eps=1e-6, qkv_bias=True),
    # C3: Llama-3.1-8B
    "llama-3.1-8b": ModelConfig("Llama-3.1-8B", d=4096, n_layers=32, ffn=14336, n_heads=32, n_kv=8,
                                vocab=128256, rope_theta=500000.0, norm_eps=1e-5, rope_llama3=True),
    # C4: Qwen2.5-32B
    "qwen2.5-32b": ModelConfig("Qwen2.5-32B", d=5120, n_layers=64, ffn=27648, n_heads=40, n_kv=8,
                               vocab=152064, rope_theta=1000000.0, norm_eps=1e-6, qkv_bias=True),
}


@dataclass(frozen=True)
class AdapterSpec:
    """One packed adapter: rank, raw alpha, sequences per step, learning rate."""
    rank: int
    alpha: float
    batch: int
    lr: float
    weight_decay: float = 0.0


# The bench configurations of SURVEY.md section 8(d).
def bench_adapters(cfg_name: str) -> tuple[list[AdapterSpec], int]:
    mults = [0.25, 1.0, 2.0, 4.0]
    lrs = [2e-5, 5e-5, 1e-4, 2e-4, 4e-4]
    if cfg_name in ("tiny", "tiny-qwen"):
        ranks, batch, s = [8, 16, 32, 64], [1, 2, 1, 2], 128
    elif cfg_name == "qwen2.5-3b":
        ranks, batch, s = [8, 16, 32, 64] * 2, [1, 2, 4, 1, 2, 4, 1, 2], 1024
    elif cfg_name == "llama-3.1-8b":
        ranks = [8, 16, 32, 64] * 4
        batch, s = [1, 1, 2, 4, 2, 1, 4, 1, 1, 2, 1, 4, 4, 2, 1, 1], 1024
    elif cfg_name == "qwen2.5-32b":
        ranks, batch, s = [8, 16, 32, 64] * 8, [1] * 32, 1024
    else:
        raise KeyError(cfg_name)
    specs = [AdapterSpec(rank=r, alpha=r * mults[i % 4], batch=b, lr=lrs[i % 5])
             for i, (r, b) in enumerate(zip(ranks, batch))]
    return specs, s


class BaseWeights:
    """Frozen bf16 base model (random init N(0, 0.02^2), seed 0; norms = 1).
    Projection weights use the nn.Linear layout [h_out][h_in] (K-major operand)."""

    def __init__(self, cfg: ModelConfig, device="cuda", seed: int = 0, std: float = 0.02,
                 shard: TPShard | None = None):
        """``shard``: keep only this tensor-parallel rank's slices (tp.py).  Every tensor
        is drawn at its full shape from the same RNG stream and then sliced, so the
        shards of a TP group are exact slices of the unsharded model."""
        self.cfg = cfg
        self.shard = shard or TPShard()
        sh = self.shard
        g = torch.Generator(device=device).manual_seed(seed)

        def rnd(*shape):
            return (torch.randn(*shape, generator=g, device=device) * std).to(bf16)

        self.embed = rnd(cfg.vocab, cfg.d)    # replicated (token gather)
        self.layers = []
        for _ in range(cfg.n_layers):
            lw = {}
            for t in cfg.targets():
                rows, cols = sh.weight_slice(t.name, t.h_in, t.h_out)
                lw[t.name] = rnd(t.h_out, t.h_in)[rows, cols].contiguous()
            lw["attn_norm"] = torch.ones(cfg.d, device=device, dtype=bf16)
            lw["mlp_norm"] = torch.ones(cfg.d, device=device, dtype=bf16)
            if cfg.qkv_bias:
                for t in cfg.targets()[:3]:
                    lw[t.name + "_bias"] = rnd(t.h_out)[sh.span(t.h_out)].contiguous()
            self.layers.append(lw)
        self.final_norm = torch.ones(cfg.d, device=device, dtype=bf16)
        vs = sh.span(cfg.vocab)
        # vocabulary-parallel lm_head: rows [v0, v0 + V/tp) of [V][d]
        self.lm_head = self.embed[vs] if cfg.tied else rnd(cfg.vocab, cfg.d)[vs].contiguous()
        self.vocab_start = vs.start

    def nbytes(self) -> int:
        n = self.embed.numel() + self.final_norm.numel()
        if self.lm_head.data_ptr() != self.embed.data_ptr():
            n += self.lm_head.numel()
        for lw in self.layers:
            n += sum(v.numel() for v in lw.values())
        return 2 * n


def rope_tables(cfg: ModelConfig, seq_len: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    hd = cfg.head_dim
    inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float64, device=device) / hd))
    if cfg.rope_llama3:  # Llama-3.1 frequency scaling (factor 8, low/high freq 1/4, orig ctx 8192)
        factor, lo, hi, orig = 8.0, 1.0, 4.0, 8192.0
        wavelen = 2 * math.pi / inv
        smooth = (orig / wavelen - lo) / (hi - lo)
        scaled = torch.where(wavelen > orig / lo, inv / factor, inv)
        mid = (wavelen <= orig / lo) & (wavelen >= orig / hi)
        scaled = torch.where(mid, (1 - smooth) * inv / factor + smooth * inv, scaled)
        inv = scaled
    pos = torch.arange(seq_len, dtype=torch.float64, device=device)
    ang = torch.outer(pos, inv)
    return ang.cos().float().contiguous(), ang.sin().float().contiguous()


@dataclass
class _LayerSave:
    h_in: torch.Tensor
    rstd1: torch.Tensor
    h_mid: torch.Tensor
    rstd2: torch.Tensor
    attn_graph: tuple
    attn_out: torch.Tensor
    g: torch.Tensor
    u: torch.Tensor
    hs: dict = field(default_factory=dict)
    x1: torch.Tensor | None = None     # normed inputs, kept when memory allows (else recomputed)
    x2: torch.Tensor | None = None


class PackedLoraTrainer:
    """One packed job: n heterogeneous adapters trained concurrently on one frozen base."""

    def __init__(self, cfg: ModelConfig, specs: Sequence[AdapterSpec], seq_len: int, device="cuda",
                 base: BaseWeights | None = None, ce_chunk: int = 4096, adapter_seeds=None,
                 a_scale: float | None = None, b_std: float | Sequence[float] = 0.02, tp: Comm | None = None,
                 save_normed: bool | None = None, sequence_parallel: bool = True, tp_fused: bool = False,
                 tp_chunks: int = 4, fuse_swiglu: bool = True, fuse_dual: bool = True,
                 fuse_swiglu_bwd: bool = True, overlap_k5: bool | None = None):
        """``tp``: a communicator over this job's tensor-parallel group (tp.py).  With
        tp.world > 1 every weight and adapter factor is this rank's Megatron shard and
        the step inserts the collectives described in tp.py; ``sequence_parallel`` (used
        when tp divides T) also shards the residual stream over tokens.
        ``save_normed``: keep the normed layer inputs for the backward (None: when the
        activation estimate leaves headroom on the device).  ``tp_chunks``: token chunks of
        the TP all-reduce / GEMM overlap; ``tp_fused``: row-parallel GEMMs reduce into the
        owner's buffer over peer memory (opt-in, unmeasured on NVLink); ``fuse_swiglu``:
        gate/up GEMM with the SwiGLU forward in its epilogue; ``fuse_dual``: K4 (dH) and K3
        (dB) of every target in one pass over dY (ops.lora_dual) instead of two;
        ``fuse_swiglu_bwd``: the SwiGLU backward and the down projection's dA in one kernel
        (ops.swiglu_bwd_segred: the activation never goes to HBM); ``overlap_k5``: the dA
        segment reductions (K5, off the critical path: only the optimizer reads dA) run on a
        side stream beside the input-gradient GEMMs (None = off: within noise at T = 32768,
        4096 and 8192 per rank, profiles/r2_overlap_k5_ab.log)."""
        self.cfg = cfg
        self.tp = tp if (tp is not None and tp.world > 1) else None
        self.shard = TPShard(tp.rank, tp.world) if self.tp is not None else TPShard()
        g = self.shard.world
        if cfg.n_heads % g or cfg.n_kv % g:
            raise ValueError(f"tp={g} must divide n_heads={cfg.n_heads} and n_kv={cfg.n_kv}")
        self.H_l, self.KV_l = cfg.n_heads // g, cfg.n_kv // g
        self.targets = [Target(t.name, t.h_in, t.h_out // g) if self.shard.kind(t.name) == "col"
                        else Target(t.name, t.h_in // g, t.h_out) for t in cfg.targets()]
        self.specs = list(specs)
        self.s = seq_len
        self.device = torch.device(device)
        tokens = [sp.batch * seq_len for sp in specs]
        self.meta: PackMeta = build_meta([sp.rank for sp in specs], tokens, [sp.alpha for sp in specs]).to(
            self.device)
        self.T = self.meta.total_tokens
        # Megatron sequence parallelism under TP: the residual stream, norms and their saved
        # activations hold only this rank's T/tp token rows; all-gather before the column-
        # parallel projections, reduce-scatter after the row-parallel ones (tp.py)
        self.sp = self.tp is not None and sequence_parallel and self.T % g == 0
        self.Tl = self.T // g if self.sp else self.T
        self.r0 = self.shard.rank * self.Tl if self.sp else 0
        self.base = base or BaseWeights(cfg, self.device, shard=self.shard)
        if self.base.shard != self.shard:
            raise ValueError("base weights are sharded for a different tensor-parallel position")
        self.bank = AdapterBank(self.meta, cfg.n_layers, self.targets, [sp.lr for sp in specs],
                                [sp.weight_decay for sp in specs], device=self.device, seeds=adapter_seeds,
                                a_scale=a_scale, b_std=b_std, full_targets=cfg.targets(),
                                shard=self.shard if self.tp is not None else None)
        self.cos, self.sin = rope_tables(cfg, seq_len, self.device)
        self.ce_chunk = int(ce_chunk)   # tokens per lm_head + CE chunk
        # per-token adapter id and the CE weight 1/n_i (labels exist for s-1 tokens per sequence)
        ta = torch.from_numpy(self.meta.token_adapter.astype("int64")).to(self.device)
        n_lab = torch.tensor([max(sp.batch * (seq_len - 1), 1) for sp in specs], dtype=torch.float32,
                             device=self.device)
        pos = torch.arange(self.T, device=self.device) % seq_len
        self.token_adapter = ta
        self.has_label = pos != seq_len - 1
        self.ce_weight = torch.where(self.has_label, 1.0 / n_lab[ta], torch.zeros((), device=self.device))
        self.losses = torch.zeros(self.meta.n_adapters, dtype=torch.float32, device=self.device)
        self.save_normed = self._fits_saved_norms() if save_normed is None else bool(save_normed)
        self.tp_chunks = int(tp_chunks)   # TP all-reduce / GEMM overlap depth
        self._side = None
        # fused GEMM + reduce onto owners through peer memory (opt-in, see _fused_reduce)
        self.tp_fused = bool(tp_fused and self.sp and getattr(self.tp, "supports_peer_memory", False))
        self._peer = {}
        # gate/up GEMM with the SwiGLU forward in its epilogue (CTA-pair tiles: ffn shard >= 256)
        self._fuse_swiglu = self.targets[4].h_out >= 256 and fuse_swiglu
        self._fuse_dual = bool(fuse_dual)
        self._fuse_swiglu_bwd = bool(fuse_swiglu_bwd)
        if overlap_k5 is None:
            overlap_k5 = False
        self._overlap_k5 = bool(overlap_k5) and self.tp is None
        self._k5_stream = None
        self._k5_used = False
        self._row_off_dev = torch.tensor(self.meta.row_offsets, dtype=torch.int64, device=self.device)

    # ------------------------------------------------------------------ helpers
    def activation_bytes(self, save_normed: bool) -> int:
        """Saved-activation estimate of one step (bf16): per layer h_in, h_mid, q/k/v, the
        attention output, gate/up and the 7 Hs tiles (+ the two normed inputs)."""
        cfg, T, hd = self.cfg, self.T, self.cfg.head_dim
        ffn_l = self.targets[4].h_out
        per = (2 * cfg.d * self.Tl // T + (self.H_l + 2 * self.KV_l) * hd + self.H_l * hd + 2 * ffn_l
               + 7 * self.meta.rpad64 + (2 * cfg.d if save_normed else 0))
        return 2 * T * per * cfg.n_layers

    def _fits_saved_norms(self) -> bool:
        """Keep x1/x2 from the forward (saves two RMSNorm recomputes per layer) when the
        extra activations leave >= 12 GB of headroom on the device."""
        if self.device.type != "cuda":
            return False
        free, _ = torch.cuda.mem_get_info(self.device)
        return free - self.activation_bytes(True) > 12e9

    def _lin_fwd(self, layer: int, tname: str, x: torch.Tensor, w: torch.Tensor, residual=None):
        a_sh = self.bank.shadow_of(layer, tname, "A")
        bt_sh = self.bank.shadow_of(layer, tname, "B")
        y, hs = ops.linear_fwd(self.meta, x, w, True, a_sh, bt_sh, residual=residual)
        return y, hs

    def _row_fwd(self, layer: int, tname: str, x: torch.Tensor, w: torch.Tensor):
        """Row-parallel target (o, down).  Under TP the output Y_s = X_s W_s^T + Hs_s B^T is a
        partial sum reduced per token chunk on a side stream, overlapping the next chunk's
        GEMM (see _overlapped; with sequence parallelism the rank's token shard is
        returned); the partial Hs is all-reduced after the last chunk read it."""
        if self.tp is None:
            return self._lin_fwd(layer, tname, x, w)
        bank, meta = self.bank, self.meta
        hs = torch.empty((self.T, meta.rpad64), dtype=bf16, device=self.device)
        ops.shrink(meta, x, bank.shadow_of(layer, tname, "A"), hs)
        y_part = torch.empty((self.T, w.shape[0]), dtype=bf16, device=self.device)
        bt = bank.shadow_of(layer, tname, "B")
        y = self._overlapped(lambda m, out=y_part: ops.linear_expand(m, x, w, True, bt, hs, y_out=out,
                                                                     residual=None if out is y_part else out),
                             y_part, extra=(hs,))
        return y, hs

    def _overlapped(self, launch, y: torch.Tensor, extra=()):
        """TP: enqueue launch(sub_pack) per token chunk of the pair-tile list on the current
        stream and reduce that chunk's rows of the partial y on the side stream as soon as
        its GEMM is done (NCCL of chunk c overlaps the GEMM of chunk c+1); then all-reduce
        `extra` there and make the current stream wait for the side stream.
        Without sequence parallelism the chunks are all-reduced and y is returned; with it
        the chunks are the ranks' token shards, each reduced onto its owner (ncclReduce),
        and this rank's [T/tp][d] shard of the sum is returned (a view of y) -- or, when a
        shard boundary falls inside a pair tile, one GEMM then a reduce-scatter."""
        cur = torch.cuda.current_stream()
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
        side = self._side
        wide = y.shape[1] >= 256   # pair-GEMM path (sub-packs only restrict pair tiles)
        out = y
        if self.tp_fused and wide and self.meta.shard_tile_chunks(self.shard.world) is not None:
            return self._fused_reduce(launch, y, extra)
        if self.sp:
            chunks = self.meta.shard_launches(self.shard.world, self.tp_chunks) if wide else None
            if chunks is None:
                launch(self.meta)
                out = torch.empty((self.Tl, y.shape[1]), dtype=y.dtype, device=y.device)
                ev = torch.cuda.Event()
                ev.record(cur)
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    self.tp.reduce_scatter_(out, y)
            else:   # launches of whole shards; each shard reduced onto its owner after its launch
                for sub, shards in chunks:
                    launch(sub)
                    ev = torch.cuda.Event()
                    ev.record(cur)
                    side.wait_event(ev)
                    with torch.cuda.stream(side):
                        for owner, r0, r1 in shards:
                            self.tp.reduce_(y[r0:r1], owner)
                out = y[self.r0:self.r0 + self.Tl]
        else:
            chunks = self.meta.tile_chunks(self.tp_chunks) if wide else [(self.meta, 0, self.T)]
            for sub, r0, r1 in chunks:
                launch(sub)
                ev = torch.cuda.Event()
                ev.record(cur)
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    self.tp.all_reduce_(y[r0:r1])
        with torch.cuda.stream(side):
            for t in extra:
                self.tp.all_reduce_(t)
        done = torch.cuda.Event()
        done.record(side)
        cur.wait_event(done)
        return out

    def _prefetch_normed(self, h, rstd, w):
        """Recompute rmsnorm(h) and (sequence parallel) all-gather it -- on the side stream
        when TP is active, so it overlaps the compute issued meanwhile; _await joins it."""
        if not self.sp:
            return ("ready", ew.rmsnorm_apply(h, rstd, w))
        cur = torch.cuda.current_stream()
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
        side = self._side
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            x = self._gather(ew.rmsnorm_apply(h, rstd, w))
            ev = torch.cuda.Event()
            ev.record(side)
        x.record_stream(cur)   # consumed on the compute stream
        return ("pending", x, ev)

    def _await(self, pre):
        if pre[0] == "ready":
            return pre[1]
        torch.cuda.current_stream().wait_event(pre[2])
        return pre[1]

    def _fused_reduce(self, launch, y: torch.Tensor, extra=()):
        """Row-parallel GEMM fused with the reduce onto the owning rank, over peer memory:
        every rank runs the GEMM tiles of owner c's token shard with its epilogue in
        reduce-add mode aimed at owner c's buffer (a TMA reduce-add of each finished
        bf16 tile into the peer's memory over NVLink), so the transfer rides the GEMM tile
        by tile and no separate collective touches the data.  Owners zero their rows, a
        barrier, the GEMMs (owners visited in rank-rotated order to spread the links),
        a barrier; the owner's rows are its shard of the sum.  Two buffers per width
        alternate (the consumer of one output runs before the buffer is reused)."""
        d = y.shape[1]
        slot = self._peer.setdefault(("next", d), 0)
        self._peer[("next", d)] = slot ^ 1
        if (d, slot) not in self._peer:
            self._peer[(d, slot)] = self.tp.peer_buffers((self.T, d), y.dtype)
        buf, peers = self._peer[(d, slot)]
        chunks = self.meta.shard_tile_chunks(self.shard.world)
        own = buf[self.r0:self.r0 + self.Tl]
        own.zero_()
        self.tp.barrier_()
        g, r = self.shard.world, self.shard.rank
        for j in range(g):
            c = (r + j) % g
            launch(chunks[c][0], peers[c])      # epilogue: reduce-add into rank c's rows
        self.tp.barrier_()
        for t in extra:
            self.tp.all_reduce_(t)
        return own

    def _gather(self, x_s: torch.Tensor) -> torch.Tensor:
        """Sequence parallelism: every rank's [T/tp][d] token shard -> the full [T][d]."""
        if not self.sp:
            return x_s
        full = torch.empty((self.T, x_s.shape[1]), dtype=x_s.dtype, device=x_s.device)
        self.tp.all_gather_(full, x_s)
        return full

    def _lin_bwd(self, layer: int, tname: str, x, w, hs, dy, need_dx=True, dx_residual=None, dx_out=None):
        """Backward of one packed LoRA linear (reference lorapack.py:202-231): Cases 2 + 1 as
        the fused dY pass, Case 3 (K5), Case 4 (K6) -- or ops.linear_bwd's four kernels."""
        bank, meta = self.bank, self.meta
        if self._fuse_dual and meta.nb == 1:
            dh = torch.empty((self.T, meta.rpad64), dtype=bf16, device=self.device)
            self._dy_pass(layer, (tname,), (dy,), (hs,), (dh,))                                  # K4 + K3
            self._k5(lambda: ops.segred(meta, x, dh, bank.region_flat(bank.G, layer, tname, "A")), x, dh)  # K5
            if not need_dx:
                return None
            return ops.linear_expand(meta, dy, w, False, bank.shadow_of(layer, tname, "A"), dh,    # K6
                                     y_out=dx_out, residual=dx_residual)
        return ops.linear_bwd(meta, x, w, True, bank.shadow_of(layer, tname, "A"),
                              bank.shadow_of(layer, tname, "B"), hs, dy,
                              bank.region_flat(bank.G, layer, tname, "A"),
                              bank.region_flat(bank.G, layer, tname, "B"),
                              dx_out=dx_out, need_dx=need_dx, dx_residual=dx_residual)

    def _group_fwd(self, layer: int, names, x: torch.Tensor, biases=None, parts=None):
        """Forward of targets sharing the input x (q/k/v or gate/up): ONE K2a launch reads
        x once for every target's Hs, then ONE grouped K1 GEMM (K2b fused) for all targets
        -- per row part when x arrives in parts (sequence-parallel all-gather, see
        _gather_parts: each part's kernels wait only for that part's rows)."""
        bank, meta, lw = self.bank, self.meta, self.base.layers[layer]
        hss = [torch.empty((self.T, meta.rpad64), dtype=bf16, device=self.device) for _ in names]
        a_shs = [bank.shadow_of(layer, nm, "A") for nm in names]
        bt_shs = [bank.shadow_of(layer, nm, "B") for nm in names]
        ws = [lw[nm] for nm in names]
        if parts is None:
            ops.shrink_multi(meta, x, a_shs, hss)
            return ops.linear_expand_group(meta, x, ws, bt_shs, hss, biases=biases), hss
        ys = [torch.empty((self.T, w.shape[0]), dtype=bf16, device=self.device) for w in ws]
        cur = torch.cuda.current_stream()
        for sub, ev in parts:
            cur.wait_event(ev)
            ops.shrink_multi(sub, x, a_shs, hss)
            ops.linear_expand_group(sub, x, ws, bt_shs, hss, biases=biases, y_outs=ys)
        return ys, hss

    def _gate_up_swiglu(self, layer: int, x: torch.Tensor, parts=None):
        """gate/up with the SwiGLU forward in the GEMM epilogue (per row part, as _group_fwd)."""
        bank, meta, lw = self.bank, self.meta, self.base.layers[layer]
        hs_g = torch.empty((self.T, meta.rpad64), dtype=bf16, device=self.device)
        hs_u = torch.empty_like(hs_g)
        a_shs = [bank.shadow_of(layer, "gate", "A"), bank.shadow_of(layer, "up", "A")]
        bts = (bank.shadow_of(layer, "gate", "B"), bank.shadow_of(layer, "up", "B"))
        if parts is None:
            ops.shrink_multi(meta, x, a_shs, [hs_g, hs_u])
            g, u, act = ops.linear_gate_up_swiglu(meta, x, lw["gate"], lw["up"], *bts, hs_g, hs_u)
            return g, u, act, hs_g, hs_u
        ffn = lw["gate"].shape[0]
        outs = tuple(torch.empty((self.T, ffn), dtype=bf16, device=self.device) for _ in range(3))
        cur = torch.cuda.current_stream()
        for sub, ev in parts:
            cur.wait_event(ev)
            ops.shrink_multi(sub, x, a_shs, [hs_g, hs_u])
            ops.linear_gate_up_swiglu(sub, x, lw["gate"], lw["up"], *bts, hs_g, hs_u, outs=outs)
        return (*outs, hs_g, hs_u)

    def _gather_parts(self, x_s: torch.Tensor):
        """Sequence-parallel forward all-gather of the normed input, overlapped with its
        consumers: the shards are broadcast from their owners on the side stream in the
        ``tp_chunks`` launch groups; returns (x_full, [(sub_pack, event)]) so the
        column-parallel kernels of a group start as soon as its rows arrived -- or
        (x_full, None) after a plain all-gather when the tile lists cannot be cut at
        the shard boundaries."""
        if not self.sp:
            return x_s, None
        groups = self.meta.shard_launches_rows(self.shard.world, self.tp_chunks)
        if groups is None or x_s.shape[1] % 8:
            return self._gather(x_s), None
        cur = torch.cuda.current_stream()
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
        side = self._side
        x = torch.empty((self.T, x_s.shape[1]), dtype=x_s.dtype, device=self.device)
        x[self.r0:self.r0 + self.Tl].copy_(x_s)
        side.wait_stream(cur)
        parts = []
        with torch.cuda.stream(side):
            for sub, shards in groups:
                for owner, r0, r1 in shards:
                    self.tp.broadcast_(x[r0:r1], owner)
                ev = torch.cuda.Event()
                ev.record(side)
                parts.append((sub, ev))
        x.record_stream(side)
        return x, parts

    def _k5(self, fn, *tensors) -> None:
        """Run the dA reduction ``fn`` (K5) in stream order, or -- with overlap_k5 -- on the
        side stream after the work issued so far (joined before the optimizer step)."""
        if not self._overlap_k5:
            fn()
            return
        cur = torch.cuda.current_stream()
        if self._k5_stream is None:
            self._k5_stream = torch.cuda.Stream(device=self.device)
        self._k5_stream.wait_stream(cur)
        with torch.cuda.stream(self._k5_stream):
            fn()
        for t in tensors:
            t.record_stream(self._k5_stream)
        self._k5_used = True

    def _dy_pass(self, layer: int, names, dys, hss, dhs) -> None:
        """Cases 2 and 1 of the reference backward (lorapack.py:225, :224) for the targets
        ``names`` (one, or the q/k/v / gate/up group): dH = alpha dY B^T into ``dhs`` and
        dB^T = Hs^T dY into the grad regions -- one fused pass over every dY in one launch
        (K4 + K3, ops.lora_dual) or the two separate kernels per target."""
        bank, meta = self.bank, self.meta
        bts = [bank.shadow_of(layer, nm, "B") for nm in names]
        gs = [bank.region_flat(bank.G, layer, nm, "B") for nm in names]
        if self._fuse_dual and meta.nb == 1:
            ops.lora_dual(meta, list(dys), bts, list(hss), list(dhs), gs)
        else:
            for dy, bt, hs, dh, g in zip(dys, bts, hss, dhs, gs):
                ops.shrink(meta, dy, bt, dh)        # K4 (Case 2)
                ops.segred(meta, dy, hs, g)         # K3 (Case 1)

    def _group_bwd(self, layer: int, names, x: torch.Tensor, hss, dys, need_dx: bool = True):
        """Backward of targets sharing the input x: per target K4 dH and K3 dB; ONE grouped
        K6 launch sums every target's input gradient in one fp32 accumulator; ONE K5
        launch for every dA (x read once).  Column-parallel under TP: dH_s and dX_s are
        partial -- both are all-reduced here (dX per token chunk, overlapping the GEMM),
        dH before dA (tp.py)."""
        bank, meta, lw = self.bank, self.meta, self.base.layers[layer]
        dhs = [torch.empty((self.T, meta.rpad64), dtype=bf16, device=self.device) for _ in names]
        self._dy_pass(layer, names, dys, hss, dhs)                                          # K4 + K3
        dx = None
        ws, ashs = [lw[nm] for nm in names], [bank.shadow_of(layer, nm, "A") for nm in names]
        if need_dx and self.tp is not None:   # partial dX_s: chunked all-reduce overlapping the GEMM
            dx_part = torch.empty((self.T, x.shape[1]), dtype=bf16, device=self.device)
            dx = self._overlapped(
                lambda m, out=dx_part: ops.linear_dx_group(m, list(dys), ws, ashs, dhs, x.shape[1], dx_out=out,
                                                           dx_residual=None if out is dx_part else out),
                dx_part, extra=dhs)
        else:
            if need_dx:   # K6 (Case 4) for every target in one accumulator
                dx = ops.linear_dx_group(meta, list(dys), ws, ashs, dhs, x.shape[1])
            self._reduce(*dhs)
        self._k5(lambda: ops.segred_multi(meta, x, dhs, [bank.region_flat(bank.G, layer, nm, "A") for nm in names]),
                 x, *dhs)                                                                           # K5
        return dx

    def _token_major(self, x: torch.Tensor) -> torch.Tensor:
        """[B][H][s][hd]-shaped attention tensor -> [T][H*hd]: a free view when the
        attention kernel already produced token-major memory, else one layout-change pass."""
        B, H, s, hd = x.shape
        xt = x.transpose(1, 2)
        if xt.is_contiguous():
            return xt.view(B * s, H * hd)
        return ew.rope(xt, self.cos, self.sin, s, rotate=False)

    def _reduce(self, *ts):
        if self.tp is not None:
            for t in ts:
                self.tp.all_reduce_(t)

    # ------------------------------------------------------------------ forward
    def _layer_fwd(self, layer: int, h_prev: torch.Tensor, delta: torch.Tensor | None
                   ) -> tuple[torch.Tensor, torch.Tensor, _LayerSave]:
        """h = h_prev + delta (the previous layer's down-projection output, added inside
        the fused add+RMSNorm); returns (h_mid, down_out) -- this layer's output is their
        sum, materialised by the next layer's (or the final) add+RMSNorm."""
        cfg, lw = self.cfg, self.base.layers[layer]
        T, hd, H, KV, s = self.T, cfg.head_dim, self.H_l, self.KV_l, self.s
        B = T // s
        if delta is None:
            h = h_prev
            x1, rstd1 = ew.rmsnorm_fwd(h, lw["attn_norm"], cfg.norm_eps)
        else:
            h, x1, rstd1 = ew.add_rmsnorm_fwd(h_prev, delta, lw["attn_norm"], cfg.norm_eps)
        x1, parts = self._gather_parts(x1)   # sequence parallel: the token shards -> all T rows
        biases = [lw["q_bias"], lw["k_bias"], lw["v_bias"]] if cfg.qkv_bias else None   # added in the epilogue
        (q, k, v), (hs_q, hs_k, hs_v) = self._group_fwd(layer, ("q", "k", "v"), x1, biases, parts)
        x1_keep = x1 if self.save_normed else None
        del x1
        ew.rope(q.view(B, s, H, hd), self.cos, self.sin, s, out=q)        # in place
        ew.rope(k.view(B, s, KV, hd), self.cos, self.sin, s, out=k)
        qg = q.view(B, s, H, hd).transpose(1, 2).detach().requires_grad_()
        kg = k.view(B, s, KV, hd).transpose(1, 2).detach().requires_grad_()
        vg = v.view(B, s, KV, hd).transpose(1, 2).detach().requires_grad_()
        with torch.enable_grad():
            og = F.scaled_dot_product_attention(qg, kg, vg, is_causal=True, enable_gqa=(KV != H))
        attn = self._token_major(og.detach())                                           # [T][H*hd]
        o_out, hs_o = self._row_fwd(layer, "o", attn, lw["o"])   # TP: Y and Hs all-reduced (row-parallel)
        h_mid, x2, rstd2 = ew.add_rmsnorm_fwd(h, o_out, lw["mlp_norm"], cfg.norm_eps)
        del o_out
        x2, parts = self._gather_parts(x2)
        if self._fuse_swiglu:   # gate/up GEMM with the SwiGLU forward in its epilogue
            g, u, act, hs_g, hs_u = self._gate_up_swiglu(layer, x2, parts)
        else:
            (g, u), (hs_g, hs_u) = self._group_fwd(layer, ("gate", "up"), x2, parts=parts)
            act = ew.swiglu_fwd(g, u)
        x2_keep = x2 if self.save_normed else None
        del x2
        d_out, hs_d = self._row_fwd(layer, "down", act, lw["down"])
        save = _LayerSave(h_in=h, rstd1=rstd1, h_mid=h_mid, rstd2=rstd2, attn_graph=(qg, kg, vg, og),
                          attn_out=attn, g=g, u=u,
                          hs={"q": hs_q, "k": hs_k, "v": hs_v, "o": hs_o, "gate": hs_g, "up": hs_u, "down": hs_d},
                          x1=x1_keep, x2=x2_keep)
        return h_mid, d_out, save

    # ------------------------------------------------------------------ backward
    def _layer_bwd(self, layer: int, sv: _LayerSave, dh: torch.Tensor, need_dx: bool) -> torch.Tensor:
        cfg, lw = self.cfg, self.base.layers[layer]
        T, hd, H, KV, s = self.T, cfg.head_dim, self.H_l, self.KV_l, self.s
        B = T // s
        # MLP: h_out = h_mid + down(swiglu(gate(x2), up(x2))).  The down projection's
        # Cases 2/1/4 run first; the SwiGLU backward re-emits the activation in the same
        # pass (no separate recompute), then Case 3 dA_down = act^T dH.
        bank, meta = self.bank, self.meta
        # sequence parallel, normed inputs not kept: start re-gathering x2 and x1 on the side
        # stream now, so the all-gathers overlap the down / o projection backward below
        pre2 = self._prefetch_normed(sv.h_mid, sv.rstd2, lw["mlp_norm"]) if sv.x2 is None else None
        pre1 = self._prefetch_normed(sv.h_in, sv.rstd1, lw["attn_norm"]) if sv.x1 is None else None
        dh_s = dh
        dh = self._gather(dh_s)   # sequence parallel: the row-parallel output gradient on all T rows
        dh_down = torch.empty((T, meta.rpad64), dtype=bf16, device=self.device)
        self._dy_pass(layer, ("down",), (dh,), (sv.hs["down"],), (dh_down,))                 # K4 + K3
        d_act = ops.linear_expand(meta, dh, lw["down"], False, bank.shadow_of(layer, "down", "A"), dh_down)  # K6
        del dh
        if self._fuse_swiglu_bwd and meta.nb == 1:   # SwiGLU bwd + K5 in one pass: act stays on chip
            dg, du = ops.swiglu_bwd_segred(meta, d_act, sv.g, sv.u, dh_down,
                                           bank.region_flat(bank.G, layer, "down", "A"), out_g=sv.g, out_u=sv.u)
            del d_act
        else:
            act = torch.empty_like(sv.g)
            dg, du = ew.swiglu_bwd(d_act, sv.g, sv.u, out_g=sv.g, out_u=sv.u, act_out=act)  # in place over g, u
            del d_act
            ops.segred(meta, act, dh_down, bank.region_flat(bank.G, layer, "down", "A"))     # K5
            del act
        del dh_down
        x2 = sv.x2 if sv.x2 is not None else self._await(pre2)
        sv.x2 = None
        dx2 = self._group_bwd(layer, ("up", "gate"), x2, (sv.hs["up"], sv.hs["gate"]), (du, dg))
        del dg, du, x2
        d_mid = ew.rmsnorm_bwd(dx2, sv.h_mid, sv.rstd2, lw["mlp_norm"], residual_grad=dh_s, out=dx2)
        # attention: h_mid = h_in + o(attn(rope(q(x1)), rope(k(x1)), v(x1)))
        d_attn = self._lin_bwd(layer, "o", sv.attn_out, lw["o"], sv.hs["o"], self._gather(d_mid))
        qg, kg, vg, og = sv.attn_graph
        dq, dk, dv = torch.autograd.grad(og, (qg, kg, vg), d_attn.view(B, s, H, hd).transpose(1, 2))
        del d_attn
        dq = ew.rope(dq.transpose(1, 2), self.cos, self.sin, s, inverse=True)      # [T][H*hd]
        dk = ew.rope(dk.transpose(1, 2), self.cos, self.sin, s, inverse=True)
        dv = self._token_major(dv)
        x1 = sv.x1 if sv.x1 is not None else self._await(pre1)
        sv.x1 = None
        dx1 = self._group_bwd(layer, ("v", "k", "q"), x1, (sv.hs["v"], sv.hs["k"], sv.hs["q"]), (dv, dk, dq),
                              need_dx=need_dx)
        del dq, dk, dv, x1
        if not need_dx:   # first layer: the embedding is frozen, no input gradient
            return None
        return ew.rmsnorm_bwd(dx1, sv.h_in, sv.rstd1, lw["attn_norm"], residual_grad=d_mid, out=dx1)

    # ------------------------------------------------------------------ loss head
    def _head(self, h_prev: torch.Tensor, delta: torch.Tensor, tokens: torch.Tensor) -> torch.Tensor:
        """Final (add+)norm + lm_head + per-adapter-mean CE, chunked over tokens; returns
        d h.  Writes per-adapter losses into self.losses."""
        cfg = self.cfg
        h, xf, rstd = ew.add_rmsnorm_fwd(h_prev, delta, self.base.final_norm, cfg.norm_eps)
        xf = self._gather(xf)
        dxf = torch.empty_like(xf)
        labels = torch.roll(tokens, -1)
        tok_loss = torch.empty(self.T, dtype=torch.float32, device=self.device)
        for c0 in range(0, self.T, self.ce_chunk):
            c1 = min(self.T, c0 + self.ce_chunk)
            logits = ops.gemm(xf[c0:c1], self.base.lm_head, True)
            if self.tp is None:
                ew.cross_entropy(logits, labels[c0:c1], self.ce_weight[c0:c1], tok_loss[c0:c1])
            else:   # vocabulary-parallel CE: per-row (max, sumexp, label logit) across the TP group
                v0 = self.base.vocab_start
                st = ew.ce_stats(logits, labels[c0:c1], v0)
                m = st[:, 0].contiguous()
                self.tp.all_reduce_(m, "max")
                sl = torch.stack((st[:, 1] * torch.exp(st[:, 0] - m), st[:, 2]), 1)
                self.tp.all_reduce_(sl)
                lse = m + torch.log(sl[:, 0])
                w = self.ce_weight[c0:c1]
                ew.ce_apply(logits, labels[c0:c1], v0, lse, w)
                tok_loss[c0:c1] = w * (lse - sl[:, 1])
            ops.gemm(logits, self.base.lm_head, False, out=dxf[c0:c1])   # dX = dlogits @ W_lm
            del logits
        if self.sp:   # partial over the vocabulary shards -> this rank's token shard of the sum
            dxf_s = torch.empty((self.Tl, dxf.shape[1]), dtype=bf16, device=self.device)
            self.tp.reduce_scatter_(dxf_s, dxf)
            dxf = dxf_s
        else:
            self._reduce(dxf)
        # per-adapter sums over contiguous segments (deterministic prefix-sum differences)
        cs = torch.cumsum(tok_loss.double(), 0)
        cs = torch.cat((cs.new_zeros(1), cs))
        ro = self._row_off_dev
        self.losses.copy_((cs[ro[1:]] - cs[ro[:-1]]).float())
        return ew.rmsnorm_bwd(dxf, h, rstd, self.base.final_norm, out=dxf)

    # ------------------------------------------------------------------ step
    def forward_backward(self, tokens: torch.Tensor) -> torch.Tensor:
        """Full packed forward + backward; fills bank.G; returns per-adapter losses (device)."""
        h = self.base.embed[tokens[self.r0:self.r0 + self.Tl]]   # sequence parallel: own token rows
        delta = None
        saves = []
        for layer in range(self.cfg.n_layers):
            h, delta, sv = self._layer_fwd(layer, h, delta)
            saves.append(sv)
        dh = self._head(h, delta, tokens)
        del h, delta
        for layer in reversed(range(self.cfg.n_layers)):
            sv = saves.pop()
            dh = self._layer_bwd(layer, sv, dh, need_dx=layer > 0)
            del sv
        if self._k5_used:   # the side stream's dA reductions before anything reads the grads
            torch.cuda.current_stream().wait_stream(self._k5_stream)
            self._k5_used = False
        return self.losses

    def step(self, tokens: torch.Tensor) -> torch.Tensor:
        """forward + backward + fused per-adapter AdamW (K7)."""
        losses = self.forward_backward(tokens)
        self.bank.adamw_step()
        return losses

    def graphed(self, tokens: torch.Tensor, warmup: int = 2) -> "GraphedStep":
        """This trainer's step (forward + backward + AdamW) captured as one CUDA graph
        (see GraphedStep).  ``warmup`` eager steps run first (they train)."""
        return GraphedStep(self, tokens, warmup)

    # ------------------------------------------------------------------ data
    def synthetic_tokens(self, seed_base: int = 1000, seeds: Sequence[int] | None = None) -> torch.Tensor:
        """tokens ~ U{0..V-1}, seed 1000+i per adapter; ``seeds``
        overrides the per-adapter seeds (a rank of a planner split keeps the seeds of its
        adapters' positions in the whole workload)."""
        parts = []
        for i, sp in enumerate(self.specs):
            g = torch.Generator(device="cpu").manual_seed(seed_base + i if seeds is None else int(seeds[i]))
            parts.append(torch.randint(0, self.cfg.vocab, (sp.batch * self.s,), generator=g))
        return torch.cat(parts)


class GraphedStep:
    """A packed training step replayed from a CUDA graph.

    Every launch of ``PackedLoraTrainer.step`` -- ~1.3k libplora kernels (tensor maps
    and LPT schedules baked into their parameters), cuDNN attention, the norms, the CE
    chunks and the fused AdamW (per-adapter step counts on the device, adapters.py) --
    is captured once and replayed with one ``cudaGraphLaunch``: no per-kernel host work
    and no launch gaps.  That is what keeps a small per-GPU share of a planner split
    (T = 4096 tokens at 8 GPUs, where the eager host enqueue takes as long as the GPU
    step) device-bound.  Shapes, adapters and the pack are fixed; new tokens are copied
    into the static input buffer.  Capture uses a private memory pool (the eager step's
    cached blocks are released first)."""

    def __init__(self, trainer: PackedLoraTrainer, tokens: torch.Tensor, warmup: int = 2):
        self.trainer = trainer
        self.tokens = tokens.detach().clone()
        side = torch.cuda.Stream(device=trainer.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):       # warm-up off the capture stream (allocator, cuDNN plans)
            for _ in range(warmup):
                trainer.step(self.tokens)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize(trainer.device)
        torch.cuda.empty_cache()
        self.graph = torch.cuda.CUDAGraph()
        launches0 = ops.launch_count()
        with torch.cuda.graph(self.graph):
            self.losses = trainer.step(self.tokens)
        self.launches_per_step = ops.launch_count() - launches0
        trainer.bank.step_count -= 1        # the capture enqueued nothing; replays count on the device

    def step(self, tokens: torch.Tensor | None = None) -> torch.Tensor:
        """One replay (after copying ``tokens`` into the static input); returns the
        per-adapter losses (device tensor, overwritten by the next replay)."""
        if tokens is not None:
            self.tokens.copy_(tokens, non_blocking=True)
        self.graph.replay()
        ops.count_launches(self.launches_per_step)
        self.trainer.bank.step_count += 1
        return self.losses
