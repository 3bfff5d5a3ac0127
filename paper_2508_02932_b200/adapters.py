"""Adapter state for a packed job: fp32 master weights, gradients and Adam moments
plus the bf16 compute shadows the kernels read -- all in flat HBM buffers.

Layout:
  * one *region* per (layer, target, A|B).  A region of a target with input
    width h_in and output width h_out holds, for every adapter i, the block
    A_i [h_in][rpad16_i] (down-projection, reference ``down`` d x r) or
    B_i^T [h_out][rpad16_i] (up-projection transposed, reference ``up`` r x k),
    adapter blocks back to back (offset rows * rpad_off[i]).  The zero padding
    columns r_i..rpad16_i stay exactly zero through training (their gradient is
    identically zero and AdamW keeps 0 at 0).
  * fp32 P (master), G (grad), M, V share that layout: the per-adapter AdamW
    kernel (K7) streams them once per step.
  * bf16 shadows: A_sh [n][h_in][64nb] and Bt_sh [n][h_out][64nb] per target
    (rank padded to 64 so one TMA box covers it); rewritten by K7.

Memory per parameter: 16 B fp32 state + 2 B shadow (x rpad64/rpad16).
Reference: costmodel.py:56-58 (GRAD_COPIES=1, OPT_COPIES=2) models exactly this
state; the per-config learning rate is workload.py:135-136,144.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from .meta import PackMeta


@dataclass(frozen=True)
class Target:
    name: str
    h_in: int
    h_out: int


@dataclass
class Region:
    layer: int
    target: str
    kind: str        # "A" or "B"
    rows: int        # h_in for A, h_out for B
    p_off: int       # element offset into P/G/M/V
    sh_off: int      # element offset into the bf16 shadow buffer


class AdapterBank:
    """All adapters' LoRA state for one packed job on one device."""

    def __init__(self, meta: PackMeta, n_layers: int, targets: Sequence[Target], lrs: Sequence[float],
                 weight_decay: float | Sequence[float] = 0.0, device="cuda",
                 betas=(0.9, 0.999), eps: float = 1e-8, seeds: Sequence[int] | None = None,
                 init: str = "bench", a_scale: float | None = None, b_std: float | Sequence[float] = 0.02,
                 chunk_elems: int = 8192, full_targets: Sequence[Target] | None = None, shard=None):
        self.meta = meta
        self.n = meta.n_adapters
        self.n_layers = n_layers
        self.targets = list(targets)
        # tensor parallel (tp.py): ``targets`` are this rank's local shapes; the initial
        # values are drawn at the full shapes (same RNG stream as an unsharded bank) and
        # sliced, so TP shards are exact slices of the unsharded adapters.
        self.full_targets = list(full_targets) if full_targets is not None else self.targets
        self.shard = shard
        self.device = torch.device(device)
        self.betas = betas
        self.eps = eps
        self.step_count = 0
        R16 = meta.rpad16_total
        R64 = meta.rpad64
        regions: dict[tuple[int, str, str], Region] = {}
        p_off = sh_off = 0
        for layer in range(n_layers):
            for t in self.targets:
                for kind, rows in (("A", t.h_in), ("B", t.h_out)):
                    regions[(layer, t.name, kind)] = Region(layer, t.name, kind, rows, p_off, sh_off)
                    p_off += rows * R16
                    sh_off += self.n * rows * R64
        self.regions = regions
        self.numel = p_off
        self.shadow_numel = sh_off
        dev = self.device
        self.P = torch.zeros(p_off, dtype=torch.float32, device=dev)
        self.G = torch.zeros(p_off, dtype=torch.float32, device=dev)
        self.M = torch.zeros(p_off, dtype=torch.float32, device=dev)
        self.V = torch.zeros(p_off, dtype=torch.float32, device=dev)
        self.shadow = torch.zeros(sh_off, dtype=torch.bfloat16, device=dev)
        wd = [float(weight_decay)] * self.n if np.isscalar(weight_decay) else [float(w) for w in weight_decay]
        self.hp = torch.tensor([[float(lr), w, 0.0, 0.0] for lr, w in zip(lrs, wd)], dtype=torch.float32,
                               device=dev)
        self.chunks = self._build_chunks(chunk_elems)
        self.trainable_params = sum(r.rows for r in regions.values()) * sum(meta.ranks)
        self._init(seeds or [100 + i for i in range(self.n)], init, a_scale, b_std)

    # ------------------------------------------------------------------ views
    def block(self, buf: torch.Tensor, layer: int, target: str, kind: str, i: int) -> torch.Tensor:
        """Adapter i's [rows][rpad16_i] block of a fp32 buffer (P, G, M or V)."""
        reg = self.regions[(layer, target, kind)]
        ro = self.meta.rpad_off
        s = reg.p_off + reg.rows * int(ro[i])
        return buf[s: s + reg.rows * int(ro[i + 1] - ro[i])].view(reg.rows, int(ro[i + 1] - ro[i]))

    def region_flat(self, buf: torch.Tensor, layer: int, target: str, kind: str) -> torch.Tensor:
        reg = self.regions[(layer, target, kind)]
        return buf[reg.p_off: reg.p_off + reg.rows * self.meta.rpad16_total]

    def shadow_of(self, layer: int, target: str, kind: str) -> torch.Tensor:
        """bf16 shadow [n][rows][64nb] of one region (A_sh or Bt_sh)."""
        reg = self.regions[(layer, target, kind)]
        R64 = self.meta.rpad64
        return self.shadow[reg.sh_off: reg.sh_off + self.n * reg.rows * R64].view(self.n, reg.rows, R64)

    def down(self, layer: int, target: str, i: int) -> torch.Tensor:
        """Reference-layout A_i (d x r) view of the master weights."""
        return self.block(self.P, layer, target, "A", i)[:, : self.meta.ranks[i]]

    def up(self, layer: int, target: str, i: int) -> torch.Tensor:
        """Reference-layout B_i (r x k) of the master weights (a transposed view)."""
        return self.block(self.P, layer, target, "B", i)[:, : self.meta.ranks[i]].t()

    # ------------------------------------------------------------------ setup
    def _build_chunks(self, chunk_elems: int) -> torch.Tensor:
        m = self.meta
        R64 = m.rpad64
        rows_list = []
        for reg in self.regions.values():
            for i in range(self.n):
                rp = int(m.rpad_off[i + 1] - m.rpad_off[i])
                step = max(1, chunk_elems // rp)
                base_p = reg.p_off + reg.rows * int(m.rpad_off[i])
                base_s = reg.sh_off + i * reg.rows * R64
                r0 = np.arange(0, reg.rows, step, dtype=np.int64)
                nr = np.minimum(step, reg.rows - r0)
                c = np.empty((len(r0), 4), dtype=np.int64)
                c[:, 0] = base_p + r0 * rp
                c[:, 1] = base_s + r0 * R64
                c[:, 2] = nr | (np.int64(rp) << 32)
                c[:, 3] = np.int64(i) | (np.int64(R64) << 32)
                rows_list.append(c)
        table = np.concatenate(rows_list, axis=0)
        return torch.from_numpy(table).to(self.device)

    def _init(self, seeds, init: str, a_scale, b_std):
        """A_i ~ U(+-1/sqrt(h_in)), B_i ~ N(0, b_std^2) (nonzero, so Case 3 is exercised
        from step 1), seeded per adapter."""
        m = self.meta
        b_stds = [float(b_std)] * self.n if np.isscalar(b_std) else [float(b) for b in b_std]
        for i, seed in enumerate(seeds):
            g = torch.Generator(device=self.device).manual_seed(int(seed))
            for layer in range(self.n_layers):
                for t, ft in zip(self.targets, self.full_targets):
                    r = m.ranks[i]
                    bound = a_scale if a_scale is not None else 1.0 / math.sqrt(ft.h_in)
                    a = (torch.rand(ft.h_in, r, generator=g, device=self.device) * 2 - 1) * bound
                    b = torch.randn(ft.h_out, r, generator=g, device=self.device) * b_stds[i]
                    if self.shard is not None:
                        a = a[self.shard.lora_rows(t.name, "A", ft.h_in, ft.h_out)]
                        b = b[self.shard.lora_rows(t.name, "B", ft.h_in, ft.h_out)]
                    self.block(self.P, layer, t.name, "A", i)[:, :r] = a
                    self.block(self.P, layer, t.name, "B", i)[:, :r] = b
        self.refresh_shadow()

    def refresh_shadow(self):
        """Rewrite every bf16 shadow from the fp32 masters (K7 does this after each step)."""
        m = self.meta
        for (layer, tname, kind), reg in self.regions.items():
            sh = self.shadow_of(layer, tname, kind)
            sh.zero_()
            for i in range(self.n):
                rp = int(m.rpad_off[i + 1] - m.rpad_off[i])
                sh[i, :, :rp] = self.block(self.P, layer, tname, kind, i).to(torch.bfloat16)

    def set_adapter(self, layer: int, target: str, i: int, down: torch.Tensor, up: torch.Tensor):
        """Load reference-layout A (d x r) and B (r x k) for adapter i (updates the shadow)."""
        r = self.meta.ranks[i]
        self.block(self.P, layer, target, "A", i)[:, :r] = down.to(self.P)
        self.block(self.P, layer, target, "B", i)[:, :r] = up.t().to(self.P)
        for kind in ("A", "B"):
            rp = int(self.meta.rpad_off[i + 1] - self.meta.rpad_off[i])
            self.shadow_of(layer, target, kind)[i, :, :rp] = self.block(self.P, layer, target, kind, i).to(
                torch.bfloat16)

    # ------------------------------------------------------------------ optimizer
    def adamw_step(self):
        """K7: one fused per-adapter AdamW launch over every region of every adapter.  The
        step counts live on the device (hp[i].z, incremented here by a device op), so the
        launch sequence is replayable by a CUDA graph (model.GraphedStep)."""
        from . import ops

        self.step_count += 1
        self.hp[:, 2] += 1.0
        ops.adamw(self.chunks, self.P, self.G, self.M, self.V, self.shadow, self.hp, 0,
                  self.betas[0], self.betas[1], self.eps, algo_params=self.trainable_params)

    def state_bytes(self) -> int:
        return 4 * 4 * self.numel + 2 * self.shadow_numel

    # ------------------------------------------------------------------ checkpoint pool
    def export_adapter(self, i: int) -> dict[str, torch.Tensor]:
        """PEFT-layout state dict of adapter i (lora_A = A^T [r][h_in], lora_B = B^T [h_out][r])."""
        out = {}
        names = {"q": "self_attn.q_proj", "k": "self_attn.k_proj", "v": "self_attn.v_proj",
                 "o": "self_attn.o_proj", "gate": "mlp.gate_proj", "up": "mlp.up_proj", "down": "mlp.down_proj"}
        for layer in range(self.n_layers):
            for t in self.targets:
                pre = f"base_model.model.model.layers.{layer}.{names.get(t.name, t.name)}"
                out[f"{pre}.lora_A.weight"] = self.down(layer, t.name, i).t().contiguous().cpu()
                out[f"{pre}.lora_B.weight"] = self.up(layer, t.name, i).t().contiguous().cpu()
        return out
