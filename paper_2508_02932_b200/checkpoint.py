"""Checkpoint pool (PLoRA's "Checkpoint Pool"; absent from the reference):
when a packed job finishes, every adapter it trained is written out on its own, in the
PEFT layout, so each hyper-parameter configuration of a sweep leaves a standalone
LoRA checkpoint.

  <dir>/<config id>/adapter_model.safetensors   lora_A = A^T [r][h_in], lora_B = B^T [h_out][r]
  <dir>/<config id>/adapter_config.json         r, lora_alpha, target_modules, ...

Scaling: the reference computes y = x W + alpha (x A) B with the RAW alpha
(lorapack.py:8); PEFT scales by lora_alpha / r, so lora_alpha = alpha * r is written
(raw_alpha is recorded beside it).  Tensor-parallel jobs: the sharded factors
(column-parallel B, row-parallel A) are all-gathered over the job's TP group and rank 0
writes the files.
"""

from __future__ import annotations

import json
from pathlib import Path

import torch

PEFT_NAMES = {"q": "self_attn.q_proj", "k": "self_attn.k_proj", "v": "self_attn.v_proj", "o": "self_attn.o_proj",
              "gate": "mlp.gate_proj", "up": "mlp.up_proj", "down": "mlp.down_proj"}


def _full_factor(trainer, layer: int, target: str, kind: str, i: int) -> torch.Tensor:
    """Adapter i's fp32 master block [rows][r] of (layer, target, kind), gathered over the
    TP group when this rank holds only a shard."""
    bank = trainer.bank
    r = trainer.meta.ranks[i]
    blk = bank.block(bank.P, layer, target, kind, i)[:, :r].contiguous()
    tp = trainer.tp
    if tp is None or trainer.shard.replicated(target, kind):
        return blk
    full = torch.empty((blk.shape[0] * tp.world, r), dtype=blk.dtype, device=blk.device)
    tp.all_gather_(full, blk)
    return full


def adapter_state(trainer, i: int) -> dict:
    """PEFT-layout state dict (CPU fp32) of adapter i of a PackedLoraTrainer (TP-aware)."""
    out = {}
    for layer in range(trainer.cfg.n_layers):
        for t in trainer.cfg.targets():
            pre = f"base_model.model.model.layers.{layer}.{PEFT_NAMES.get(t.name, t.name)}"
            a = _full_factor(trainer, layer, t.name, "A", i)      # A   [h_in][r]
            b = _full_factor(trainer, layer, t.name, "B", i)      # B^T [h_out][r]
            out[f"{pre}.lora_A.weight"] = a.t().contiguous().cpu()
            out[f"{pre}.lora_B.weight"] = b.contiguous().cpu()
    return out


def save_adapter(trainer, i: int, directory, config_id: str | None = None, extra: dict | None = None):
    """Write adapter i as <directory>/<config_id> (PEFT files); on TP jobs every rank must
    call it (collective), rank 0 writes.  Returns the output directory (or None on other ranks)."""
    from safetensors.torch import save_file

    state = adapter_state(trainer, i)
    if trainer.tp is not None and trainer.tp.rank != 0:
        return None
    spec = trainer.specs[i]
    out = Path(directory) / (config_id or f"adapter{i}")
    out.mkdir(parents=True, exist_ok=True)
    save_file(state, str(out / "adapter_model.safetensors"))
    cfg = {"peft_type": "LORA", "task_type": "CAUSAL_LM", "base_model_name_or_path": trainer.cfg.name,
           "r": spec.rank, "lora_alpha": spec.alpha * spec.rank, "raw_alpha": spec.alpha, "lora_dropout": 0.0,
           "bias": "none", "target_modules": [PEFT_NAMES[t.name].split(".")[-1] for t in trainer.cfg.targets()],
           "learning_rate": spec.lr, "optimizer_steps": int(trainer.bank.hp[i, 2].item())}
    cfg.update(extra or {})
    (out / "adapter_config.json").write_text(json.dumps(cfg, indent=1))
    return out


def load_adapter(directory) -> tuple[dict, dict]:
    """(state dict, adapter_config) of a saved adapter."""
    from safetensors.torch import load_file

    d = Path(directory)
    return load_file(str(d / "adapter_model.safetensors")), json.loads((d / "adapter_config.json").read_text())


def restore_adapter(trainer, i: int, state: dict):
    """Load a PEFT-layout state into adapter i of an (unsharded) trainer."""
    for layer in range(trainer.cfg.n_layers):
        for t in trainer.cfg.targets():
            pre = f"base_model.model.model.layers.{layer}.{PEFT_NAMES.get(t.name, t.name)}"
            a = state[f"{pre}.lora_A.weight"].to(trainer.device)
            b = state[f"{pre}.lora_B.weight"].to(trainer.device)
            trainer.bank.set_adapter(layer, t.name, i, a.t(), b.t())
