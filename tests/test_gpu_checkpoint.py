"""Checkpoint pool: per-adapter export in PEFT layout
(lora_A = A^T [r][h_in], lora_B = B^T [h_out][r]) round-trips into a fresh bank."""

import pytest
import torch

from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters

pytestmark = pytest.mark.gpu


def test_export_import_round_trip(tmp_path):
    specs, s = bench_adapters("tiny")
    tr = PackedLoraTrainer(PRESETS["tiny"], specs, s, device="cuda")
    tok = tr.synthetic_tokens().cuda()
    for _ in range(2):
        tr.step(tok)
    sd = tr.bank.export_adapter(2)
    path = tmp_path / "adapter2.pt"
    torch.save(sd, path)
    loaded = torch.load(path)
    fresh = PackedLoraTrainer(PRESETS["tiny"], [specs[2]], s, device="cuda", base=tr.base)
    names = {"q": "self_attn.q_proj", "k": "self_attn.k_proj", "v": "self_attn.v_proj", "o": "self_attn.o_proj",
             "gate": "mlp.gate_proj", "up": "mlp.up_proj", "down": "mlp.down_proj"}
    for layer in range(2):
        for t in PRESETS["tiny"].targets():
            pre = f"base_model.model.model.layers.{layer}.{names[t.name]}"
            a, b = loaded[f"{pre}.lora_A.weight"], loaded[f"{pre}.lora_B.weight"]
            assert a.shape == (specs[2].rank, t.h_in) and b.shape == (t.h_out, specs[2].rank)
            fresh.bank.set_adapter(layer, t.name, 0, a.t().cuda(), b.t().cuda())
    r0, r1 = tr.meta.row_offsets[2], tr.meta.row_offsets[3]
    l_packed = tr.forward_backward(tok)[2].item()
    l_solo = fresh.forward_backward(tok[r0:r1].contiguous())[0].item()
    assert abs(l_packed - l_solo) <= 1e-3 * abs(l_packed)


def test_checkpoint_pool_files_round_trip(tmp_path):
    """save_adapter writes PEFT files (safetensors + adapter_config.json with
    lora_alpha = raw alpha * r); restore_adapter into a solo trainer reproduces the
    adapter's packed loss."""
    from paper_2508_02932_b200.checkpoint import load_adapter, restore_adapter, save_adapter
    specs, s = bench_adapters("tiny")
    tr = PackedLoraTrainer(PRESETS["tiny"], specs, s, device="cuda")
    tok = tr.synthetic_tokens().cuda()
    for _ in range(2):
        tr.step(tok)
    out = save_adapter(tr, 1, tmp_path, config_id="cfg-1")
    state, cfg = load_adapter(out)
    assert cfg["r"] == specs[1].rank and cfg["lora_alpha"] == specs[1].alpha * specs[1].rank
    assert cfg["optimizer_steps"] == 2 and len(cfg["target_modules"]) == 7
    solo = PackedLoraTrainer(PRESETS["tiny"], [specs[1]], s, device="cuda", base=tr.base)
    restore_adapter(solo, 0, state)
    r0, r1 = tr.meta.row_offsets[1], tr.meta.row_offsets[2]
    l_packed = tr.forward_backward(tok)[1].item()
    l_solo = solo.forward_backward(tok[r0:r1].contiguous())[0].item()
    assert abs(l_packed - l_solo) <= 1e-3 * abs(l_packed)
