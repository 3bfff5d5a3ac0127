"""bench.py multi-GPU plumbing: the planner split of the workload over the ranks, the
self-launch of N ranks (torch.distributed.run) and the reference arm -- on CPU; the
GPU run of two ranks sharing one device is marked gpu."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2508_02932_b200.model import bench_adapters  # noqa: E402
from paper_2508_02932_b200.sweep.jobsplit import split_adapters  # noqa: E402


def _bench(*args, env=None, timeout=300):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, env=e, cwd=ROOT)


@pytest.mark.parametrize("cfg", ["tiny", "qwen2.5-3b", "llama-3.1-8b"])
@pytest.mark.parametrize("gpus", [1, 2, 4, 8])
def test_split_covers_every_adapter_once(cfg, gpus):
    specs, _ = bench_adapters(cfg)
    sp = split_adapters(cfg, gpus)
    assert len(sp.adapters) == gpus
    flat = sorted(i for a in sp.adapters for i in a)
    assert flat == list(range(len(specs)))
    # placement: every job on its own device, all in the first (only) batch
    assert len(sp.queue.batches) == 1
    devs = sorted(d for j in sp.queue.jobs() for d in sp.placement.devices[j.id])
    assert devs == list(range(len(sp.queue.jobs())))


def test_c3_split_balances_tokens():
    """C3's 32 sequences: 16 / 8 / 4 per GPU at 2 / 4 / 8 GPUs (LPT on the calibrated load)."""
    specs, _ = bench_adapters("llama-3.1-8b")
    for gpus, per in ((2, 16), (4, 8), (8, 4)):
        sp = split_adapters("llama-3.1-8b", gpus)
        assert [sum(specs[i].batch for i in a) for a in sp.adapters] == [per] * gpus


def test_split_is_deterministic():
    assert split_adapters("llama-3.1-8b", 8) == split_adapters("llama-3.1-8b", 8)


def test_relaunch_two_ranks_reference_arm():
    """--gpus 2 outside torchrun starts two ranks; rank 0 alone prints the reference line
    and uses every host thread although torchrun exports OMP_NUM_THREADS=1."""
    r = _bench("--gpus", "2", "--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "1")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["cores"] == (os.cpu_count() or 1)
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_mismatch_fails_loudly():
    r = _bench("--gpus", "1", "--impl", "reference", "--config", "tiny", env={"WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=2" in (r.stderr + r.stdout)


@pytest.mark.gpu
def test_two_ranks_split_on_one_gpu():
    """The planner-split multi-GPU bench path end to end: two ranks (sharing the one GPU of
    the box, so the control plane falls back to gloo), each training its placed job."""
    r = _bench("--gpus", "2", "--config", "tiny", "--steps", "2", "--warmup", "1", "--no-cpu-baseline",
               timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["parallelism"].startswith("planner-split")
    ranks = d["ranks"]
    assert [x["rank"] for x in ranks] == [0, 1] and all(x["world"] == 2 for x in ranks)
    assert sorted(i for x in ranks for i in x["adapters"]) == [0, 1, 2, 3]
    assert sum(x["tokens"] for x in ranks) == 768
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
