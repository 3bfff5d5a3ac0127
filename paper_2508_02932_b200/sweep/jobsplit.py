"""The planner's split of one packed workload (a bench configuration) over the GPUs
of a box: which adapters every rank trains.

PLoRA's job-level parallelism (reference planner.py:124-130,
simulator.py:109-125): adapters are independent, so a packed workload spread over g
GPUs is g independent packed jobs with no data-path collective.  ``split_adapters``
turns the bench adapters (model.bench_adapters) into planner configurations, costs
them with the B200-calibrated time model (``B200_TIME_MODEL``, fitted from the C5
profile run, profiles/r1s2_sweep_c5.json: base 18.6 ms, 2.76e-8 s per unit of load
r*b*s + 1024*b*s, rel-RMSE 0.019) and the trainer's memory model, packs them with
``plan_split`` and places the jobs with ``place`` (job k -> device k).
"""

from __future__ import annotations

from dataclasses import dataclass

from .costmodel import MemoryContext, TimeModel
from .planner import JobQueue, Placement, place, plan_split
from .workload import STATE_BYTES_PLORA, GpuPool, LoraConfig, model_spec_from_config

# (base seconds, seconds per unit of load, token weight) -- profiles/r1s2_sweep_c5.json
B200_TIME_MODEL = (0.018605064705778624, 2.7642496096777574e-08, 1024.0)
# saved activations per token of the packed trainer (measured peak at T = 32768, C3)
ACT_BYTES_PER_TOKEN = 2.95e6


def b200_time_model(gpu_count: int) -> TimeModel:
    b, m, w = B200_TIME_MODEL
    return TimeModel(coeffs={d: (b * d, m * d) for d in (1, 2, 4, 8) if d <= max(1, gpu_count)}, token_weight=w)


def adapter_configs(cfg_name: str) -> list:
    """The bench adapters of ``cfg_name`` as planner configurations ``<cfg>-a<i>``."""
    from ..model import bench_adapters

    specs, s = bench_adapters(cfg_name)
    return [LoraConfig(f"{cfg_name}-a{i:02d}", rank=sp.rank, alpha=float(sp.alpha), batch_size=sp.batch,
                       learning_rate=sp.lr, seq_len=s, train_steps=50) for i, sp in enumerate(specs)]


def memory_context(cfg_name: str, gpu_count: int, configs, mem_gb: float = 178.0) -> MemoryContext:
    from ..model import PRESETS

    half = ACT_BYTES_PER_TOKEN / 2 / 2
    model = model_spec_from_config(PRESETS[cfg_name], c_prec=2, act_coeffs=(0.0, half, half),
                                   state_bytes=STATE_BYTES_PLORA)
    return MemoryContext(model, GpuPool(gpu_count, int(mem_gb * 1e9), load_factor=0.9), configs)


@dataclass(frozen=True)
class Split:
    queue: JobQueue
    placement: Placement
    adapters: tuple          # per device: tuple of bench-adapter indices (ascending)

    def describe(self) -> str:
        return "planner-split " + "/".join(str(len(a)) for a in self.adapters)


def split_adapters(cfg_name: str, gpu_count: int, mem_gb: float = 178.0) -> Split:
    """Adapters per device for ``gpu_count`` GPUs (every adapter exactly once)."""
    configs = adapter_configs(cfg_name)
    index = {c.id: i for i, c in enumerate(configs)}
    tm = b200_time_model(gpu_count)
    mem = memory_context(cfg_name, gpu_count, configs, mem_gb)
    queue = plan_split(gpu_count, configs, tm, mem)
    pl = place(queue, gpu_count)
    per_dev: list = [() for _ in range(gpu_count)]
    for job in queue.jobs():
        (dev,) = pl.devices[job.id]
        per_dev[dev] = tuple(sorted(index[c] for c in job.configs))
    return Split(queue=queue, placement=pl, adapters=tuple(per_dev))
