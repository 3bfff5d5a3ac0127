"""Packed multi-LoRA training throughput (tokens/s, summed over adapters) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama-3.1-8b] [--impl ours|reference]

Workload (BASELINE.json configs[2]): Llama-3.1-8B shapes,
random-init frozen bf16 base, 16 packed LoRA adapters on all 7 targets (ranks
8/16/32/64 x4, raw alpha = r*{0.25,1,2,4}, b_i in {1,2,4} sequences of 1024 tokens,
T = 32768 tokens/step/GPU), synthetic uniform tokens.  One step = forward +
backward + fused per-adapter AdamW.  Multi-GPU: one process per GPU, each rank
trains its own independent packed job (the planner's job-level parallelism; no
data-path collective) -> "scaling": "weak".

--impl reference times the reference algorithm (the oracle port of
lorasweep.packed_forward/packed_backward, numpy fp64, all host cores) on a bounded
sample of the same workload (the 7 LoRA linears of one layer at 1/16 of the tokens,
scaled linearly to the full model and step).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "packed LoRA training tokens/sec/GPU (sum over adapters); sweep makespan vs CPU ref"


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"tflops_burst": d["bf16_tflops"], "tflops_sustained": d["bf16_tflops_sustained"],
                "hbm_gbs": d["hbm_gbs"], "source": "measured"}
    return {"tflops_burst": 1590.0, "tflops_sustained": 1400.0, "hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference(cfg_name: str, frac: float | None = None) -> dict:
    """Reference CPU path (oracle port of lorasweep.packed_forward/backward, fp64
    numpy/OpenBLAS on all host cores) over the 7 LoRA linears of ONE layer at a
    fraction f of the step's tokens; throughput scaled by 1/(L) (cost linear in T)."""
    import numpy as np

    from oracle import lorapack_oracle as O
    from paper_2508_02932_b200.model import PRESETS, bench_adapters

    cfg = PRESETS[cfg_name]
    specs, s = bench_adapters(cfg_name)
    if frac is None:
        frac = {"tiny": 1.0, "qwen2.5-3b": 1 / 8, "llama-3.1-8b": 1 / 16, "qwen2.5-32b": 1 / 32}[cfg_name]
    rng = np.random.default_rng(0)
    toks = [max(1, int(sp.batch * s * frac)) for sp in specs]
    T = sum(toks)
    work = []
    for t in cfg.targets():
        downs = [rng.uniform(-1, 1, (t.h_in, sp.rank)) / np.sqrt(t.h_in) for sp in specs]
        ups = [rng.standard_normal((sp.rank, t.h_out)) * 0.02 for sp in specs]
        xs = [rng.standard_normal((n, t.h_in)) for n in toks]
        dys = [rng.standard_normal((n, t.h_out)) for n in toks]
        w = rng.standard_normal((t.h_in, t.h_out)) * 0.02
        work.append((O.pack(downs, ups, [sp.alpha for sp in specs], xs), w, dys))
    # warm the BLAS threads on a small problem, then time the layer once
    O.packed_backward(*work[0][:2], work[0][2]) if T <= 4096 else O.packed_forward(work[0][0], work[0][1])
    t0 = time.perf_counter()
    for p, w, dys in work:
        O.packed_forward(p, w)
        O.packed_backward(p, w, dys)
    dt = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        blas = max((i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"), default=1)
    except Exception:  # pragma: no cover
        blas = os.cpu_count() or 1
    tok_s = T / (dt * cfg.n_layers)
    return {"value": tok_s, "unit": "tokens/s", "cores": int(blas), "kind": "port",
            "sample": (f"oracle port of lorasweep packed_forward+packed_backward (fp64 numpy, {blas} BLAS threads), "
                       f"7 LoRA linears of 1 of {cfg.n_layers} layers at {T} tokens (1/{round(1 / frac)} of the "
                       f"{sum(sp.batch for sp in specs) * s}-token step), {dt:.2f} s, scaled by 1/L; attention, norms, "
                       f"lm_head and optimizer excluded (the reference implements none)"),
            "host_cpus": os.cpu_count()}


def dropin_api_sample(cfg_name: str) -> dict:
    """The reference-facing operator API itself (paper_2508_02932_b200.lorapack:
    pack_adapters -> packed_forward -> packed_backward, float64 numpy in and out, the
    device path in between) on the SAME sample as cpu_baseline (7 LoRA linears of one
    layer at 1/16 of the step's tokens), scaled by 1/L the same way -- an API-for-API
    comparison with the reference arm.  The drop-in is stateless (base weight and
    adapters cross PCIe on every call, as numpy arrays in the reference signature), so
    it is transfer-bound; the training path keeps everything resident."""
    import numpy as np

    from paper_2508_02932_b200 import lorapack as L
    from paper_2508_02932_b200.model import PRESETS, bench_adapters

    cfg = PRESETS[cfg_name]
    specs, s = bench_adapters(cfg_name)
    frac = {"tiny": 1.0, "qwen2.5-3b": 1 / 8, "llama-3.1-8b": 1 / 16, "qwen2.5-32b": 1 / 32}[cfg_name]
    rng = np.random.default_rng(0)
    toks = [max(1, int(sp.batch * s * frac)) for sp in specs]
    T = sum(toks)
    work = []
    for t in cfg.targets():
        ads = [L.AdapterWeights(rng.uniform(-1, 1, (t.h_in, sp.rank)) / np.sqrt(t.h_in),
                                rng.standard_normal((sp.rank, t.h_out)) * 0.02, sp.alpha) for sp in specs]
        xs = [rng.standard_normal((n, t.h_in)) for n in toks]
        dys = [rng.standard_normal((n, t.h_out)) for n in toks]
        work.append((ads, xs, rng.standard_normal((t.h_in, t.h_out)) * 0.02, dys))
    for ads, xs, w, dys in work:   # warm-up: library load, first launches, pinned host blocks per shape
        packed = L.pack_adapters(ads, xs)
        L.packed_forward(packed, w)
        L.packed_backward(packed, w, dys)
    t0 = time.perf_counter()
    for ads, xs, w, dys in work:
        packed = L.pack_adapters(ads, xs)
        L.packed_forward(packed, w)
        L.packed_backward(packed, w, dys)
    dt = time.perf_counter() - t0
    return {"value": T / (dt * cfg.n_layers), "unit": "tokens/s",
            "sample": f"lorapack drop-in (numpy fp64 in/out), same 7-linear {T}-token sample as cpu_baseline, "
                      f"{dt:.2f} s, scaled by 1/L"}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    base = cpu_reference(args.config)
    from paper_2508_02932_b200.model import PRESETS, bench_adapters
    specs, s = bench_adapters(args.config)
    T = sum(sp.batch for sp in specs) * s
    # per step: the sampled layer's work, scaled; --steps/--warmup bound the run
    vals = [base["value"]]
    for _ in range(max(0, args.steps - 1)):
        if time.perf_counter() - _T0 > 120:
            break
        vals.append(cpu_reference(args.config)["value"])
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": len(vals),
            "warmup": args.warmup, "ms_per_step": 1000.0 * T / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{PRESETS[args.config].name} packed LoRA, {len(specs)} adapters, T={T}",
                       "model": PRESETS[args.config].name, "global_batch": T // s, "seq_len": s,
                       "parallelism": "cpu"},
            "cpu_baseline": {**base, "value": v},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


_T0 = time.perf_counter()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="llama-3.1-8b")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tp", type=int, default=None,
                    help="tensor-parallel degree per packed job (config C4 default: all GPUs); "
                         "world/tp independent jobs run side by side")
    ap.add_argument("--tp-comm", default="torch", choices=["torch", "abi"],
                    help="TP all-reduce through torch.distributed (NCCL) or libplora's C-ABI (plora_tp_*, NCCL)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
    import torch
    import torch.distributed as dist

    from paper_2508_02932_b200 import _lib, ops
    from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters

    from paper_2508_02932_b200.tp import AbiNcclComm, DistComm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _lib.check(_lib.lib().plora_device_check(), "device check")

    cfg = PRESETS[args.config]
    tp = args.tp or (world if args.config == "qwen2.5-32b" else 1)
    if world % tp:
        raise SystemExit(f"--tp {tp} must divide the world size {world}")
    if args.config == "qwen2.5-32b" and tp < 8:
        raise SystemExit("C4 (Qwen2.5-32B, 32 adapters) needs a tensor-parallel group of 8 GPUs "
                         "(one 180 GB B200 holds a TP=8 shard: tools/c4_shard_bench.py)")
    n_jobs = world // tp
    job = rank // tp
    comm = None
    if tp > 1:   # one NCCL group per packed job (Megatron TP over NVLink), jobs side by side
        groups = [dist.new_group(list(range(j * tp, (j + 1) * tp))) for j in range(n_jobs)]
        if args.tp_comm == "abi":
            comm = AbiNcclComm(rank - job * tp, tp, group=groups[job])
        else:
            comm = DistComm(groups[job])
    specs, s = bench_adapters(args.config)
    n = len(specs)
    trainer = PackedLoraTrainer(cfg, specs, s, device="cuda", adapter_seeds=[100 + i + 1000 * job for i in range(n)],
                                tp=comm)
    T = trainer.T
    tokens_host = trainer.synthetic_tokens(seed_base=1000 + 100000 * job).pin_memory()
    tokens = tokens_host.to("cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        trainer.step(tokens)
    barrier()

    # ---------------------------------------------------------------- timed region (device)
    timer = ops.KernelTimer()
    launches0 = ops.launch_count()
    profile_range = os.environ.get("PLORA_PROFILE_RANGE") == "1"   # ncu --profile-from-start off
    with ClockSampler(local) as clocks:
        barrier()
        if profile_range:
            torch.cuda.profiler.start()
        ops.set_timer(timer)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            trainer.step(tokens)
        e1.record()
        ops.set_timer(None)
        barrier()
        if profile_range:
            torch.cuda.profiler.stop()
    launches = ops.launch_count() - launches0
    ms = e0.elapsed_time(e1)
    kstats = timer.summary()
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    value = n_jobs * T * args.steps / (ms_max / 1000.0)
    losses_dev = trainer.losses.clone()

    # ---------------------------------------------------------------- end-to-end (public API, host buffers)
    barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(args.steps):
        tokens.copy_(tokens_host, non_blocking=True)
        losses_host = trainer.step(tokens).cpu()
    e3.record()
    barrier()
    ms_e2e = e2.elapsed_time(e3)
    if world > 1:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    e2e_value = n_jobs * T * args.steps / (ms_e2e / 1000.0)

    peaks = _peaks()
    g = kstats.get("gemm", {"ms": 0.0, "flops": 0.0, "launches": 0})
    achieved = g["flops"] / (g["ms"] / 1000.0) / 1e12 if g["ms"] else 0.0
    traffic = None
    prof = ROOT / "profiles" / "gemm_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    kernels = {}
    shapes = {}
    for kind, d in kstats.items():
        sec = d["ms"] / 1000.0
        if "[" in kind:   # per-shape GEMM detail
            shapes[kind[kind.index("[") + 1:-1]] = {"launches": d["launches"], "ms": round(d["ms"], 2),
                                                   "tflops": round(d["flops"] / sec / 1e12, 1)}
            continue
        kernels[kind] = {"launches": d["launches"], "ms_total": round(d["ms"], 3),
                         "share_of_step": round(d["ms"] / ms, 4)}
        if d["flops"]:
            kernels[kind]["tflops"] = round(d["flops"] / sec / 1e12, 1)
        if d["bytes"]:
            kernels[kind]["hbm_gbs"] = round(d["bytes"] / sec / 1e9, 1)
            kernels[kind]["hbm_frac"] = round(d["bytes"] / sec / 1e9 / peaks["hbm_gbs"], 3)
    base_tf = value / world * cfg.base_flops_per_token() / 1e12   # per GPU
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.tp is not None or tp == 1 else "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform tokens, random-init weights)",
        "config": {"workload": f"{cfg.name} packed LoRA training, {n} adapters (ranks 8/16/32/64), all 7 targets, "
                               f"T={T} tokens/step/GPU, fwd+bwd+per-adapter AdamW",
                   "model": cfg.name, "global_batch": n_jobs * T // s, "seq_len": s,
                   "parallelism": f"jobs{n_jobs}" + (f"xtp{tp}" if tp > 1 else ""),
                   "adapters": n, "l2": "working set (~100 GB activations) >> 126 MB L2; no flush needed"},
        "roofline": {"bound": "tensor", "kernel": "tcgen05 base GEMM + fused LoRA expand (K1/K2b/K6, lm_head)",
                     "achieved": round(achieved, 1), "peak": peaks["tflops_sustained"], "unit": "TFLOP/s",
                     "frac": round(achieved / peaks["tflops_sustained"], 4), "traffic": traffic,
                     "peak_source": f"{peaks['source']} bf16 sustained (kernel timed inside a long step)",
                     "step_base_gemm_tflops": round(base_tf, 1),
                     "step_frac_of_burst_peak": round(base_tf / peaks["tflops_burst"], 4)},
        "kernels": kernels,
        "gemm_shapes": shapes,
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": tokens_host.numel() * tokens_host.element_size(),
                "d2h_bytes_per_step": losses_host.numel() * losses_host.element_size()},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "losses": [round(float(x), 4) for x in losses_dev.tolist()],
        "mem_peak_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference(args.config)
        line["dropin_api"] = dropin_api_sample(args.config)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
