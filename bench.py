"""Packed multi-LoRA training throughput (tokens/s, summed over adapters) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama-3.1-8b]
                    [--scaling split|weak] [--impl ours|reference]

Workload (BASELINE.json configs[2]): Llama-3.1-8B shapes,
random-init frozen bf16 base, 16 packed LoRA adapters on all 7 targets (ranks
8/16/32/64 x4, raw alpha = r*{0.25,1,2,4}, b_i in {1,2,4} sequences of 1024 tokens,
T = 32768 tokens/step), synthetic uniform tokens.  One step = forward + backward +
fused per-adapter AdamW.

Multi-GPU (one process per GPU; ``--gpus N`` outside torchrun starts the N ranks
itself): by default the planner splits the workload's adapters over the N GPUs
(sweep/jobsplit.py: ``plan_split`` + ``place``, BASELINE configs[2] "via planner"),
so rank r trains the packed job placed on device r -- independent jobs, no data-path
collective, fixed total work ("scaling": "strong"); ``--scaling weak`` replicates the
whole workload on every GPU.  ``--config qwen2.5-32b`` (C4) runs one tensor-parallel
job over all GPUs (tp.py, NCCL).  value = tokens of all ranks / the max over ranks of
the device-timed region.

--impl reference times the reference's own CPU implementation (lorasweep from
baseline/_ref: pack_adapters + packed_forward + packed_backward, numpy fp64, all host
cores) on a bounded sample of the same workload (the 7 LoRA linears of one layer at
1/16 of the tokens, scaled linearly to the full model and step).
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


def _ref_lorapack():
    """The reference's own lorapack (lorasweep installed into baseline/_ref, git-ignored,
    travels to the box) -- or None when it is not installed."""
    ref = ROOT / "baseline" / "_ref"
    if (ref / "lorasweep" / "lorapack.py").exists() and str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import lorasweep.lorapack as RL   # noqa: N812
    except ImportError:
        return None
    return RL


def _cpu_sample(cfg_name: str, frac: float | None):
    """The bounded CPU sample of one training step: the 7 LoRA linears of ONE layer at a
    fraction f of the step's tokens (fp64, seeded)."""
    import numpy as np

    from paper_2508_02932_b200.model import PRESETS, bench_adapters

    cfg = PRESETS[cfg_name]
    specs, s = bench_adapters(cfg_name)
    if frac is None:
        frac = {"tiny": 1.0, "tiny-qwen": 1.0, "qwen2.5-3b": 1 / 8, "llama-3.1-8b": 1 / 16,
                "qwen2.5-32b": 1 / 32}[cfg_name]
    rng = np.random.default_rng(0)
    toks = [max(1, int(sp.batch * s * frac)) for sp in specs]
    work = []
    for t in cfg.targets():
        downs = [rng.uniform(-1, 1, (t.h_in, sp.rank)) / np.sqrt(t.h_in) for sp in specs]
        ups = [rng.standard_normal((sp.rank, t.h_out)) * 0.02 for sp in specs]
        xs = [rng.standard_normal((n, t.h_in)) for n in toks]
        dys = [rng.standard_normal((n, t.h_out)) for n in toks]
        w = rng.standard_normal((t.h_in, t.h_out)) * 0.02
        work.append((downs, ups, [float(sp.alpha) for sp in specs], xs, w, dys))
    return cfg, specs, s, frac, toks, work


def _all_host_threads() -> None:
    """torchrun exports OMP_NUM_THREADS=1; the CPU reference uses every host core."""
    try:
        import numpy  # noqa: F401  (load OpenBLAS first: threadpoolctl only sees loaded libraries)
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=os.cpu_count() or 1, user_api="blas")
    except Exception:  # pragma: no cover
        pass


def _blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        return int(max((i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"),
                       default=1))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


class CpuReference:
    """The reference CPU path of one step, as a bounded sample: lorasweep's own
    ``pack_adapters`` -> ``packed_forward`` -> ``packed_backward`` (pkg/src/lorasweep/
    lorapack.py:128-231, fp64 numpy/OpenBLAS on every host core) over the 7 LoRA linears
    of one layer at 1/16 (C3) of the step's tokens; tokens/s are scaled by 1/L (the cost
    is linear in T and in the layer count).  Uses the real reference from baseline/_ref
    ("kind": "reference"); without it, the oracle port (oracle/lorapack_oracle.py,
    "kind": "port")."""

    def __init__(self, cfg_name: str, frac: float | None = None):
        self.cfg, self.specs, self.s, self.frac, toks, work = _cpu_sample(cfg_name, frac)
        self.T = sum(toks)
        self.RL = _ref_lorapack()
        if self.RL is not None:
            RL = self.RL
            self.kind = "reference"
            self.work = [([RL.AdapterWeights(a, b, al) for a, b, al in zip(downs, ups, alphas)], xs, w, dys)
                         for downs, ups, alphas, xs, w, dys in work]
        else:
            from oracle import lorapack_oracle as O
            self.kind = "port"
            self.O = O
            self.work = [(O.pack(downs, ups, alphas, xs), w, dys) for downs, ups, alphas, xs, w, dys in work]

    def step(self) -> float:
        """One sample step; returns its wall seconds."""
        t0 = time.perf_counter()
        if self.kind == "reference":
            RL = self.RL
            for ads, xs, w, dys in self.work:
                packed = RL.pack_adapters(ads, xs)
                RL.packed_forward(packed, w)
                RL.packed_backward(packed, w, dys)
        else:
            for p, w, dys in self.work:
                self.O.packed_forward(p, w)
                self.O.packed_backward(p, w, dys)
        return time.perf_counter() - t0

    def tok_s(self, dt: float) -> float:
        return self.T / (dt * self.cfg.n_layers)

    def describe(self, dt: float) -> str:
        what = ("lorasweep (the reference, baseline/_ref) pack_adapters+packed_forward+packed_backward"
                if self.kind == "reference" else "oracle port of lorasweep packed_forward+packed_backward")
        step_tokens = sum(sp.batch for sp in self.specs) * self.s
        return (f"{what} (fp64 numpy, {_blas_threads()} BLAS threads), 7 LoRA linears of 1 of {self.cfg.n_layers} "
                f"layers at {self.T} tokens (1/{round(1 / self.frac)} of the {step_tokens}-token step), "
                f"{dt:.2f} s per sample, scaled by 1/L; attention, norms, lm_head and optimizer excluded "
                f"(the reference implements none)")


def cpu_reference(cfg_name: str, frac: float | None = None) -> dict:
    """cpu_baseline: one warm-up sample, then the best of two timed samples."""
    _all_host_threads()
    ref = CpuReference(cfg_name, frac)
    ref.step()
    dt = min(ref.step(), ref.step())
    return {"value": ref.tok_s(dt), "unit": "tokens/s", "cores": _blas_threads(), "kind": ref.kind,
            "sample": ref.describe(dt), "host_cpus": os.cpu_count()}


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
    """--impl reference: the reference's CPU implementation of the path (module doc).
    Each step is one bounded sample (one layer's 7 LoRA linears at 1/16 of the tokens),
    so ms_per_step is the sample's measured time; value is the tokens/s of the whole
    model that the sample implies (x 1/L).  Under torchrun only rank 0 runs."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    _all_host_threads()
    ref = CpuReference(args.config)
    for _ in range(args.warmup):
        ref.step()
    dts = []
    for _ in range(max(1, args.steps)):
        dts.append(ref.step())
        if time.perf_counter() - _T0 > 240:   # keep the arm within a few minutes
            break
    dt = sum(dts) / len(dts)
    v = ref.tok_s(dt)
    s = ref.s
    T = sum(sp.batch for sp in ref.specs) * s
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": len(dts),
            "warmup": args.warmup, "ms_per_step": 1000.0 * dt, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{ref.cfg.name} packed LoRA, {len(ref.specs)} adapters, T={T}",
                       "model": ref.cfg.name, "global_batch": T // s, "seq_len": s, "parallelism": "cpu",
                       "step": f"one bounded sample: 7 LoRA linears of 1 layer at {ref.T} tokens"},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": _blas_threads(), "kind": ref.kind,
                             "sample": ref.describe(dt), "host_cpus": os.cpu_count()},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


_T0 = time.perf_counter()


def _relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: start N ranks (one process per GPU) on this node
    through torch.distributed.run, exactly as the driver does, and pass rank 0's line
    through."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def job_for_rank(cfg_name: str, world: int, rank: int, scaling: str) -> tuple[list, list, str]:
    """(bench-adapter indices, all-adapter count, parallelism tag) of this rank's packed job.
    split (default): the planner's one-batch split of the workload over the world
    (sweep/jobsplit.py: plan_split + place), so rank r trains the job placed on device r;
    weak: every rank trains the whole workload (independent replicas)."""
    from paper_2508_02932_b200.model import bench_adapters

    n = len(bench_adapters(cfg_name)[0])
    if world == 1 or scaling == "weak":
        return list(range(n)), n, f"jobs{world}" if world > 1 else "jobs1"
    from paper_2508_02932_b200.sweep.jobsplit import split_adapters

    sp = split_adapters(cfg_name, world)
    return list(sp.adapters[rank]), n, sp.describe()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="llama-3.1-8b")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="split", choices=["split", "weak"],
                    help="split: the planner splits the workload's adapters over the GPUs (one packed job "
                         "per GPU, fixed total work); weak: every GPU trains the whole workload")
    ap.add_argument("--tp", type=int, default=None,
                    help="tensor-parallel degree per packed job (config C4 default: all GPUs); "
                         "world/tp independent jobs run side by side")
    ap.add_argument("--tp-comm", default="torch", choices=["torch", "abi"],
                    help="TP all-reduce through torch.distributed (NCCL) or libplora's C-ABI (plora_tp_*, NCCL)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fuse-dual", action="store_true", help="separate K4 / K3 kernels (A/B of the fused dY pass)")
    ap.add_argument("--overlap-k5", action="store_true", help="dA reductions on a side stream (A/B)")
    ap.add_argument("--graph", dest="graph", action="store_true", default=True,
                    help="time the step replayed from one CUDA graph (model.GraphedStep; default)")
    ap.add_argument("--eager", dest="graph", action="store_false", help="time the eager step instead")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        raise SystemExit(_relaunch(args))
    if args.config == "qwen2.5-32b":
        # the 64-layer TP shard peaks at ~154 GB eagerly; a captured graph's private pool does
        # not fit beside it (profiles/r2_c4_shard_projection.log): C4 times the eager step
        args.graph = False
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU")
    if args.impl == "reference":
        run_reference(args)
        return

    os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
    import torch
    import torch.distributed as dist

    from paper_2508_02932_b200 import _lib, ops
    from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters
    from paper_2508_02932_b200.tp import AbiNcclComm, DistComm

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    device = local % max(1, ndev)
    shared = world > ndev          # several ranks on one GPU (test runs): NCCL refuses that
    torch.cuda.set_device(device)
    backend = "gloo" if shared else "nccl"
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
    _lib.check(_lib.lib().plora_device_check(), "device check")

    cfg = PRESETS[args.config]
    tp = args.tp or (world if args.config == "qwen2.5-32b" else 1)
    if world % tp:
        raise SystemExit(f"--tp {tp} must divide the world size {world}")
    if args.config == "qwen2.5-32b" and tp < 8:
        raise SystemExit("C4 (Qwen2.5-32B, 32 adapters) needs a tensor-parallel group of 8 GPUs "
                         "(one 180 GB B200 holds a TP=8 shard: tools/c4_shard_bench.py)")
    if tp > 1 and shared:
        raise SystemExit("tensor-parallel jobs need one GPU per rank")
    n_jobs = world // tp
    job = rank // tp
    comm = None
    all_specs, s = bench_adapters(args.config)
    if tp > 1:   # one NCCL group per packed job (Megatron TP over NVLink), jobs side by side
        groups = [dist.new_group(list(range(j * tp, (j + 1) * tp))) for j in range(n_jobs)]
        if args.tp_comm == "abi":
            comm = AbiNcclComm(rank - job * tp, tp, group=groups[job])
        else:
            comm = DistComm(groups[job])
        mine, parallelism = list(range(len(all_specs))), f"jobs{n_jobs}xtp{tp}"
        scaling = "weak" if args.tp is not None else "strong"
        seed_off = 1000 * job
    else:
        mine, _, parallelism = job_for_rank(args.config, world, rank, args.scaling)
        scaling = "weak" if (args.scaling == "weak" or world == 1) else "strong"
        seed_off = 1000 * rank if args.scaling == "weak" else 0
    specs = [all_specs[i] for i in mine]
    trainer = None
    T = 0
    if specs:
        trainer = PackedLoraTrainer(cfg, specs, s, device="cuda", adapter_seeds=[100 + i + seed_off for i in mine],
                                    tp=comm, fuse_dual=not args.no_fuse_dual,
                                    overlap_k5=True if args.overlap_k5 else None)
        T = trainer.T
        tokens_host = trainer.synthetic_tokens(seeds=[1000 + i + 100 * seed_off for i in mine]).pin_memory()
        tokens = tokens_host.to("cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    for _ in range(args.warmup):
        if trainer is not None:
            trainer.step(tokens)
    barrier()

    def timed_region(run, steps, sample_clocks=None):
        """Device time (ms) of `steps` calls of run() between barriers + synchronize, max
        over ranks (CUDA events on the launching stream)."""
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            run()
        e1.record()
        barrier()
        return e0.elapsed_time(e1)

    # ---------------------------------------------------------------- eager timed region (plain eager step)
    # With PLORA_PROFILE_RANGE=1 (ncu --profile-from-start off) this region is the profiled one and
    # its libplora launches carry the per-launch timer (PLORA_RECORDS_OUT: records for
    # tools/dram_by_shape.py, matched launch by launch with ncu's list).
    profile_range = os.environ.get("PLORA_PROFILE_RANGE") == "1"
    timer = ops.KernelTimer() if profile_range else None
    launches0 = ops.launch_count()
    if profile_range:
        barrier()
        torch.cuda.profiler.start()
    ops.set_timer(timer)
    with ClockSampler(device) as clocks_eager:
        ms_eager = timed_region(lambda: trainer.step(tokens) if trainer is not None else None, args.steps)
    ops.set_timer(None)
    if profile_range:
        torch.cuda.profiler.stop()
    launches_eager = ops.launch_count() - launches0
    if timer is not None and os.environ.get("PLORA_RECORDS_OUT") and rank == 0:
        Path(os.environ["PLORA_RECORDS_OUT"]).write_text(json.dumps(timer.dump()))
    ms_eager_max = max_over_ranks(ms_eager)
    # tokens processed by the whole job: a TP group's ranks share one job's tokens
    tokens_all = sum_over_ranks(float(T) if (tp == 1 or rank % tp == 0) else 0.0)

    # ---------------------------------------------------------------- per-launch kernel stats
    # The step captured as a CUDA graph with every libplora launch bracketed by event-record
    # nodes (KernelTimer(external=True)) and replayed: per-launch device times with no host
    # enqueue gaps (the eager step's host work per launch is as long as a small LoRA kernel,
    # so eager per-launch events time the host).  Source of roofline, kernels, gemm_shapes.
    kstats, kstats_mode = None, None
    if trainer is not None and args.graph and not shared:
        try:
            kt = ops.KernelTimer(external=True)
            ops.set_timer(kt)
            try:
                tg = trainer.graphed(tokens, warmup=0)
            finally:
                ops.set_timer(None)
            tg.step()                          # warm replay
            torch.cuda.synchronize()
            kstats = {}
            for _ in range(max(1, min(args.steps, 3))):
                tg.step()
                for key, d in kt.summary().items():
                    acc = kstats.setdefault(key, {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0})
                    for f in acc:
                        acc[f] += d[f]
            kstats_steps = max(1, min(args.steps, 3))
            kstats_mode = f"cuda graph with event-record nodes around every libplora launch, {kstats_steps} replays"
            del tg, kt
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
        except Exception as exc:   # noqa: BLE001 -- fall back to the eager per-launch timer
            kstats, kstats_mode = None, f"graph timer failed ({type(exc).__name__}: {str(exc)[:120]}); eager"
            ops.set_timer(None)
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
    if kstats is None:
        kt = ops.KernelTimer()
        ops.set_timer(kt)
        timed_region(lambda: trainer.step(tokens) if trainer is not None else None, args.steps)
        ops.set_timer(None)
        kstats = kt.summary()
        kstats_steps = args.steps
        kstats_mode = (kstats_mode or "") + "eager step with every libplora launch bracketed by CUDA events"
        del kt
    # ---------------------------------------------------------------- the step as one CUDA graph
    graphed = None
    if trainer is not None and args.graph and not shared:
        try:
            graphed = trainer.graphed(tokens, warmup=1)
        except Exception as exc:   # noqa: BLE001 -- reported in the line; the eager GPU step remains
            graph_error = f"{type(exc).__name__}: {exc}"[:300]
            graphed = None
            torch.cuda.synchronize()
        else:
            graph_error = None
    else:
        graph_error = "disabled" if not args.graph else ("ranks share a device (gloo)" if shared else None)
    use_graph = max_over_ranks(0.0 if (graphed is not None or trainer is None) else 1.0) == 0.0 and args.graph \
        and not shared
    step_fn = graphed.step if (use_graph and graphed is not None) else (lambda t=None: trainer.step(tokens))

    # ---------------------------------------------------------------- timed region (device): the headline value
    launches0 = ops.launch_count()
    with ClockSampler(device) as clocks:
        ms = timed_region(lambda: step_fn() if trainer is not None else None, args.steps)
    launches = ops.launch_count() - launches0
    ms_max = max_over_ranks(ms)
    value = tokens_all * args.steps / (ms_max / 1000.0)
    losses_dev = trainer.losses.clone() if trainer is not None else torch.zeros(0)

    # ---------------------------------------------------------------- end-to-end (public API, host buffers)
    losses_host = torch.zeros(0)

    def e2e_step():
        nonlocal losses_host
        if trainer is not None:
            tokens.copy_(tokens_host, non_blocking=True)
            losses_host = (graphed.step(tokens) if (use_graph and graphed is not None) else trainer.step(tokens)).cpu()

    ms_e2e = max_over_ranks(timed_region(e2e_step, args.steps))
    e2e_value = tokens_all * args.steps / (ms_e2e / 1000.0)

    peaks = _peaks()
    g = kstats.get("gemm", {"ms": 0.0, "flops": 0.0, "launches": 0})
    achieved = g["flops"] / (g["ms"] / 1000.0) / 1e12 if g["ms"] else 0.0
    kernels, shapes, lora_shapes = {}, {}, {}
    for kind, d in kstats.items():
        sec = d["ms"] / 1000.0
        if kind.startswith("gemm["):   # per-shape GEMM detail
            shapes[kind[kind.index("[") + 1:-1]] = {"launches": d["launches"], "ms": round(d["ms"], 2),
                                                   "tflops": round(d["flops"] / sec / 1e12, 1)}
            continue
        if "[" in kind:                # per-shape LoRA-kernel detail (shrink[K..], segred[M..])
            lora_shapes[kind] = {"launches": d["launches"], "ms": round(d["ms"], 2),
                                 "hbm_gbs": round(d["bytes"] / sec / 1e9, 1) if sec else 0.0}
            continue
        kernels[kind] = {"launches": d["launches"], "ms_total": round(d["ms"], 3),
                         "share_of_step": round(d["ms"] / kstats_steps / (ms / args.steps), 4) if ms else 0.0}
        if d["flops"]:
            kernels[kind]["tflops"] = round(d["flops"] / sec / 1e12, 1)
        if d["bytes"]:
            kernels[kind]["hbm_gbs"] = round(d["bytes"] / sec / 1e9, 1)
            kernels[kind]["hbm_frac"] = round(d["bytes"] / sec / 1e9 / peaks["hbm_gbs"], 3)
    if "dual" in kernels:
        kernels["dual"]["note"] = ("K4+K3 fused: bytes = ONE pass over dY (the separate kernels stream it twice); "
                                   "paced by the tensor pipe / smem operand reads, not DRAM (profiles/r2_lora_ncu.md)")
    useful = useful_flops(cfg, specs, s, tp) if specs else {"base": 0.0, "lora": 0.0, "attention": 0.0}
    useful_all = {k: sum_over_ranks(v) for k, v in useful.items()}   # this rank's share, summed
    per_rank = {"rank": rank, "device": device, "world": dist.get_world_size() if world > 1 else 1,
                "backend": backend if world > 1 else None, "adapters": mine, "tokens": T,
                "ms_per_step": round(ms / args.steps, 2),
                "tokens_per_s": round(T * args.steps / (ms / 1000.0), 1) if ms and T else 0.0,
                "gemm_tflops": round(achieved, 1), "gemm_frac": round(achieved / peaks["tflops_sustained"], 4),
                "step_base_tflops": round(useful["base"] * args.steps / (ms / 1000.0) / 1e12, 1) if ms else 0.0}
    ranks = [per_rank]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, per_rank)
    base_tf = sum(r["step_base_tflops"] for r in ranks) / len(ranks)   # per GPU
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform tokens, random-init weights)",
        "config": {"workload": f"{cfg.name} packed LoRA training, {len(all_specs)} adapters (ranks 8/16/32/64), "
                               f"all 7 targets, {sum(sp.batch for sp in all_specs) * s} tokens/step per job, "
                               f"fwd+bwd+per-adapter AdamW",
                   "model": cfg.name, "global_batch": int(tokens_all) // s, "seq_len": s,
                   "parallelism": parallelism, "adapters": len(all_specs),
                   "l2": "working set (~100 GB activations) >> 126 MB L2; no flush needed"},
        "roofline": {"bound": "tensor", "kernel": "tcgen05 base GEMM + fused LoRA expand (K1/K2b/K6, lm_head)",
                     "achieved": round(achieved, 1), "peak": peaks["tflops_sustained"], "unit": "TFLOP/s",
                     "frac": round(achieved / peaks["tflops_sustained"], 4), "traffic": _traffic(),
                     "traffic_by_shape": _dram_by_shape(peaks["hbm_gbs"]) if args.config == "llama-3.1-8b" else None,
                     "peak_source": f"{peaks['source']} bf16 sustained (kernel timed inside a long step)",
                     "step_base_gemm_tflops": round(base_tf, 1),
                     "step_frac_of_burst_peak": round(base_tf / peaks["tflops_burst"], 4)},
        "useful_tflops_per_gpu": {k: round(v * args.steps / (ms_max / 1000.0) / 1e12 / world, 1)
                                  for k, v in useful_all.items()},
        "kernels": kernels,
        "gemm_shapes": shapes,
        "lora_shapes": lora_shapes,
        "e2e": {"value": e2e_value, "unit": "tokens/s",
                "h2d_bytes_per_step": (tokens_host.numel() * tokens_host.element_size()) if trainer is not None else 0,
                "d2h_bytes_per_step": losses_host.numel() * losses_host.element_size()},
        "gpu_launches": launches,
        "step_mode": ("cuda_graph" if use_graph else "eager") + ("" if graph_error is None else
                                                                 f" (graph not used: {graph_error})"),
        "eager": {"value": tokens_all * args.steps / (ms_eager_max / 1000.0), "ms_per_step": ms_eager_max / args.steps,
                  "gpu_launches": launches_eager, "clocks": clocks_eager.summary()},
        "kernel_stats": {"mode": kstats_mode, "steps": kstats_steps,
                         "note": "source of roofline, kernels, gemm_shapes and lora_shapes"},
        "clocks": clocks.summary(),
        "losses": [round(float(x), 4) for x in losses_dev.tolist()],
        "mem_peak_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1),
    }
    if world > 1:
        line["ranks"] = ranks
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference(args.config)
        line["dropin_api"] = dropin_api_sample(args.config)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def useful_flops(cfg, specs, s: int, tp: int = 1) -> dict:
    """Useful FLOPs of one step of a packed job, this rank's share (1/tp of the job):
    base = 4 (sum_layers sum_targets h_in h_out + d V) per token (forward X W + backward
    dY W^T; the frozen base has no dW); lora = 6 r_i sum(h_in +
    h_out) L per token of adapter i (reference lora_flop, costmodel.py:168-178);
    attention = causal SDPA, 2 forward + 4 backward matmuls of 2 s^2 hd / 2 per head,
    sequence and layer."""
    T = sum(sp.batch for sp in specs) * s
    base = cfg.base_flops_per_token() * T
    lora = cfg.lora_flops_per_token_per_rank() * sum(sp.rank * sp.batch * s for sp in specs)
    seqs = sum(sp.batch for sp in specs)
    attn = 6 * 2.0 * s * s * cfg.head_dim / 2 * cfg.n_heads * seqs * cfg.n_layers
    return {"base": base / tp, "lora": lora / tp, "attention": attn / tp}   # one rank's share


def _traffic():
    """ncu DRAM bytes per launch of the dominant GEMM launch of the timed step
    (profiles/gemm_traffic.json, written from the step's own ncu capture)."""
    prof = ROOT / "profiles" / "gemm_traffic.json"
    if not prof.exists():
        return None
    try:
        return json.loads(prof.read_text()).get("dram_bytes_per_launch")
    except Exception:
        return None


def _dram_by_shape(hbm_peak_gbs: float):
    """DRAM bytes over algorithmic bytes per launch shape of one timed C3 step, from its
    committed ncu launch list (profiles/r2_c3_step_dram_by_shape.json, tools/dram_by_shape.py),
    and for the HBM-bound LoRA / optimizer shapes the algorithmic bytes over ncu's launch
    duration (serialised, no launch gap) as a fraction of the HBM peak -- beside the in-graph
    event timing of `kernels`, which includes each launch's ramp-up and gap."""
    prof = ROOT / "profiles" / "r2_c3_step_dram_by_shape.json"
    try:
        d = json.loads(prof.read_text())
        return {"source": "profiles/r2_c3_step_dram_by_shape.json (ncu, one timed C3 step)",
                "dram_over_algo": {k: v["dram_over_algo"] for k, v in d.items()},
                "hbm_frac_ncu": {k: round(v["algo_gb_per_launch"] / (v["ncu_ms_per_launch"] * 1e-3) / hbm_peak_gbs, 3)
                                 for k, v in d.items() if not k.startswith("gemm")}}
    except Exception:
        return None


if __name__ == "__main__":
    main()
