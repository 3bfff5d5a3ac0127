"""Sweep vocabulary: hyper-parameter configurations, base-model and pool descriptions.

Field-for-field compatible with the reference's value types
(pkg/src/lorasweep/workload.py:53-164) so that planner inputs and outputs can
be exchanged with ``lorasweep`` (same config-id content hash, same grid order).
Only what the planner, the cost model and the engine need is kept here; the
reference's JSON document ingestion is reproduced in ``parse_workload``.
"""

from __future__ import annotations

import hashlib
import itertools
import json
from dataclasses import dataclass, replace
from typing import Any, Mapping, Sequence

__all__ = [
    "WorkloadSyntaxError", "WorkloadValidationError", "TargetModule", "ModelSpec", "GpuPool",
    "ShardingSpec", "LoraConfig", "ProfileRecord", "WorkloadSpec", "config_id", "enumerate_grid",
    "validate_config", "validate_model", "validate_pool", "validate_sharding", "parse_workload",
    "serialize_workload", "workload_digest", "model_spec_from_config", "STATE_BYTES_PLORA",
]

MAX_TARGETS = 7
ZERO_LEVELS = (0, 1, 2, 3)


class WorkloadSyntaxError(ValueError):
    """Malformed input document (reference workload.py:45-46)."""


class WorkloadValidationError(ValueError):
    """Well-formed input that violates an invariant (reference workload.py:49-50)."""


@dataclass(frozen=True)
class TargetModule:
    name: str
    h_in: int
    h_out: int


@dataclass(frozen=True)
class ModelSpec:
    """Base model as seen by the memory model (reference workload.py:60-84)."""

    name: str
    n_layers: int
    target_modules: tuple
    base_param_count: int
    c_prec: int
    embed_act_coeff: float = 0.0
    attn_act_coeff: float = 0.0
    mlp_act_coeff: float = 0.0
    # B200 extension (default: the reference's c_prec for
    # everything): bytes per adapter parameter of (params, grads, one optimizer moment).
    # The packed trainer keeps fp32 masters + a bf16 shadow, fp32 grads and fp32 AdamW
    # moments: (6, 4, 4) -- see STATE_BYTES_PLORA.
    state_bytes: tuple | None = None

    @property
    def act_coeff_sum(self) -> float:
        return self.embed_act_coeff + self.attn_act_coeff + self.mlp_act_coeff

    @property
    def min_projection_dim(self) -> int:
        return min(min(t.h_in, t.h_out) for t in self.target_modules)


@dataclass(frozen=True)
class GpuPool:
    gpu_count: int
    mem_per_gpu: int
    load_factor: float = 1.0

    @property
    def memory_budget(self) -> float:
        return self.load_factor * self.mem_per_gpu


@dataclass(frozen=True)
class ShardingSpec:
    d_tp: int = 1
    d_pp: int = 1
    d_fsdp: int = 1
    zero_level: int = 0

    @property
    def model_shards(self) -> int:
        return self.d_tp * self.d_pp

    @classmethod
    def tensor_parallel(cls, degree: int) -> "ShardingSpec":
        return cls(d_tp=degree)


@dataclass(frozen=True)
class LoraConfig:
    id: str
    rank: int
    alpha: float
    batch_size: int
    learning_rate: float
    seq_len: int
    train_steps: int


@dataclass(frozen=True)
class ProfileRecord:
    parallelism_degree: int
    packed_ranks: tuple
    packed_batch_sizes: tuple
    seq_len: int
    iter_time_s: float


@dataclass(frozen=True)
class WorkloadSpec:
    model: ModelSpec
    pool: GpuPool
    configs: tuple
    profiles: tuple = ()

    def config_ids(self) -> tuple:
        return tuple(c.id for c in self.configs)


def config_id(rank: int, alpha: float, batch_size: int, learning_rate: float, seq_len: int,
              train_steps: int) -> str:
    """Content hash of the hyper-parameter tuple; identical to the reference's ids
    (workload.py:167-178) so queues/reports interoperate."""
    fields = (str(int(rank)), repr(float(alpha)), str(int(batch_size)), repr(float(learning_rate)),
              str(int(seq_len)), str(int(train_steps)))
    return "cfg-" + hashlib.sha256("|".join(fields).encode()).hexdigest()[:12]


def enumerate_grid(learning_rates: Sequence[float], batch_sizes: Sequence[int], ranks: Sequence[int],
                   alphas: Sequence[float], template: LoraConfig) -> list:
    """Cartesian grid in (lr, batch, rank, alpha) order (reference workload.py:187-212)."""
    for name, vals in (("learning_rates", learning_rates), ("batch_sizes", batch_sizes),
                       ("ranks", ranks), ("alphas", alphas)):
        if not len(vals):
            raise WorkloadValidationError(f"empty range list for '{name}'")
    grid = []
    for lr, bs, r, a in itertools.product(learning_rates, batch_sizes, ranks, alphas):
        grid.append(replace(template, rank=int(r), alpha=float(a), batch_size=int(bs), learning_rate=float(lr),
                            id=config_id(r, a, bs, lr, template.seq_len, template.train_steps)))
    return grid


def validate_config(cfg: LoraConfig, model: ModelSpec) -> list:
    errs = []
    for attr in ("rank", "batch_size", "seq_len", "train_steps"):
        if getattr(cfg, attr) < 1:
            errs.append(f"{attr} must be >= 1 (got {getattr(cfg, attr)})")
    for attr in ("alpha", "learning_rate"):
        if not getattr(cfg, attr) > 0:
            errs.append(f"{attr} must be > 0 (got {getattr(cfg, attr)})")
    if cfg.rank >= 1:
        for t in model.target_modules:
            lim = min(t.h_in, t.h_out)
            if cfg.rank > lim:
                errs.append(f"rank {cfg.rank} exceeds projection dimension {lim} (target '{t.name}')")
    return errs


def validate_model(model: ModelSpec) -> list:
    errs = []
    if model.n_layers < 1:
        errs.append(f"n_layers must be >= 1 (got {model.n_layers})")
    if not model.target_modules:
        errs.append("at least one target module must be enabled")
    if len(model.target_modules) > MAX_TARGETS:
        errs.append(f"at most {MAX_TARGETS} target modules allowed (got {len(model.target_modules)})")
    for t in model.target_modules:
        if t.h_in < 1 or t.h_out < 1:
            errs.append(f"target '{t.name}' dimensions must be positive (got {t.h_in}x{t.h_out})")
    if model.base_param_count < 0:
        errs.append("base_param_count must be >= 0")
    if model.c_prec < 1:
        errs.append(f"c_prec must be a positive byte count (got {model.c_prec})")
    if model.state_bytes is not None and (len(model.state_bytes) != 3 or min(model.state_bytes) < 1):
        errs.append(f"state_bytes must be three positive byte counts (got {model.state_bytes})")
    for attr in ("embed_act_coeff", "attn_act_coeff", "mlp_act_coeff"):
        if getattr(model, attr) < 0:
            errs.append(f"{attr} must be >= 0")
    return errs


def validate_pool(pool: GpuPool) -> list:
    errs = []
    if pool.gpu_count < 1:
        errs.append(f"gpu_count must be >= 1 (got {pool.gpu_count})")
    if pool.mem_per_gpu <= 0:
        errs.append(f"mem_per_gpu must be > 0 (got {pool.mem_per_gpu})")
    if not 0 < pool.load_factor <= 1:
        errs.append(f"load_factor must be in (0, 1] (got {pool.load_factor})")
    return errs


def validate_sharding(shard: ShardingSpec) -> list:
    errs = [f"{a} must be >= 1 (got {getattr(shard, a)})" for a in ("d_tp", "d_pp", "d_fsdp")
            if getattr(shard, a) < 1]
    if shard.zero_level not in ZERO_LEVELS:
        errs.append(f"invalid ZeRO level {shard.zero_level} (expected one of {ZERO_LEVELS})")
    if shard.model_shards > 1 and shard.zero_level != 0:
        errs.append("tensor/pipeline sharding cannot be combined with ZeRO sharding")
    if shard.d_fsdp > 1 and shard.zero_level == 0:
        errs.append("d_fsdp > 1 requires a ZeRO level")
    return errs


STATE_BYTES_PLORA = (6, 4, 4)   # fp32 master + bf16 shadow, fp32 grad, fp32 m / v (adapters.py)


def model_spec_from_config(cfg, c_prec: int = 2, act_coeffs=(0.0, 0.0, 0.0), state_bytes=None) -> ModelSpec:
    """ModelSpec of a ``model.ModelConfig`` preset (all 7 LoRA targets); pass
    ``state_bytes=STATE_BYTES_PLORA`` to cost adapter state as the packed trainer stores it."""
    targets = tuple(TargetModule(t.name, t.h_in, t.h_out) for t in cfg.targets())
    base = cfg.n_layers * sum(t.h_in * t.h_out for t in cfg.targets()) + cfg.vocab * cfg.d * (1 if cfg.tied else 2)
    return ModelSpec(name=cfg.name, n_layers=cfg.n_layers, target_modules=targets, base_param_count=base,
                     c_prec=c_prec, embed_act_coeff=act_coeffs[0], attn_act_coeff=act_coeffs[1],
                     mlp_act_coeff=act_coeffs[2], state_bytes=tuple(state_bytes) if state_bytes else None)


# ------------------------------------------------------------------ document I/O
def _field(obj: Mapping, key: str, kind, where: str, default=...):
    if key not in obj:
        if default is not ...:
            return default
        raise WorkloadValidationError(f"{where}: missing field '{key}'")
    v = obj[key]
    if kind in (int, float) and isinstance(v, bool):
        v = None
    if kind is float:
        if not isinstance(v, (int, float)):
            raise WorkloadValidationError(f"{where}: field '{key}' must be a number")
        return float(v)
    if kind is int:
        if not isinstance(v, int):
            raise WorkloadValidationError(f"{where}: field '{key}' must be an integer")
        return v
    names = {dict: "an object", list: "an array", str: "a string"}
    if not isinstance(v, kind):
        raise WorkloadValidationError(f"{where}: field '{key}' must be {names.get(kind, kind.__name__)}")
    return v


def _state_bytes(m: Mapping):
    """Optional model.state_bytes (B200 extension): [param, grad, optimizer-moment] bytes."""
    if "state_bytes" not in m:
        return None
    v = m["state_bytes"]
    if not (isinstance(v, list) and len(v) == 3 and all(isinstance(x, int) and not isinstance(x, bool) for x in v)):
        raise WorkloadValidationError("model: state_bytes must be a list of three integers")
    return tuple(v)


def parse_workload(text: str) -> WorkloadSpec:
    """Parse a workload JSON document (reference workload.py:415-450)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise WorkloadSyntaxError(f"invalid JSON at line {e.lineno}, column {e.colno}: {e.msg}") from e
    if not isinstance(doc, dict):
        raise WorkloadValidationError("top level must be an object")
    m = _field(doc, "model", dict, "workload")
    targets = []
    for i, t in enumerate(_field(m, "target_modules", list, "model")):
        w = f"model.target_modules[{i}]"
        if not isinstance(t, dict):
            raise WorkloadValidationError(f"{w}: must be an object")
        targets.append(TargetModule(_field(t, "name", str, w), _field(t, "h_in", int, w), _field(t, "h_out", int, w)))
    co = _field(m, "activation_coeffs", dict, "model", {})
    model = ModelSpec(_field(m, "name", str, "model"), _field(m, "n_layers", int, "model"), tuple(targets),
                      _field(m, "base_param_count", int, "model"), _field(m, "c_prec", int, "model"),
                      *(_field(co, k, float, "model.activation_coeffs", 0.0) for k in ("embed", "attn", "mlp")),
                      state_bytes=_state_bytes(m))
    if validate_model(model):
        raise WorkloadValidationError("model: " + "; ".join(validate_model(model)))
    p = _field(doc, "pool", dict, "workload")
    pool = GpuPool(_field(p, "gpu_count", int, "pool"), _field(p, "mem_per_gpu", int, "pool"),
                   _field(p, "load_factor", float, "pool", 1.0))
    if validate_pool(pool):
        raise WorkloadValidationError("pool: " + "; ".join(validate_pool(pool)))
    defaults = _field(doc, "defaults", dict, "workload", {})
    raw = _field(doc, "configs", list, "workload")
    if not raw:
        raise WorkloadValidationError("configs: at least one configuration is required")
    configs, seen = [], set()
    for i, c in enumerate(raw):
        w = f"configs[{i}]"
        if not isinstance(c, dict):
            raise WorkloadValidationError(f"{w}: must be an object")

        def pick(key, kind):
            if key in c:
                return _field(c, key, kind, w)
            if key in defaults:
                return _field(defaults, key, kind, "defaults")
            raise WorkloadValidationError(f"{w}: missing field '{key}' (no default given)")

        vals = dict(rank=pick("rank", int), alpha=pick("alpha", float), batch_size=pick("batch_size", int),
                    learning_rate=pick("learning_rate", float), seq_len=pick("seq_len", int),
                    train_steps=pick("train_steps", int))
        cid = c.get("id")
        if cid is None:
            cid = config_id(**vals)
        elif not isinstance(cid, str) or not cid:
            raise WorkloadValidationError(f"{w}: field 'id' must be a non-empty string")
        cfg = LoraConfig(id=cid, **vals)
        if cid in seen:
            raise WorkloadValidationError(f"{w}: duplicate id '{cid}'")
        seen.add(cid)
        if validate_config(cfg, model):
            raise WorkloadValidationError(f"config '{cid}': " + "; ".join(validate_config(cfg, model)))
        configs.append(cfg)
    profiles = []
    for i, r in enumerate(_field(doc, "profiles", list, "workload", [])):
        w = f"profiles[{i}]"
        if not isinstance(r, dict):
            raise WorkloadValidationError(f"{w}: must be an object")
        rec = ProfileRecord(_field(r, "degree", int, w), tuple(int(x) for x in _field(r, "ranks", list, w)),
                            tuple(int(x) for x in _field(r, "batch_sizes", list, w)), _field(r, "seq_len", int, w),
                            _field(r, "iter_time_s", float, w))
        if not rec.packed_ranks or len(rec.packed_ranks) != len(rec.packed_batch_sizes):
            raise WorkloadValidationError(f"{w}: ranks and batch_sizes must be equal-length, non-empty lists")
        if rec.iter_time_s <= 0:
            raise WorkloadValidationError(f"{w}: iter_time_s must be > 0")
        if rec.parallelism_degree < 1:
            raise WorkloadValidationError(f"{w}: degree must be >= 1")
        profiles.append(rec)
    return WorkloadSpec(model, pool, tuple(configs), tuple(profiles))


def _as_doc(spec: WorkloadSpec) -> dict:
    m = spec.model
    return {
        "model": {"name": m.name, "n_layers": m.n_layers,
                  "target_modules": [{"name": t.name, "h_in": t.h_in, "h_out": t.h_out} for t in m.target_modules],
                  "base_param_count": m.base_param_count, "c_prec": m.c_prec,
                  "activation_coeffs": {"embed": m.embed_act_coeff, "attn": m.attn_act_coeff,
                                        "mlp": m.mlp_act_coeff},
                  **({"state_bytes": list(m.state_bytes)} if m.state_bytes else {})},
        "pool": {"gpu_count": spec.pool.gpu_count, "mem_per_gpu": spec.pool.mem_per_gpu,
                 "load_factor": spec.pool.load_factor},
        "configs": [{"id": c.id, "rank": c.rank, "alpha": c.alpha, "batch_size": c.batch_size,
                     "learning_rate": c.learning_rate, "seq_len": c.seq_len, "train_steps": c.train_steps}
                    for c in spec.configs],
        "profiles": [{"degree": p.parallelism_degree, "ranks": list(p.packed_ranks),
                      "batch_sizes": list(p.packed_batch_sizes), "seq_len": p.seq_len,
                      "iter_time_s": p.iter_time_s} for p in spec.profiles],
    }


def serialize_workload(spec: WorkloadSpec) -> str:
    return json.dumps(_as_doc(spec), indent=2) + "\n"


def workload_digest(spec: WorkloadSpec) -> str:
    return hashlib.sha256(json.dumps(_as_doc(spec), separators=(",", ":"), sort_keys=True).encode()).hexdigest()
