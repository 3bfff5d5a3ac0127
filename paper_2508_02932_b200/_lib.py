"""ctypes binding of libplora.so (the C-ABI declared in include/plora.h).

The shared library is built in-tree by ``paper_2508_02932_b200.build``.  There
is deliberately no fallback: if the library is missing or fails to load, every
operator raises ``PloraError`` (the product path never silently drops to CPU
math).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(os.environ.get("PLORA_LIB", "")).resolve() if os.environ.get("PLORA_LIB") else \
    Path(__file__).resolve().parent / "libplora.so"   # PLORA_LIB: A/B experiments with another build

# Every symbol include/plora.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "plora_abi_version",
    "plora_lora_workspace_bytes",
    "plora_last_error",
    "plora_device_check",
    "plora_meta_build",
    "plora_meta_max_mtiles",
    "plora_gemm_bf16",
    "plora_linear_fwd",
    "plora_lora_shrink",
    "plora_lora_segred",
    "plora_lora_shrink_multi",
    "plora_lora_segred_multi",
    "plora_lora_dual_workspace_bytes",
    "plora_lora_dual",
    "plora_swiglu_bwd_segred",
    "plora_linear_expand",
    "plora_linear_expand_group",
    "plora_add_row_bias",
    "plora_linear_dx_group",
    "plora_linear_gate_up_swiglu",
    "plora_linear_bwd",
    "plora_adamw",
    "plora_rmsnorm_fwd",
    "plora_add_rmsnorm_fwd",
    "plora_rmsnorm_bwd",
    "plora_swiglu_fwd",
    "plora_swiglu_bwd",
    "plora_rope",
    "plora_cross_entropy",
    "plora_ce_stats",
    "plora_ce_apply",
    "plora_tp_get_unique_id",
    "plora_tp_comm_init",
    "plora_tp_comm_destroy",
    "plora_tp_allreduce",
    "plora_tp_allgather",
    "plora_tp_reducescatter",
    "plora_tp_reduce",
    "plora_tp_broadcast",
)

ABI_VERSION = 9


class PloraError(RuntimeError):
    """Raised when a libplora entry point reports failure (or cannot be loaded)."""


class PackStruct(ctypes.Structure):
    """Mirror of ``plora_pack_t`` (include/plora.h)."""

    _fields_ = [
        ("n_adapters", ctypes.c_int32),
        ("n_mtiles", ctypes.c_int32),
        ("total_tokens", ctypes.c_int64),
        ("nb", ctypes.c_int32),
        ("rpad16_total", ctypes.c_int32),
        ("d_mtiles", ctypes.c_void_p),
        ("d_row_off", ctypes.c_void_p),
        ("d_ranks", ctypes.c_void_p),
        ("d_rpad_off", ctypes.c_void_p),
        ("d_alpha", ctypes.c_void_p),
        ("n_ptiles", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("d_ptiles", ctypes.c_void_p),
        ("h_row_off", ctypes.c_void_p),
        ("d_ws", ctypes.c_void_p),
        ("ws_bytes", ctypes.c_int64),
    ]


_lock = threading.Lock()
_lib: ctypes.CDLL | None = None

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f32 = ctypes.c_float
_p64 = ctypes.POINTER(ctypes.c_int64)
_p32 = ctypes.POINTER(ctypes.c_int32)

_SIGNATURES = {
    "plora_abi_version": ([], ctypes.c_int),
    "plora_lora_workspace_bytes": ([], _i64),
    "plora_last_error": ([], ctypes.c_char_p),
    "plora_device_check": ([], ctypes.c_int),
    "plora_meta_build": ([_i32, _p64, _p64, _p64, _p64, _p32, _p32, _i32, _p32, _p32, _p32, _p32],
                         ctypes.c_int),
    "plora_meta_max_mtiles": ([_i32, _p64], _i32),
    "plora_gemm_bf16": ([_vp, _i64, _i64, _i64, _vp, _vp, _i32, _vp, _i64, _vp], ctypes.c_int),
    "plora_linear_fwd": ([_vp, ctypes.POINTER(PackStruct), _vp, _i64, _i64, _vp, _i32, _vp, _vp,
                          _vp, _vp, _i64, _vp], ctypes.c_int),
    "plora_lora_shrink": ([_vp, ctypes.POINTER(PackStruct), _i64, _vp, _vp, _vp], ctypes.c_int),
    "plora_lora_segred": ([_vp, ctypes.POINTER(PackStruct), _i64, _vp, _vp, _vp], ctypes.c_int),
    "plora_lora_shrink_multi": ([_vp, ctypes.POINTER(PackStruct), _i64, _vp, _i32, ctypes.POINTER(_vp),
                                 ctypes.POINTER(_vp)], ctypes.c_int),
    "plora_lora_segred_multi": ([_vp, ctypes.POINTER(PackStruct), _i64, _vp, _i32, ctypes.POINTER(_vp),
                                 ctypes.POINTER(_vp)], ctypes.c_int),
    "plora_lora_dual_workspace_bytes": ([ctypes.POINTER(PackStruct), _i32, _p64, _p32], _i64),
    "plora_lora_dual": ([_vp, ctypes.POINTER(PackStruct), _i32, _p64, _p32, ctypes.POINTER(_vp),
                         ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp, _i64],
                        ctypes.c_int),
    "plora_swiglu_bwd_segred": ([_vp, ctypes.POINTER(PackStruct), _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
                                ctypes.c_int),
    "plora_linear_expand": ([_vp, ctypes.POINTER(PackStruct), _vp, _i64, _i64, _vp, _i32, _vp, _vp,
                             _vp, _i64, _vp], ctypes.c_int),
    "plora_linear_expand_group": ([_vp, ctypes.POINTER(PackStruct), _vp, _i64, _i32, _p64, ctypes.POINTER(_vp),
                                   _i32, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                   ctypes.POINTER(_vp)], ctypes.c_int),
    "plora_add_row_bias": ([_vp, _i64, _i64, _vp, _i64, _vp], ctypes.c_int),
    "plora_linear_dx_group": ([_vp, ctypes.POINTER(PackStruct), _i32, ctypes.POINTER(_vp), _p64, ctypes.POINTER(_vp),
                               _i32, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64, _vp, _i64, _vp], ctypes.c_int),
    "plora_linear_gate_up_swiglu": ([_vp, ctypes.POINTER(PackStruct), _vp, _i64, _i64] + [_vp] * 9, ctypes.c_int),
    "plora_linear_bwd": ([_vp, ctypes.POINTER(PackStruct), _vp, _i64, _i64, _vp, _i32, _vp, _vp,
                          _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp], ctypes.c_int),
    "plora_adamw": ([_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _f32, _f32, _f32, _i64],
                    ctypes.c_int),
    "plora_rmsnorm_fwd": ([_vp, _i64, _i64, _vp, _vp, _f32, _vp, _vp, _i32], ctypes.c_int),
    "plora_add_rmsnorm_fwd": ([_vp, _i64, _i64, _vp, _vp, _vp, _f32, _vp, _vp, _vp], ctypes.c_int),
    "plora_rmsnorm_bwd": ([_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "plora_swiglu_fwd": ([_vp, _i64, _vp, _vp, _vp], ctypes.c_int),
    "plora_swiglu_bwd": ([_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "plora_rope": ([_vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _i64, _i64, _i64, _i32, _i32],
                   ctypes.c_int),
    "plora_cross_entropy": ([_vp, _i64, _i64, _vp, _vp, _vp, _vp], ctypes.c_int),
    "plora_ce_stats": ([_vp, _i64, _i64, _vp, _vp, _i64, _vp], ctypes.c_int),
    "plora_ce_apply": ([_vp, _i64, _i64, _vp, _vp, _i64, _vp, _vp], ctypes.c_int),
    "plora_tp_get_unique_id": ([ctypes.c_char_p], ctypes.c_int),
    "plora_tp_comm_init": ([ctypes.POINTER(_vp), ctypes.c_char_p, _i32, _i32], ctypes.c_int),
    "plora_tp_comm_destroy": ([_vp], ctypes.c_int),
    "plora_tp_allreduce": ([_vp, _vp, _vp, _i64, _i32, _i32], ctypes.c_int),
    "plora_tp_allgather": ([_vp, _vp, _vp, _vp, _i64, _i32], ctypes.c_int),
    "plora_tp_reducescatter": ([_vp, _vp, _vp, _vp, _i64, _i32], ctypes.c_int),
    "plora_tp_reduce": ([_vp, _vp, _vp, _i64, _i32, _i32], ctypes.c_int),
    "plora_tp_broadcast": ([_vp, _vp, _vp, _i64, _i32, _i32], ctypes.c_int),
}


def lib() -> ctypes.CDLL:
    """Load (once) and return the libplora handle; raises PloraError if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise PloraError(
                f"{LIB_PATH} not built; run `python -m paper_2508_02932_b200.build` "
                "(or __graft_entry__.build())")
        try:
            handle = ctypes.CDLL(str(LIB_PATH))
        except OSError as exc:  # pragma: no cover - depends on the host
            raise PloraError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (argtypes, restype) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.argtypes = argtypes
            fn.restype = restype
        if handle.plora_abi_version() != ABI_VERSION:
            raise PloraError("libplora ABI version mismatch; rebuild the extension")
        _lib = handle
        return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().plora_last_error().decode(errors="replace")
        raise PloraError(f"{what} failed ({status}): {msg}")
