"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/plora.h declares (no compute calls without a GPU)."""

import re
from pathlib import Path

from paper_2508_02932_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "plora.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"PLORA_API\s+[\w\s\*]*?\b(plora_\w+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    assert set(syms) == set(_lib.EXPORTS), syms


def test_library_loads_and_exports_everything():
    lib = _lib.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.plora_abi_version() == _lib.ABI_VERSION


def test_device_check_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        return
    assert _lib.lib().plora_device_check() != 0
    assert _lib.lib().plora_last_error()


def test_invalid_arguments_return_status_and_message():
    """Nothing throws across the ABI: a NULL or empty pack is
    rejected with a nonzero status and a plora_last_error() message, before any CUDA call."""
    import ctypes
    lib = _lib.lib()
    rc = lib.plora_linear_fwd(None, None, None, 64, 64, None, 1, None, None, None, None, 64, None)
    assert rc != 0 and b"pack is NULL" in lib.plora_last_error()
    empty = _lib.PackStruct()
    rc = lib.plora_lora_segred(None, ctypes.byref(empty), 64, None, None, None)
    assert rc != 0 and b"no adapters" in lib.plora_last_error()
    rc = lib.plora_linear_bwd(None, None, None, 64, 64, None, 1, None, None, None, None, None, None, 64, None,
                              None, None)
    assert rc != 0 and b"pack is NULL" in lib.plora_last_error()
