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


def test_fused_dy_pass_plan_on_host():
    """plora_lora_dual_workspace_bytes plans the fused K3+K4 pass on the host (no device
    memory is touched): the C3 pack (16 adapters, T = 32768) takes the fused path with
    fp32 partials of about a third of dY's bytes; rank blocks > 1 and k % 128 != 0 run
    the separate kernels (0)."""
    import ctypes

    import numpy as np

    from paper_2508_02932_b200 import ops
    from paper_2508_02932_b200.meta import build_meta

    lib = _lib.lib()

    def plan(ranks, tokens, k):
        meta = build_meta(ranks, tokens, [1.0] * len(ranks))
        s = _lib.PackStruct()
        s.n_adapters, s.n_mtiles, s.total_tokens = len(ranks), len(meta.mtiles), meta.total_tokens
        s.nb, s.rpad16_total = meta.nb, meta.rpad16_total
        for f in ("d_mtiles", "d_row_off", "d_ranks", "d_rpad_off", "d_alpha"):   # never dereferenced
            setattr(s, f, 16)
        h_row = np.ascontiguousarray(meta.row_offsets, dtype=np.int64)
        s.h_row_off = h_row.ctypes.data
        karr = (ctypes.c_int64 * 1)(k)
        return int(lib.plora_lora_dual_workspace_bytes(ctypes.byref(s), 1, karr, ops._h_rpad(meta))), meta

    c3_tokens = [x * 1024 for x in [1, 1, 2, 4, 2, 1, 4, 1, 1, 2, 1, 4, 4, 2, 1, 1]]
    ws, meta = plan([8, 16, 32, 64] * 4, c3_tokens, 4096)
    dy_bytes = 2 * meta.total_tokens * 4096
    assert 0.15 * dy_bytes < ws < 0.5 * dy_bytes, (ws, dy_bytes)
    assert plan([8, 100], [4096, 4096], 4096)[0] == 0  # rank > 64: two rank blocks
    assert plan([8, 16, 32, 64] * 4, c3_tokens, 4000)[0] == 0   # k not a multiple of 128
    assert np.all(np.diff(meta.rpad_off) % 16 == 0)
