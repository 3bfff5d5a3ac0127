import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "lorapack_golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100a (B200) CUDA device")


def load_golden():
    """Yield (name, case-dict) for every golden case generated from the real reference."""
    z = np.load(GOLDEN)
    for name in z["__cases__"]:
        name = str(name)
        keys = [k for k in z.files if k.startswith(name + "/")]
        case = {k.split("/", 1)[1]: z[k] for k in keys}
        case["rank_offsets"] = tuple(int(v) for v in case["rank_offsets"])
        case["row_offsets"] = tuple(int(v) for v in case["row_offsets"])
        case["alphas"] = tuple(float(v) for v in case["alphas"])
        for k in ("w", "down_block", "up_block", "inputs", "upstream"):
            case[k] = case[k].astype(np.float64)
        yield name, case


def split_rows(arr, row_offsets):
    return [arr[row_offsets[i]:row_offsets[i + 1]] for i in range(len(row_offsets) - 1)]


def split_cols(arr, rank_offsets):
    return [arr[:, rank_offsets[i]:rank_offsets[i + 1]] for i in range(len(rank_offsets) - 1)]


@pytest.fixture(scope="session")
def golden_cases():
    return list(load_golden())


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
