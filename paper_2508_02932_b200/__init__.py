"""paper_2508_02932_b200 -- B200-native (sm_100a) packed multi-LoRA training hot path.

Drop-in for the reference's packed-LoRA operator API (``lorasweep.lorapack``):
the names below keep the reference's signatures; the arithmetic runs in the
tcgen05/TMA kernels of libplora.so (see include/plora.h).
"""

__version__ = "0.1.0"

from .lorapack import (  # noqa: F401
    AdapterWeights,
    GradCheckReport,
    PackedAdapters,
    adapter_backward,
    adapter_forward,
    grad_check,
    pack_adapters,
    packed_backward,
    packed_forward,
    unpack_adapters,
)
