"""Time the CUTLASS CuTe-DSL Blackwell FMHA backward example (library code shipped in the
image under flashinfer/data/cutlass/examples) on the C3 attention shape, for comparison with
cuDNN's SDPA backward (tools/attn_cudnn_split.py)."""
import os
import sys

D = "/opt/prime-rl/.venv/lib/python3.12/site-packages/flashinfer/data/cutlass/examples/python/CuTeDSL/blackwell"
sys.path.insert(0, D)
sys.path.insert(0, os.path.dirname(D))
import cutlass  # noqa: E402
import fmha_bwd  # noqa: E402

us = fmha_bwd.run(1024, 1024, 32, 8, 128, 32, True, False, cutlass.BFloat16, cutlass.Float32, (128, 128), 0.0,
                  (-1, -1), 3, 20, True, False)
flops = 2.5 * 4 * 32 * 32 * 1024 * 1024 * 128 / 2
print(f"cute fmha bwd (b=32, s=1024, h_q=32, h_k=8, d=128, causal): {us:.1f} us, {flops / us / 1e6:.0f} TF/s")
