"""tcgen05 GEMM engine (K1/K6 path) vs a torch fp32 reference of the same bf16 operands."""

import pytest
import torch

from paper_2508_02932_b200 import ops

pytestmark = pytest.mark.gpu

SHAPES = [(128, 256, 64), (300, 200, 136), (1000, 1024, 1024), (257, 4096, 512), (4096, 1024, 4096),
          (64, 64, 64), (130, 136, 72)]


def _ref(a, w, kmajor, res=None):
    out = a.float() @ (w.float().t() if kmajor else w.float())
    if res is not None:
        out = out + res.float()
    return out


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("kmajor", [True, False])
def test_gemm_matches_torch(M, N, K, kmajor):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) if kmajor else
         torch.randn(K, N, device="cuda", generator=g)).to(torch.bfloat16)
    out = ops.gemm(a, w, kmajor)
    ref = _ref(a, w, kmajor)
    err = (out.float() - ref).norm() / ref.norm()
    assert err < 8e-3, float(err)


def test_gemm_residual_and_ldo():
    M, N, K = 384, 512, 256
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    res = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    out = ops.gemm(a, w, True, residual=res)
    ref = _ref(a, w, True, res)
    assert ((out.float() - ref).norm() / ref.norm()) < 8e-3


def test_gemm_bit_stable_across_runs():
    a = torch.randn(512, 1024, device="cuda").to(torch.bfloat16)
    w = torch.randn(768, 1024, device="cuda").to(torch.bfloat16)
    o1 = ops.gemm(a, w, True)
    o2 = ops.gemm(a, w, True)
    assert torch.equal(o1, o2)
