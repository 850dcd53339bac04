"""The library's GEMM kernels (tcgen05 1-SM, tcgen05 2-SM cluster pair, weight-major 2-SM, SIMT) through the
sv_debug_gemm test hook, against the plain definition C = A B^T evaluated in fp64 on the host.

Inputs are bf16, so products are exact in fp32; only the fp32 accumulation rounds. The bound
used is the standard recursive-summation one, |C - C*| <= gamma_K * sum_k |a_k b_k| with
gamma_K = K u / (1 - K u), u = 2^-24 (any summation order satisfies it)."""
import numpy as np
import pytest
import torch

import synth
from paper_2604_09562_b200 import sv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lane():
    cfg = synth.TOY.with_(max_batch=64, max_slots=8, n_pages=16)
    w = synth.model_weights(cfg, seed=0)
    return sv.Lane(cfg, {k: v.cuda() for k, v in w.items()})


@pytest.mark.parametrize("variant", [1, 2, 3, 5, 0])
@pytest.mark.parametrize("M,N,K", [(1, 300, 64), (200, 1000, 4096), (576, 6144, 4096),
                                   (130, 4096 + 64 + 7, 512), (576, 520, 14336)])
def test_gemm_against_definition(lane, variant, M, N, K):
    if variant == 3 and M * N * K > 2e9:
        pytest.skip("SIMT GEMM checked on the smaller shapes only")
    g = torch.Generator().manual_seed(M * 7919 + N * 31 + K)
    a = torch.randn(M, K, generator=g).to(torch.bfloat16)
    b = (torch.randn(N, K, generator=g) * 0.05).to(torch.bfloat16)
    c = torch.full((M, N), float("nan"), device="cuda")
    lane.debug_gemm(a.cuda(), b.cuda(), c, variant)
    torch.cuda.synchronize()
    A, B = a.double().numpy(), b.double().numpy()
    exact = A @ B.T
    mag = np.abs(A) @ np.abs(B).T
    u = 2.0 ** -24
    gamma = K * u / (1 - K * u)
    got = c.cpu().double().numpy()
    assert np.isfinite(got).all()
    bad = np.abs(got - exact) > gamma * mag + 1e-30
    assert not bad.any(), f"{bad.sum()} elements outside the fp32 summation bound"
