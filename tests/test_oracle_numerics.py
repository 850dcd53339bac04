"""Pins for oracle/numerics.py: bf16 round-to-nearest-even."""
import numpy as np
import torch

from oracle.numerics import round_bf16, is_bf16


def test_matches_torch_cast_on_fp32_inputs():
    # for fp32-representable inputs torch's fp32->bf16 cast is a single RNE rounding
    g = torch.Generator().manual_seed(0)
    x = torch.randn(200000, generator=g) * torch.exp(torch.randn(200000, generator=g) * 8)
    x = torch.cat([x, torch.tensor([0.0, -0.0, 1e-39, -3e-40, 3.3e38, 65504.0])])
    ref = x.to(torch.bfloat16).to(torch.float64).numpy()
    got = round_bf16(x.to(torch.float64).numpy())
    assert np.array_equal(ref, got)


def test_ties_to_even():
    ulp = 2.0 ** -7
    assert round_bf16(1.0 + ulp / 2) == 1.0                 # tie -> even (mantissa 0)
    assert round_bf16(1.0 + 3 * ulp / 2) == 1.0 + 2 * ulp   # tie -> even (mantissa 2)
    assert round_bf16(1.0 + ulp / 2 + 2.0 ** -30) == 1.0 + ulp
    assert round_bf16(-(1.0 + ulp / 2)) == -1.0
    assert round_bf16(255.5 * 2.0 ** -6) == 4.0             # tie at the top of [2,4): carry to 4


def test_identity_on_bf16_values():
    v = torch.randn(10000).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(round_bf16(v), v)
    assert is_bf16(v).all()


def test_direct_rounding_from_fp64_is_single_rounding():
    # 1 + 2^-8 + 2^-40 is above the tie in fp64 but rounds to the tie in fp32;
    # the oracle rounds the exact value once (up), not via fp32 (which would tie to even).
    x = 1.0 + 2.0 ** -8 + 2.0 ** -40
    assert round_bf16(x) == 1.0 + 2.0 ** -7
