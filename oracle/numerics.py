"""Rounding to bfloat16, written out from the IEEE definition.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

bf16(x) = round-to-nearest-even of x to 8 significant bits with fp32's 8-bit
exponent range (SURVEY.md §8(c) step 1 notes: "bf16(.) is round-to-nearest-even
to bfloat16, applied exactly where the GPU feeds an MMA operand or stores to
the KV cache"). The oracle rounds its fp64 value DIRECTLY to bf16 (one
rounding), because the exact value it models is the fp64 one.

Subnormal bf16 results (|x| < 2^-126) are rounded on the same 2^-133 grid as
the smallest subnormal, exactly as IEEE prescribes; overflow goes to +-inf.

Pinned by: tests/test_oracle_numerics.py — agreement with torch's fp32->bf16
cast on fp32-representable inputs (single rounding there), hand-written
halfway cases (ties to even), and exactness on bf16-representable values.
"""
import numpy as np


def round_bf16(x):
    """Round fp64 values to the nearest bf16 value (ties to even); returns fp64."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    finite = np.isfinite(x)
    xf = x[finite]
    ax = np.abs(xf)
    # exponent of each value (ax = m * 2^e, m in [1,2)); zero handled separately
    with np.errstate(divide="ignore"):
        e = np.floor(np.log2(np.where(ax > 0, ax, 1.0)))
    # correct possible off-by-one of log2 near powers of two
    e = np.where(np.ldexp(1.0, e.astype(np.int64)) > ax, e - 1, e)
    e = np.where(np.ldexp(1.0, (e + 1).astype(np.int64)) <= ax, e + 1, e)
    e = np.maximum(e, -126.0)          # subnormal range shares the 2^-133 quantum
    quantum = np.ldexp(1.0, (e - 7).astype(np.int64))   # 8 significant bits
    scaled = ax / quantum                                # exact (power of two)
    r = np.round(scaled)                                 # numpy rounds half to even
    res = r * quantum
    res = np.where(res >= 2.0 ** 128, np.inf, res)       # overflow
    res = np.where(ax == 0, 0.0, res)
    out[finite] = np.copysign(res, xf)
    out[~finite] = x[~finite]
    return out


def is_bf16(x):
    """True where x is exactly representable in bf16."""
    x = np.asarray(x, dtype=np.float64)
    return round_bf16(x) == x
