"""Philox4x32-10 counter-based RNG and the uniform mapping used by the verifier.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Source of the definition: north_star asks for "counter-based Philox RNG (so
draws are reproducible)"; the paper has no RNG. The
generator is Philox4x32 with 10 rounds (Salmon et al., Random123), with the
cuRAND multiplier / Weyl constants:

    M0 = 0xD2511F53, M1 = 0xCD9E8D57, W0 = 0x9E3779B9, W1 = 0xBB67AE85
    round:  (hi0, lo0) = M0 * c0 ; (hi1, lo1) = M1 * c2
            c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    key bump between rounds: k0 += W0, k1 += W1  (10 rounds, 9 bumps)

Counter layout (our reading S7, R7):
    key     = (seed & 0xffffffff, seed >> 32)
    counter = (z, rid & 0xffffffff, rid >> 32, purpose << 28 | x >> 2)
    ACCEPT: purpose 0, x = 0, output lane 0
    RACE:   purpose 1, output lane x & 3
Uniform: U = ((w >> 9) + 0.5) * 2**-23  in (0, 1). (SURVEY.md proposed >> 8 and
2^-24, but (n + 1/2) 2^-24 needs 25 significant bits for n >= 2^23 and is not
exact in fp32; the 23-bit lattice is exact in fp32 and fp64 — DESIGN.md R7.)

Pinned by: tests/test_oracle_philox.py — Random123 known-answer vectors
(tests/golden/philox_kat.txt), scalar-vs-vectorised agreement, and the
uniform mapping worked value U(0,0,0,ACCEPT) = ((0x6627e8d5 >> 9) + 0.5) 2^-23.
"""
import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF

ACCEPT = 0
RACE = 1


def philox4x32_10(ctr, key):
    """Scalar Philox4x32-10 on python ints. ctr: 4 words, key: 2 words."""
    c0, c1, c2, c3 = (int(v) & MASK32 for v in ctr)
    k0, k1 = (int(v) & MASK32 for v in key)
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK32
        hi1, lo1 = p1 >> 32, p1 & MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return (c0, c1, c2, c3)


def philox4x32_10_np(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10; all arguments broadcastable uint32-valued arrays.

    Returns four uint64 arrays holding 32-bit words. Same rounds as the scalar
    version above (products formed exactly in uint64).
    """
    c0 = np.asarray(c0, dtype=np.uint64)
    c1 = np.asarray(c1, dtype=np.uint64)
    c2 = np.asarray(c2, dtype=np.uint64)
    c3 = np.asarray(c3, dtype=np.uint64)
    k0 = np.asarray(k0, dtype=np.uint64)
    k1 = np.asarray(k1, dtype=np.uint64)
    c0, c1, c2, c3, k0, k1 = np.broadcast_arrays(c0, c1, c2, c3, k0, k1)
    m32 = np.uint64(MASK32)
    for r in range(10):
        if r > 0:
            k0 = (k0 + np.uint64(W0)) & m32
            k1 = (k1 + np.uint64(W1)) & m32
        p0 = np.uint64(M0) * c0
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & m32
        hi1, lo1 = p1 >> np.uint64(32), p1 & m32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def word_to_uniform(w):
    """U = ((w >> 9) + 0.5) * 2^-23 (exact in fp32 and fp64)."""
    w = np.asarray(w, dtype=np.uint64)
    return ((w >> np.uint64(9)).astype(np.float64) + 0.5) * (2.0 ** -23)


def uniform_accept(seed, rid, z):
    """u_j = U(seed, rid, z, ACCEPT): scalar float."""
    ctr = (z, rid & MASK32, (rid >> 32) & MASK32, (ACCEPT << 28) | 0)
    w = philox4x32_10(ctr, (seed & MASK32, (seed >> 32) & MASK32))[0]
    return ((w >> 9) + 0.5) * (2.0 ** -23)


def uniform_race(seed, rid, z, vocab):
    """U(seed, rid, z, RACE, x) for x = 0..vocab-1 (fp64 array)."""
    x = np.arange(vocab, dtype=np.uint64)
    c3 = (np.uint64(RACE << 28)) | (x >> np.uint64(2))
    words = philox4x32_10_np(z & MASK32, rid & MASK32, (rid >> 32) & MASK32, c3,
                             seed & MASK32, (seed >> 32) & MASK32)
    lane = (x & np.uint64(3)).astype(np.int64)
    w = np.choose(lane, words)
    return word_to_uniform(w)


def uniform_accept_rank(seed, rid, z, s):
    """Accept uniform of the s-th sibling tried at sequence index z (tree drafts, R30):
    counter (z, rid_lo, rid_hi, ACCEPT << 28 | s >> 2), output lane s & 3 — the RACE layout with
    x = s. s = 0 is uniform_accept(seed, rid, z): a chain is a tree of only-children."""
    ctr = (z, rid & MASK32, (rid >> 32) & MASK32, (ACCEPT << 28) | (int(s) >> 2))
    w = philox4x32_10(ctr, (seed & MASK32, (seed >> 32) & MASK32))[int(s) & 3]
    return ((w >> 9) + 0.5) * (2.0 ** -23)
