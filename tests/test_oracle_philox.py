"""Pins for oracle/philox.py (pins P7/P7b)."""
import os

import numpy as np

from oracle import philox

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def _kat():
    rows = []
    for line in open(GOLD):
        line = line.split("#")[0].strip()
        if not line:
            continue
        w = [int(x, 16) for x in line.split()]
        rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


def test_known_answer_vectors_scalar():
    for ctr, key, out in _kat():
        assert list(philox.philox4x32_10(ctr, key)) == out


def test_known_answer_vectors_vectorised():
    for ctr, key, out in _kat():
        got = philox.philox4x32_10_np(*[np.array([c]) for c in ctr], key[0], key[1])
        assert [int(g[0]) for g in got] == out


def test_vectorised_matches_scalar_random_counters():
    rng = np.random.default_rng(7)
    c = rng.integers(0, 2**32, size=(4, 200), dtype=np.uint64)
    k = rng.integers(0, 2**32, size=(2,), dtype=np.uint64)
    got = philox.philox4x32_10_np(c[0], c[1], c[2], c[3], k[0], k[1])
    for i in range(200):
        ref = philox.philox4x32_10([int(c[j, i]) for j in range(4)], [int(k[0]), int(k[1])])
        assert tuple(int(g[i]) for g in got) == ref


def test_uniform_worked_value():
    # U(seed=0, rid=0, z=0, ACCEPT) = ((0x6627e8d5 >> 9) + 0.5) * 2^-23 (KAT word 0; R7)
    assert philox.uniform_accept(0, 0, 0) == 0.39904648065567017
    assert philox.uniform_accept(0, 0, 0) == ((0x6627E8D5 >> 9) + 0.5) * 2.0 ** -23


def test_uniform_range_and_lattice():
    u = philox.uniform_race(123, 456, 789, 4096)
    assert np.all(u > 0) and np.all(u < 1)
    # on the (n + 1/2) 2^-23 lattice, exactly representable in fp32
    n = u * 2**23 - 0.5
    assert np.all(n == np.round(n))
    assert np.all(u.astype(np.float32).astype(np.float64) == u)


def test_race_lanes_share_one_call_per_four_entries():
    # entries 4m..4m+3 are the four output words of one Philox call
    seed, rid, z = 99, (5 << 32) | 17, 1000
    u = philox.uniform_race(seed, rid, z, 16)
    for m in range(4):
        ctr = (z, rid & 0xFFFFFFFF, rid >> 32, (philox.RACE << 28) | m)
        words = philox.philox4x32_10(ctr, (seed & 0xFFFFFFFF, seed >> 32))
        for lane in range(4):
            assert u[4 * m + lane] == ((words[lane] >> 9) + 0.5) * 2.0 ** -23


def test_uniform_distribution_moments():
    u = philox.uniform_race(1, 2, 3, 200000)
    assert abs(u.mean() - 0.5) < 0.005
    assert abs(u.var() - 1 / 12) < 0.002
