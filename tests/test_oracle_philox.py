"""Pins for oracle/philox.py (reading Q4): Random123 known answers and the
closed form of the multiply-high integer map."""
import os

import numpy as np

from oracle.philox import draw, philox4x32_10, uniform_int

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def _kat():
    rows = []
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        v = [int(x, 16) for x in line.split()]
        rows.append((v[:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answers():
    rows = _kat()
    assert len(rows) == 3
    for ctr, key, want in rows:
        got = philox4x32_10(*ctr, *key)
        assert [int(x) for x in got] == want


def test_philox_vectorised_matches_scalar():
    rng = np.random.default_rng(11)
    c = rng.integers(0, 2**32, size=(4, 64), dtype=np.uint64)
    k = rng.integers(0, 2**32, size=(2, 64), dtype=np.uint64)
    vec = philox4x32_10(c[0], c[1], c[2], c[3], k[0], k[1])
    for i in range(64):
        sc = philox4x32_10(int(c[0, i]), int(c[1, i]), int(c[2, i]), int(c[3, i]),
                           int(k[0, i]), int(k[1, i]))
        assert [int(x[i]) for x in vec] == [int(x) for x in sc]


def test_draw_counter_layout():
    # draw(seed, h, v, s) = word s&3 of philox(ctr=(s>>2, 0, v, h), key=(lo, hi))
    seed = 0x123456789ABCDEF0
    for h, v, s in [(0, 0, 0), (1, 7, 3), (2, 123456, 5), (0, 2**31 - 1, 13)]:
        words = philox4x32_10(s >> 2, 0, v, h, seed & 0xFFFFFFFF, seed >> 32)
        assert int(draw(seed, h, v, s)) == int(words[s & 3])


def test_uniform_int_range_and_preimage_closed_form():
    # t = floor(u (j+1) / 2^32).  Closed form: the smallest u mapping to t is
    # ceil(t 2^32 / (j+1)), so preimage sizes differ by at most one.
    for j in [0, 1, 2, 4, 6, 9, 14, 24, 1000, 2**20 + 7, 2**31 - 1]:
        for t in sorted({0, 1, j // 2, j}):
            if t > j:
                continue
            u_lo = -(-(t << 32) // (j + 1))
            assert int(uniform_int(u_lo, j)) == t
            if u_lo > 0:
                assert int(uniform_int(u_lo - 1, j)) == t - 1
        sizes = {(-(-((t + 1) << 32) // (j + 1))) - (-(-(t << 32) // (j + 1))) for t in range(min(j + 1, 64))}
        assert max(sizes) - min(sizes) <= 1
        assert int(uniform_int(2**32 - 1, j)) == j
        assert int(uniform_int(0, j)) == 0
