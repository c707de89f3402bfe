"""Philox4x32-10 counter-based RNG (oracle side, numpy, vectorised).

Reading Q4: the paper does not name an RNG (Eq.2, P:240-244,
only says neighbours are chosen "at a given probability").  We fix
Philox4x32-10 (Salmon et al., SC'11, "Parallel random numbers: as easy as
1, 2, 3") so that a node's draws depend only on (rng_seed, hop, node, draw
index) -- rank-, order- and device-independent.

Pinned by the Random123 known-answer vectors (tests/golden/philox_kat.txt).
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)
S32 = np.uint64(32)


def _u(x):
    return np.asarray(x, dtype=np.uint64) & MASK


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Ten Philox4x32 rounds.  Arguments broadcast; returns 4 uint64 arrays.

    One round (Random123 philox4x32round):
        (hi0, lo0) = M0 * c0 ; (hi1, lo1) = M1 * c2
        c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    with the key bumped by (W0, W1) between rounds.
    """
    c0, c1, c2, c3, k0, k1 = (_u(x) for x in (c0, c1, c2, c3, k0, k1))
    c0, c1, c2, c3, k0, k1 = np.broadcast_arrays(c0, c1, c2, c3, k0, k1)
    for r in range(10):
        if r:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> S32, p0 & MASK
        hi1, lo1 = p1 >> S32, p1 & MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def draw(rng_seed: int, hop, node, s):
    """32-bit draw number s for (hop, node) -- DESIGN.md reading Q4.

    word (s & 3) of Philox4x32-10(ctr = (s >> 2, 0, node, hop),
    key = (lo32(rng_seed), hi32(rng_seed))).  This equals
    curand_init(rng_seed, (hop << 32) | node, s, &st); curand(&st).
    """
    rng_seed = int(rng_seed) & 0xFFFFFFFFFFFFFFFF
    s = np.asarray(s, dtype=np.uint64)
    node = np.asarray(node, dtype=np.uint64)
    hop = np.asarray(hop, dtype=np.uint64)
    out = philox4x32_10(s >> np.uint64(2), 0, node, hop,
                        rng_seed & 0xFFFFFFFF, rng_seed >> 32)
    w = (s & np.uint64(3)).astype(np.int64)
    w = np.broadcast_to(w, out[0].shape)
    stacked = np.stack(out, axis=0)
    return np.take_along_axis(stacked, w[None, ...], axis=0)[0]


def uniform_int(u32, j):
    """Integer in [0, j] from a 32-bit draw: floor(u32 * (j+1) / 2^32).

    Multiply-high with no rejection (reading Q4); bias <= (j+1)/2^32.
    """
    u32 = np.asarray(u32, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    return (u32 * (j + np.uint64(1))) >> S32
