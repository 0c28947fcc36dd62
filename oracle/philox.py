"""Philox4x32-10 counter-based generator, vectorised numpy (test infrastructure).

Salmon et al. 2011 ("Parallel random numbers: as easy as 1, 2, 3"); constants
M0 = 0xD2511F53, M1 = 0xCD9E8D57, Weyl W0 = 0x9E3779B9, W1 = 0xBB67AE85, ten
rounds, first round with the unbumped key.  Pinned by the Random123 known-answer
vectors in tests/golden/philox_kat.txt.

Counter layout and Box-Muller are readings of SURVEY §8c1-2 / Q10:
  key     = (seed_lo, seed_hi)
  counter = (index, slot | stream << 16, frame_lo, frame_hi)
  u1 = (x + 1) 2^-32 in (0, 1],  u2 = x' 2^-32,
  (g1, g2) = sqrt(-2 ln u1) (cos 2 pi u2, sin 2 pi u2)
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK = np.uint64(0xFFFFFFFF)

STREAM_FIELD = 0
STREAM_OUTPUT_NOISE = 1


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10; inputs broadcastable uint32-valued arrays / ints."""
    c0, c1, c2, c3 = [np.asarray(c, dtype=np.uint64) & MASK for c in (c0, c1, c2, c3)]
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    c0, c1, c2, c3 = c0.copy(), c1.copy(), c2.copy(), c3.copy()
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0)), lo1, (hi0 ^ c3 ^ np.uint64(k1)), lo0
    return c0, c1, c2, c3


def box_muller(xa, xb):
    """(g1, g2) standard normals from two uint32 words (float64)."""
    u1 = (np.asarray(xa, dtype=np.float64) + 1.0) * 2.0 ** -32
    u2 = np.asarray(xb, dtype=np.float64) * 2.0 ** -32
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.cos(2.0 * np.pi * u2), r * np.sin(2.0 * np.pi * u2)


def gaussians(index, slot, stream, frame, seed):
    """Four Philox words -> ((g_a1, g_a2), (g_b1, g_b2)) for counter (index, slot|stream<<16, frame)."""
    seed = int(seed)
    frame = int(frame)
    x0, x1, x2, x3 = philox4x32_10(index, (int(slot) | (int(stream) << 16)), frame & 0xFFFFFFFF,
                                   (frame >> 32) & 0xFFFFFFFF, seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    return box_muller(x0, x1), box_muller(x2, x3)
