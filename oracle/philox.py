"""Philox4x32-10 counter-based generator, written from its published definition.

Reading Z6: the paper names no RNG (P:278, P:287 only say
"sampled with replacement"); BASELINE.json's north star fixes Philox4x32-10
keyed on (seed, iteration).  Definition (Salmon, Moraes, Dror, Shaw, SC'11,
"Parallel random numbers: as easy as 1, 2, 3"): 10 rounds of
    (hi0, lo0) = mulhilo32(0xD2511F53, c0); (hi1, lo1) = mulhilo32(0xCD9E8D57, c2)
    c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
with the key bumped by the Weyl constants (0x9E3779B9, 0xBB67AE85) before
every round but the first.  Pinned by the published known-answer vectors in
tests/golden/philox4x32_10_kat.txt.
Vectorised with numpy uint64 arithmetic (32x32 -> 64-bit products are exact).
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)
S32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0, k1, rounds: int = 10):
    """Return the four uint32 output words (as uint64 arrays) for counters (c0..c3), key (k0, k1)."""
    c = [np.asarray(x, dtype=np.uint64) & MASK32 for x in (c0, c1, c2, c3)]
    k0 = np.asarray(k0, dtype=np.uint64) & MASK32
    k1 = np.asarray(k1, dtype=np.uint64) & MASK32
    for r in range(rounds):
        if r > 0:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> S32, p0 & MASK32
        hi1, lo1 = p1 >> S32, p1 & MASK32
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return c


def philox_u64(j, stream: int, purpose: int, seed: int):
    """u = x1 * 2^32 + x0 for counter (j lo, j hi, stream, purpose), key (seed lo, seed hi) (reading Z6)."""
    j = np.asarray(j, dtype=np.uint64)
    x = philox4x32_10(j & MASK32, j >> S32, np.uint64(stream & 0xFFFFFFFF),
                      np.uint64(purpose & 0xFFFFFFFF),
                      np.uint64(seed & 0xFFFFFFFF), np.uint64((seed >> 32) & 0xFFFFFFFF))
    return (x[1] << S32) | x[0], x


def mulhi64(u, W: int):
    """floor(u * W / 2^64) exactly, for uint64 arrays u and a Python int 0 <= W < 2^64."""
    u = np.asarray(u, dtype=np.uint64)
    W = int(W)
    uh, ul = u >> S32, u & MASK32
    Wh, Wl = np.uint64(W >> 32), np.uint64(W & 0xFFFFFFFF)
    ll = ul * Wl
    lh = ul * Wh
    hl = uh * Wl
    hh = uh * Wh
    mid = (ll >> S32) + (lh & MASK32) + (hl & MASK32)
    return hh + (lh >> S32) + (hl >> S32) + (mid >> S32)
