"""numpy restatement of the action sampler (TEST INFRASTRUCTURE ONLY -- see oracle/__init__).

beastpipe sample_actions (model.py:218-221) is Gumbel-max: argmax(logits + Gumbel noise).
The kernels draw the noise from Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random
numbers: as easy as 1, 2, 3", SC'11; round constants M0 = 0xD2511F53, M1 = 0xCD9E8D57, Weyl
key increments 0x9E3779B9 / 0xBB67AE85) keyed by the 64-bit seed, counter (row lo, row hi,
column // 4, 0), word column % 4; u = ((w >> 8) + 1/2) 2^-24, noise = -log(-log u)
(include/beast_b200.h bp_sample_actions_f32).  This restates that draw so tests can pin the
keying bit-exactly (the Philox words) and the argmax up to float32 log rounding.
"""
from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 over uint32 arrays; returns the four output words."""
    c = [np.asarray(x, dtype=np.uint32) for x in (c0, c1, c2, c3)]
    k0, k1 = np.uint32(k0), np.uint32(k1)
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = M0 * c[0].astype(np.uint64)
            p1 = M1 * c[2].astype(np.uint64)
            hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & MASK).astype(np.uint32)
            hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & MASK).astype(np.uint32)
            c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
            k0 = np.uint32(k0 + W0)
            k1 = np.uint32(k1 + W1)
    return c


def gumbel_words(seed: int, n: int, A: int) -> np.ndarray:
    """Philox words (n, A) uint32 of rows 0..n-1, columns 0..A-1."""
    rows = np.arange(n, dtype=np.uint64)
    out = np.empty((n, A), dtype=np.uint32)
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    for j0 in range(0, A, 4):
        w = philox4x32_10((rows & MASK).astype(np.uint32), (rows >> np.uint64(32)).astype(np.uint32),
                          np.full(n, j0 // 4, np.uint32), np.zeros(n, np.uint32), k0, k1)
        for q in range(min(4, A - j0)):
            out[:, j0 + q] = w[q]
    return out


def sample_actions(logits: np.ndarray, seed: int, greedy: bool = False) -> np.ndarray:
    """Gumbel-max (float64 noise) with the kernels' keying; greedy: argmax."""
    logits = np.asarray(logits, dtype=np.float64)
    if greedy:
        return logits.argmax(-1).astype(np.int64)
    w = gumbel_words(seed, logits.shape[0], logits.shape[1])
    u = ((w >> np.uint32(8)).astype(np.float64) + 0.5) * 2.0 ** -24
    return (logits + -np.log(-np.log(u))).argmax(-1).astype(np.int64)
