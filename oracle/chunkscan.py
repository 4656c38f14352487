"""CPU mirror of the B200 fast-mode residual-diagonal scan and inverse-CDF sampling
(paper_2410_03969_b200/csrc/sampling.cu), including its row-sharded protocol.

TEST INFRASTRUCTURE ONLY.  The reference's cumulative_sums is a strictly sequential
sum (rng.hpp:67-75, restated in rpc_oracle.c); the GPU's fast mode uses a fixed
two-level association instead.  This module restates that fixed
order in plain Python floats (IEEE binary64, one rounding per add) so tests can check
(a) the GPU sampler bit-for-bit, (b) the sharded protocol (chunk totals allgathered,
owner shard resolves the draw) against the unsharded one, and (c) agreement with the
reference's sequential sampler on the same draws.
"""
from __future__ import annotations

import bisect

import numpy as np

KCHUNK = 4096
THREADS = 256
EPT = 16


def u01(z: int) -> float:
    return float(z >> 11) * (2.0 ** -53)


def splitmix64_draw(seed: int, n: int) -> int:
    M = (1 << 64) - 1
    z = (seed + (n + 1) * 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def chunk_local(uc) -> list:
    """local_i for the valid elements of one chunk (sampling.cu chunk_scan_core)."""
    n_valid = len(uc)
    pad = [float(v) for v in uc] + [0.0] * (KCHUNK - n_valid)
    s = []
    for t in range(THREADS):
        acc = 0.0
        row = []
        for e in range(EPT):
            acc = acc + pad[t * EPT + e]
            row.append(acc)
        s.append(row)
    bases, b = [], 0.0
    for t in range(THREADS):
        bases.append(b)
        b = b + s[t][EPT - 1]
    return [bases[i // EPT] + s[i // EPT][i % EPT] for i in range(n_valid)]


def chunk_totals(u_shard) -> list:
    out = []
    for c0 in range(0, len(u_shard), KCHUNK):
        loc = chunk_local(u_shard[c0:c0 + KCHUNK])
        out.append(loc[-1])
    return out


def chunk_ends(totals) -> list:
    ends, off = [], 0.0
    for t in totals:
        off = off + t
        ends.append(off)
    return ends


def locate(ends, r: float):
    """(chunk, mode, target) for one draw: mode 0 = first cumsum > target,
    mode 1 = clamp to N-1 then walk back over the zero plateau (rng.hpp:88-94)."""
    nc = len(ends)
    target = r * ends[-1]
    c = bisect.bisect_right(ends, target)
    if c == nc:
        c = nc - 1
        while c > 0 and ends[c] == ends[c - 1]:
            c -= 1
        return c, 1, target
    return c, 0, target


def resolve(uc, off: float, mode: int, target: float) -> int:
    """Row inside the chunk for a located draw (sampling.cu sample_kernel)."""
    loc = chunk_local(uc)
    if mode == 0:
        for i, v in enumerate(loc):
            if off + v > target:
                return i
        return 0
    best, prev = -1, off
    for i, v in enumerate(loc):
        cum = off + v
        if cum > prev:
            best = i
        prev = cum
    return max(best, 0)


def sample(u, seed: int, draw0: int, b: int) -> list:
    """Unsharded fast-mode sampler over the global u."""
    u = [float(v) for v in np.asarray(u, dtype=np.float64)]
    ends = chunk_ends(chunk_totals(u))
    out = []
    for j in range(b):
        c, mode, target = locate(ends, u01(splitmix64_draw(seed, draw0 + j)))
        off = ends[c - 1] if c else 0.0
        out.append(c * KCHUNK + resolve(u[c * KCHUNK:(c + 1) * KCHUNK], off, mode, target))
    return out
