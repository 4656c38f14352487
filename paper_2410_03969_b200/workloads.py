"""Seeded synthetic point sets for the BASELINE.json configurations.

Host-side input generation only (the reference's analog is datasets.hpp; its
configs are synthetic, no dataset is involved).  Every generator is driven by
the reference's SplitMix64 stream (rng.hpp:27-42) evaluated vectorised as a
counter: draw t (0-based) of seed s is mix64(s + (t+1)*0x9e3779b97f4a7c15).
Normals use the reference's Box-Muller map (rng.hpp:57-64: two uniforms per
normal, u1 redrawn only when it is exactly 0, which has probability 2^-53 and
is asserted absent).  Points are filled row by row (point i, then coordinate
j), as datasets.hpp:168-177 does.

Returned arrays are N x d float64 in C (row-major) order; the C-ABI accepts
either layout through its `ld`/layout arguments.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_counter(seed: int, start: int, count: int) -> np.ndarray:
    """Draws [start, start+count) of SplitMix64(seed) as uint64."""
    with np.errstate(over="ignore"):
        t = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + t * _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniforms(seed: int, start: int, count: int) -> np.ndarray:
    z = splitmix64_counter(seed, start, count)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normals(seed: int, start: int, count: int) -> np.ndarray:
    """count standard normals from draws [start, start + 2*count)."""
    u = uniforms(seed, start, 2 * count)
    u1, u2 = u[0::2], u[1::2]
    if np.any(u1 <= 0.0):  # rng.hpp:61 redraw case; probability 2^-53 per normal
        raise RuntimeError("Box-Muller redraw case hit; pick another data seed")
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    d: int
    kernel: str        # "gaussian" | "l1laplace"
    sigma: float
    k: int
    b: int
    seed: int = 0      # algorithm seed (RunConfig::seed)
    data_seed: int = 0

    def points(self, n: int | None = None) -> np.ndarray:
        return GENERATORS[self.name](n or self.n, self.d, self.data_seed)


def gen_c1(n, d, seed):
    """C1: i.i.d. N(0,1) (make_gaussian_cloud, datasets.hpp:168-177)."""
    return normals(seed, 0, n * d).reshape(n, d)


def gen_c2(n, d, seed, n_comp=10):
    """C2: 10-component Gaussian mixture; means ~ N(0, 4I) (std 2), labels
    uniform via next_u64() % 10, unit covariance.  Draw layout: means use
    draws [0, 2*n_comp*d), labels the next n draws, point noise the rest."""
    means = 2.0 * normals(seed, 0, n_comp * d).reshape(n_comp, d)
    off = 2 * n_comp * d
    labels = (splitmix64_counter(seed, off, n) % np.uint64(n_comp)).astype(np.int64)
    off += n
    return means[labels] + normals(seed, off, n * d).reshape(n, d)


def gen_c3(n, d, seed):
    """C3: uniform on [0,1)^d via next_double (rng.hpp:40-42)."""
    return uniforms(seed, 0, n * d).reshape(n, d)


def gen_c4(n, d, seed):
    """C4: N(0,1) with coordinate j (1-based) scaled by 1/sqrt(j)."""
    x = normals(seed, 0, n * d).reshape(n, d)
    return x / np.sqrt(np.arange(1, d + 1, dtype=np.float64))


def gen_c5(n, d, seed):
    """C5: chemistry-like non-negative descriptors: 0 w.p. 0.7 else Exp(1)
    = -log(1 - U).  Draw 2t decides the zero, draw 2t+1 the magnitude."""
    u = uniforms(seed, 0, 2 * n * d)
    zero = u[0::2] < 0.7
    mag = -np.log1p(-u[1::2])
    return np.where(zero, 0.0, mag).reshape(n, d)


GENERATORS = {"C1": gen_c1, "C2": gen_c2, "C3": gen_c3, "C4": gen_c4, "C5": gen_c5}

# BASELINE.json "configs", in order.
CONFIGS = {
    "C1": Workload("C1", 20_000, 10, "gaussian", float(np.sqrt(10.0)), 200, 40),
    "C2": Workload("C2", 200_000, 20, "gaussian", float(np.sqrt(20.0)), 1000, 120),
    "C3": Workload("C3", 200_000, 50, "l1laplace", 5.0, 1000, 120),
    "C4": Workload("C4", 1_000_000, 30, "gaussian", 3.0, 1000, 120),
    "C5": Workload("C5", 2_000_000, 100, "l1laplace", 10.0, 4000, 200),
}
