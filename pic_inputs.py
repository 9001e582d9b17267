"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds none of the method's arithmetic (no deposit, solve, gather,
push, key or sort) and imports neither ``oracle`` nor the product package.  It
only draws particle states with the structure of the paper's workload
(P:140-146): positions with the Landau-perturbed density
prod_d (1 + alpha cos(k x_d)) / L on [0, L)^3 (drawn here by rejection sampling
with numpy's PCG64, *not* by the method's Philox/Newton sampler), velocities
standard normal.  Arrays are float64 of shape (6, np): x, y, z, vx, vy, vz.
"""
from __future__ import annotations

import numpy as np


def landau_state(n: int, ppc: int, k: float = 0.5, alpha: float = 0.05, seed: int = 1,
                 L: float | None = None, np_: int | None = None) -> np.ndarray:
    """Landau-perturbed positions + Maxwellian velocities (rejection sampling)."""
    if L is None:
        L = 2.0 * np.pi / k
    if np_ is None:
        np_ = ppc * n ** 3
    rng = np.random.Generator(np.random.PCG64(seed))
    xv = np.empty((6, np_), dtype=np.float64)
    for d in range(3):
        out = np.empty(0)
        while out.size < np_:
            m = int((np_ - out.size) * 1.2) + 16
            x = rng.random(m) * L
            acc = rng.random(m) * (1.0 + alpha) < 1.0 + alpha * np.cos(k * x)
            out = np.concatenate([out, x[acc]])
        xv[d] = out[:np_]
    xv[3:] = rng.standard_normal((3, np_))
    # guard: every coordinate in [0, L)
    xv[:3] = np.where(xv[:3] >= L, 0.0, xv[:3])
    return xv


def random_grid(n: int, seed: int = 1, mean: float = 0.0) -> np.ndarray:
    """A random (N, N, N) float64 grid (e.g. an injected charge density)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((n, n, n)) + mean


def random_field(n: int, seed: int = 1) -> np.ndarray:
    """A random (3, N, N, N) float64 vector field (e.g. an injected E)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((3, n, n, n))


def random_weights(np_: int, seed: int = 1) -> np.ndarray:
    """Standard-normal float64 weights (NUFFT type-1 inputs)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal(np_)


def random_spectrum(n: int, seed: int = 1) -> np.ndarray:
    """A random complex128 (N, N, N) mode array (NUFFT type-2 inputs)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((n, n, n)) + 1j * rng.standard_normal((n, n, n))
