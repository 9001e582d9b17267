"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element, on the same seeded inputs (pic_inputs).  Tolerances (SURVEY §8(c.4),
BASELINE.json north_star):
  keys, permutation, push given an identical field ... bit-exact
  rho after scatter .................................. 1e-14 of max|rho|
  E after solve (same rho) ........................... 1e-12 of max|E|
  W_x per step ....................................... 1e-10 relative
  x, v after 20 steps ................................ 1e-12 (periodic |dx|/L, |dv|/max(|v|,1))
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from pic_inputs import landau_state, random_grid, random_field

pytestmark = pytest.mark.gpu

K = 0.5
L = 2 * np.pi / K
DT = 0.05


@pytest.fixture(scope="module")
def Sim():
    import torch
    from paper_2605_05469_b200 import Simulation

    torch.cuda.set_device(0)
    return Simulation


def dist(a, b):
    """(max periodic |dx|/L, max |dv|/max(|v|,1)) between two (6, np) states."""
    dx = np.abs(a[:3] - b[:3])
    dx = np.minimum(dx, L - dx) / L
    dv = np.abs(a[3:] - b[3:]) / np.maximum(np.abs(b[3:]), 1.0)
    return dx.max(initial=0.0), dv.max(initial=0.0)


def test_sampler_matches_oracle_sampler(Sim):
    """Init (D#10/D#11): identical Philox uniforms; positions/velocities to a few ulp."""
    n, ppc = 16, 8
    sim = Sim(n=n, ppc=ppc, seed=7, half_kick=False)
    g = sim.get_particles()
    ref = O.sample_landau(ppc * n ** 3, K, L, 0.05, 7)
    ref, _ = O.sort(n, L, ref)
    dx, dv = dist(g, ref)
    assert dx < 1e-14 and dv < 1e-13, (dx, dv)


def test_init_half_kick_matches_oracle(Sim):
    n, ppc = 16, 8
    sim = Sim(n=n, ppc=ppc, seed=3, half_kick=True)
    g = sim.get_particles()
    ref = O.init_state(n, ppc, seed=3, half_kick_=True)
    dx, dv = dist(g, ref)
    assert dx < 1e-14 and dv < 1e-12, (dx, dv)


@pytest.mark.parametrize("n,ppc,alpha", [(16, 8, 0.05), (32, 3, 0.5), (16, 1, 0.9)])
def test_sort_keys_and_permutation_bit_exact(Sim, n, ppc, alpha):
    """Import (any order) -> stable sort by cell key: keys and perm bit-exact; includes
    empty cells (alpha = 0.9, ppc = 1) and ragged per-cell counts."""
    xv = landau_state(n, ppc, alpha=alpha, seed=n + ppc)
    sim = Sim(n=n, ppc=ppc, half_kick=False)
    sim.set_particles(xv)
    keys, perm = sim.keys_perm()
    xs, rperm = O.sort(n, L, xv)
    assert np.array_equal(perm, rperm)
    assert np.array_equal(keys, O.keys(n, L, xs))
    assert np.array_equal(sim.get_particles(), xs)


def test_deposit_matches_oracle(Sim):
    n, ppc = 32, 8
    xv = landau_state(n, ppc, seed=11)
    sim = Sim(n=n, ppc=ppc, half_kick=False)
    sim.set_particles(xv)
    rho = sim.get_grid(0)
    ref = O.deposit(n, L, O.sort(n, L, xv)[0], -L ** 3 / xv.shape[1])
    assert np.max(np.abs(rho - ref)) <= 1e-14 * np.max(np.abs(ref))
    assert abs(rho.sum() * (L / n) ** 3 + L ** 3) < 1e-12 * L ** 3   # charge conservation


def test_deposit_special_positions(Sim):
    """Particles exactly on nodes, at cell centres, on x = 0 and just below L."""
    n, ppc = 16, 1
    h = L / n
    rng = np.random.default_rng(0)
    idx = rng.integers(0, n, size=(3, n ** 3))
    xv = np.zeros((6, n ** 3))
    xv[:3] = idx * h
    xv[:3, ::3] += 0.5 * h
    xv[0, 1::7] = np.nextafter(L, 0)
    xv[1, 2::5] = 0.0
    xv[3:] = rng.standard_normal((3, n ** 3))
    sim = Sim(n=n, ppc=ppc, half_kick=False)
    sim.set_particles(xv)
    rho = sim.get_grid(0)
    ref = O.deposit(n, L, O.sort(n, L, xv)[0], -L ** 3 / xv.shape[1])
    assert np.max(np.abs(rho - ref)) <= 1e-14 * np.max(np.abs(ref))


@pytest.mark.parametrize("n", [16, 64, 128, 256])
def test_solve_matches_oracle(Sim, n):
    """Element-wise solve parity.  At 128^3 and 256^3 every persistent CTA of the x / y
    passes handles several tiles, so the cp.async next-tile prefetch path runs under the
    element-wise check (at 64^3 each CTA gets at most one tile)."""
    rho = random_grid(n, seed=n, mean=-1.0)
    sim = Sim(n=n, ppc=1, half_kick=False)
    E, wx, w = sim.solve_injected(rho)
    with O.threads(min(16, os.cpu_count() or 1)):     # OpenMP mode: the same per-line FFT arithmetic
        ref, _ = O.solve_fft(n, L, rho)
    assert np.max(np.abs(E - ref)) <= 1e-12 * np.max(np.abs(ref))
    rwx, rw = O.field_energy(n, L, ref)
    assert abs(wx - rwx) <= 1e-12 * rwx and abs(w - rw) <= 1e-12 * rw


def test_solve_single_mode_closed_form(Sim):
    """S:210 on the GPU: rho = cos(k1 y) => E_y = sin(k1 y)/k1."""
    n = 32
    k1 = 2 * np.pi / L
    y = np.arange(n) * L / n
    rho = np.broadcast_to(np.cos(k1 * y)[None, :, None], (n, n, n)).copy()
    sim = Sim(n=n, ppc=1, half_kick=False)
    E, _, _ = sim.solve_injected(rho)
    want = np.broadcast_to((np.sin(k1 * y) / k1)[None, :, None], (n, n, n))
    assert np.max(np.abs(E[1] - want)) < 1e-12
    assert np.max(np.abs(E[0])) < 1e-12 and np.max(np.abs(E[2])) < 1e-12


@pytest.mark.parametrize("n,ppc", [(16, 8), (32, 2)])
def test_push_bit_exact_given_identical_field(Sim, n, ppc):
    """Gather + push + wrap + sort with an injected E: bit-exact (D#17)."""
    xv = landau_state(n, ppc, seed=3)
    xv[3:] *= 5.0                                   # large moves: many wraps
    E = random_field(n, seed=4)
    sim = Sim(n=n, ppc=ppc, half_kick=False)
    sim.set_particles(xv)
    sim.push_injected(E)
    g = sim.get_particles()
    xs, _ = O.sort(n, L, xv)
    Ep = O.gather(n, L, xs, E)
    ref = O.push(L, xs, Ep, -DT, DT)
    ref, rperm = O.sort(n, L, ref)
    assert np.array_equal(g, ref)
    _, perm = sim.keys_perm()
    assert np.array_equal(perm, rperm)


@pytest.mark.parametrize("n,ppc,seed", [(16, 8, 1), (32, 8, 2), (64, 4, 3)])
def test_twenty_step_parity(Sim, n, ppc, seed):
    """BJ: 20 steps, W_x within 1e-10 relative each step; x, v within 1e-12."""
    xv = landau_state(n, ppc, seed=seed)
    sim = Sim(n=n, ppc=ppc, half_kick=False)
    sim.set_particles(xv)
    ex = sim.step(20)
    g = sim.get_particles()
    ref, rex, _, _ = O.run(n, L, DT, xv, 20)
    assert np.all(np.abs(ex - rex) <= 1e-10 * rex), np.max(np.abs(ex - rex) / rex)
    dx, dv = dist(g, ref)
    assert dx <= 1e-12 and dv <= 1e-12, (dx, dv)
    wx, w = sim.field_energy()
    assert wx == ex[-1] and w >= wx


def test_pic_init_then_steps_match_oracle(Sim):
    """The whole public path: pic_init (sampler + half kick) then 10 steps vs the oracle
    run from the oracle's own sampler (D#11: init agrees to ulps, not bits)."""
    n, ppc = 16, 8
    sim = Sim(n=n, ppc=ppc, seed=9)
    ex = sim.step(10)
    ref0 = O.init_state(n, ppc, seed=9)
    _, rex, _, _ = O.run(n, L, DT, ref0, 10)
    assert np.all(np.abs(ex - rex) <= 1e-9 * rex)


def test_steps_zero_and_errors(Sim):
    from paper_2605_05469_b200 import PicError

    sim = Sim(n=16, ppc=1, half_kick=False)
    assert sim.step(0).size == 0
    bad = landau_state(16, 1, seed=2)
    bad[0, 0] = L            # out of [0, L)
    with pytest.raises(PicError):
        sim.set_particles(bad)
    sim.step(1)              # context still usable after EINVAL
