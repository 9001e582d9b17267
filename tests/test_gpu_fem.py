"""GPU parity of the matrix-free Q1 FEM solver (P:183-195, P:226,
P:260; D#33) against oracle_solve_fem / oracle_run_fem on the same seeded inputs.  The
GPU applies the assembled 27-point stencil, the oracle the element loop: the two agree
up to summation order, as do the dot products, so
  iteration counts ........................... equal
  phi, E after one solve (same rho) .......... 1e-10 of max |.|
  W_x per step (20 steps) .................... 1e-10 relative
  x, v after 20 steps ........................ 1e-12
and, beyond the oracle's sizes, the residual of the GPU's phi recomputed with torch."""
import itertools

import numpy as np
import pytest

from oracle import oracle as O
from pic_inputs import landau_state, random_grid

pytestmark = pytest.mark.gpu

K = 0.5
L = 2 * np.pi / K
DT = 0.05


@pytest.fixture(scope="module")
def Sim():
    import torch
    from paper_2605_05469_b200 import Simulation

    torch.cuda.set_device(0)

    def make(**kw):
        return Simulation(solver="fem", **kw)

    return make


def dist(a, b):
    dx = np.abs(a[:3] - b[:3])
    dx = np.minimum(dx, L - dx) / L
    dv = np.abs(a[3:] - b[3:]) / np.maximum(np.abs(b[3:]), 1.0)
    return dx.max(initial=0.0), dv.max(initial=0.0)


@pytest.mark.parametrize("n,tol", [(16, 1e-4), (32, 1e-4), (32, 1e-10)])
def test_fem_solve_matches_oracle(Sim, n, tol):
    rho = random_grid(n, seed=n + 1, mean=-1.0)
    sim = Sim(n=n, ppc=1, half_kick=False, pcg_tol=tol)
    E, wx, w = sim.solve_injected(rho)
    it, _, _, rel = sim.pcg_stats()
    phi = sim.get_phi()
    rE, rphi, rit, rrel = O.solve_fem(n, L, rho, tol=tol)
    assert it == rit and it > 0, (it, rit)
    assert abs(rel - rrel) <= 1e-6 * rrel
    assert np.max(np.abs(phi - rphi)) <= 1e-10 * np.max(np.abs(rphi))
    assert np.max(np.abs(E - rE)) <= 1e-10 * np.max(np.abs(rE))
    rwx, rw = O.field_energy(n, L, rE)
    assert abs(wx - rwx) <= 1e-10 * rwx and abs(w - rw) <= 1e-10 * rw


@pytest.mark.parametrize("n,ppc,seed", [(16, 8, 1), (32, 4, 2)])
def test_fem_twenty_step_parity(Sim, n, ppc, seed):
    xv = landau_state(n, ppc, seed=seed)
    sim = Sim(n=n, ppc=ppc, half_kick=False)
    sim.set_particles(xv)
    ex = sim.step(20)
    _, tot, ns, _ = sim.pcg_stats()
    g = sim.get_particles()
    ref, rex, _, _, rits = O.run_fem(n, L, DT, xv, 20)
    assert ns == 20 and tot == int(rits.sum()), (tot, rits)
    assert np.all(np.abs(ex - rex) <= 1e-10 * rex), np.max(np.abs(ex - rex) / rex)
    dx, dv = dist(g, ref)
    assert dx <= 1e-12 and dv <= 1e-12, (dx, dv)


def test_fem_residual_property_at_128(Sim):
    """128^3 x 2 ppc: ||b - A phi|| <= 1e-4 ||b|| with b = h^3 rho - mean and A the
    Q1 stiffness stencil, recomputed with torch on the GPU."""
    import torch

    n = 128
    h = L / n
    sim = Sim(n=n, ppc=2, seed=5)
    sim.step(2)
    rho = torch.from_numpy(sim.get_grid(0)).cuda()
    sim.solve_injected(sim.get_grid(0))
    phi = torch.from_numpy(sim.get_phi()).cuda()
    b = h ** 3 * rho
    b = b - b.mean()
    Ap = torch.zeros_like(phi)
    for off in itertools.product((-1, 0, 1), repeat=3):
        m = sum(abs(o) for o in off)
        wgt = {0: 8 / 3, 1: 0.0, 2: -1 / 6, 3: -1 / 12}[m] * h
        if wgt:
            Ap += wgt * torch.roll(phi, shifts=tuple(-o for o in off), dims=(0, 1, 2))
    assert (torch.linalg.norm(b - Ap) / torch.linalg.norm(b)).item() <= 1e-4


def test_fem_pic_init_then_steps_match_oracle(Sim):
    n, ppc = 16, 8
    sim = Sim(n=n, ppc=ppc, seed=9)
    ex = sim.step(10)
    ref0, phi0 = O.init_state_fem(n, ppc, seed=9)
    _, rex, _, _, _ = O.run_fem(n, L, DT, ref0, 10, phi0=phi0)
    assert np.all(np.abs(ex - rex) <= 1e-9 * rex)
