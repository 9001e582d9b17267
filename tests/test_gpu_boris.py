"""GPU parity of the external-field push (Eq. 1, 3-4: P:97; D#32):
uniform E_ext added to the gathered field, the Boris scheme when B_ext != 0.  The
push given an identical field is bit-exact against oracle_push_ext (the same
operation order, fma where the oracle writes fma); whole runs match oracle_run_ext
to the BJ tolerances."""
import numpy as np
import pytest

from oracle import oracle as O
from pic_inputs import landau_state, random_field

pytestmark = pytest.mark.gpu

K = 0.5
L = 2 * np.pi / K
DT = 0.05
B = (0.3, -0.4, 1.5)
EX = (0.1, 0.0, -0.05)


@pytest.fixture(scope="module")
def Sim():
    import torch
    from paper_2605_05469_b200 import Simulation

    torch.cuda.set_device(0)
    return Simulation


def dist(a, b):
    dx = np.abs(a[:3] - b[:3])
    dx = np.minimum(dx, L - dx) / L
    dv = np.abs(a[3:] - b[3:]) / np.maximum(np.abs(b[3:]), 1.0)
    return dx.max(initial=0.0), dv.max(initial=0.0)


@pytest.mark.parametrize("b_ext,e_ext", [(B, (0, 0, 0)), ((0, 0, 0), EX), (B, EX)])
def test_push_with_external_fields_bit_exact(Sim, b_ext, e_ext):
    n, ppc = 16, 8
    xv = landau_state(n, ppc, seed=3)
    xv[3:] *= 3.0
    E = random_field(n, seed=4)
    sim = Sim(n=n, ppc=ppc, half_kick=False, b_ext=b_ext, e_ext=e_ext)
    sim.set_particles(xv)
    sim.push_injected(E)
    g = sim.get_particles()
    xs, _ = O.sort(n, L, xv)
    Ep = O.gather(n, L, xs, E)
    ref, _ = O.sort(n, L, O.push_ext(L, xs, Ep, DT, b_ext=b_ext, e_ext=e_ext))
    assert np.array_equal(g, ref)


@pytest.mark.parametrize("n,ppc", [(16, 8), (32, 4)])
def test_twenty_steps_with_external_fields(Sim, n, ppc):
    xv = landau_state(n, ppc, seed=7)
    sim = Sim(n=n, ppc=ppc, half_kick=False, b_ext=B, e_ext=EX)
    sim.set_particles(xv)
    ex = sim.step(20)
    g = sim.get_particles()
    ref, rex, _ = O.run_ext(n, L, DT, xv, 20, b_ext=B, e_ext=EX)
    assert np.all(np.abs(ex - rex) <= 1e-10 * rex), np.max(np.abs(ex - rex) / rex)
    dx, dv = dist(g, ref)
    assert dx <= 1e-12 and dv <= 1e-12, (dx, dv)


def test_boris_speed_conserved_on_gpu(Sim):
    """S:158 on the GPU: E = 0 (injected), B = (0, 0, 1): |v| conserved to 1e-13 over
    500 pushes."""
    n, ppc = 16, 1
    xv = landau_state(n, ppc, seed=5)
    s0 = np.sort(np.linalg.norm(xv[3:], axis=0))
    sim = Sim(n=n, ppc=ppc, half_kick=False, b_ext=(0.0, 0.0, 1.0))
    sim.set_particles(xv)
    E0 = np.zeros((3, n, n, n))
    for _ in range(500):
        sim.push_injected(E0)
    s1 = np.sort(np.linalg.norm(sim.get_particles()[3:], axis=0))
    assert np.max(np.abs(s1 / s0 - 1.0)) < 1e-13
