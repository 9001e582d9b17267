"""GPU parity of the FD-PCG solver (BJ config 5; D#26-D#31):
the CUDA path through the C ABI against the CPU oracle (oracle_solve_pcg /
oracle_run_pcg) on the same seeded inputs.  Both sides run the same iteration;
only the dot products' summation order differs (D#31), so
  iteration counts ........................... equal
  phi, E after one solve (same rho) .......... 1e-10 of max |.|
  W_x per step (20 steps) .................... 1e-10 relative
  x, v after 20 steps ........................ 1e-12 (periodic |dx|/L, |dv|/max(|v|,1))
and, at sizes the oracle cannot run, the defining property of the solve: the
residual of the GPU's phi, recomputed with torch on the GPU, is <= tol ||b||.
"""
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
        return Simulation(solver="pcg", **kw)

    return make


def dist(a, b):
    dx = np.abs(a[:3] - b[:3])
    dx = np.minimum(dx, L - dx) / L
    dv = np.abs(a[3:] - b[3:]) / np.maximum(np.abs(b[3:]), 1.0)
    return dx.max(initial=0.0), dv.max(initial=0.0)


@pytest.mark.parametrize("n,tol", [(16, 1e-4), (32, 1e-4), (32, 1e-10), (64, 1e-6)])
def test_pcg_solve_matches_oracle(Sim, n, tol):
    rho = random_grid(n, seed=n, mean=-1.0)
    sim = Sim(n=n, ppc=1, half_kick=False, pcg_tol=tol)
    E, wx, w = sim.solve_injected(rho)
    it, _, _, rel = sim.pcg_stats()
    phi = sim.get_phi()
    rE, rphi, rit, rrel = O.solve_pcg(n, L, rho, tol=tol)
    assert it == rit and it > 0, (it, rit)
    assert abs(rel - rrel) <= 1e-6 * rrel
    assert np.max(np.abs(phi - rphi)) <= 1e-10 * np.max(np.abs(rphi))
    assert np.max(np.abs(E - rE)) <= 1e-10 * np.max(np.abs(rE))
    rwx, rw = O.field_energy(n, L, rE)
    assert abs(wx - rwx) <= 1e-10 * rwx and abs(w - rw) <= 1e-10 * rw


def test_pcg_zero_and_constant_rho(Sim):
    """rho constant => b = 0 => phi = 0, E = 0 with 0 iterations."""
    n = 16
    sim = Sim(n=n, ppc=1, half_kick=False)
    E, wx, w = sim.solve_injected(np.full((n, n, n), -1.0))
    it, _, _, _ = sim.pcg_stats()
    assert it == 0 and np.all(E == 0) and wx == 0 and w == 0


def test_pcg_single_mode_discrete_closed_form(Sim):
    """rho = cos(k1 y): phi = cos(k1 y)/lambda_h, E_y = sin(k1 y) sin(k1 h)/(h lambda_h)
    with lambda_h = (4/h^2) sin^2(k1 h/2) (D#26, D#30), at tol 1e-12."""
    n = 32
    h = L / n
    k1 = 2 * np.pi / L
    y = np.arange(n) * h
    rho = np.broadcast_to(np.cos(k1 * y)[None, :, None], (n, n, n)).copy()
    sim = Sim(n=n, ppc=1, half_kick=False, pcg_tol=1e-12)
    E, _, _ = sim.solve_injected(rho)
    lam = (4 / h ** 2) * np.sin(k1 * h / 2) ** 2
    want = np.broadcast_to((np.sin(k1 * y) * np.sin(k1 * h) / (h * lam))[None, :, None], (n, n, n))
    assert np.max(np.abs(E[1] - want)) < 1e-10
    assert np.max(np.abs(E[0])) < 1e-10 and np.max(np.abs(E[2])) < 1e-10


@pytest.mark.parametrize("n,ppc,seed", [(16, 8, 1), (32, 8, 2), (64, 2, 3)])
def test_pcg_twenty_step_parity(Sim, n, ppc, seed):
    """BJ: 20 PCG-PIC steps (warm start, tol 1e-4): W_x within 1e-10 relative each step,
    x, v within 1e-12, the same iteration counts."""
    xv = landau_state(n, ppc, seed=seed)
    sim = Sim(n=n, ppc=ppc, half_kick=False)
    sim.set_particles(xv)
    ex = sim.step(20)
    _, tot, ns, _ = sim.pcg_stats()
    g = sim.get_particles()
    ref, rex, _, _, rits = O.run_pcg(n, L, DT, xv, 20)
    assert ns == 20 and tot == int(rits.sum()), (tot, rits)
    assert np.all(np.abs(ex - rex) <= 1e-10 * rex), np.max(np.abs(ex - rex) / rex)
    dx, dv = dist(g, ref)
    assert dx <= 1e-12 and dv <= 1e-12, (dx, dv)


def test_pcg_pic_init_then_steps_match_oracle(Sim):
    """pic_init with the PCG solver (sampler + PCG half kick from phi = 0) then 10 steps
    vs the oracle's init_state_pcg + run_pcg (D#11: init agrees to ulps)."""
    n, ppc = 16, 8
    sim = Sim(n=n, ppc=ppc, seed=9)
    ex = sim.step(10)
    ref0, phi0 = O.init_state_pcg(n, ppc, seed=9)
    _, rex, _, _, _ = O.run_pcg(n, L, DT, ref0, 10, phi0=phi0)
    assert np.all(np.abs(ex - rex) <= 1e-9 * rex)


def test_pcg_residual_property_at_256(Sim):
    """At 256^3 x 2 ppc (beyond the oracle's budget): after each of 3 steps the GPU's
    phi satisfies ||b - A phi|| <= 1e-4 ||b|| with b = rho - mean(rho), recomputed with
    torch on the GPU from pic_get_grid; the central-difference E of that phi equals
    the library's E (D#30)."""
    import torch

    n = 256
    h = L / n
    sim = Sim(n=n, ppc=2, seed=5)
    for _ in range(3):
        sim.step(1)
        it, _, _, rel = sim.pcg_stats()
        # the state after the step is deposited; re-solving it from phi_prev is not what
        # we check -- fetch rho of the solved state by solving it again from phi = 0
        rho = torch.from_numpy(sim.get_grid(0)).cuda()
        E, _, _ = sim.solve_injected(sim.get_grid(0))
        phi = torch.from_numpy(sim.get_phi()).cuda()
        b = rho - rho.mean()
        s = sum(torch.roll(phi, sh, dims=a) for a in range(3) for sh in (1, -1))
        r = b - (6 * phi - s) / h ** 2
        assert (torch.linalg.norm(r) / torch.linalg.norm(b)).item() <= 1e-4
        Ex = (torch.roll(phi, 1, dims=2) - torch.roll(phi, -1, dims=2)) * (0.5 * n / L)
        Et = torch.from_numpy(E[0]).cuda()
        assert (Ex - Et).abs().max().item() <= 1e-12 * Et.abs().max().item()
        assert it >= 0


def test_pcg_landau_damping_rate_on_gpu(Sim):
    """P:231-232 with the PCG solver (tol 1e-4 still shows the analytic rate):
    256^3 x 8 ppc, alpha = 0.05, 260 steps; W_x peak slope within 10% of
    2 gamma and spacing within 5% of pi/omega_r (D#20, D#21)."""
    from landau_fit import dispersion_root, fit_damping_rate

    w = dispersion_root(0.5)
    sim = Sim(n=256, ppc=8, seed=1)
    ex = sim.step(260)
    t = np.arange(260) * DT
    slope, npk, tp = fit_damping_rate(t, ex, t_max=12.0)
    assert npk >= 3
    assert abs(slope - 2 * w.imag) < 0.10 * abs(2 * w.imag), slope
    assert abs(np.mean(np.diff(tp)) - np.pi / w.real) < 0.05 * np.pi / w.real


@pytest.mark.parametrize("n,inner,outer", [(16, 4, 2), (64, 4, 2), (32, 3, 1), (128, 1, 1)])
def test_pcg_blocked_passes_bit_identical_to_half_sweeps(Sim, n, inner, outer, monkeypatch):
    """The temporally blocked SSOR passes (k_ssor_tb, default) reproduce the
    one-kernel-per-half-sweep path (PIC_PCG_TB=0): same colour order and the same
    arithmetic per half-sweep (D#28), including pass counts that are not a multiple
    of 4; only the (r, z) sum is taken in another order, so the CG iterates agree to
    rounding (equal iteration counts, phi and E to 1e-12)."""
    rho = random_grid(n, seed=3 * n, mean=-1.0)
    out = []
    for tb in ("1", "0"):
        monkeypatch.setenv("PIC_PCG_TB", tb)
        sim = Sim(n=n, ppc=1, half_kick=False, pcg_inner=inner, pcg_outer=outer, pcg_tol=1e-8)
        E, _, _ = sim.solve_injected(rho)
        out.append((sim.get_phi(), E, sim.pcg_stats()[0]))
        sim.close()
    assert out[0][2] == out[1][2] and out[0][2] > 0
    for a, b in ((out[0][0], out[1][0]), (out[0][1], out[1][1])):
        assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))
    if (inner, outer) == (4, 2):
        _, rphi, rit, _ = O.solve_pcg(n, L, rho, tol=1e-8)
        assert rit == out[0][2]
        assert np.max(np.abs(out[0][0] - rphi)) <= 1e-10 * np.max(np.abs(rphi))


def test_pcg_nonconvergence_is_reported_not_poisoning(Sim):
    """pcg_maxit reached -> PIC_ENONCONV with the last iterate's field kept; the context
    stays usable (D#29, include/pic.h)."""
    from paper_2605_05469_b200 import PicError
    from paper_2605_05469_b200._binding import PIC_ENONCONV

    n = 32
    sim = Sim(n=n, ppc=2, half_kick=False, pcg_tol=1e-14, pcg_maxit=2)
    sim.set_particles(landau_state(n, 2, seed=1))
    with pytest.raises(PicError) as e:
        sim.step(1)
    assert e.value.status == PIC_ENONCONV
    it, tot, ns, rel = sim.pcg_stats()
    assert it == -1 and tot == 2 and rel > 1e-14
    E = sim.get_grid(1)
    assert np.all(np.isfinite(E)) and np.max(np.abs(E)) > 0
