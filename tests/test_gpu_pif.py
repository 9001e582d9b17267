"""GPU parity of the Particle-in-Fourier solve and its NUFFTs (include/pif.h; P:197-221,
Appendix A; readings D#34-D#37) against oracle/nufft.py on
the same seeded inputs.  Both sides use the same window (ES, w = ceil(log10 1/eps) + 2,
beta = 2.30 w, sigma = 2) and differ only in rounding order (atomic spreading order,
cuFFT vs numpy FFT, libm ulps), so
  type 1 vs oracle nufft1 ..................... 1e-11 of sum |f|
  type 2 vs oracle nufft2 ..................... 1e-11 of sum |f^|
  PIF E at particles / energies vs oracle ...... 1e-10 of max |E| / relative
and, at sizes beyond the oracle's, sampled modes against the direct NUDFT sum (within
eps sum |f|) and the closed-form field and energy of a lattice-sampled cosine density."""
import numpy as np
import pytest

from oracle import nufft as U
from pic_inputs import landau_state, random_spectrum, random_weights

pytestmark = pytest.mark.gpu

L = 4 * np.pi


@pytest.fixture(scope="module")
def torch_dev():
    import torch

    torch.cuda.set_device(0)
    return torch


def _x(torch, xv):
    return torch.from_numpy(np.ascontiguousarray(xv[:3])).cuda()


@pytest.mark.parametrize("binned", [True, False])
@pytest.mark.parametrize("N,np_,eps", [(16, 3000, 1e-4), (32, 777, 1e-4), (8, 500, 1e-6), (16, 0, 1e-4),
                                       (64, 300, 1e-4), (8, 400, 1e-2)])
def test_type1_matches_oracle(torch_dev, N, np_, eps, binned):
    from paper_2605_05469_b200 import PifSolver

    torch = torch_dev
    xv = landau_state(4, 1, L=L, np_=max(np_, 1), seed=3)[:, :np_]
    f = random_weights(np_, seed=4)
    P = PifSolver(N, L, eps, np_max=np_ if binned else 0)
    g = P.type1(_x(torch, xv), torch.from_numpy(f).cuda()).cpu().numpy()
    if np_ == 0:
        assert np.all(g == 0)
        return
    ref = U.nufft1(xv[:3], f, N, L, eps)
    assert np.abs(g - ref).max() <= 1e-11 * np.abs(f).sum()
    assert np.abs(g - U.nudft1(xv[:3], f, N, L)).max() <= eps * np.abs(f).sum()


@pytest.mark.parametrize("binned", [True, False])
@pytest.mark.parametrize("N,np_", [(16, 400), (32, 123), (8, 333)])
def test_type2_matches_oracle(torch_dev, N, np_, binned):
    from paper_2605_05469_b200 import PifSolver

    torch = torch_dev
    xv = landau_state(4, 1, L=L, np_=np_, seed=5)
    fh = random_spectrum(N, seed=6)
    P = PifSolver(N, L, 1e-4, np_max=np_ if binned else 0)
    g = P.type2(torch.from_numpy(fh).cuda(), _x(torch, xv)).cpu().numpy()
    ref = U.nufft2(fh, xv[:3], L, 1e-4)
    assert np.abs(g - ref).max() <= 1e-11 * np.abs(fh).sum()
    assert np.abs(g - U.nudft2(fh, xv[:3], L)).max() <= 1e-4 * np.abs(fh).sum()


@pytest.mark.parametrize("binned", [True, False])
@pytest.mark.parametrize("N,ppc", [(16, 2), (8, 8)])
def test_pif_solve_matches_oracle(torch_dev, N, ppc, binned):
    from paper_2605_05469_b200 import PifSolver

    torch = torch_dev
    Lk = 2 * np.pi / 0.5
    xv = landau_state(N, ppc, L=Lk, seed=7)
    npart = xv.shape[1]
    q = np.full(npart, -Lk ** 3 / npart)          # D#2 macro charge
    P = PifSolver(N, Lk, 1e-4, np_max=npart if binned else 0)
    E, W = P.solve(_x(torch, xv), torch.from_numpy(q).cuda())
    E = E.cpu().numpy()
    Eo, Wo, _ = U.pif_solve(xv[:3], q, N, Lk, 1e-4)
    assert np.abs(E - Eo).max() <= 1e-10 * np.abs(Eo).max()
    assert np.allclose(W, Wo, rtol=1e-10, atol=0)


@pytest.mark.parametrize("band", [(0.30, 0.45), (0.9, 1.0)])
def test_pif_solve_particles_in_a_z_band(torch_dev, band):
    """Particles confined to a z band (the decomposed PIF's rank shares; the second band
    wraps its window tiles through z = 0): the fine-grid x and y passes skip the planes no
    bin tile reaches, exactly -- E at the particles, energies and type 1 vs the oracle."""
    from paper_2605_05469_b200 import PifSolver

    torch = torch_dev
    N = 32
    Lk = 2 * np.pi / 0.5
    rng = np.random.default_rng(13)
    npart = 6000
    xv = np.concatenate([rng.random((2, npart)) * Lk,
                         (band[0] + (band[1] - band[0]) * rng.random((1, npart))) * Lk,
                         rng.standard_normal((3, npart))])
    xv[2] = np.minimum(xv[2], np.nextafter(Lk, 0))
    q = np.full(npart, -Lk ** 3 / npart)
    P = PifSolver(N, Lk, 1e-4, np_max=npart)
    E, W = P.solve(_x(torch, xv), torch.from_numpy(q).cuda())
    Eo, Wo, _ = U.pif_solve(xv[:3], q, N, Lk, 1e-4)
    assert np.abs(E.cpu().numpy() - Eo).max() <= 1e-10 * np.abs(Eo).max()
    assert np.allclose(W, Wo, rtol=1e-10, atol=0)
    f = random_weights(npart, seed=14)
    g = P.type1(_x(torch, xv), torch.from_numpy(f).cuda()).cpu().numpy()
    assert np.abs(g - U.nufft1(xv[:3], f, N, Lk, 1e-4)).max() <= 1e-11 * np.abs(f).sum()


def test_pif_cosine_lattice_closed_form_at_size(torch_dev):
    """2^21 particles on a 128^3 lattice, weights h^3 (1 + alpha cos(k1 x)), N = 64 modes:
    E_x = alpha sin(k1 x) / k1, E_y = E_z = 0, W_x = alpha^2 L^3 / (4 k1^2)."""
    from paper_2605_05469_b200 import PifSolver

    torch = torch_dev
    Nl, alpha = 128, 0.05
    k1 = 2 * np.pi / L
    h = L / Nl
    g = torch.arange(Nl, dtype=torch.float64, device="cuda") * h + 0.21 * h
    Z, Y, X = torch.meshgrid(g, g, g, indexing="ij")
    x = torch.stack([X.reshape(-1), Y.reshape(-1), Z.reshape(-1)]).contiguous()
    q = (h ** 3 * (1 + alpha * torch.cos(k1 * x[0]))).contiguous()
    P = PifSolver(64, L, 1e-4, np_max=x.shape[1])
    E, W = P.solve(x, q)
    scale = alpha / k1
    assert (E[0] - alpha * torch.sin(k1 * x[0]) / k1).abs().max().item() < 1e-4 * scale
    assert E[1:].abs().max().item() < 1e-4 * scale
    assert abs(W[0] - alpha ** 2 * L ** 3 / (4 * k1 ** 2)) < 1e-4 * W[0]


def test_type1_sampled_modes_at_size(torch_dev):
    """128^3 x 8 Landau particles, N = 128: 6 sampled modes against the direct sum (Eq. p2f)."""
    from paper_2605_05469_b200 import PifSolver

    torch = torch_dev
    N = 128
    Lk = 2 * np.pi / 0.5
    xv = landau_state(N, 8, L=Lk, seed=11)
    f = random_weights(xv.shape[1], seed=12)
    P = PifSolver(N, Lk, 1e-4, np_max=xv.shape[1])
    g = P.type1(_x(torch, xv), torch.from_numpy(f).cuda()).cpu().numpy()
    modes = [(0, 0, 0), (1, 0, 0), (0, -1, 2), (-64, 5, 63), (17, -33, -64), (63, 63, 63)]
    ref = U.nudft1_modes(xv[:3], f, Lk, modes)
    got = np.array([g[n[2] + N // 2, n[1] + N // 2, n[0] + N // 2] for n in modes])
    assert np.abs(got - ref).max() <= 1e-4 * np.abs(f).sum()


@pytest.mark.parametrize("binned", [True, False])
@pytest.mark.parametrize("N,ppc,nsteps", [(8, 4, 10), (16, 1, 3)])
def test_pif_step_matches_oracle_run(torch_dev, N, ppc, nsteps, binned):
    """pic_pif_step vs oracle pif_run (PIF solve + the PIC leapfrog push + wrap), Landau
    alpha = 0.3: W_x per step 1e-9 relative, x (periodic) and v within 1e-9 after the steps;
    total momentum conserved (1e-11)."""
    from paper_2605_05469_b200 import PifSolver

    torch = torch_dev
    Lk = 2 * np.pi / 0.5
    xv = landau_state(N, ppc, L=Lk, seed=23, alpha=0.3)
    npart = xv.shape[1]
    q = np.full(npart, -Lk ** 3 / npart)
    P = PifSolver(N, Lk, 1e-4, np_max=npart if binned else 0)
    x = torch.from_numpy(np.ascontiguousarray(xv[:3])).cuda()
    v = torch.from_numpy(np.ascontiguousarray(xv[3:])).cuda()
    ex = P.step(x, v, torch.from_numpy(q).cuda(), nsteps=nsteps, qm=-1.0, dt=0.05)
    xo, exo = U.pif_run(N, Lk, 0.05, xv, q, nsteps)
    assert np.allclose(ex, exo, rtol=1e-9, atol=0)
    dx = np.abs(x.cpu().numpy() - xo[:3])
    dx = np.minimum(dx, Lk - dx)
    assert dx.max() < 1e-9 * Lk
    assert np.abs(v.cpu().numpy() - xo[3:]).max() < 1e-9
    assert np.abs(v.cpu().numpy().sum(axis=1) - xv[3:].sum(axis=1)).max() < 1e-11 * np.abs(xv[3:]).sum()


def test_binned_equals_atomic_path_at_size(torch_dev):
    """128^3 x 8 Landau particles, N = 128: the binned (tile) and the atomic paths of the PIF
    solve agree to rounding (1e-11 of max |E|), and a particle count above np_max falls back."""
    from paper_2605_05469_b200 import PifSolver

    torch = torch_dev
    Lk = 2 * np.pi / 0.5
    xv = landau_state(128, 8, L=Lk, seed=31)
    npart = xv.shape[1]
    x = _x(torch, xv)
    q = torch.full((npart,), -Lk ** 3 / npart, dtype=torch.float64, device="cuda")
    Eb, Wb = PifSolver(128, Lk, 1e-4, np_max=npart).solve(x, q)
    Ea, Wa = PifSolver(128, Lk, 1e-4).solve(x, q)
    Es, Ws = PifSolver(128, Lk, 1e-4, np_max=npart // 2).solve(x, q)
    scale = Ea.abs().max().item()
    assert (Eb - Ea).abs().max().item() < 1e-11 * scale
    assert np.allclose(Wb, Wa, rtol=1e-11) and np.allclose(Ws, Wa, rtol=1e-11)


def test_pif_landau_damping_rate(torch_dev):
    """P:140-146, P:231-232 with the PIF scheme: 16^3 modes, 128^3 x 8 Landau
    particles (alpha = 0.05), backward half kick, 260 steps of pic_pif_step: the slope of the
    W_x peaks for t <= 12 within 10% of 2 gamma of the dispersion relation and their spacing
    within 5% of pi / omega_r (D#20, D#21)."""
    from landau_fit import dispersion_root, fit_damping_rate
    from paper_2605_05469_b200 import PifSolver

    torch = torch_dev
    Lk = 2 * np.pi / 0.5
    xv = landau_state(128, 8, L=Lk, seed=41)
    npart = xv.shape[1]
    x = torch.from_numpy(np.ascontiguousarray(xv[:3])).cuda()
    v = torch.from_numpy(np.ascontiguousarray(xv[3:])).cuda()
    q = torch.full((npart,), -Lk ** 3 / npart, dtype=torch.float64, device="cuda")
    P = PifSolver(16, Lk, 1e-4, np_max=npart)
    E, _ = P.solve(x, q)
    v -= (-1.0) * 0.5 * 0.05 * E          # v_{-1/2} = v_0 - (q/m) dt/2 E(x_0) (D#9)
    ex = P.step(x, v, q, nsteps=260, qm=-1.0, dt=0.05)
    w = dispersion_root(0.5)
    t = np.arange(260) * 0.05
    slope, npk, tp = fit_damping_rate(t, ex, t_max=12.0)
    assert npk >= 5
    assert abs(slope - 2 * w.imag) < 0.10 * abs(2 * w.imag), slope
    assert abs(np.mean(np.diff(tp)) - np.pi / w.real) < 0.05 * np.pi / w.real


def test_one_pass_gather_equals_two_pass(torch_dev, monkeypatch):
    """Binned PIF solve: the one-pass gather of (E_x + i E_y, E_z) from two fine grids equals
    the two-pass gather (PIC_PIF_SPLIT_INTERP=1) to rounding."""
    from paper_2605_05469_b200 import PifSolver

    torch = torch_dev
    Lk = 2 * np.pi / 0.5
    xv = landau_state(32, 8, L=Lk, seed=43)
    npart = xv.shape[1]
    x = _x(torch, xv)
    q = torch.full((npart,), -Lk ** 3 / npart, dtype=torch.float64, device="cuda")
    E1, W1 = PifSolver(32, Lk, 1e-4, np_max=npart).solve(x, q)
    monkeypatch.setenv("PIC_PIF_SPLIT_INTERP", "1")
    E2, W2 = PifSolver(32, Lk, 1e-4, np_max=npart).solve(x, q)
    assert (E1 - E2).abs().max().item() <= 1e-13 * E2.abs().max().item()
    assert np.allclose(W1, W2, rtol=1e-13)
