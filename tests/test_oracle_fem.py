"""Pins of the matrix-free Q1 FEM solve of the oracle (
SURVEY §8(f) NEXT-4; reading D#33).

Not the oracle re-typed: the element stiffness is pinned to its closed form (1/3 on the
diagonal, 0 for edge neighbours, -1/12 for face-diagonal and opposite vertices, times h),
the element-loop operator to the assembled 27-point stencil applied with numpy rolls,
the CG solve to the spectral pseudo-inverse of that stencil (numpy FFT), the discrete
solution to second-order convergence, and the whole loop to the Landau damping rate.
"""
import itertools

import numpy as np

from oracle import oracle as O
from pic_inputs import landau_state, random_grid
from landau_fit import dispersion_root, fit_damping_rate

K = 0.5
L = 2 * np.pi / K


def _stencil27(n):
    """Assembled Q1 stiffness stencil (x h): centre 8/3, faces 0, edges -1/6, corners -1/12."""
    out = []
    for off in itertools.product((-1, 0, 1), repeat=3):
        m = sum(abs(o) for o in off)
        w = {0: 8 / 3, 1: 0.0, 2: -1 / 6, 3: -1 / 12}[m]
        if w != 0.0:
            out.append((off, w))
    return out


def _apply_np(n, x):
    h = L / n
    y = np.zeros_like(x)
    for (dz, dy, dx), w in _stencil27(n):
        y += w * h * np.roll(x, (-dz, -dy, -dx), axis=(0, 1, 2))
    return y


def _pinv_np(n, b):
    h = L / n
    ker = np.zeros((n, n, n))
    for (dz, dy, dx), w in _stencil27(n):
        ker[dz % n, dy % n, dx % n] += w * h
    lam = np.fft.fftn(ker).real
    bh = np.fft.fftn(b)
    lam[0, 0, 0] = 1.0
    xh = bh / lam
    xh[0, 0, 0] = 0.0
    return np.fft.ifftn(xh).real


def test_element_stiffness_closed_form():
    for h in (1.0, 0.3):
        Ae = O.fem_element_stiffness(h)
        want = np.zeros((8, 8))
        for i in range(8):
            for j in range(8):
                d = bin(i ^ j).count("1")
                want[i, j] = {0: 1 / 3, 1: 0.0, 2: -1 / 12, 3: -1 / 12}[d] * h
        assert np.max(np.abs(Ae - want)) < 1e-14
        assert np.array_equal(Ae, Ae.T)
        assert np.max(np.abs(Ae.sum(axis=1))) < 1e-15


def test_element_loop_equals_assembled_stencil():
    """the matrix-free element loop equals the assembled operator (here its
    closed-form 27-point stencil), annihilates constants and is symmetric."""
    n = 8
    x = random_grid(n, 1)
    assert np.max(np.abs(O.fem_apply(n, L, x) - _apply_np(n, x))) < 1e-12 * np.max(np.abs(x))
    assert np.max(np.abs(O.fem_apply(n, L, np.full((n, n, n), 3.0)))) < 1e-13
    y = random_grid(n, 2)
    a = (O.fem_apply(n, L, x) * y).sum()
    b = (x * O.fem_apply(n, L, y)).sum()
    assert abs(a - b) < 1e-12 * abs(a)


def test_fem_cg_matches_spectral_pseudo_inverse():
    """CG at tol 1e-12 on a random mean-zero load == A^+ b (numpy FFT) to 1e-9."""
    n = 16
    b = random_grid(n, 3)
    b -= b.mean()
    x, it, rel = O.fem_cg(n, L, b, tol=1e-12)
    assert it > 0 and rel <= 1e-12
    ref = _pinv_np(n, b)
    x -= x.mean()
    assert np.max(np.abs(x - ref)) < 1e-9 * np.max(np.abs(ref))


def test_fem_solve_second_order_and_zero():
    """rho = cos(k1 x): phi vs cos(k1 x)/k1^2 converges at order 2 +- 0.15 from
    N = 16 to 32 (Table 1: (p+1)-order with p = 1); rho constant -> phi = 0."""
    k1 = 2 * np.pi / L
    err = []
    for n in (16, 32):
        x = np.arange(n) * L / n
        rho = np.broadcast_to(np.cos(k1 * x)[None, None, :], (n, n, n)).copy()
        _, phi, it, _ = O.solve_fem(n, L, rho, tol=1e-12)
        err.append(np.max(np.abs(phi - phi.mean() - rho / k1 ** 2)))
    assert abs(np.log2(err[0] / err[1]) - 2.0) < 0.15
    E, phi, it, _ = O.solve_fem(16, L, np.full((16, 16, 16), -1.0))
    # b = 0 up to the rounding of its mean (a constant: the operator's nullspace) -> E = 0
    assert np.ptp(phi) < 1e-9 * max(1.0, np.max(np.abs(phi))) and np.max(np.abs(E)) < 1e-12


def test_fem_residual_and_warm_start():
    """P:226 / P:260: ||b - A phi|| <= 1e-4 ||b|| (recomputed with the numpy stencil); a
    converged warm start needs no iteration."""
    n = 16
    xv = landau_state(n, 8, seed=3)
    rho = O.deposit(n, L, xv, -L ** 3 / xv.shape[1])
    h3 = (L / n) ** 3
    b = h3 * rho - (h3 * rho).mean()
    _, phi, it, rel = O.solve_fem(n, L, rho)
    res = np.linalg.norm(b - _apply_np(n, phi)) / np.linalg.norm(b)
    assert it > 0 and res <= 1e-4 and abs(res - rel) < 1e-8
    _, _, it2, _ = O.solve_fem(n, L, rho, phi0=phi)
    assert it2 == 0


def test_landau_damping_rate_oracle_fem():
    """the FEM loop (plain CG, tol 1e-4, warm start) shows the analytic rate:
    slope within 10% of 2 gamma, spacing within 5% (16^3 x 128 ppc, alpha = 0.1, D#21)."""
    n = 16
    w = dispersion_root(0.5)
    xv = O.init_state(n, 128, alpha=0.1, seed=1)
    _, ex, _, _, its = O.run_fem(n, L, 0.05, xv, 200)
    t = np.arange(200) * 0.05
    slope, npk, tp = fit_damping_rate(t, ex, t_max=10.0)
    assert npk >= 3 and np.all(its >= 0)
    assert abs(slope - 2 * w.imag) < 0.10 * abs(2 * w.imag)
    assert abs(np.mean(np.diff(tp)) - np.pi / w.real) < 0.05 * np.pi / w.real
