"""Pins of the FD-PCG Poisson solve of the oracle (BJ config 5).

Like tests/test_oracle.py, nothing here compares the oracle with itself: the
stencil is pinned by closed forms (nullspace, impulse response, the discrete
eigenvalue of a Fourier mode), the preconditioner by the properties CG needs
(symmetry, positivity) and by its limit (SSOR iterated to convergence is the
pseudo-inverse, computed independently with numpy's FFT and the discrete
symbol), PCG by that independent spectral solve, by Krylov theory (one
iteration for an eigenvector right-hand side), by an independently computed
residual and by the Landau damping rate.  D#26-D#31 = DESIGN.md readings.
"""
import numpy as np
import pytest

from oracle import oracle as O
from pic_inputs import landau_state, random_grid
from landau_fit import dispersion_root, fit_damping_rate

K = 0.5
L = 2 * np.pi / K


def _grid(n):
    x = np.arange(n) * L / n
    z, y, xx = np.meshgrid(x, x, x, indexing="ij")
    return xx, y, z


def _discrete_symbol(n):
    """lambda(k) = sum_d (4/h^2) sin^2(k_d h/2): the eigenvalues of -Delta_h (periodic)."""
    h = L / n
    m = np.fft.fftfreq(n, d=1.0 / n)
    s = (4 / h ** 2) * np.sin(np.pi * m / n) ** 2
    sz, sy, sx = np.meshgrid(s, s, s, indexing="ij")
    return sx + sy + sz


def _pinv_spectral(n, b):
    """A^+ b by numpy FFT: divide by the discrete symbol, zero mode removed."""
    lam = _discrete_symbol(n)
    bh = np.fft.fftn(b)
    lam[0, 0, 0] = 1.0
    xh = bh / lam
    xh[0, 0, 0] = 0.0
    return np.fft.ifftn(xh).real


def _lap_np(n, x):
    h = L / n
    s = sum(np.roll(x, sh, axis=a) for a in range(3) for sh in (1, -1))
    return (6 * x - s) / h ** 2


# ------------------------------------------------------------ stencil -------
def test_laplacian_nullspace_and_impulse():
    """A(const) = 0; a unit impulse gives 6/h^2 at the centre, -1/h^2 at the six faces."""
    n = 8
    h = L / n
    assert np.max(np.abs(O.laplacian_fd(n, L, np.full((n, n, n), 2.5)))) < 1e-12
    x = np.zeros((n, n, n))
    x[3, 4, 0] = 1.0                     # ix = 0: the x neighbour wraps to ix = n - 1
    y = O.laplacian_fd(n, L, x)
    assert y[3, 4, 0] == pytest.approx(6 / h ** 2, rel=1e-14)
    for idx in [(2, 4, 0), (4, 4, 0), (3, 3, 0), (3, 5, 0), (3, 4, 1), (3, 4, n - 1)]:
        assert y[idx] == pytest.approx(-1 / h ** 2, rel=1e-14)
    assert np.count_nonzero(y) == 7


@pytest.mark.parametrize("modes", [(1, 0, 0), (0, 3, 0), (2, 1, 5), (4, 4, 4)])
def test_laplacian_fourier_mode_eigenvalue(modes):
    """cos(k.x) -> (sum_d (4/h^2) sin^2(k_d h/2)) cos(k.x), node-wise to 1e-12."""
    n = 8
    h = L / n
    X = _grid(n)
    kv = [2 * np.pi * m / L for m in modes]
    f = np.cos(sum(k * c for k, c in zip(kv, X)))
    lam = sum((4 / h ** 2) * np.sin(k * h / 2) ** 2 for k in kv)
    y = O.laplacian_fd(n, L, f)
    assert np.max(np.abs(y - lam * f)) < 1e-12 * max(lam, 1.0)


def test_laplacian_symmetric():
    """<A x, y> = <x, A y> for random x, y, 1e-12 relative."""
    n = 16
    x, y = random_grid(n, 1), random_grid(n, 2)
    a = (O.laplacian_fd(n, L, x) * y).sum()
    b = (x * O.laplacian_fd(n, L, y)).sum()
    assert abs(a - b) < 1e-12 * np.sqrt((O.laplacian_fd(n, L, x) ** 2).sum() * (y ** 2).sum())


# ----------------------------------------------------------- SSOR -----------
def test_ssor_symmetric_positive_definite():
    """D#28: the palindromic red-black sweep sequence makes M^-1 symmetric, and
    0 < omega < 2 makes it positive definite (CG's requirement)."""
    n = 8
    rng = np.random.default_rng(7)
    for _ in range(10):
        r = rng.standard_normal((n, n, n))
        s = rng.standard_normal((n, n, n))
        r -= r.mean()
        s -= s.mean()
        Mr = O.ssor(n, L, r)
        Ms = O.ssor(n, L, s)
        assert abs((Mr * s).sum() - (r * Ms).sum()) < 1e-12 * np.sqrt((Mr ** 2).sum() * (s ** 2).sum())
        assert (r * Mr).sum() > 0


def test_ssor_iterated_converges_to_pseudo_inverse():
    """SSOR is a convergent splitting for 0 < omega < 2: many outer sweeps give
    A^+ r up to a constant (numpy spectral inverse of the discrete symbol)."""
    n = 8
    r = random_grid(n, 3)
    r -= r.mean()
    z = O.ssor(n, L, r, outer=300)
    ref = _pinv_spectral(n, r)
    z -= z.mean()
    assert np.max(np.abs(z - ref)) < 1e-10 * np.max(np.abs(ref))


def test_ssor_reduces_the_error_of_one_sweep_pair():
    """One symmetric sweep pair (inner = outer = 1) from 0 is a contraction: the
    A-norm error of z vs A^+ r is below that of z = 0."""
    n = 16
    r = random_grid(n, 4)
    r -= r.mean()
    ref = _pinv_spectral(n, r)
    z = O.ssor(n, L, r, inner=1, outer=1)
    z -= z.mean()
    e1, e0 = z - ref, -ref
    assert (e1 * _lap_np(n, e1)).sum() < 0.8 * (e0 * _lap_np(n, e0)).sum()


# ------------------------------------------------------------ PCG -----------
def test_pcg_matches_spectral_solve_at_tight_tolerance():
    """random mean-zero b; PCG at tol 1e-12 == A^+ b (numpy FFT) to 1e-9."""
    n = 16
    b = random_grid(n, 5)
    b -= b.mean()
    x, it, rel = O.pcg(n, L, b, tol=1e-12)
    assert it > 0 and rel <= 1e-12
    x -= x.mean()
    ref = _pinv_spectral(n, b)
    assert np.max(np.abs(x - ref)) < 1e-9 * np.max(np.abs(ref))


def test_pcg_eigenvector_rhs_converges_in_one_iteration():
    """b an eigenvector of A: unpreconditioned CG from 0 is exact after one
    iteration (x = b / lambda_h)."""
    n = 16
    h = L / n
    X = _grid(n)
    k1 = 2 * np.pi / L
    b = np.cos(k1 * X[0])
    x, it, rel = O.pcg(n, L, b, tol=1e-10, precond=0)
    lam = (4 / h ** 2) * np.sin(k1 * h / 2) ** 2
    assert it == 1
    assert np.max(np.abs(x - b / lam)) < 1e-12 / lam


def test_pcg_residual_is_within_tolerance_and_preconditioner_helps():
    """||b - A x|| <= 1e-4 ||b|| (residual recomputed with numpy); P:260 / S:291:
    SSOR(pi/2, 4, 2) needs fewer iterations than plain CG on a Landau charge density."""
    n = 32
    xv = landau_state(n, 8, seed=3)
    rho = O.deposit(n, L, xv, -L ** 3 / xv.shape[1])
    b = rho - rho.mean()
    x, it_p, rel = O.pcg(n, L, b)
    res = np.linalg.norm(b - _lap_np(n, x)) / np.linalg.norm(b)
    assert res <= 1e-4 and abs(res - rel) < 1e-8
    _, it_cg, _ = O.pcg(n, L, b, precond=0)
    assert 0 < it_p < it_cg


def test_pcg_zero_rhs_and_warm_start():
    """S:266 / S:302: b = 0 -> x = 0 with 0 iterations; a converged warm start needs 0
    iterations, and warm-starting step 2 of a Landau run never needs more than cold."""
    n = 16
    x, it, _ = O.pcg(n, L, np.zeros((n, n, n)), x0=np.ones((n, n, n)))
    assert it == 0 and np.all(x == 0)
    xv = landau_state(n, 8, seed=8)
    q = -L ** 3 / xv.shape[1]
    rho0 = O.deposit(n, L, xv, q)
    E0, phi0, it0, _ = O.solve_pcg(n, L, rho0)
    _, _, it_again, _ = O.solve_pcg(n, L, rho0, phi0=phi0)
    assert it_again == 0
    Ep = O.gather(n, L, xv, E0)
    xv1 = O.push(L, xv, Ep, -0.05, 0.05)
    rho1 = O.deposit(n, L, xv1, q)
    _, _, it_warm, _ = O.solve_pcg(n, L, rho1, phi0=phi0)
    _, _, it_cold, _ = O.solve_pcg(n, L, rho1)
    assert it_warm <= it_cold


def test_gradient_central_closed_form():
    """D#30: phi = cos(k1 x_d) -> E_d = sin(k1 x_d) sin(k1 h)/h, other components 0."""
    n = 16
    h = L / n
    X = _grid(n)
    k1 = 2 * np.pi / L * 3
    for d in range(3):
        E = O.gradient_central(n, L, np.cos(k1 * X[d]))
        want = np.sin(k1 * X[d]) * np.sin(k1 * h) / h
        assert np.max(np.abs(E[d] - want)) < 1e-12
        for e in range(3):
            if e != d:
                assert np.max(np.abs(E[e])) < 1e-12


def test_pcg_solve_second_order_convergence():
    """S:300 / Table 1 ("2nd order"): rho = cos(k1 x) -> the error of phi vs
    cos(k1 x)/k1^2 falls by 4 (rate 2.0 +- 0.15) from N = 16 to N = 32."""
    k1 = 2 * np.pi / L
    err = []
    for n in (16, 32):
        X = _grid(n)
        rho = np.cos(k1 * X[0])
        _, phi, it, _ = O.solve_pcg(n, L, rho, tol=1e-12)
        assert it > 0
        err.append(np.max(np.abs(phi - phi.mean() - rho / k1 ** 2)))
    rate = np.log2(err[0] / err[1])
    assert abs(rate - 2.0) < 0.15


def test_pcg_run_momentum_and_determinism():
    """Total momentum is conserved when A phi = b holds: sum_i rho_i (D phi)_i = 0 for
    the antisymmetric central difference D commuting with the symmetric A (so with a
    converged solve, tol 1e-10, sum_j v_j is conserved to rounding as for the FFT
    loop); the runs are bitwise reproducible, and the warm start keeps the
    iteration counts of later steps at or below the first."""
    n = 16
    xv = landau_state(n, 8, seed=21)
    xs, ex, tot, phi, its = O.run_pcg(n, L, 0.05, xv, 6, tol=1e-10)
    assert np.max(np.abs(xs[3:].sum(axis=1) - xv[3:].sum(axis=1))) < 1e-10 * np.abs(xv[3:]).sum()
    xs, ex, tot, phi, its = O.run_pcg(n, L, 0.05, xv, 6)
    xs2, ex2, tot2, phi2, its2 = O.run_pcg(n, L, 0.05, xv, 6)
    assert np.array_equal(xs, xs2) and np.array_equal(ex, ex2) and np.array_equal(its, its2)
    assert np.all(its >= 0) and np.all(its[1:] <= its[0])
    assert np.all(ex > 0) and np.all(tot >= ex)


def test_landau_damping_rate_oracle_pcg():
    """P:231-232 (all four schemes show the analytic rate at tol 1e-4): the
    PCG loop's E_x-energy peaks decay at 2 gamma (+-10%), spacing pi/omega_r (+-5%).
    Same input as the FFT pin (D#21): 16^3 x 128 ppc, alpha = 0.1."""
    n = 16
    w = dispersion_root(0.5)
    xv, phi = O.init_state_pcg(n, 128, alpha=0.1, seed=1)
    _, ex, _, _, its = O.run_pcg(n, L, 0.05, xv, 200, phi0=phi)
    t = np.arange(200) * 0.05
    slope, npk, tp = fit_damping_rate(t, ex, t_max=10.0)
    assert npk >= 3 and np.all(its >= 0)
    assert abs(slope - 2 * w.imag) < 0.10 * abs(2 * w.imag)
    assert abs(np.mean(np.diff(tp)) - np.pi / w.real) < 0.05 * np.pi / w.real
