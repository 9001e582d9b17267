"""Pins of the NUFFT / PIF oracle (oracle/nufft.py; Appendix A P:423-467;
SURVEY §8(f) NEXT-2; readings D#34-D#37).

The pins are not the oracle re-typed: the NUDFTs are pinned to closed forms (one
particle at the origin / at L/2, one mode) and to numpy's FFT on the coarse lattice
(particles on nodes); the NUFFTs to the NUDFTs within the accuracy eps the window
is chosen for (eps = 1e-4) and to exact adjointness; the window transform to
adaptive quadrature (scipy); the PIF solve to the closed-form field and energy of a
cosine density sampled on a lattice, and to equal-and-opposite forces of a mirrored pair.
"""
import numpy as np
import pytest
from scipy import integrate

from oracle import nufft as U

L = 4 * np.pi


def _pts(rng, n):
    return rng.uniform(0, L, (3, n))


def test_nudft1_single_particle_closed_forms():
    """x = 0 -> f^ = q everywhere; x = (L/2, 0, 0) -> f^(n) = q (-1)^{n_x}."""
    N = 8
    q = 0.7
    a = U.nudft1(np.zeros((3, 1)), np.array([q]), N, L)
    assert np.allclose(a, q, atol=1e-15)
    b = U.nudft1(np.array([[L / 2], [0.0], [0.0]]), np.array([q]), N, L)
    sign = (-1.0) ** U.modes_1d(N)
    assert np.allclose(b, q * np.broadcast_to(sign[None, None, :], b.shape), atol=1e-13)
    i = N // 2 + 1  # n_x = 1
    assert abs(b[N // 2, N // 2, i] - (-q)) < 1e-13


def test_nudft_on_lattice_is_numpy_fft():
    """Particles on coarse nodes x = i h: Eq. (p2f) is the DFT of the node-impulse field
    (numpy fftn), Eq. (f2p) the unnormalised inverse DFT (numpy ifftn x N^3)."""
    N = 8
    h = L / N
    rng = np.random.default_rng(3)
    idx = rng.integers(0, N, (3, 40))
    f = rng.standard_normal(40)
    x = idx * h
    grid = np.zeros((N, N, N))
    np.add.at(grid, (idx[2], idx[1], idx[0]), f)
    ref = np.fft.fftshift(np.fft.fftn(grid))           # index n + N/2, n ascending
    assert np.allclose(U.nudft1(x, f, N, L), ref, atol=1e-11)
    fh = rng.standard_normal((N, N, N)) + 1j * rng.standard_normal((N, N, N))
    g = np.fft.ifftn(np.fft.ifftshift(fh)) * N ** 3
    assert np.allclose(U.nudft2(fh, x, L), g[idx[2], idx[1], idx[0]], atol=1e-10)


def test_nudft2_single_mode_and_adjoint():
    """one coefficient c at k0 -> c e^{i k0 . x}; <nudft1 w, g> = <w, nudft2 g>."""
    N = 8
    rng = np.random.default_rng(4)
    x = _pts(rng, 30)
    fh = np.zeros((N, N, N), dtype=complex)
    c = 0.3 - 1.1j
    n0 = (2, -3, 1)  # (n_x, n_y, n_z)
    fh[n0[2] + N // 2, n0[1] + N // 2, n0[0] + N // 2] = c
    k0 = 2 * np.pi / L * np.array(n0)
    assert np.allclose(U.nudft2(fh, x, L), c * np.exp(1j * (k0 @ x)), atol=1e-13)
    w = rng.standard_normal(30)
    g = rng.standard_normal((N, N, N)) + 1j * rng.standard_normal((N, N, N))
    lhs = np.vdot(U.nudft1(x, w, N, L), g)
    rhs = np.vdot(w, U.nudft2(g, x, L))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


@pytest.mark.parametrize("N,eps", [(8, 1e-3), (16, 1e-4), (12, 1e-4), (8, 1e-6)])
def test_nufft1_within_eps_of_nudft(N, eps):
    """max |nufft1 - nudft1| <= eps sum |w| (several seeds, ragged N = 12)."""
    for seed in range(3):
        rng = np.random.default_rng(100 + seed)
        x = _pts(rng, 150)
        f = rng.standard_normal(150)
        err = np.abs(U.nufft1(x, f, N, L, eps) - U.nudft1(x, f, N, L)).max()
        assert err <= eps * np.abs(f).sum()


@pytest.mark.parametrize("N,eps", [(8, 1e-3), (16, 1e-4), (8, 1e-6)])
def test_nufft2_within_eps_of_nudft(N, eps):
    """max |nufft2 - nudft2| <= eps sum |f^|."""
    rng = np.random.default_rng(7)
    x = _pts(rng, 25)
    fh = rng.standard_normal((N, N, N)) + 1j * rng.standard_normal((N, N, N))
    err = np.abs(U.nufft2(fh, x, L, eps) - U.nudft2(fh, x, L)).max()
    assert err <= eps * np.abs(fh).sum()


def test_nufft_exact_adjoint_and_linear():
    """the discrete type-2 pipeline is the adjoint of type 1 (1e-12), linear."""
    N = 8
    rng = np.random.default_rng(8)
    x = _pts(rng, 60)
    w = rng.standard_normal(60)
    g = rng.standard_normal((N, N, N)) + 1j * rng.standard_normal((N, N, N))
    a = U.nufft1(x, w, N, L, 1e-2)
    b = U.nufft2(g, x, L, 1e-2)
    assert abs(np.vdot(a, g) - np.vdot(w, b)) <= 1e-12 * abs(np.vdot(a, g))
    w2 = rng.standard_normal(60)
    assert np.allclose(U.nufft1(x, 2 * w - w2, N, L), 2 * U.nufft1(x, w, N, L) - U.nufft1(x, w2, N, L),
                       atol=1e-12 * np.abs(w).sum())
    assert np.all(U.nufft1(x, np.zeros(60), N, L) == 0)
    assert np.all(U.nufft2(np.zeros((N, N, N), complex), x, L) == 0)


def test_window_transform_matches_adaptive_quadrature():
    """D: psi^(n) = int psi(2t/w) cos(2 pi n t / M) dt, against scipy.integrate.quad."""
    N, w = 16, 6
    M = 2 * N
    beta = U.beta_of(w)
    for n in (0, 3, N // 2):
        f = lambda t: np.exp(beta * (np.sqrt(max(0.0, 1 - (2 * t / w) ** 2)) - 1)) * np.cos(2 * np.pi * n * t / M)
        ref, _ = integrate.quad(f, -w / 2, w / 2, limit=400, epsabs=1e-15, epsrel=1e-13)
        assert abs(U.psi_hat(np.array([n]), w, M)[0] - ref) <= 1e-9 * abs(ref)
    assert U.window_width(1e-4) == 6 and U.window_width(1e-3) <= U.window_width(1e-6)
    with pytest.raises(ValueError):
        U.window_width(1e-20)


def _cos_lattice(N_lat, alpha, k1):
    """Particles on a lattice of spacing L / N_lat, weights q_j = h^3 (1 + alpha cos(k1 x_j)):
    the density 1 + alpha cos(k1 x) sampled exactly (no aliasing below N_lat / 2)."""
    h = L / N_lat
    g = np.arange(N_lat) * h + 0.37 * h
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    x = np.stack([X.ravel(), Y.ravel(), Z.ravel()])
    q = h ** 3 * (1 + alpha * np.cos(k1 * x[0]))
    return x, q


def test_pif_cosine_density_closed_form():
    """rho = 1 + alpha cos(k1 x) -> E_x = alpha sin(k1 x) / k1, E_y = E_z = 0,
    W_x = alpha^2 L^3 / (4 k1^2) (D#8, D#35, D#37); NUFFT error at eps = 1e-4."""
    alpha, k1 = 0.3, 2 * np.pi / L
    x, q = _cos_lattice(12, alpha, k1)
    E, W, _ = U.pif_solve(x, q, 8, L, eps=1e-8)
    assert np.abs(E[0] - alpha * np.sin(k1 * x[0]) / k1).max() < 1e-6
    assert np.abs(E[1:]).max() < 1e-6
    assert abs(W[0] - alpha ** 2 * L ** 3 / (4 * k1 ** 2)) < 1e-6 * W[0]
    assert W[1] < 1e-12 and W[2] < 1e-12


def test_pif_mirrored_pair_forces_opposite_and_exact_hook():
    """two equal charges mirrored about the centre -> E(x_1) = -E(x_2) (momentum);
    the NUFFT solve agrees with the NUDFT test hook to eps (1e-4) x scale."""
    N = 8
    c = np.array([L / 2] * 3)
    d = np.array([0.9, -0.4, 1.3])
    x = np.stack([c + d, c - d], axis=1)
    q = np.array([1.0, 1.0])
    E, _, _ = U.pif_solve(x, q, N, L, eps=1e-4)
    Ee, _, _ = U.pif_solve(x, q, N, L, exact=True)
    scale = np.abs(Ee).max()
    assert np.abs(Ee[:, 0] + Ee[:, 1]).max() < 1e-12 * scale
    assert np.abs(E[:, 0] + E[:, 1]).max() < 2e-4 * scale
    assert np.abs(E - Ee).max() < 1e-4 * scale * 10


def test_pif_run_conserves_momentum_and_streams_freely():
    """P:203-214 + P:124-137: equal charges, type 2 the exact adjoint of type 1 ->
    sum_j E(x_j) = L^-3 sum_k conj(rho^) (-i k rho^ / |k|^2) = 0 (antisymmetric in k), so
    total momentum is conserved to rounding; a uniform lattice (alpha = 0) feels no field
    and streams freely (x + n v dt, wrapped)."""
    from pic_inputs import landau_state

    Lk = 2 * np.pi / 0.5
    xv = landau_state(4, 4, L=Lk, seed=21, alpha=0.3)
    q = np.full(xv.shape[1], -Lk ** 3 / xv.shape[1])
    p0 = xv[3:].sum(axis=1)
    xs, ex = U.pif_run(4, Lk, 0.05, xv, q, 3)
    assert np.abs(xs[3:].sum(axis=1) - p0).max() < 1e-11 * np.abs(xv[3:]).sum()
    assert np.all(ex > 0)
    h = Lk / 4
    g = np.arange(4) * h + 0.5 * h
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    lat = np.zeros((6, 64))
    lat[:3] = np.stack([X.ravel(), Y.ravel(), Z.ravel()])
    lat[3] = 0.7
    ql = np.full(64, -Lk ** 3 / 64)
    xs, ex = U.pif_run(4, Lk, 0.05, lat, ql, 2)
    assert np.abs(xs[3] - 0.7).max() < 1e-12 and np.all(ex < 1e-20)
    assert np.abs(xs[0] - np.mod(lat[0] + 2 * 0.05 * 0.7, Lk)).max() < 1e-12
