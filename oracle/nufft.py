"""Plain numpy oracle of the NUFFT type 1 / type 2 and the Particle-in-Fourier field solve.

TEST INFRASTRUCTURE ONLY: only tests/, ``__graft_entry__.smoke()`` and ``bench.py``
(its ``cpu_baseline`` leg and ``--impl reference``) may import this module.  The product
package ``paper_2605_05469_b200`` never imports it, and the two share no code.

Citation key: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n, "D#k" = DESIGN.md reading k.

What it computes (P:197-221 Particle-in-Fourier, Appendix A):

* ``nudft1`` / ``nudft2``: the NUDFTs of Eq. (p2f) / (f2p) written out as
  direct sums, O(N_p N_m).
* ``nufft1``: Eq. (type1nufft), f^ = D chi F C f, in the paper's order:
  C spreads the weights onto the oversampled grid of M = sigma N points per dimension
  (sigma = 2) with a compact window (D#34: the "exponential of semicircle"
  psi(z) = exp(beta (sqrt(1 - z^2) - 1)), |z| <= 1, w fine-grid points of support,
  beta = 2.30 w); F is the unnormalised forward FFT on the M^3 grid (numpy); chi keeps
  the N^3 modes of K_N; D divides by the window's Fourier transform at those
  modes, computed by Gauss-Legendre quadrature.
* ``nufft2``: Eq. (type2nufft), f = C^T F^-1 chi^T D f^: the same steps
  reversed (the exact adjoint of ``nufft1``; F^-1 unnormalised, e^{+i}).
* ``pif_solve``: P:203-214. rho^ = nufft1(x, q); phi^ = rho^ / |k|^2 (D#8 sign, the
  k = 0 mode removed, D#3); E^ = -i k phi^; E(x_j) = L^-3 nufft2(E^)(x_j) (D#35: the
  1 / L^3 of the Fourier series of a periodic field, absent from P:214); the modes on
  the unpaired -N/2 planes of K_N are dropped from E^ (D#36) so E is real.
  W_d = 1 / (2 L^3) sum_k |E^_d(k)|^2 (D#37, Parseval for the truncated series).

Array conventions: positions ``x`` of shape (3, np) in [0, L); mode arrays of shape
(N, N, N) indexed [nz + N/2, ny + N/2, nx + N/2] (n ascending from -N/2); vector mode
arrays (3, N, N, N).  Fine grid (M, M, M) indexed [lz, ly, lx].
"""
from __future__ import annotations

import numpy as np

SIGMA = 2  # oversampling factor ("sigma = 2 is commonly chosen")


def window_width(eps: float) -> int:
    """D#34: w = ceil(log10(1/eps)) + 2 fine-grid points of support (sigma = 2); 1e-4 -> 6."""
    if not 1e-14 <= eps < 1:
        raise ValueError("eps must be in [1e-14, 1)")
    return int(np.ceil(np.log10(1.0 / eps))) + 2


def beta_of(w: int) -> float:
    """D#34: ES shape parameter beta = 2.30 w at sigma = 2."""
    return 2.30 * w


def psi(z: np.ndarray, beta: float) -> np.ndarray:
    """ES window psi(z) = exp(beta (sqrt(1 - z^2) - 1)) on |z| <= 1, 0 outside (D#34)."""
    z = np.asarray(z, dtype=np.float64)
    out = np.zeros_like(z)
    m = np.abs(z) <= 1.0
    out[m] = np.exp(beta * (np.sqrt(1.0 - z[m] * z[m]) - 1.0))
    return out


def psi_hat(n: np.ndarray, w: int, M: int, nq: int = 64) -> np.ndarray:
    """Fourier transform of the window at integer modes n (the entries of D):
    psi^(n) = int_{-w/2}^{w/2} psi(2t/w) e^{-2 pi i n t / M} dt
            = (w/2) int_{-1}^{1} psi(z) cos(pi n w z / M) dz   (psi even),
    by Gauss-Legendre quadrature with nq nodes."""
    z, a = np.polynomial.legendre.leggauss(nq)
    n = np.asarray(n, dtype=np.float64)
    vals = psi(z, beta_of(w))
    return (w / 2.0) * np.cos(np.pi * np.outer(n, z) * w / M) @ (a * vals)


def modes_1d(N: int) -> np.ndarray:
    """n in [-N/2, N/2 - 1] ascending."""
    return np.arange(-N // 2, N // 2)


def nudft1(x: np.ndarray, f: np.ndarray, N: int, L: float) -> np.ndarray:
    """Eq. (p2f): f^(k) = sum_j f_j exp(-i k . x_j), k in K_N; direct double loop
    over modes (vectorised over particles)."""
    n = modes_1d(N)
    k = 2 * np.pi / L * n
    ex = np.exp(-1j * np.outer(k, x[0]))  # (N, np)
    ey = np.exp(-1j * np.outer(k, x[1]))
    ez = np.exp(-1j * np.outer(k, x[2]))
    out = np.zeros((N, N, N), dtype=np.complex128)
    for a in range(N):
        for b in range(N):
            out[a, b, :] = ex @ (ez[a] * ey[b] * f)
    return out


def nudft2(fhat: np.ndarray, x: np.ndarray, L: float) -> np.ndarray:
    """Eq. (f2p): f(x_j) = sum_k f^(k) exp(+i k . x_j); direct sums, per particle."""
    N = fhat.shape[0]
    k = 2 * np.pi / L * modes_1d(N)
    out = np.zeros(x.shape[1], dtype=np.complex128)
    for j in range(x.shape[1]):
        ex = np.exp(1j * k * x[0, j])
        ey = np.exp(1j * k * x[1, j])
        ez = np.exp(1j * k * x[2, j])
        out[j] = np.einsum("abc,a,b,c->", fhat, ez, ey, ex)
    return out


def _spread_weights(xd: np.ndarray, M: int, L: float, w: int):
    """For one dimension: the w fine-grid indices (mod M) each point touches and the window
    values psi((l - u) / (w/2)) there, u = x M / L the fine-grid coordinate; l runs over the
    w integers with |l - u| <= w/2 (l0 = ceil(u - w/2))."""
    u = xd * (M / L)
    l0 = np.ceil(u - w / 2.0).astype(np.int64)
    ls = l0[:, None] + np.arange(w)[None, :]
    vals = psi((ls - u[:, None]) / (w / 2.0), beta_of(w))
    return np.mod(ls, M), vals


def spread(x: np.ndarray, f: np.ndarray, N: int, L: float, w: int) -> np.ndarray:
    """C: the M^3 fine grid b_l = sum_j f_j psi_x psi_y psi_z, periodic wrap."""
    M = SIGMA * N
    grid = np.zeros((M, M, M), dtype=np.complex128)
    ix, wx = _spread_weights(x[0], M, L, w)
    iy, wy = _spread_weights(x[1], M, L, w)
    iz, wz = _spread_weights(x[2], M, L, w)
    for j in range(x.shape[1]):
        blk = f[j] * wz[j][:, None, None] * wy[j][None, :, None] * wx[j][None, None, :]
        grid[np.ix_(iz[j], iy[j], ix[j])] += blk
    return grid


def interp(grid: np.ndarray, x: np.ndarray, N: int, L: float, w: int) -> np.ndarray:
    """C^T: f_j = sum_l g_l psi_x psi_y psi_z over the w^3 points of x_j."""
    M = SIGMA * N
    ix, wx = _spread_weights(x[0], M, L, w)
    iy, wy = _spread_weights(x[1], M, L, w)
    iz, wz = _spread_weights(x[2], M, L, w)
    out = np.zeros(x.shape[1], dtype=np.complex128)
    for j in range(x.shape[1]):
        blk = grid[np.ix_(iz[j], iy[j], ix[j])]
        out[j] = np.einsum("abc,a,b,c->", blk, wz[j], wy[j], wx[j])
    return out


def _deconv(N: int, w: int) -> np.ndarray:
    """D: 1 / (psi^(n_x) psi^(n_y) psi^(n_z)) on K_N, shape (N, N, N)."""
    p = 1.0 / psi_hat(modes_1d(N), w, SIGMA * N)
    return p[:, None, None] * p[None, :, None] * p[None, None, :]


def _chi_index(N: int) -> np.ndarray:
    """chi: the fine-grid frequency index n mod M of each n in K_N."""
    return np.mod(modes_1d(N), SIGMA * N)


def nufft1(x: np.ndarray, f: np.ndarray, N: int, L: float, eps: float = 1e-4) -> np.ndarray:
    """Eq. (type1nufft): f^ = D chi F C f."""
    w = window_width(eps)
    b = spread(x, f, N, L, w)                                   # C
    B = np.fft.fftn(b)                                          # F (e^{-i}, unnormalised)
    c = _chi_index(N)
    sel = B[np.ix_(c, c, c)]                                    # chi
    return sel * _deconv(N, w)                                  # D


def nufft2(fhat: np.ndarray, x: np.ndarray, L: float, eps: float = 1e-4) -> np.ndarray:
    """Eq. (type2nufft): f = C^T F^-1 chi^T D f^ (F^-1 = e^{+i}, unnormalised)."""
    N = fhat.shape[0]
    M = SIGMA * N
    w = window_width(eps)
    G = np.zeros((M, M, M), dtype=np.complex128)
    c = _chi_index(N)
    G[np.ix_(c, c, c)] = fhat * _deconv(N, w)                   # chi^T D
    g = np.fft.ifftn(G) * float(M) ** 3                         # F^-1, unnormalised
    return interp(g, x, N, L, w)                                # C^T


def k_vectors(N: int, L: float):
    """k_d = 2 pi n_d / L on K_N, broadcastable to (N, N, N) [nz, ny, nx]."""
    k = 2 * np.pi / L * modes_1d(N)
    return k[None, None, :], k[None, :, None], k[:, None, None]


def pif_fields_hat(rho_hat: np.ndarray, L: float) -> np.ndarray:
    """phi^ = rho^ / |k|^2 (D#8; k = 0 removed, D#3), E^ = -i k phi^; modes on
    the unpaired -N/2 planes dropped (D#36).  Returns E^ of shape (3, N, N, N)."""
    N = rho_hat.shape[0]
    kx, ky, kz = k_vectors(N, L)
    k2 = kx * kx + ky * ky + kz * kz
    phi = np.zeros_like(rho_hat)
    nz = k2 != 0
    phi[nz] = rho_hat[nz] / np.broadcast_to(k2, rho_hat.shape)[nz]
    Eh = np.stack([-1j * kx * phi, -1j * ky * phi, -1j * kz * phi])
    Eh[:, 0, :, :] = 0.0                                        # n_z = -N/2
    Eh[:, :, 0, :] = 0.0                                        # n_y = -N/2
    Eh[:, :, :, 0] = 0.0                                        # n_x = -N/2
    return Eh


def pif_energy(E_hat: np.ndarray, L: float) -> np.ndarray:
    """D#37: W_d = 1 / (2 L^3) sum_k |E^_d(k)|^2 = 1/2 int E_d^2 dx of the truncated series."""
    return np.array([0.5 / L ** 3 * np.sum(np.abs(E_hat[d]) ** 2) for d in range(3)])


def pif_solve(x: np.ndarray, q: np.ndarray, N: int, L: float, eps: float = 1e-4, exact: bool = False):
    """the PIF field solve.  Returns (E at particles (3, np) real, W (3,), E^).
    ``exact`` replaces both NUFFTs with the direct NUDFTs (test hook)."""
    rho_hat = nudft1(x, q, N, L) if exact else nufft1(x, q, N, L, eps)
    Eh = pif_fields_hat(rho_hat, L)
    E = np.zeros((3, x.shape[1]))
    for d in range(3):
        v = nudft2(Eh[d], x, L) if exact else nufft2(Eh[d], x, L, eps)
        E[d] = v.real / L ** 3
    return E, pif_energy(Eh, L), Eh


def nudft1_modes(x: np.ndarray, f: np.ndarray, L: float, modes) -> np.ndarray:
    """Eq. (p2f) at a list of integer modes (n_x, n_y, n_z) only: sum_j f_j e^{-i k . x_j}
    (the sampled full-size check)."""
    out = []
    for n in modes:
        k = 2 * np.pi / L * np.asarray(n, dtype=np.float64)
        out.append(np.sum(f * np.exp(-1j * (k[0] * x[0] + k[1] * x[1] + k[2] * x[2]))))
    return np.array(out)


def pif_run(N: int, L: float, dt: float, xv: np.ndarray, q: np.ndarray, nsteps: int, eps: float = 1e-4):
    """The PIF time loop (Fig. 1, with the PIF solve of P:203-214 in place of
    deposit + solve + gather): each step E = pif_solve(x_n), W_x(t_n) recorded (D#12), then
    the leapfrog kick-drift-wrap of the PIC oracle (q/m = -1, D#2, D#9).
    Returns (xv after nsteps, W_x[nsteps])."""
    from oracle import oracle as O

    xs = np.ascontiguousarray(xv, dtype=np.float64).copy()
    ex = np.zeros(nsteps)
    for s in range(nsteps):
        E, W, _ = pif_solve(xs[:3], q, N, L, eps)
        ex[s] = W[0]
        xs = O.push(L, xs, E, -dt, dt)
    return xs, ex
