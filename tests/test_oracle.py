"""Pins of the CPU oracle (oracle/oracle.c) against the paper and the mathematics.

Nothing here compares the oracle with itself: every check is a published
value, a closed form, an invariant, brute force, or an independent library
routine (numpy's FFT / stable argsort).  Citations: P:n = PAPER.md line n,
S:n = SPEC.md line n, D#k = DESIGN.md reading k.
"""
import os

import numpy as np
import pytest
from scipy import stats

from oracle import oracle as O
from pic_inputs import landau_state, random_grid, random_field
from landau_fit import dispersion_root, fit_damping_rate

K = 0.5
L = 2 * np.pi / K
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------- RNG ------
def test_philox_known_answers():
    """Random123 published vectors (golden/philox4x32_10_kat.txt)."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt"))
            if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(t, 16) for t in r]
        out = O.philox(v[0:4], v[4:6])
        assert list(out) == v[6:10]


def test_uniforms_are_53bit_grid_and_counter_based():
    u = O.uniforms(7, 12345)
    assert np.all((u >= 0) & (u < 1))
    assert np.all(u * 2.0 ** 53 == np.floor(u * 2.0 ** 53))
    assert np.array_equal(u, O.uniforms(7, 12345))          # pure function of (seed, j)
    assert not np.array_equal(u, O.uniforms(7, 12346))
    assert not np.array_equal(u, O.uniforms(8, 12345))


def test_uniforms_word_layout_matches_random123_kat():
    """SURVEY c.1 Init 1 / D#10: (seed 0, particle j 0, block b 0) is the first Random123
    vector (counter 0, key 0 -> r0..r3, golden/philox4x32_10_kat.txt), so u_0 and u_1 must
    be ((r0 | r1 << 32) >> 11) 2^-53 and ((r2 | r3 << 32) >> 11) 2^-53.  A swapped word
    order, a wrong shift or a dropped high word fails here."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt"))
            if l.strip() and not l.startswith("#")]
    r = [int(t, 16) for t in rows[0][6:10]]
    assert [int(t, 16) for t in rows[0][:6]] == [0] * 6
    u = O.uniforms(0, 0)
    w0 = r[0] | (r[1] << 32)
    w1 = r[2] | (r[3] << 32)
    assert u[0] == (w0 >> 11) * 2.0 ** -53
    assert u[1] == (w1 >> 11) * 2.0 ** -53
    # written out from the published words: 0xe169c58d6627e8d5 >> 11, 0x9b00dbd8bc57ac4c >> 11
    assert u[0] == 0x1C2D38B1ACC4FD * 2.0 ** -53 and u[1] == 0x13601B7B178AF5 * 2.0 ** -53


def test_sampler_alpha0_is_uniform_ks():
    """alpha = 0 degenerates to uniform; KS below the 1% critical value."""
    xv = O.sample_landau(200_000, K, L, 0.0, 3)
    for d in range(3):
        stat = stats.kstest(xv[d] / L, "uniform").statistic
        assert stat < 1.63 / np.sqrt(xv.shape[1])


def test_sampler_landau_density_chi2():
    """64-bin histogram of x vs (1 + alpha cos kx)/L, chi-square p > 0.001."""
    n = 1_000_000
    xv = O.sample_landau(n, K, L, 0.05, 5)
    edges = np.linspace(0, L, 65)
    cdf = (edges + (0.05 / K) * np.sin(K * edges)) / L
    expected = np.diff(cdf) * n
    for d in range(3):
        obs, _ = np.histogram(xv[d], edges)
        p = stats.chisquare(obs, expected).pvalue
        assert p > 1e-3
        assert np.all(xv[d] >= 0) and np.all(xv[d] < L)


def test_sampler_velocity_moments():
    """mean within 5/sqrt(n) of 0, variance within 5 sqrt(2/n) of 1."""
    n = 400_000
    xv = O.sample_landau(n, K, L, 0.05, 11)
    for d in range(3, 6):
        assert abs(xv[d].mean()) < 5 / np.sqrt(n)
        assert abs(xv[d].var() - 1) < 5 * np.sqrt(2 / n)


def test_dispersion_root_golden():
    """The analytic damping rate the physics pins use (golden/landau_k0p5.txt)."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "landau_k0p5.txt"))
            if l.strip() and not l.startswith("#")]
    wr, g = map(float, rows[0])
    w = dispersion_root(0.5)
    assert abs(w.real - wr) < 1e-6 and abs(w.imag - g) < 1e-6


def test_damping_fitter_on_synthetic_series():
    """e^{2 gamma t} sin^2(omega t) must give slope 2 gamma to 1%."""
    t = np.arange(0, 20, 0.05)
    W = np.exp(2 * -0.1533 * t) * np.sin(1.4 * t) ** 2
    slope, npk, _ = fit_damping_rate(t, W)
    assert npk >= 3 and abs(slope - 2 * -0.1533) < 0.01 * 0.3066


# ---------------------------------------------------------- keys / sort -----
def test_cell_index_edges():
    n = 16
    inv_h = n / L
    assert O.cell_index(0.0, inv_h, n) == 0
    assert O.cell_index(np.nextafter(L, 0), inv_h, n) == n - 1      # D#5 clamp
    h = L / n
    assert O.cell_index(3 * h + 0.5 * h, inv_h, n) == 3


def test_morton_key_is_bijective_and_blocked():
    """D#14: Morton order; each aligned run of 8^l keys is a (2^l)^3 cube."""
    n = 16
    ks = np.array([[[O.morton_key(ix, iy, iz, n) for ix in range(n)] for iy in range(n)]
                   for iz in range(n)])
    assert sorted(ks.ravel().tolist()) == list(range(n ** 3))
    assert O.morton_key(1, 0, 0, n) == 1 and O.morton_key(0, 1, 0, n) == 2
    assert O.morton_key(0, 0, 1, n) == 4
    inv = np.zeros((n ** 3, 3), dtype=int)
    for iz in range(n):
        for iy in range(n):
            for ix in range(n):
                inv[ks[iz, iy, ix]] = (ix, iy, iz)
    for side in (2, 4, 8):
        run = side ** 3
        for start in range(0, n ** 3, run):
            c = inv[start:start + run]
            assert np.all(c.max(0) - c.min(0) == side - 1)
            assert np.all(c.min(0) % side == 0)


def test_sort_equals_numpy_stable_argsort():
    n = 16
    xv = landau_state(n, 8, seed=4)
    keys = O.keys(n, L, xv)
    xs, perm = O.sort(n, L, xv)
    ref = np.argsort(keys, kind="stable")
    assert np.array_equal(perm, ref.astype(np.uint32))
    assert np.array_equal(xs, xv[:, ref])
    assert np.all(np.diff(O.keys(n, L, xs).astype(np.int64)) >= 0)


# ----------------------------------------------------------- scatter --------
def test_deposit_particle_on_node():
    """a particle exactly on a node gives that node q/h^3, others 0."""
    n = 8
    h = L / n
    xv = np.zeros((6, 1))
    xv[:3, 0] = [2 * h, 3 * h, 5 * h]
    rho = O.deposit(n, L, xv, q=1.0)
    assert rho[5, 3, 2] == pytest.approx(1 / h ** 3, rel=1e-14)
    rho[5, 3, 2] = 0
    assert np.all(rho == 0)


def test_deposit_particle_at_cell_centre_and_wrap():
    """each of the 8 corners gets q/(8 h^3); the last cell wraps to node 0."""
    n = 8
    h = L / n
    xv = np.zeros((6, 1))
    xv[:3, 0] = [(n - 0.5) * h, 0.5 * h, 3.5 * h]
    rho = O.deposit(n, L, xv, q=1.0)
    for iz in (3, 4):
        for iy in (0, 1):
            for ix in (n - 1, 0):
                assert rho[iz, iy, ix] == pytest.approx(1 / (8 * h ** 3), rel=1e-13)
    assert np.count_nonzero(rho) == 8


def test_deposit_charge_conservation():
    """S:135/S:140 and BJ: sum rho h^3 = N_p q = -L^3 within 1e-12."""
    n = 16
    xv = landau_state(n, 8, seed=2)
    q = -L ** 3 / xv.shape[1]
    rho = O.deposit(n, L, xv, q)
    total = rho.sum() * (L / n) ** 3
    assert abs(total - (-L ** 3)) < 1e-12 * L ** 3


def test_gather_constant_and_linear():
    """constant field reproduced (partition of unity, to a few ulp: the
    eight weight products sum to 1 only up to rounding); linear reproduced in a cell."""
    n = 8
    h = L / n
    rng = np.random.default_rng(0)
    xv = np.zeros((6, 100))
    xv[:3] = rng.random((3, 100)) * (n - 1) * h        # stay off the periodic seam
    E = np.full((3, n, n, n), 0.75)
    Ep = O.gather(n, L, xv, E)
    np.testing.assert_allclose(Ep, 0.75, rtol=4e-16, atol=0)
    iz, iy, ix = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    E = np.stack([ix * h * 2.0 + 1.0, iy * h * -3.0, iz * h * 0.5 + ix * h])
    Ep = O.gather(n, L, xv, E)
    x, y, z = xv[0], xv[1], xv[2]
    np.testing.assert_allclose(Ep[0], 2 * x + 1, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(Ep[1], -3 * y, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(Ep[2], 0.5 * z + x, rtol=1e-13, atol=1e-13)


def test_scatter_gather_adjointness():
    """sum_nodes scatter(q, x) G h^3 = sum_j q gather(G, x_j), 1e-12."""
    n = 16
    xv = landau_state(n, 2, seed=9)
    G = random_field(n, seed=3)[0]
    q = 0.37
    lhs = (O.deposit(n, L, xv, q) * G).sum() * (L / n) ** 3
    rhs = q * O.gather(n, L, xv, np.stack([G, G, G]))[0].sum()
    assert abs(lhs - rhs) < 1e-12 * abs(rhs) + 1e-12


# -------------------------------------------------------------- solve -------
@pytest.mark.parametrize("n", [8, 16])
def test_solve_fft_equals_brute_force_dft(n):
    """BJ: FFT solve == O(N^6) direct DFT solve to 1e-13 (relative to max)."""
    rho = random_grid(n, seed=n)
    Ef, imf = O.solve_fft(n, L, rho)
    Ed, imd = O.solve_dft(n, L, rho)
    assert np.max(np.abs(Ef - Ed)) < 1e-13 * np.max(np.abs(Ed))
    assert imf < 1e-13 * np.max(np.abs(Ef)) and imd < 1e-12 * np.max(np.abs(Ed))


def _numpy_spectral_solve(n, rho):
    """Independent library path: numpy.fft with the D#6 Nyquist reading."""
    rh = np.fft.fftn(rho)
    m = np.fft.fftfreq(n, d=1.0 / n)          # 0..N/2-1, -N/2..-1
    kv = 2 * np.pi * m / L
    kz, ky, kx = np.meshgrid(kv, kv, kv, indexing="ij")
    k2 = kx ** 2 + ky ** 2 + kz ** 2
    k2[0, 0, 0] = 1.0
    out = []
    for d, kd in enumerate((kx, ky, kz)):
        eh = -1j * kd * rh / k2
        eh[0, 0, 0] = 0
        sl = [slice(None)] * 3
        sl[2 - d] = n // 2
        eh[tuple(sl)] = 0
        out.append(np.fft.ifftn(eh).real)
    return np.stack(out)


def test_solve_fft_equals_numpy_fft():
    n = 32
    rho = random_grid(n, seed=5, mean=-1.0)
    E, _ = O.solve_fft(n, L, rho)
    ref = _numpy_spectral_solve(n, rho)
    assert np.max(np.abs(E - ref)) < 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_solve_single_mode(axis):
    """rho = cos(k1 x_d) => E_d = sin(k1 x_d)/k1, other components 0."""
    n = 16
    k1 = 2 * np.pi / L
    x = np.arange(n) * L / n
    shape = [1, 1, 1]
    shape[2 - axis] = n
    rho = np.broadcast_to(np.cos(k1 * x).reshape(shape), (n, n, n)).copy()
    E, imag = O.solve_fft(n, L, rho)
    want = np.broadcast_to((np.sin(k1 * x) / k1).reshape(shape), (n, n, n))
    assert np.max(np.abs(E[axis] - want)) < 1e-12
    for d in range(3):
        if d != axis:
            assert np.max(np.abs(E[d])) < 1e-12
    assert imag < 1e-12


def test_solve_constant_linearity_translation_gauss():
    n = 16
    c = np.full((n, n, n), 3.5)
    E0, _ = O.solve_fft(n, L, c)
    assert np.max(np.abs(E0)) < 1e-12
    r1, r2 = random_grid(n, 1), random_grid(n, 2)
    E1, _ = O.solve_fft(n, L, r1)
    E2, _ = O.solve_fft(n, L, r2)
    E12, _ = O.solve_fft(n, L, 2.0 * r1 - 0.5 * r2)
    assert np.max(np.abs(E12 - (2 * E1 - 0.5 * E2))) < 1e-11
    Es, _ = O.solve_fft(n, L, np.roll(r1, (1, 2, 3), axis=(0, 1, 2)))
    assert np.max(np.abs(Es - np.roll(E1, (1, 2, 3), axis=(1, 2, 3)))) < 1e-11
    assert np.max(np.abs(E1.mean(axis=(1, 2, 3)))) < 1e-13
    # Gauss's law in spectral space, i k . E^ = rho^ - mean, on modes with no Nyquist index
    m = np.fft.fftfreq(n, d=1.0 / n)
    kv = 2 * np.pi * m / L
    kz, ky, kx = np.meshgrid(kv, kv, kv, indexing="ij")
    div = 1j * (kx * np.fft.fftn(E1[0]) + ky * np.fft.fftn(E1[1]) + kz * np.fft.fftn(E1[2]))
    rh = np.fft.fftn(r1)
    mask = np.ones((n, n, n), bool)
    mask[n // 2, :, :] = mask[:, n // 2, :] = mask[:, :, n // 2] = False
    mask[0, 0, 0] = False
    assert np.max(np.abs(div[mask] - rh[mask])) < 1e-10 * np.max(np.abs(rh))
    # total momentum: sum_i rho_i E_i = 0 (SURVEY c.3 "Whole step")
    for d in range(3):
        assert abs((r1 * E1[d]).sum()) < 1e-12 * np.sqrt((r1 ** 2).sum() * (E1[d] ** 2).sum())


def test_field_energy_closed_forms():
    """E_x = sin(k1 x) on N=32 => 1/2 L^3/2; constant c => 1/2 c^2 L^3."""
    n = 32
    k1 = 2 * np.pi / L
    x = np.arange(n) * L / n
    E = np.zeros((3, n, n, n))
    E[0] = np.sin(k1 * x)[None, None, :]
    wx, w = O.field_energy(n, L, E)
    assert wx == pytest.approx(0.5 * L ** 3 / 2, rel=1e-12) and w == pytest.approx(wx, rel=1e-15)
    E = np.full((3, n, n, n), 1.5)
    wx, w = O.field_energy(n, L, E)
    assert wx == pytest.approx(0.5 * 1.5 ** 2 * L ** 3, rel=1e-12)
    assert w == pytest.approx(3 * wx, rel=1e-12)


# --------------------------------------------------------- push / wrap ------
def test_push_free_streaming_and_constant_kick():
    """S:156-157."""
    xv = np.zeros((6, 3))
    xv[:3] = 1.0
    xv[3:] = [[0.5, -0.25, 1.0]] * 3
    out = O.push(L, xv, np.zeros((3, 3)), -0.05, 0.05)
    assert np.all(out[3:] == xv[3:])
    np.testing.assert_allclose(out[:3], 1.0 + xv[3:] * 0.05, rtol=0, atol=1e-15)
    Ep = np.zeros((3, 3))
    Ep[0] = 1.0
    out = O.push(L, xv, Ep, -0.05, 0.05)                 # q/m = -1 => v_x decreases by dt
    np.testing.assert_allclose(out[3], xv[3] - 0.05, rtol=0, atol=1e-15)


def test_half_kick_single_mode_closed_form():
    """S:180 / D#9: the backward half kick is v_{-1/2} = v_0 - (q/m) E(x_0) dt/2 = v_0 + E dt/2.

    Particles sit exactly on the nodes of a 16^3 grid, c_i = 2 + cos(pi i_x / 2) of them on
    every node of x-plane i_x (integers 3, 2, 1, 2), so the CIC deposit is exactly
    rho = (q/h^3)(2 + cos(k4 x)) with k4 = 2 pi 4 / L and q = -L^3/N_p = -h^3/2.
    The k = 0 mode is removed, so E_x = -(1/2) sin(k4 x)/k4 and E_y = E_z = 0
    (P:175 with D#8), and a particle on a node gathers its node's value exactly.  Hence
    v_x changes by -(dt/4) sin(k4 x)/k4: a sign slip or a missing 1/2 fails here."""
    n, dt = 16, 0.05
    h = L / n
    pos = []
    for iz in range(n):
        for iy in range(n):
            for ix in range(n):
                c = 2 + [1, 0, -1, 0][ix % 4]
                pos += [(ix * h, iy * h, iz * h)] * c
    pos = np.array(pos).T
    assert pos.shape[1] == 2 * n ** 3
    rng = np.random.default_rng(3)
    xv = np.concatenate([pos, rng.standard_normal((3, pos.shape[1]))])
    out = O.half_kick(n, L, dt, xv)
    assert np.array_equal(out[:3], xv[:3])                       # x unchanged
    k4 = 2 * np.pi * 4 / L
    ex = -0.5 * np.sin(k4 * xv[0]) / k4
    np.testing.assert_allclose(out[3] - xv[3], ex * dt / 2, rtol=0, atol=1e-13)
    np.testing.assert_allclose(out[4:] - xv[4:], 0.0, rtol=0, atol=1e-13)
    assert np.abs(out[3] - xv[3]).max() > 0.9 * 0.25 * dt / k4   # the odd planes do move


def test_wrap_cases():
    """x = L -> 0; x = -0.3h -> L - 0.3h; in-range unchanged bitwise."""
    h = L / 16
    assert O.wrap(L, L) == 0.0
    assert O.wrap(-0.3 * h, L) == pytest.approx(L - 0.3 * h, abs=1e-15)
    for x in (0.0, 1.234, np.nextafter(L, 0)):
        assert O.wrap(x, L) == x
    assert O.wrap(-1e-300, L) == 0.0        # rounds to L -> 0


def test_mirrored_particles_equal_opposite_forces():
    """two particles mirrored about the domain centre feel opposite forces."""
    n = 16
    c = L / 2
    p = np.array([c + 1.1, c - 0.7, c + 2.3])
    xv = np.zeros((6, 2))
    xv[:3, 0] = p
    xv[:3, 1] = 2 * c - p
    rho = O.deposit(n, L, xv, -1.0)
    E, _ = O.solve_fft(n, L, rho)
    Ep = O.gather(n, L, xv, E)
    assert np.max(np.abs(Ep[:, 0] + Ep[:, 1])) < 1e-10
    assert np.max(np.abs(Ep)) > 1e-4


# ----------------------------------------------------------- whole step -----
def test_run_momentum_conservation_and_determinism():
    """SURVEY c.3: total momentum sum_j v_j is conserved to rounding; runs are bitwise reproducible."""
    n = 16
    xv = landau_state(n, 8, seed=21)
    xs, ex, tot, perm = O.run(n, L, 0.05, xv, 10, want_perm=True)
    p0 = xv[3:].sum(axis=1)
    p1 = xs[3:].sum(axis=1)
    assert np.max(np.abs(p1 - p0)) < 1e-10 * np.abs(xv[3:]).sum()
    xs2, ex2, tot2, perm2 = O.run(n, L, 0.05, xv, 10, want_perm=True)
    assert np.array_equal(xs, xs2) and np.array_equal(ex, ex2) and np.array_equal(perm, perm2)
    assert np.all(ex > 0) and np.all(tot >= ex)
    assert np.all((xs[:3] >= 0) & (xs[:3] < L))
    assert np.all(np.diff(O.keys(n, L, xs).astype(np.int64)) >= 0)   # canonical order


@pytest.mark.parametrize("threads", [3, 8])
def test_openmp_deterministic_mode(threads):
    """SURVEY c.1/c.5 "OpenMP-deterministic mode": with T threads the sort is still the
    stable sort (numpy's stable argsort), the two-colour slab deposit conserves charge
    exactly and equals the serial deposit up to summation order, and whole runs are
    bitwise reproducible at fixed T and agree with the serial mode within the BJ
    tolerances (energies 1e-10, x, v 1e-12, permutation bit-exact)."""
    n = 32
    xv = landau_state(n, 8, seed=23)
    keys = O.keys(n, L, xv)
    with O.threads(threads):
        assert O.get_threads() == threads
        xs, perm = O.sort(n, L, xv)
        assert np.array_equal(perm, np.argsort(keys, kind="stable").astype(np.uint32))
        q = -L ** 3 / xv.shape[1]
        rho = O.deposit(n, L, xs, q)
        h = L / n
        assert rho.sum() * h ** 3 == pytest.approx(-L ** 3, rel=1e-12)
    rho_ref = O.deposit(n, L, xs, q)
    assert np.abs(rho - rho_ref).max() <= 1e-14 * np.abs(rho_ref).max()
    with O.threads(threads):
        a = O.run(n, L, 0.05, xv, 5, want_perm=True)
        b = O.run(n, L, 0.05, xv, 5, want_perm=True)
    assert O.get_threads() == 1
    for u, v in zip(a, b):
        assert np.array_equal(u, v)                    # deterministic for a fixed thread count
    s = O.run(n, L, 0.05, xv, 5, want_perm=True)
    assert np.array_equal(a[3], s[3])
    assert np.all(np.abs(a[1] - s[1]) <= 1e-10 * s[1])
    dx = np.abs(a[0][:3] - s[0][:3])
    assert np.minimum(dx, L - dx).max() / L <= 1e-12
    assert (np.abs(a[0][3:] - s[0][3:]) / np.maximum(np.abs(s[0][3:]), 1)).max() <= 1e-12


def test_alpha0_no_growth():
    """alpha = 0 at 16^3 x 8: no growth above 10x W_x(0) over 100 steps."""
    n = 16
    xv = O.init_state(n, 8, alpha=0.0, seed=3)
    _, ex, _, _ = O.run(n, L, 0.05, xv, 100)
    assert np.max(ex) < 10 * ex[0]


def test_landau_damping_rate_oracle():
    """P:231-232, BJ: the E_x energy peaks decay at 2 gamma = -0.3067 (+-10%) and are
    spaced pi/omega_r = 2.219 (+-5%).  Input (D#21): 16^3 x 128 ppc, alpha = 0.1 so
    the t <= 10 window stays above the shot-noise floor on a CPU-budget run."""
    n = 16
    w = dispersion_root(0.5)
    xv = O.init_state(n, 128, alpha=0.1, seed=1)
    _, ex, _, _ = O.run(n, L, 0.05, xv, 200)
    t = np.arange(200) * 0.05
    slope, npk, tp = fit_damping_rate(t, ex, t_max=10.0)
    assert npk >= 3
    assert abs(slope - 2 * w.imag) < 0.10 * abs(2 * w.imag)
    assert abs(np.mean(np.diff(tp)) - np.pi / w.real) < 0.05 * np.pi / w.real
