"""Pins of the oracle's external-field push (Eq. 1, Eq. 3-4: P:97; S:153;
SURVEY §8(f) NEXT-3; reading D#32): the Boris scheme for uniform B_ext and E_ext.

The pins are closed forms of the discrete Boris map, not the oracle re-typed:
a pure magnetic kick is a rotation about B by theta = 2 atan(|q/m| |B| dt / 2)
(so |v| is conserved and v after N steps is R(N theta) v0, the positions the sum
of the rotated velocities); the E x B drift velocity E x B / |B|^2 is a fixed
point of the map; B = 0 reduces to the leapfrog kick; a uniform E_ext alone is a
constant acceleration (q/m) E_ext.
"""
import numpy as np
import pytest

from oracle import oracle as O

K = 0.5
L = 2 * np.pi / K
DT = 0.05


def _state(v, x=None):
    v = np.asarray(v, dtype=np.float64)
    npart = v.shape[1]
    xv = np.zeros((6, npart))
    xv[:3] = L / 2 if x is None else x
    xv[3:] = v
    return xv


def _rot_z(theta):
    c, s = np.cos(theta), np.sin(theta)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def test_boris_conserves_speed_over_1000_steps():
    """E = 0, B = (0, 0, 1): |v| conserved to 1e-13 relative over 1000 steps."""
    rng = np.random.default_rng(1)
    xv = _state(rng.standard_normal((3, 64)))
    s0 = np.linalg.norm(xv[3:], axis=0)
    for _ in range(1000):
        xv = O.push_ext(L, xv, np.zeros((3, 64)), DT, b_ext=[0.0, 0.0, 1.0])
    assert np.max(np.abs(np.linalg.norm(xv[3:], axis=0) / s0 - 1.0)) < 1e-13


@pytest.mark.parametrize("b0", [0.5, 1.0, 4.0])
def test_boris_rotation_closed_form(b0):
    """E = 0, B = b0 z: each step rotates v_perp by theta = 2 atan(b0 dt / 2) in the
    positive sense (q/m = -1: dv/dt = -v x B); v_z is untouched; x advances by the
    rotated velocities (drift after the kick)."""
    v0 = np.array([[0.7], [-0.2], [0.3]])
    x0 = np.array([[1.0], [2.0], [3.0]])
    xv = _state(v0, x0)
    theta = 2 * np.arctan(b0 * DT / 2)
    x = x0[:, 0].copy()
    for k in range(1, 201):
        xv = O.push_ext(L, xv, np.zeros((3, 1)), DT, b_ext=[0.0, 0.0, b0])
        vk = _rot_z(k * theta) @ v0[:, 0]
        x = x + vk * DT
        assert np.max(np.abs(xv[3:, 0] - vk)) < 1e-12
        assert xv[5, 0] == v0[2, 0]
    assert np.max(np.abs(xv[:3, 0] - np.mod(x, L))) < 1e-11


def test_boris_rotation_about_an_oblique_field():
    """The rotation is about B for any direction: v . B is conserved and the angle
    between successive perpendicular parts is 2 atan(|B| dt / 2)."""
    B = np.array([0.3, -0.4, 1.2])
    b = B / np.linalg.norm(B)
    v0 = np.array([[1.0], [0.5], [-0.25]])
    xv = _state(v0)
    xv1 = O.push_ext(L, xv, np.zeros((3, 1)), DT, b_ext=B)
    v1 = xv1[3:, 0]
    assert abs(v1 @ b - v0[:, 0] @ b) < 1e-15
    p0 = v0[:, 0] - (v0[:, 0] @ b) * b
    p1 = v1 - (v1 @ b) * b
    ang = np.arctan2(np.cross(p0, p1) @ b, p0 @ p1)
    assert abs(ang - 2 * np.arctan(np.linalg.norm(B) * DT / 2)) < 1e-13


def test_exb_drift_is_a_fixed_point():
    """E_ext = (E0, 0, 0), B = (0, 0, B0): v = E x B / |B|^2 = (0, -E0/B0, 0) stays
    exactly (to rounding) the velocity of the Boris map for 100 steps."""
    E0, B0 = 0.2, 1.5
    vd = np.cross([E0, 0, 0], [0, 0, B0]) / B0 ** 2
    xv = _state(vd.reshape(3, 1))
    for _ in range(100):
        xv = O.push_ext(L, xv, np.zeros((3, 1)), DT, b_ext=[0, 0, B0], e_ext=[E0, 0, 0])
    assert np.max(np.abs(xv[3:, 0] - vd)) < 1e-14


def test_zero_B_is_the_leapfrog_kick_and_E_ext_accelerates():
    """B = 0: exactly oracle_push; E_ext alone adds (q/m) E_ext dt per step."""
    rng = np.random.default_rng(2)
    xv = _state(rng.standard_normal((3, 16)), rng.random((3, 16)) * L)
    Ep = rng.standard_normal((3, 16))
    assert np.array_equal(O.push_ext(L, xv, Ep, DT), O.push(L, xv, Ep, -DT, DT))
    out = O.push_ext(L, xv, np.zeros((3, 16)), DT, e_ext=[1.0, -2.0, 0.5])
    np.testing.assert_allclose(out[3:] - xv[3:], -DT * np.array([[1.0], [-2.0], [0.5]]) + 0 * xv[3:],
                               rtol=0, atol=1e-15)


def test_run_ext_with_magnetic_field_conserves_kinetic_plus_field_energy_trend():
    """A whole loop with B_ext (16^3 x 8): the magnetic force does no work, so the total
    energy (kinetic + W) drifts no more than in the B = 0 run over 20 steps (leapfrog
    noise only), and the loop stays deterministic."""
    from pic_inputs import landau_state

    n = 16
    xv = landau_state(n, 8, seed=4)
    q = L ** 3 / xv.shape[1]                 # |macro charge| = macro mass (q/m = -1)

    def total(x, w):
        return 0.5 * q * (x[3:] ** 2).sum() + w

    xs0, _, w0 = O.run_ext(n, L, DT, xv, 20)
    xsb, _, wb = O.run_ext(n, L, DT, xv, 20, b_ext=[0.0, 0.0, 2.0])
    xsb2, _, _ = O.run_ext(n, L, DT, xv, 20, b_ext=[0.0, 0.0, 2.0])
    assert np.array_equal(xsb, xsb2)
    e_start = total(xv, w0[0])
    drift0 = abs(total(xs0, w0[-1]) - e_start) / e_start
    driftb = abs(total(xsb, wb[-1]) - e_start) / e_start
    assert driftb < max(5 * drift0, 1e-3)
    assert not np.array_equal(xs0, xsb)
