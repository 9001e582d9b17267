"""ctypes wrapper over the plain-C PIC oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this module.  The product package ``paper_2605_05469_b200`` never imports it,
and the two share no code.

Array conventions follow oracle/oracle.h: particle state ``xv`` is a
C-contiguous float64 array of shape (6, np) (x, y, z, vx, vy, vz); grids are
(N, N, N) float64 indexed [iz, iy, ix]; vector fields are (3, N, N, N).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-ffp-contract=off: fma only where written)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        dp = C.POINTER(C.c_double)
        u32p = C.POINTER(C.c_uint32)
        i32, i64, u64, dbl = C.c_int32, C.c_int64, C.c_uint64, C.c_double
        sig = {
            "oracle_philox4x32_10": (None, [u32p, u32p, u32p]),
            "oracle_set_threads": (None, [i32]),
            "oracle_get_threads": (i32, []),
            "oracle_uniforms": (None, [u64, u64, dp]),
            "oracle_sample_landau": (None, [i64, dbl, dbl, dbl, u64, dp]),
            "oracle_cell_index": (i32, [dbl, dbl, i32]),
            "oracle_morton_key": (C.c_uint32, [i32, i32, i32, i32]),
            "oracle_keys": (None, [i32, dbl, i64, dp, u32p]),
            "oracle_sort": (None, [i32, dbl, i64, dp, u32p]),
            "oracle_deposit": (None, [i32, dbl, i64, dp, dbl, dp]),
            "oracle_solve_fft": (dbl, [i32, dbl, dp, dp]),
            "oracle_solve_dft": (dbl, [i32, dbl, dp, dp]),
            "oracle_field_energy": (None, [i32, dbl, dp, dp, dp]),
            "oracle_gather": (None, [i32, dbl, i64, dp, dp, dp]),
            "oracle_push": (None, [dbl, i64, dp, dp, dbl, dbl]),
            "oracle_wrap": (dbl, [dbl, dbl]),
            "oracle_run": (None, [i32, dbl, dbl, i64, dp, i32, dp, dp, u32p]),
            "oracle_half_kick": (None, [i32, dbl, dbl, i64, dp]),
            "oracle_laplacian_fd": (None, [i32, dbl, dp, dp]),
            "oracle_ssor": (None, [i32, dbl, dp, dp, dbl, i32, i32]),
            "oracle_pcg": (i32, [i32, dbl, dp, dp, dbl, i32, dbl, i32, i32, i32, dp]),
            "oracle_gradient_central": (None, [i32, dbl, dp, dp]),
            "oracle_solve_pcg": (i32, [i32, dbl, dp, dp, dp, dbl, dbl, i32, i32, i32, dp]),
            "oracle_run_pcg": (None, [i32, dbl, dbl, i64, dp, i32, dp, dp, dp, dbl, dbl, i32, i32,
                                      i32, C.POINTER(C.c_int32)]),
            "oracle_half_kick_pcg": (None, [i32, dbl, dbl, i64, dp, dp, dbl, dbl, i32, i32, i32]),
            "oracle_boris_coeffs": (None, [dbl, dp, dp, dp]),
            "oracle_fem_element_stiffness": (None, [dbl, dp]),
            "oracle_fem_apply": (None, [i32, dbl, dp, dp]),
            "oracle_fem_cg": (i32, [i32, dbl, dp, dp, dbl, i32, dp]),
            "oracle_solve_fem": (i32, [i32, dbl, dp, dp, dp, dbl, i32, dp]),
            "oracle_half_kick_fem": (None, [i32, dbl, dbl, i64, dp, dp, dbl, i32]),
            "oracle_run_fem": (None, [i32, dbl, dbl, i64, dp, i32, dp, dp, dp, dbl, i32, C.POINTER(C.c_int32)]),
            "oracle_push_ext": (None, [dbl, i64, dp, dp, dbl, dp, dp]),
            "oracle_run_ext": (None, [i32, dbl, dbl, i64, dp, i32, dp, dp, dp, dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _dp(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _up(a):
    if a is None:
        return None
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def set_threads(t: int) -> None:
    """1 = serial parity mode (default); T > 1 = OpenMP-deterministic mode (SURVEY c.5)."""
    lib().oracle_set_threads(int(t))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


class threads:
    """with threads(T): ... runs the oracle in the OpenMP-deterministic mode, then restores."""

    def __init__(self, t: int):
        self.t = t

    def __enter__(self):
        self.old = get_threads()
        set_threads(self.t)
        return self

    def __exit__(self, *a):
        set_threads(self.old)


def philox(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_up(c), _up(k), _up(out))
    return out


def uniforms(seed: int, j: int) -> np.ndarray:
    u = np.zeros(8)
    lib().oracle_uniforms(seed, j, _dp(u))
    return u


def sample_landau(np_: int, k: float, L: float, alpha: float, seed: int) -> np.ndarray:
    xv = np.zeros((6, np_))
    lib().oracle_sample_landau(np_, k, L, alpha, seed, _dp(xv))
    return xv


def cell_index(x: float, inv_h: float, n: int) -> int:
    return lib().oracle_cell_index(x, inv_h, n)


def morton_key(ix: int, iy: int, iz: int, n: int) -> int:
    return lib().oracle_morton_key(ix, iy, iz, n)


def keys(n: int, L: float, xv: np.ndarray) -> np.ndarray:
    out = np.zeros(xv.shape[1], dtype=np.uint32)
    lib().oracle_keys(n, L, xv.shape[1], _dp(xv), _up(out))
    return out


def sort(n: int, L: float, xv: np.ndarray):
    """Stable sort by cell key, in place on a copy; returns (xv_sorted, perm)."""
    xs = np.ascontiguousarray(xv, dtype=np.float64).copy()
    perm = np.zeros(xs.shape[1], dtype=np.uint32)
    lib().oracle_sort(n, L, xs.shape[1], _dp(xs), _up(perm))
    return xs, perm


def deposit(n: int, L: float, xv: np.ndarray, q: float) -> np.ndarray:
    xv = np.ascontiguousarray(xv, dtype=np.float64)
    rho = np.zeros((n, n, n))
    lib().oracle_deposit(n, L, xv.shape[1], _dp(xv), q, _dp(rho))
    return rho


def solve_fft(n: int, L: float, rho: np.ndarray):
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    E = np.zeros((3, n, n, n))
    imag = lib().oracle_solve_fft(n, L, _dp(rho), _dp(E))
    return E, imag


def solve_dft(n: int, L: float, rho: np.ndarray):
    assert n <= 16
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    E = np.zeros((3, n, n, n))
    imag = lib().oracle_solve_dft(n, L, _dp(rho), _dp(E))
    return E, imag


def field_energy(n: int, L: float, E: np.ndarray):
    E = np.ascontiguousarray(E, dtype=np.float64)
    wx, w = C.c_double(), C.c_double()
    lib().oracle_field_energy(n, L, _dp(E), C.byref(wx), C.byref(w))
    return wx.value, w.value


def gather(n: int, L: float, xv: np.ndarray, E: np.ndarray) -> np.ndarray:
    xv = np.ascontiguousarray(xv, dtype=np.float64)
    E = np.ascontiguousarray(E, dtype=np.float64)
    Ep = np.zeros((3, xv.shape[1]))
    lib().oracle_gather(n, L, xv.shape[1], _dp(xv), _dp(E), _dp(Ep))
    return Ep


def push(L: float, xv: np.ndarray, Ep: np.ndarray, qm_dt: float, dt: float) -> np.ndarray:
    out = np.ascontiguousarray(xv, dtype=np.float64).copy()
    Ep = np.ascontiguousarray(Ep, dtype=np.float64)
    lib().oracle_push(L, out.shape[1], _dp(out), _dp(Ep), qm_dt, dt)
    return out


def wrap(x: float, L: float) -> float:
    return lib().oracle_wrap(x, L)


def run(n: int, L: float, dt: float, xv: np.ndarray, nsteps: int, want_perm: bool = False):
    """Canonicalise then run nsteps PIC steps.  Returns (xv, W_x[n], W[n], perm_last)."""
    xs = np.ascontiguousarray(xv, dtype=np.float64).copy()
    ex = np.zeros(max(nsteps, 1))
    tot = np.zeros(max(nsteps, 1))
    perm = np.zeros(xs.shape[1], dtype=np.uint32) if want_perm else None
    lib().oracle_run(n, L, dt, xs.shape[1], _dp(xs), nsteps, _dp(ex), _dp(tot), _up(perm))
    return xs, ex[:nsteps], tot[:nsteps], perm


def half_kick(n: int, L: float, dt: float, xv: np.ndarray) -> np.ndarray:
    out = np.ascontiguousarray(xv, dtype=np.float64).copy()
    lib().oracle_half_kick(n, L, dt, out.shape[1], _dp(out))
    return out


def init_state(n: int, ppc: int, k: float = 0.5, alpha: float = 0.05, seed: int = 1,
               dt: float = 0.05, half_kick_: bool = True, L: float | None = None):
    """Oracle version of pic_init: sample, canonicalise, optional backward half kick."""
    if L is None:
        L = 2.0 * np.pi / k
    np_ = ppc * n ** 3
    xv = sample_landau(np_, k, L, alpha, seed)
    xv, _ = sort(n, L, xv)
    if half_kick_:
        xv = half_kick(n, L, dt, xv)
    return xv


# ------------------------------------------------ FD-PCG solve (BJ config 5) ----
# P:179-181, P:226 (tol 1e-4), P:260 (SSOR: 4 inner, 2 outer, damping pi/2; warm start).
PCG_DEFAULTS = dict(tol=1e-4, omega=np.pi / 2, inner=4, outer=2, maxit=1000)


def laplacian_fd(n: int, L: float, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros((n, n, n))
    lib().oracle_laplacian_fd(n, L, _dp(x), _dp(y))
    return y


def ssor(n: int, L: float, r: np.ndarray, omega=np.pi / 2, inner=4, outer=2) -> np.ndarray:
    r = np.ascontiguousarray(r, dtype=np.float64)
    z = np.zeros((n, n, n))
    lib().oracle_ssor(n, L, _dp(r), _dp(z), omega, inner, outer)
    return z


def pcg(n: int, L: float, b: np.ndarray, x0=None, tol=1e-4, precond=1, omega=np.pi / 2, inner=4,
        outer=2, maxit=1000):
    """Returns (x, iterations (-1: not converged), relative residual)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros((n, n, n)) if x0 is None else np.ascontiguousarray(x0, dtype=np.float64).copy()
    rel = C.c_double()
    it = lib().oracle_pcg(n, L, _dp(b), _dp(x), tol, precond, omega, inner, outer, maxit, C.byref(rel))
    return x, it, rel.value


def gradient_central(n: int, L: float, phi: np.ndarray) -> np.ndarray:
    phi = np.ascontiguousarray(phi, dtype=np.float64)
    E = np.zeros((3, n, n, n))
    lib().oracle_gradient_central(n, L, _dp(phi), _dp(E))
    return E


def solve_pcg(n: int, L: float, rho: np.ndarray, phi0=None, tol=1e-4, omega=np.pi / 2, inner=4,
              outer=2, maxit=1000):
    """Returns (E, phi, iterations, relative residual)."""
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    phi = np.zeros((n, n, n)) if phi0 is None else np.ascontiguousarray(phi0, dtype=np.float64).copy()
    E = np.zeros((3, n, n, n))
    rel = C.c_double()
    it = lib().oracle_solve_pcg(n, L, _dp(rho), _dp(phi), _dp(E), tol, omega, inner, outer, maxit,
                                C.byref(rel))
    return E, phi, it, rel.value


def run_pcg(n: int, L: float, dt: float, xv: np.ndarray, nsteps: int, phi0=None, tol=1e-4,
            omega=np.pi / 2, inner=4, outer=2, maxit=1000):
    """oracle_run with the PCG solve.  Returns (xv, W_x[n], W[n], phi, iterations[n])."""
    xs = np.ascontiguousarray(xv, dtype=np.float64).copy()
    ex = np.zeros(max(nsteps, 1))
    tot = np.zeros(max(nsteps, 1))
    phi = np.zeros((n, n, n)) if phi0 is None else np.ascontiguousarray(phi0, dtype=np.float64).copy()
    its = np.zeros(max(nsteps, 1), dtype=np.int32)
    lib().oracle_run_pcg(n, L, dt, xs.shape[1], _dp(xs), nsteps, _dp(ex), _dp(tot), _dp(phi), tol, omega,
                         inner, outer, maxit, its.ctypes.data_as(C.POINTER(C.c_int32)))
    return xs, ex[:nsteps], tot[:nsteps], phi, its[:nsteps]


def init_state_pcg(n: int, ppc: int, k: float = 0.5, alpha: float = 0.05, seed: int = 1,
                   dt: float = 0.05, L: float | None = None, tol=1e-4, omega=np.pi / 2, inner=4,
                   outer=2, maxit=1000):
    """pic_init with the PCG solver: sample, canonicalise, half kick with the PCG field
    (phi from 0).  Returns (xv, phi) -- phi is the warm start of the first step."""
    if L is None:
        L = 2.0 * np.pi / k
    np_ = ppc * n ** 3
    xv = sample_landau(np_, k, L, alpha, seed)
    xv, _ = sort(n, L, xv)
    phi = np.zeros((n, n, n))
    lib().oracle_half_kick_pcg(n, L, dt, xv.shape[1], _dp(xv), _dp(phi), tol, omega, inner, outer, maxit)
    return xv, phi


# ------------------------------- external fields, Boris push ----
def _vec3(v):
    return np.ascontiguousarray(np.zeros(3) if v is None else v, dtype=np.float64)


def boris_coeffs(dt: float, b_ext):
    t, s = np.zeros(3), np.zeros(3)
    lib().oracle_boris_coeffs(dt, _dp(_vec3(b_ext)), _dp(t), _dp(s))
    return t, s


def push_ext(L: float, xv: np.ndarray, Ep: np.ndarray, dt: float, b_ext=None, e_ext=None) -> np.ndarray:
    out = np.ascontiguousarray(xv, dtype=np.float64).copy()
    Ep = np.ascontiguousarray(Ep, dtype=np.float64)
    b, e = _vec3(b_ext), _vec3(e_ext)
    lib().oracle_push_ext(L, out.shape[1], _dp(out), _dp(Ep), dt, _dp(b), _dp(e))
    return out


def run_ext(n: int, L: float, dt: float, xv: np.ndarray, nsteps: int, b_ext=None, e_ext=None):
    """oracle.run with uniform external fields.  Returns (xv, W_x[n], W[n])."""
    xs = np.ascontiguousarray(xv, dtype=np.float64).copy()
    ex = np.zeros(max(nsteps, 1))
    tot = np.zeros(max(nsteps, 1))
    b, e = _vec3(b_ext), _vec3(e_ext)
    lib().oracle_run_ext(n, L, dt, xs.shape[1], _dp(xs), nsteps, _dp(ex), _dp(tot), _dp(b), _dp(e))
    return xs, ex[:nsteps], tot[:nsteps]


# ---------------------------------- matrix-free Q1 FEM solve ----
def fem_element_stiffness(h: float) -> np.ndarray:
    Ae = np.zeros((8, 8))
    lib().oracle_fem_element_stiffness(h, _dp(Ae))
    return Ae


def fem_apply(n: int, L: float, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros((n, n, n))
    lib().oracle_fem_apply(n, L, _dp(x), _dp(y))
    return y


def fem_cg(n: int, L: float, b: np.ndarray, x0=None, tol=1e-4, maxit=5000):
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros((n, n, n)) if x0 is None else np.ascontiguousarray(x0, dtype=np.float64).copy()
    rel = C.c_double()
    it = lib().oracle_fem_cg(n, L, _dp(b), _dp(x), tol, maxit, C.byref(rel))
    return x, it, rel.value


def solve_fem(n: int, L: float, rho: np.ndarray, phi0=None, tol=1e-4, maxit=5000):
    """Returns (E, phi, iterations, relative residual)."""
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    phi = np.zeros((n, n, n)) if phi0 is None else np.ascontiguousarray(phi0, dtype=np.float64).copy()
    E = np.zeros((3, n, n, n))
    rel = C.c_double()
    it = lib().oracle_solve_fem(n, L, _dp(rho), _dp(phi), _dp(E), tol, maxit, C.byref(rel))
    return E, phi, it, rel.value


def run_fem(n: int, L: float, dt: float, xv: np.ndarray, nsteps: int, phi0=None, tol=1e-4, maxit=5000):
    """oracle_run with the FEM solve.  Returns (xv, W_x[n], W[n], phi, iterations[n])."""
    xs = np.ascontiguousarray(xv, dtype=np.float64).copy()
    ex = np.zeros(max(nsteps, 1))
    tot = np.zeros(max(nsteps, 1))
    phi = np.zeros((n, n, n)) if phi0 is None else np.ascontiguousarray(phi0, dtype=np.float64).copy()
    its = np.zeros(max(nsteps, 1), dtype=np.int32)
    lib().oracle_run_fem(n, L, dt, xs.shape[1], _dp(xs), nsteps, _dp(ex), _dp(tot), _dp(phi), tol, maxit,
                         its.ctypes.data_as(C.POINTER(C.c_int32)))
    return xs, ex[:nsteps], tot[:nsteps], phi, its[:nsteps]


def init_state_fem(n: int, ppc: int, k: float = 0.5, alpha: float = 0.05, seed: int = 1,
                   dt: float = 0.05, L: float | None = None, tol=1e-4, maxit=5000):
    """pic_init with the FEM solver: sample, canonicalise, half kick with the FEM field."""
    if L is None:
        L = 2.0 * np.pi / k
    xv = sample_landau(ppc * n ** 3, k, L, alpha, seed)
    xv, _ = sort(n, L, xv)
    phi = np.zeros((n, n, n))
    lib().oracle_half_kick_fem(n, L, dt, xv.shape[1], _dp(xv), _dp(phi), tol, maxit)
    return xv, phi
