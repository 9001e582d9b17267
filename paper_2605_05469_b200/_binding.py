"""Thin ctypes binding of libpic.so (include/pic.h): argument marshalling only.

Every step of the PIC path runs in the CUDA kernels behind the C ABI; this
module converts Python/numpy/torch arguments to pointers and status codes to
exceptions.  PyTorch supplies the device workspace and the stream.  There is no
fallback: if libpic.so is missing or fails to load, importing the product path
raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpic.so")

PIC_OK, PIC_EINVAL, PIC_ENOMEM, PIC_ECUDA, PIC_ENCCL = 0, -1, -2, -3, -4
PIC_ENONFINITE, PIC_EOVERFLOW, PIC_EPOISONED, PIC_EUNSUPPORTED = -5, -6, -7, -8
PIC_ENONCONV = -9
STATUS_NAMES = {0: "PIC_OK", -1: "PIC_EINVAL", -2: "PIC_ENOMEM", -3: "PIC_ECUDA", -4: "PIC_ENCCL",
                -5: "PIC_ENONFINITE", -6: "PIC_EOVERFLOW", -7: "PIC_EPOISONED",
                -8: "PIC_EUNSUPPORTED", -9: "PIC_ENONCONV"}
PIC_SOLVER_FFT, PIC_SOLVER_PCG, PIC_SOLVER_FEM = 0, 1, 2
SOLVERS = {"fft": PIC_SOLVER_FFT, "pcg": PIC_SOLVER_PCG, "fem": PIC_SOLVER_FEM}

STAGES = ["fft_x_fwd", "fft_y_fwd", "fft_z_mul", "fft_y_inv", "fft_x_inv", "energy", "clear",
          "push_key", "scan", "place", "reorder_deposit", "exchange", "xpose", "pcg_ssor", "pcg_cg",
          "pcg_field"]
PIC_NSTAGES = len(STAGES)


class pic_params(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("ppc", C.c_int32),
        ("k", C.c_double),
        ("length", C.c_double),
        ("alpha", C.c_double),
        ("dt", C.c_double),
        ("seed", C.c_uint64),
        ("half_kick", C.c_int32),
        ("pgrid", C.c_int32 * 2),
        ("solver", C.c_int32),
        ("pcg_inner", C.c_int32),
        ("pcg_outer", C.c_int32),
        ("pcg_maxit", C.c_int32),
        ("pcg_tol", C.c_double),
        ("pcg_omega", C.c_double),
        ("b_ext", C.c_double * 3),
        ("e_ext", C.c_double * 3),
    ]


class PicError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


# Every symbol include/pic.h declares, with (restype, argtypes).
_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_i64p = C.POINTER(C.c_int64)
SYMBOLS = {
    "pic_params_default": (C.c_int, [C.POINTER(pic_params)]),
    "pic_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "pic_slab": (C.c_int, [C.POINTER(pic_params), C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                           C.POINTER(C.c_int32), _i64p]),
    "pic_domain": (C.c_int, [C.POINTER(pic_params), C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                             C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32), _i64p]),
    "pic_owner_ranks": (C.c_int, [C.POINTER(pic_params), C.c_int32, _dp, C.c_int64, C.POINTER(C.c_int32)]),
    "pic_gather_particles": (C.c_int, [_vp, _dp, C.c_int64, _i64p]),
    "pic_migrated": (C.c_int, [_vp, _i64p]),
    "pic_peer_transport": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "pic_workspace_bytes": (C.c_int, [C.POINTER(pic_params), C.c_int32, C.c_int32, C.POINTER(C.c_size_t)]),
    "pic_init": (C.c_int, [C.POINTER(pic_params), C.c_int32, C.c_int32, _vp, _vp, C.c_size_t, _vp,
                           C.POINTER(_vp)]),
    "pic_step": (C.c_int, [_vp, C.c_int32, _dp]),
    "pic_field_energy": (C.c_int, [_vp, _dp, _dp]),
    "pic_free": (None, [_vp]),
    "pic_last_error": (C.c_char_p, [_vp]),
    "pic_num_particles": (C.c_int, [_vp, _i64p]),
    "pic_get_particles": (C.c_int, [_vp, _dp, C.c_int64]),
    "pic_set_particles": (C.c_int, [_vp, _dp, C.c_int64]),
    "pic_get_grid": (C.c_int, [_vp, C.c_int32, _dp]),
    "pic_solve_injected": (C.c_int, [_vp, _dp, _dp, _dp, _dp]),
    "pic_push_injected": (C.c_int, [_vp, _dp]),
    "pic_get_keys_perm": (C.c_int, [_vp, _u32p, _u32p]),
    "pic_set_timing": (C.c_int, [_vp, C.c_int32]),
    "pic_get_timings": (C.c_int, [_vp, _dp, _i64p]),
    "pic_reset_timings": (C.c_int, [_vp]),
    "pic_stage_name": (C.c_char_p, [C.c_int32]),
    "pic_launches_per_step": (C.c_int, [_vp, _i64p]),
    "pic_diag_bandwidth": (C.c_int, [_vp, C.c_int32, C.c_int32, _dp, _dp]),
    "pic_pcg_stats": (C.c_int, [_vp, C.POINTER(C.c_int32), _i64p, _i64p, _dp]),
    # include/pif.h
    "pic_pif_workspace_bytes": (C.c_int, [C.c_int32, C.c_double, C.c_double, C.c_int64, C.POINTER(C.c_size_t)]),
    "pic_pif_create": (C.c_int, [C.c_int32, C.c_double, C.c_double, C.c_int64, _vp, C.c_size_t, _vp,
                                 C.POINTER(_vp)]),
    "pic_nufft_type1": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp]),
    "pic_nufft_type2": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp]),
    "pic_pif_solve": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _dp]),
    "pic_pif_step": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp, C.c_double, C.c_double, C.c_int32, _dp]),
    "pic_pif_attach_nccl": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_void_p]),
    "pic_pif_set_timing": (C.c_int, [_vp, C.c_int32]),
    "pic_pif_get_timings": (C.c_int, [_vp, _dp, _i64p]),
    "pic_pif_window": (C.c_int, [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "pic_pif_last_error": (C.c_char_p, [_vp]),
    "pic_pif_free": (None, [_vp]),
}

PIF_STAGES = ["spread", "fft", "modes", "fill", "interp", "push", "bin"]

_lib = None


def lib() -> C.CDLL:
    """Load libpic.so (raises if it is missing: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SYMBOLS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st: int, ctx=None):
    if st != PIC_OK:
        msg = lib().pic_last_error(ctx)
        raise PicError(st, msg.decode() if msg else "")


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def default_params(**kw) -> pic_params:
    p = pic_params()
    _check(lib().pic_params_default(C.byref(p)))
    for k, v in kw.items():
        if k == "pgrid":
            p.pgrid[0], p.pgrid[1] = v
        elif k in ("b_ext", "e_ext"):
            arr = getattr(p, k)
            for d in range(3):
                arr[d] = float(v[d])
        else:
            setattr(p, k, v)
    return p


def workspace_bytes(p: pic_params, rank: int = 0, nranks: int = 1) -> int:
    b = C.c_size_t()
    _check(lib().pic_workspace_bytes(C.byref(p), rank, nranks, C.byref(b)))
    return b.value


def nccl_unique_id() -> bytes:
    """128-byte NCCL id (rank 0 creates it, the caller broadcasts it)."""
    buf = (C.c_uint8 * 128)()
    _check(lib().pic_nccl_unique_id(buf))
    return bytes(buf)


def owner_ranks(xv: np.ndarray, n: int, L: float, nranks: int, pgrid=None) -> np.ndarray:
    """Owner rank of every particle of xv[6][np] (or [3][np]) -- pic_owner_ranks; pgrid =
    (Py, Pz), default z-slabs (1, nranks)."""
    xv = np.ascontiguousarray(xv, dtype=np.float64)
    p = default_params(n=n, k=2 * np.pi / L, length=L, pgrid=pgrid or (1, nranks))
    out = np.empty(xv.shape[1], dtype=np.int32)
    _check(lib().pic_owner_ranks(C.byref(p), nranks, _d(xv), xv.shape[1],
                                 out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


def slab_select(xv: np.ndarray, n: int, L: float, rank: int, nranks: int, pgrid=None) -> np.ndarray:
    """The particles of a global state xv[6][np] that rank owns (pic_owner_ranks), in
    their global order -- what each rank passes to set_particles."""
    return np.ascontiguousarray(xv[:, owner_ranks(xv, n, L, nranks, pgrid) == rank])


def domain(p: pic_params, rank: int, nranks: int):
    """(y0, ny, z0, nz, capacity) of a rank's domain (pic_domain)."""
    v = [C.c_int32() for _ in range(4)]
    cap = C.c_int64()
    _check(lib().pic_domain(C.byref(p), rank, nranks, *[C.byref(x) for x in v], C.byref(cap)))
    return tuple(x.value for x in v) + (cap.value,)


def slab(p: pic_params, rank: int, nranks: int):
    """(z0, nz, capacity) of a rank's z-slab."""
    z0, nz, cap = C.c_int32(), C.c_int32(), C.c_int64()
    _check(lib().pic_slab(C.byref(p), rank, nranks, C.byref(z0), C.byref(nz), C.byref(cap)))
    return z0.value, nz.value, cap.value


class Simulation:
    """One rank of the PIC simulation on the current CUDA device.

    ``workspace`` is a torch uint8 CUDA tensor owned by this object; the stream
    is torch's current stream at construction.
    """

    def __init__(self, n=16, ppc=8, k=0.5, alpha=0.05, dt=0.05, seed=1, half_kick=True,
                 length=0.0, device=None, rank=0, nranks=1, nccl_id: bytes | None = None,
                 solver="fft", pgrid=None, **pcg):
        """solver: "fft", "pcg" (BJ config 5) or "fem"; pcg keywords
        pcg_tol, pcg_omega, pcg_inner, pcg_outer, pcg_maxit override P:226 / P:260;
        b_ext=(bx, by, bz) / e_ext=(ex, ey, ez): uniform external fields (Eq. 1, D#32)."""
        import torch

        self.params = default_params(n=n, ppc=ppc, k=k, alpha=alpha, dt=dt, seed=seed,
                                     half_kick=int(bool(half_kick)), length=length,
                                     pgrid=tuple(pgrid) if pgrid else (1, nranks), solver=SOLVERS[solver], **pcg)
        self.solver = solver
        self.rank, self.nranks = rank, nranks
        self.y0, self.ny, self.z0, self.nz, self.capacity = domain(self.params, rank, nranks)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        nbytes = workspace_bytes(self.params, rank, nranks)
        with torch.cuda.device(self.device):
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self.stream = torch.cuda.current_stream(self.device)
        ctx = C.c_void_p()
        idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
        _check(lib().pic_init(C.byref(self.params), rank, nranks, idbuf, C.c_void_p(self.workspace.data_ptr()),
                              nbytes, C.c_void_p(self.stream.cuda_stream), C.byref(ctx)))
        self.ctx = ctx
        self.n = n
        self.L = length if length else 2 * np.pi / k

    @property
    def np(self) -> int:
        """Particles held by this rank now (changes with migration at nranks > 1)."""
        n64 = C.c_int64()
        _check(lib().pic_num_particles(self.ctx, C.byref(n64)), self.ctx)
        return n64.value

    def migrated(self) -> int:
        v = C.c_int64()
        _check(lib().pic_migrated(self.ctx, C.byref(v)), self.ctx)
        return v.value

    def peer_transport(self) -> bool:
        """True when the P > 1 exchanges are peer-memory stores (CUDA IPC over NVLink)."""
        v = C.c_int32()
        _check(lib().pic_peer_transport(self.ctx, C.byref(v)), self.ctx)
        return bool(v.value)

    # -- core --------------------------------------------------------------
    def step(self, nsteps: int = 1) -> np.ndarray:
        ex = np.zeros(max(nsteps, 1))
        _check(lib().pic_step(self.ctx, nsteps, _d(ex)), self.ctx)
        return ex[:nsteps]

    def field_energy(self):
        a, b = C.c_double(), C.c_double()
        _check(lib().pic_field_energy(self.ctx, C.byref(a), C.byref(b)), self.ctx)
        return a.value, b.value

    # -- host buffers ------------------------------------------------------
    def get_particles(self, out: np.ndarray | None = None) -> np.ndarray:
        npl = self.np
        if out is None:
            out = np.zeros((6, npl))
        assert out.shape == (6, npl)
        _check(lib().pic_get_particles(self.ctx, _d(out), npl), self.ctx)
        return out

    def diag_bandwidth(self, mode: int, reps: int = 3):
        """(ms per launch, bytes per launch) of a bandwidth probe (pic_diag_bandwidth)."""
        ms, b = C.c_double(), C.c_double()
        _check(lib().pic_diag_bandwidth(self.ctx, mode, reps, C.byref(ms), C.byref(b)), self.ctx)
        return ms.value, b.value

    def gather_particles(self, out: np.ndarray | None = None):
        """Collective: rank 0 returns every rank's particles in the global canonical order
        (pic_gather_particles); the other ranks return None."""
        tot = C.c_int64()
        _check(lib().pic_gather_particles(self.ctx, None, 0, C.byref(tot)), self.ctx)
        if self.rank == 0:
            if out is None:
                out = np.zeros((6, tot.value))
            assert out.shape == (6, tot.value) and out.flags.c_contiguous
            _check(lib().pic_gather_particles(self.ctx, _d(out), tot.value, None), self.ctx)
            return out
        _check(lib().pic_gather_particles(self.ctx, None, 0, None), self.ctx)
        return None

    def set_particles(self, xv: np.ndarray):
        xv = np.ascontiguousarray(xv, dtype=np.float64)
        assert xv.ndim == 2 and xv.shape[0] == 6
        _check(lib().pic_set_particles(self.ctx, _d(xv), xv.shape[1]), self.ctx)

    def get_grid(self, which: int) -> np.ndarray:
        out = np.zeros((self.nz, self.ny, self.n))
        _check(lib().pic_get_grid(self.ctx, which, _d(out)), self.ctx)
        return out

    def solve_injected(self, rho: np.ndarray):
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        E = np.zeros((3, self.nz, self.ny, self.n))
        a, b = C.c_double(), C.c_double()
        _check(lib().pic_solve_injected(self.ctx, _d(rho), _d(E), C.byref(a), C.byref(b)), self.ctx)
        return E, a.value, b.value

    def push_injected(self, E: np.ndarray):
        E = np.ascontiguousarray(E, dtype=np.float64)
        _check(lib().pic_push_injected(self.ctx, _d(E)), self.ctx)

    def keys_perm(self):
        """Global Morton cell keys of the current state, and the permutation of the
        latest sort (perm[i] = pre-sort index; P > 1: extended index of residents and
        arrivals)."""
        npl = self.np
        k = np.zeros(npl, dtype=np.uint32)
        p = np.zeros(npl, dtype=np.uint32)
        _check(lib().pic_get_keys_perm(self.ctx, k.ctypes.data_as(_u32p), p.ctypes.data_as(_u32p)), self.ctx)
        return k, p

    # -- timing ------------------------------------------------------------
    def set_timing(self, on: bool = True):
        _check(lib().pic_set_timing(self.ctx, int(on)), self.ctx)

    def timings(self):
        ms = np.zeros(PIC_NSTAGES)
        la = np.zeros(PIC_NSTAGES, dtype=np.int64)
        _check(lib().pic_get_timings(self.ctx, _d(ms), la.ctypes.data_as(_i64p)), self.ctx)
        return {STAGES[i]: (ms[i], int(la[i])) for i in range(PIC_NSTAGES)}

    def reset_timings(self):
        _check(lib().pic_reset_timings(self.ctx), self.ctx)

    def pcg_stats(self):
        """(iterations of the latest solve (-1: not converged), total iterations, solves,
        relative residual of the latest solve) of a PCG simulation."""
        it, tot, ns, rel = C.c_int32(), C.c_int64(), C.c_int64(), C.c_double()
        _check(lib().pic_pcg_stats(self.ctx, C.byref(it), C.byref(tot), C.byref(ns), C.byref(rel)), self.ctx)
        return it.value, tot.value, ns.value, rel.value

    def get_phi(self) -> np.ndarray:
        """phi of the latest PCG solve, this rank's slab [nz][N][N]."""
        return self.get_grid(4)

    def launches_per_step(self) -> int:
        v = C.c_int64()
        _check(lib().pic_launches_per_step(self.ctx, C.byref(v)), self.ctx)
        return v.value

    def close(self):
        if getattr(self, "ctx", None):
            lib().pic_free(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _check_pif(st: int, plan=None):
    if st != PIC_OK:
        msg = lib().pic_pif_last_error(plan)
        raise PicError(st, msg.decode() if msg else "")


class PifSolver:
    """Particle-in-Fourier field solve and the type-1 / type-2 NUFFTs (include/pif.h; P:197-221,
    P:423-467) on the current CUDA device.  Arguments are torch float64 CUDA tensors:
    positions x of shape (3, np), weights / charges (np,), spectra complex128 (N, N, N)
    indexed [nz + N/2, ny + N/2, nx + N/2].  The workspace is a torch uint8 tensor owned
    here; the stream is torch's current stream at construction."""

    def __init__(self, n: int, length: float, eps: float = 1e-4, device=None, np_max: int = 0, rank: int = 0,
                 nranks: int = 1, nccl_id: bytes | None = None):
        """np_max > 0 reserves the binned (shared-memory tile) path for up to np_max particles.
        nranks > 1: the decomposed PIF (pic_pif_attach_nccl): each rank passes its own particles,
        the modes are summed over the ranks."""
        import torch

        self.n, self.L, self.eps, self.np_max = n, float(length), float(eps), int(np_max)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        b = C.c_size_t()
        with torch.cuda.device(self.device):
            _check_pif(lib().pic_pif_workspace_bytes(n, self.L, self.eps, self.np_max, C.byref(b)))
            self.workspace = torch.empty(b.value, dtype=torch.uint8, device=self.device)
            self.stream = torch.cuda.current_stream(self.device)
        plan = C.c_void_p()
        _check_pif(lib().pic_pif_create(n, self.L, self.eps, self.np_max, C.c_void_p(self.workspace.data_ptr()),
                                        b.value,
                                        C.c_void_p(self.stream.cuda_stream), C.byref(plan)))
        self.plan = plan
        if nranks > 1:
            idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            _check_pif(lib().pic_pif_attach_nccl(self.plan, rank, nranks, idbuf), self.plan)

    def __del__(self):
        if getattr(self, "plan", None):
            lib().pic_pif_free(self.plan)
            self.plan = None

    def _pos(self, x):
        import torch

        assert x.dtype == torch.float64 and x.is_cuda and x.dim() == 2 and x.shape[0] == 3 and x.is_contiguous()
        return x.shape[1]

    def window(self):
        w, m = C.c_int32(), C.c_int32()
        _check_pif(lib().pic_pif_window(self.plan, C.byref(w), C.byref(m)), self.plan)
        return w.value, m.value

    def type1(self, x, f):
        import torch

        npart = self._pos(x)
        assert f.dtype == torch.float64 and f.is_contiguous() and f.numel() == npart
        out = torch.empty((self.n, self.n, self.n), dtype=torch.complex128, device=x.device)
        _check_pif(lib().pic_nufft_type1(self.plan, npart, C.c_void_p(x.data_ptr()), C.c_void_p(f.data_ptr()),
                                         C.c_void_p(out.data_ptr())), self.plan)
        return out

    def type2(self, fhat, x):
        import torch

        npart = self._pos(x)
        assert fhat.dtype == torch.complex128 and fhat.is_contiguous() and fhat.shape == (self.n,) * 3
        out = torch.empty(npart, dtype=torch.complex128, device=x.device)
        _check_pif(lib().pic_nufft_type2(self.plan, npart, C.c_void_p(x.data_ptr()), C.c_void_p(fhat.data_ptr()),
                                         C.c_void_p(out.data_ptr())), self.plan)
        return out

    def solve(self, x, q, E=None, energy: bool = True):
        """E at the particles (3, np) and, if ``energy``, W = (W_x, W_y, W_z) (synchronises)."""
        import torch

        npart = self._pos(x)
        assert q.dtype == torch.float64 and q.is_contiguous() and q.numel() == npart
        if E is None:
            E = torch.empty((3, npart), dtype=torch.float64, device=x.device)
        W = np.zeros(3)
        _check_pif(lib().pic_pif_solve(self.plan, npart, C.c_void_p(x.data_ptr()), C.c_void_p(q.data_ptr()),
                                       C.c_void_p(E.data_ptr()), _d(W) if energy else None), self.plan)
        return E, (W if energy else None)

    def step(self, x, v, q, nsteps: int = 1, qm: float = -1.0, dt: float = 0.05, E=None, energy: bool = True):
        """The PIF time loop (pic_pif_step): x, v (3, np) updated in place; returns W_x per step
        (synchronises) or None."""
        import torch

        npart = self._pos(x)
        assert v.dtype == torch.float64 and v.is_contiguous() and v.shape == x.shape
        assert q.dtype == torch.float64 and q.is_contiguous() and q.numel() == npart
        if E is None:
            E = torch.empty_like(x)
        ex = np.zeros(max(nsteps, 1))
        _check_pif(lib().pic_pif_step(self.plan, npart, C.c_void_p(x.data_ptr()), C.c_void_p(v.data_ptr()),
                                      C.c_void_p(q.data_ptr()), C.c_void_p(E.data_ptr()), qm, dt, nsteps,
                                      _d(ex) if energy else None), self.plan)
        return ex[:nsteps] if energy else None

    def set_timing(self, enable: bool = True):
        _check_pif(lib().pic_pif_set_timing(self.plan, int(enable)), self.plan)

    def timings(self):
        ms = np.zeros(len(PIF_STAGES))
        la = np.zeros(len(PIF_STAGES), dtype=np.int64)
        _check_pif(lib().pic_pif_get_timings(self.plan, _d(ms), la.ctypes.data_as(_i64p)), self.plan)
        return {k: (float(ms[i]), int(la[i])) for i, k in enumerate(PIF_STAGES)}
