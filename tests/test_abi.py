"""CPU-side checks of the C ABI library: it loads, exports every symbol
include/pic.h and include/pif.h declare, and its host-only entry points (parameter validation,
workspace sizing) behave as documented.  No compute call needs a GPU here."""
import os
import re

import pytest

import paper_2605_05469_b200 as pkg
from paper_2605_05469_b200 import _binding as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = "".join(open(os.path.join(ROOT, "include", h)).read() for h in ("pic.h", "pif.h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pic_[a-z_]+)\s*\(", src)))


def test_header_declares_and_library_exports_every_symbol():
    pkg.build_lib()
    L = pkg.lib()
    names = _declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(L, name), name
        assert name in B.SYMBOLS, f"binding lacks {name}"


def test_defaults_follow_the_paper():
    p = B.default_params()
    assert (p.n, p.ppc, p.k, p.alpha, p.dt, p.half_kick) == (16, 8, 0.5, 0.05, 0.05, 1)
    assert tuple(p.pgrid) == (1, 1) and p.length == 0.0


@pytest.mark.parametrize("bad", [
    dict(n=12), dict(n=8), dict(n=2048), dict(ppc=0), dict(alpha=1.0), dict(alpha=-0.1),
    dict(k=0.0), dict(dt=0.0), dict(length=5.0), dict(n=1024, ppc=8),
])
def test_invalid_parameters_rejected(bad):
    p = B.default_params(**bad)
    with pytest.raises(B.PicError) as e:
        B.workspace_bytes(p)
    assert e.value.status == B.PIC_EINVAL


def test_multi_rank_geometry():
    """z-slabs: rank r owns planes [r N/P, (r+1) N/P); Py Pz = P; P in
    {1, 2, 4, 8}; the FFT's slabs need >= 4 planes; pencils run the FFT solver only."""
    for P in (1, 2, 4, 8):
        p = B.default_params(n=64, pgrid=(1, P))
        zs = [B.slab(p, r, P) for r in range(P)]
        assert [z[0] for z in zs] == [r * 64 // P for r in range(P)]
        assert all(z[1] == 64 // P for z in zs)
        cap = zs[0][2]
        assert cap >= 8 * 64 ** 3 // P
        assert B.workspace_bytes(p, 0, P) > 48 * cap
    with pytest.raises(B.PicError) as e:
        B.workspace_bytes(B.default_params(n=64, pgrid=(1, 1)), rank=0, nranks=2)
    assert e.value.status == B.PIC_EINVAL
    with pytest.raises(B.PicError) as e:
        B.workspace_bytes(B.default_params(n=64, pgrid=(2, 2), solver=1), rank=0, nranks=4)
    assert e.value.status == B.PIC_EUNSUPPORTED
    with pytest.raises(B.PicError) as e:       # pencil rows: n / Py >= 8
        B.workspace_bytes(B.default_params(n=16, pgrid=(4, 1)), rank=0, nranks=4)
    assert e.value.status == B.PIC_EINVAL
    with pytest.raises(B.PicError) as e:
        B.workspace_bytes(B.default_params(n=16, pgrid=(1, 8)), rank=0, nranks=8)
    assert e.value.status == B.PIC_EINVAL
    with pytest.raises(B.PicError) as e:
        B.workspace_bytes(B.default_params(n=64, pgrid=(1, 3)), rank=0, nranks=3)
    assert e.value.status == B.PIC_EINVAL


def test_workspace_bytes_model():
    """Workspace = 2 x 48 B/particle state + 10 B/particle key/rank/perm + cell arrays + grids."""
    p = B.default_params(n=512, ppc=8)
    b = B.workspace_bytes(p)
    np_ = 8 * 512 ** 3
    assert 106 * np_ <= b <= 106 * np_ + 12 * 2 ** 30
    assert b < 170 * 2 ** 30     # fits one B200 (183 GB)
    # the north-star run, 1024^3 x 8 ppc on 8 z-slabs: state (1.1 x nominal slab),
    # neighbour-sized migration segments and slab grids fit every rank's B200
    p = B.default_params(n=1024, ppc=8, pgrid=(1, 8))
    np_r = 8 * 1024 ** 3 // 8
    for r in range(8):
        b = B.workspace_bytes(p, r, 8)
        assert 106 * np_r < b < 160 * 2 ** 30
    p = B.default_params(n=16, ppc=8, length=8 * 3.141592653589793)   # kL/2pi = 2
    assert B.workspace_bytes(p) > 0


def test_stage_names():
    L = pkg.lib()
    for i, s in enumerate(B.STAGES):
        assert L.pic_stage_name(i).decode() == s
    assert L.pic_stage_name(len(B.STAGES)) is None


def test_pcg_defaults_and_validation():
    """BJ config 5 defaults (P:226 tol 1e-4; P:260 SSOR pi/2, 4 inner, 2 outer); invalid
    PCG settings and non-finite external fields are PIC_EINVAL; the PCG workspace adds
    six colour-split fields (x, r, z, two p, q) of 8 B/node."""
    import math

    p = B.default_params()
    assert p.solver == B.PIC_SOLVER_FFT
    assert (p.pcg_inner, p.pcg_outer, p.pcg_maxit) == (4, 2, 10000)
    assert p.pcg_tol == 1e-4 and p.pcg_omega == math.pi / 2
    assert tuple(p.b_ext) == (0.0, 0.0, 0.0) and tuple(p.e_ext) == (0.0, 0.0, 0.0)
    for bad in (dict(pcg_tol=0.0), dict(pcg_omega=2.0), dict(pcg_omega=0.0), dict(pcg_inner=0),
                dict(pcg_outer=0), dict(pcg_maxit=0), dict(solver=3)):
        q = B.default_params(**{"solver": B.PIC_SOLVER_PCG, **bad})
        with pytest.raises(B.PicError) as e:
            B.workspace_bytes(q)
        assert e.value.status == B.PIC_EINVAL, bad
    for bad in (dict(b_ext=(0.0, float("nan"), 0.0)), dict(e_ext=(float("inf"), 0.0, 0.0))):
        with pytest.raises(B.PicError) as e:
            B.workspace_bytes(B.default_params(**bad))
        assert e.value.status == B.PIC_EINVAL
    n = 64
    fft = B.workspace_bytes(B.default_params(n=n))
    pcg = B.workspace_bytes(B.default_params(n=n, solver=B.PIC_SOLVER_PCG))
    assert 6 * 8 * n ** 3 <= pcg - fft <= 6 * 8 * n ** 3 + 8 * 4096


def test_pif_parameter_validation_without_gpu():
    """include/pif.h: invalid N (odd, < 8, > 1024), L <= 0 or eps outside [1e-14, 1) are
    rejected before any CUDA call."""
    import ctypes as C

    b = C.c_size_t()
    for n, L, eps in [(7, 1.0, 1e-4), (4, 1.0, 1e-4), (2048, 1.0, 1e-4), (16, 0.0, 1e-4), (16, 1.0, 1.5),
                      (16, 1.0, 1e-20)]:
        assert pkg.lib().pic_pif_workspace_bytes(n, L, eps, 0, C.byref(b)) == B.PIC_EINVAL
    assert pkg.lib().pic_pif_workspace_bytes(16, 1.0, 1e-4, -1, C.byref(b)) == B.PIC_EINVAL
    assert pkg.lib().pic_nufft_type1(None, 1, None, None, None) == B.PIC_EINVAL
    assert pkg.lib().pic_pif_solve(None, 1, None, None, None, None) == B.PIC_EINVAL
    assert B.PIF_STAGES == ["spread", "fft", "modes", "fill", "interp", "push", "bin"]


def test_owner_ranks_partition_by_slab():
    """pic_owner_ranks: rank = the slab of the cell plane floor(z N / L)
    clamped to N - 1 (D#5), restated here; z = L is rejected."""
    import numpy as np
    from paper_2605_05469_b200 import owner_ranks
    from paper_2605_05469_b200._binding import PicError

    n, L = 32, 4 * np.pi
    rng = np.random.default_rng(5)
    xv = rng.random((6, 10000)) * L
    xv[2, :4] = [0.0, np.nextafter(L, 0), 15.999999 * L / n, 16 * L / n]
    for world in (1, 2, 4, 8):
        own = owner_ranks(xv, n, L, world)
        iz = np.minimum(np.floor(xv[2] * (n / L)).astype(np.int64), n - 1)
        assert np.array_equal(own, iz // (n // world))
    assert list(owner_ranks(xv, n, L, 2)[:4]) == [0, 1, 0, 1]
    bad = xv.copy()
    bad[2, 7] = L
    with pytest.raises(PicError):
        owner_ranks(bad, n, L, 2)


def test_pif_sizes_rejected_on_the_host():
    """include/pif.h: the fine grid M = 2N goes through the library's own power-of-two FFT
    passes, so N must be a power of two in [8, 512] (host-only check, no GPU)."""
    import ctypes as C
    import numpy as np

    for n, ok in ((8, True), (512, True), (12, False), (1024, False), (4, False)):
        b = C.c_size_t()
        st = B.lib().pic_pif_workspace_bytes(n, 4 * np.pi, 1e-4, 0, C.byref(b))
        assert (st == 0) == ok, (n, st)


@pytest.mark.parametrize("Py,Pz", [(2, 1), (2, 2), (2, 4), (4, 2), (8, 1)])
def test_pencil_domains_partition_the_box(Py, Pz):
    """Pencils (BJ config 4): rank r = pz Py + py owns rows [py N/Py, +N/Py) and
    planes [pz N/Pz, +N/Pz); the domains tile the box; pic_owner_ranks follows the same rule
    (restated here); every rank's workspace fits a B200 at 1024^3 x 8 ppc on 8 ranks."""
    import numpy as np
    from paper_2605_05469_b200 import owner_ranks

    n, P = 64, Py * Pz
    p = B.default_params(n=n, pgrid=(Py, Pz))
    cover = np.zeros((n, n), dtype=int)
    for r in range(P):
        y0, ny, z0, nz, cap = B.domain(p, r, P)
        assert (y0, ny, z0, nz) == ((r % Py) * n // Py, n // Py, (r // Py) * n // Pz, n // Pz)
        cover[z0:z0 + nz, y0:y0 + ny] += 1
        assert cap >= 8 * n ** 3 // P
    assert np.all(cover == 1)
    L = 4 * np.pi
    rng = np.random.default_rng(7)
    xv = rng.random((6, 5000)) * L
    own = owner_ranks(xv, n, L, P, (Py, Pz))
    iy = np.minimum(np.floor(xv[1] * (n / L)).astype(int), n - 1)
    iz = np.minimum(np.floor(xv[2] * (n / L)).astype(int), n - 1)
    assert np.array_equal(own, (iz // (n // Pz)) * Py + iy // (n // Py))
    if P == 8:
        big = B.default_params(n=1024, ppc=8, pgrid=(Py, Pz))
        for r in range(P):
            assert B.workspace_bytes(big, r, P) < 170 * 2 ** 30
