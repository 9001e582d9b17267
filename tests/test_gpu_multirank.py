"""Multi-GPU z-slab decomposition against the single-domain oracle:
runs tests/mp_worker.py under torchrun on 2 (and 4, 8 when present) GPUs, with the
peer-memory transport (the default; the worker asserts it is the one in use) and
with the NCCL transport (PIC_P2P=0)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch

    return torch.cuda.device_count()


@pytest.mark.parametrize("transport", ["peer", "nccl"])
@pytest.mark.parametrize("world,n", [(2, 32), (4, 32), (8, 64)])
def test_slab_decomposition_matches_oracle(world, n, transport):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, MP_EXPECT_TRANSPORT=transport)
    if transport == "nccl":
        env["PIC_P2P"] = "0"
    else:
        env.pop("PIC_P2P", None)
    port = 29600 + 10 * world + (transport == "nccl")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mp_worker.py"), str(n), "8", "20"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MP OK" in r.stdout and f"transport={transport}" in r.stdout


@pytest.mark.parametrize("solver", ["pcg", "fem"])
@pytest.mark.parametrize("world,n", [(2, 32), (4, 32)])
def test_slab_decomposition_cg_solvers_match_oracle(world, n, solver):
    """The FD-PCG (BJ config 5) and Q1 FEM solvers on z-slabs: the stencils read the
    neighbour slabs' planes over NVLink (peer transport), the dot products are
    all-reduced; vs the single-domain oracle_run_pcg / oracle_run_fem."""
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, MP_EXPECT_TRANSPORT="peer", MP_SOLVER=solver)
    env.pop("PIC_P2P", None)
    port = 29650 + 10 * world + (solver == "fem")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mp_worker.py"), str(n), "8", "20"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MP OK" in r.stdout and f"solver={solver}" in r.stdout


@pytest.mark.parametrize("world,n,pgrid,pulls", [(2, 32, "2x1", "ce"), (4, 32, "2x2", "ce"), (4, 32, "4x1", "ce"),
                                                (4, 32, "2x2", "nccl"), (8, 64, "2x4", "ce"), (8, 64, "4x2", "ce")])
def test_pencil_decomposition_matches_oracle(world, n, pgrid, pulls):
    """Pencils over (y, z) (BJ config 4): particles and the real-space grid on
    Py x Pz domains (ghost row/plane folds and halos over NCCL, migration to the face and
    diagonal neighbours), the FFT on z-slabs after a y-group exchange (copy-engine pulls over
    the IPC mapping, or with pulls="nccl" the NCCL all-to-alls); vs the single-domain oracle
    (W_x 1e-10 every step, x, v 1e-12 after 20 steps) and the library sampler on the pencils
    vs the oracle's."""
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, MP_EXPECT_TRANSPORT="nccl", MP_PGRID=pgrid)
    env.pop("PIC_P2P", None)
    if pulls == "nccl":
        env.update(PIC_PENCIL_PULL="0", PIC_XPOSE_PULL="0")
    port = 29700 + 10 * world + int(pgrid[0]) + (5 if pulls == "nccl" else 0)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mp_worker.py"), str(n), "8", "20"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MP OK" in r.stdout and f"pgrid={pgrid}" in r.stdout


@pytest.mark.parametrize("world", [2, 4])
def test_decomposed_pif_matches_oracle(world):
    """The decomposed PIF (SURVEY §8(f) NEXT-2 on P ranks): particle shares on
    P GPUs, the selected modes all-reduced; vs oracle/nufft.py on the whole particle set (E
    1e-10, energies 1e-10, type 1 1e-11, 3 steps of the time loop W_x 1e-10, x, v 1e-12)."""
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    port = 29800 + world
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mp_pif_worker.py"), "16", "2", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MP PIF OK" in r.stdout
