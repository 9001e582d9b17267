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
