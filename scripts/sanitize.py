"""A small PIC run for compute-sanitizer (memcheck / racecheck / synccheck): 16^3 x 8 ppc,
pic_init with the half kick, 3 steps, the particle and grid exports; a PIF solve at 8^3 modes.
P > 1: run under torchrun (every rank the same, NCCL), pgrid from argv[1] ("1x2" / "2x1")."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_05469_b200 import PifSolver, Simulation, nccl_unique_id  # noqa: E402

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
ncid = None
if world > 1:
    import torch.distributed as dist

    dist.init_process_group("gloo")
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ncid = obj[0]
pg = sys.argv[1] if len(sys.argv) > 1 else f"1x{world}"
pgrid = tuple(int(v) for v in pg.split("x"))
sim = Simulation(n=16, ppc=8, seed=3, rank=rank, nranks=world, nccl_id=ncid, pgrid=pgrid)
ex = sim.step(3)
xv = sim.get_particles()
rho = sim.get_grid(0)
E = sim.get_grid(1)
k, p = sim.keys_perm()
sim.close()
if world == 1:
    x = torch.rand((3, 4096), dtype=torch.float64, device="cuda") * (4 * np.pi)
    q = torch.full((4096,), -1.0, dtype=torch.float64, device="cuda")
    P = PifSolver(8, 4 * np.pi, 1e-4, np_max=4096)
    P.solve(x, q)
torch.cuda.synchronize()
print(f"SANITIZE RUN OK rank {rank}/{world} pgrid {pgrid} W_x {ex.tolist()}", flush=True)
if world > 1:
    dist.destroy_process_group()
