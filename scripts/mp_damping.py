"""torchrun: Landau damping on P GPUs (slabs or pencils) at a size one GPU cannot hold -- e.g.
1024^3 x 4 ppc (4.3e9 particles) on 4 GPUs in 2 x 2 pencils: the W_x peak-slope fit
(tests/landau_fit.py, SURVEY c.6) and the ms per step (CUDA events, max over ranks).
Args: n ppc steps t_max [PyxPz].  Writes gpurun_out/mp_damping_<n>_<ppc>_<grid>.json (rank 0)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from landau_fit import dispersion_root, fit_damping_rate  # noqa: E402
from paper_2605_05469_b200 import Simulation, nccl_unique_id  # noqa: E402

n, ppc, steps, tmax = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
pg = tuple(int(v) for v in sys.argv[5].split("x")) if len(sys.argv) > 5 else (1, world)
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dist.init_process_group("nccl")
obj = [nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
sim = Simulation(n=n, ppc=ppc, seed=1, rank=rank, nranks=world, nccl_id=obj[0], pgrid=pg)
sim.step(2)
dist.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(sim.stream)
ex = sim.step(steps)
e1.record(sim.stream)
e1.synchronize()
ms = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device="cuda")
dist.all_reduce(ms, op=dist.ReduceOp.MAX)
if rank == 0:
    w = dispersion_root(0.5)
    t = (2 + np.arange(steps)) * 0.05
    slope, npk, tp = fit_damping_rate(t, ex, t_max=tmax)
    sp = float(np.mean(np.diff(tp)))
    r = {"n": n, "ppc": ppc, "particles": ppc * n ** 3, "gpus": world, "pgrid": list(pg), "steps": steps,
         "ms_per_step": float(ms.item()), "pushes_per_s": ppc * n ** 3 / (float(ms.item()) / 1e3),
         "slope": slope, "slope_target": 2 * w.imag, "slope_rel_err": abs(slope - 2 * w.imag) / abs(2 * w.imag),
         "peaks": npk, "peak_spacing": sp, "spacing_rel_err": abs(sp - np.pi / w.real) / (np.pi / w.real),
         "W_x": [float(v) for v in ex]}
    print(json.dumps({k: v for k, v in r.items() if k != "W_x"}), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(r, open(os.path.join(ROOT, "gpurun_out", f"mp_damping_{n}_{ppc}_{pg[0]}x{pg[1]}.json"), "w"))
sim.close()
dist.barrier()
dist.destroy_process_group()
