"""Time the PIF solve (include/pif.h) at N^3 modes x ppc particles per cell, particles in
cell order (x fastest) with uniform jitter -- the order a PIC code keeps them in."""
import sys
import time

import numpy as np
import torch

from paper_2605_05469_b200 import PifSolver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ppc = int(sys.argv[2]) if len(sys.argv) > 2 else 8
order = sys.argv[3] if len(sys.argv) > 3 else "cell"
L = 4 * np.pi
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(1)
npart = N ** 3 * ppc
h = L / N
x = torch.empty((3, npart), dtype=torch.float64, device="cuda")
cell = torch.arange(npart, device="cuda", dtype=torch.int64) // ppc
if order.startswith("random"):
    cell = cell[torch.randperm(npart, device="cuda", generator=g)]
for d, c in enumerate([cell % N, (cell // N) % N, cell // (N * N)]):
    x[d] = (c.double() + torch.rand(npart, dtype=torch.float64, device="cuda", generator=g)) * h
del cell
q = torch.full((npart,), -L ** 3 / npart, dtype=torch.float64, device="cuda")
P = PifSolver(N, L, 1e-4, np_max=0 if order.endswith('atomic') else npart)
E = torch.empty_like(x)
P.solve(x, q, E)
torch.cuda.synchronize()
P.set_timing(True)
reps = 3
t = time.time()
for _ in range(reps):
    P.solve(x, q, E, energy=False)
torch.cuda.synchronize()
wall = (time.time() - t) / reps
tm = P.timings()
print(f"N={N} ppc={ppc} np={npart} order={order} w,M={P.window()} wall {wall*1e3:.1f} ms/solve "
      f"({npart/wall:.3e} particles/s)", {k: round(v[0] / reps, 2) for k, v in tm.items()}, flush=True)
