import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2605_05469_b200 import Simulation
from pic_inputs import random_grid
n = int(sys.argv[1])
torch.cuda.set_device(0)
sim = Simulation(n=n, ppc=1, half_kick=False, solver="pcg", pcg_tol=1e-2)
rho = random_grid(n, seed=1, mean=-1.0)
E, _, _ = sim.solve_injected(rho)
print("iters", sim.pcg_stats())
