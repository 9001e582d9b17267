"""Dump W_x(t) series from the GPU path for a few configs (analysis helper)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_05469_b200 import Simulation
torch.cuda.set_device(0)
out = {}
for (n, ppc, alpha, steps) in [(128, 8, 0.05, 600), (128, 64, 0.05, 600), (64, 8, 0.05, 600), (256, 8, 0.05, 600)]:
    for seed in (1, 2):
        sim = Simulation(n=n, ppc=ppc, alpha=alpha, seed=seed)
        out[f"{n}_{ppc}_{alpha}_{seed}"] = sim.step(steps)
        sim.close()
        del sim
        torch.cuda.empty_cache()
np.savez("gpurun_out/damping_series.npz", **out)
print("ok", list(out))
