"""Landau damping at the bench size on one GPU (evidence for BJ "reproduces the damping rate"):
512^3 x 8 ppc for 400 steps (t = 20) and 1024^3 x 1 ppc for 300 steps (t = 15); the W_x
peak-slope fit of tests/landau_fit.py with the SURVEY c.6 windows, against the
dispersion root (D#20).  Writes gpurun_out/damping_large.json."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from landau_fit import dispersion_root, fit_damping_rate  # noqa: E402
from paper_2605_05469_b200 import Simulation  # noqa: E402

torch.cuda.set_device(0)
w = dispersion_root(0.5)
out = {"gamma": w.imag, "omega_r": w.real, "runs": []}
for n, ppc, steps, tmax in ((512, 8, 400, 20.0), (1024, 1, 300, 15.0)):
    sim = Simulation(n=n, ppc=ppc, seed=1)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(sim.stream)
    ex = sim.step(steps)
    ev1.record(sim.stream)
    ev1.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    sim.close()
    del sim
    torch.cuda.empty_cache()
    t = np.arange(steps) * 0.05
    slope, npk, tp = fit_damping_rate(t, ex, t_max=tmax)
    spacing = float(np.mean(np.diff(tp)))
    r = {"n": n, "ppc": ppc, "steps": steps, "t_max": tmax, "ms_per_step": ms, "slope": slope,
         "slope_target": 2 * w.imag, "slope_rel_err": abs(slope - 2 * w.imag) / abs(2 * w.imag),
         "peaks": npk, "peak_spacing": spacing, "spacing_target": float(np.pi / w.real),
         "spacing_rel_err": abs(spacing - np.pi / w.real) / (np.pi / w.real), "W_x": [float(v) for v in ex]}
    out["runs"].append(r)
    print(json.dumps({k: v for k, v in r.items() if k != "W_x"}), flush=True)
json.dump(out, open("gpurun_out/damping_large.json", "w"))
