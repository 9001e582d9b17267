"""Bandwidth probes on the live 512^3 x 8 state (pic_diag_bandwidth): what the sort's
access patterns can reach on this B200 with the real permutation of a step."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_05469_b200 import Simulation  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ppc = int(sys.argv[2]) if len(sys.argv) > 2 else 8
torch.cuda.set_device(0)
sim = Simulation(n=n, ppc=ppc, seed=1)
sim.step(3)
sim.set_timing(True)
sim.reset_timings()
sim.step(2)
st = sim.timings()
sim.set_timing(False)
out = {"n": n, "ppc": ppc, "stage_ms_per_step": {k: v[0] / 2 for k, v in st.items() if v[0] > 0}}
names = {0: "stream_copy_96B", 1: "gather_via_perm_100B", 2: "scatter4_via_perm_8B", 3: "stream_read_48B"}
for mode in (3, 0, 1, 2, 1, 0):
    ms, b = sim.diag_bandwidth(mode, reps=3)
    out[names[mode]] = {"ms": ms, "GBps": b / ms / 1e6}
print(json.dumps(out, indent=1))
