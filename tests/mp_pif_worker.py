"""torchrun worker: the decomposed PIF (pic_pif_attach_nccl; P ranks, each with its own share of
the particles, the modes all-reduced) against the single-process oracle/nufft.py on the whole
particle set.  Run:  torchrun --nproc-per-node P tests/mp_pif_worker.py [N] [ppc] [steps]

Case 1: one PIF solve -- E at every rank's particles within 1e-10 of max |E| of the oracle's
field at those particles, energies 1e-10 relative, identical on every rank.
Case 2: `steps` steps of the PIF time loop (pic_pif_step) -- W_x every step 1e-10 relative,
x and v after the steps 1e-12 (the BJ metrics).  Type 1 summed over the ranks vs nufft1.
Prints "MP PIF OK ..." on rank 0; exits non-zero on failure."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import nufft as U  # noqa: E402
from paper_2605_05469_b200 import PifSolver, nccl_unique_id  # noqa: E402
from pic_inputs import landau_state, random_weights  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    ppc = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")

    def fresh_id():
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    L, dt = 4 * np.pi, 0.05
    xv = landau_state(N, ppc, L=L, seed=21)
    npg = xv.shape[1]
    q = np.full(npg, -L ** 3 / npg)
    own = np.arange(npg) * world // npg == rank          # contiguous shares of the particle array
    x = torch.from_numpy(np.ascontiguousarray(xv[:3, own])).cuda()
    qq = torch.from_numpy(np.ascontiguousarray(q[own])).cuda()
    P = PifSolver(N, L, 1e-4, np_max=int(own.sum()), rank=rank, nranks=world, nccl_id=fresh_id())
    E, W = P.solve(x, qq)
    Eo, Wo, _ = U.pif_solve(xv[:3], q, N, L, 1e-4)
    err = np.abs(E.cpu().numpy() - Eo[:, own]).max() / np.abs(Eo).max()
    assert err <= 1e-10, f"rank {rank}: E rel err {err}"
    assert np.allclose(W, Wo, rtol=1e-10), (W, Wo)
    Ws = [None] * world
    dist.all_gather_object(Ws, [float(w) for w in W])
    assert all(w == Ws[0] for w in Ws), "every rank holds the same (global) energies"
    # type 1 summed over the ranks
    f = random_weights(npg, seed=5)
    g = P.type1(x, torch.from_numpy(np.ascontiguousarray(f[own])).cuda()).cpu().numpy()
    ref1 = U.nufft1(xv[:3], f, N, L, 1e-4)
    e1 = np.abs(g - ref1).max() / np.abs(f).sum()
    assert e1 <= 1e-11, f"type1 rel err {e1}"
    # the time loop
    v = torch.from_numpy(np.ascontiguousarray(xv[3:, own])).cuda()
    ex = P.step(x, v, qq, nsteps=steps, dt=dt)
    ref, rex = U.pif_run(N, L, dt, xv, q, steps)
    rel = np.max(np.abs(ex - rex) / rex)
    assert rel <= 1e-10, f"W_x rel err {rel}"
    got = np.concatenate([x.cpu().numpy(), v.cpu().numpy()])
    dx = np.abs(got[:3] - ref[:3, own])
    dx = np.max(np.minimum(dx, L - dx)) / L
    dv = np.max(np.abs(got[3:] - ref[3:, own]) / np.maximum(np.abs(ref[3:, own]), 1.0))
    assert dx <= 1e-12 and dv <= 1e-12, (dx, dv)
    errs = [None] * world
    dist.all_gather_object(errs, (err, e1, rel, dx, dv))
    if rank == 0:
        m = np.max(np.array(errs), axis=0)
        print(f"MP PIF OK P={world} N={N} ppc={ppc} particles={npg} | solve E rel {m[0]:.1e} type1 {m[1]:.1e} | "
              f"{steps} steps: W_x rel {m[2]:.1e} dx/L {m[3]:.1e} dv {m[4]:.1e}", flush=True)
    del P
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
