"""torchrun worker: the z-slab decomposition (P ranks, NCCL) against the single-domain
CPU oracle.  Run:  torchrun --nproc-per-node P tests/mp_worker.py [n] [ppc] [steps]

Case 1 (import): every rank imports its slab's particles of one seeded global state
(pic_inputs), runs `steps` PIC steps; rank 0 gathers the states, merges them in
global key order and compares with oracle.run on the whole box: W_x every step
1e-10 relative, x and v 1e-12, global keys sorted, particle count
conserved, migration happened.
Case 2 (init): pic_init's own sampler on P ranks + 10 steps vs the oracle's sampler
(D#11: ulp-level init differences) -- W_x 1e-9.
Prints one line "MP OK ..." on success (rank 0); exits non-zero on failure.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2605_05469_b200 import Simulation, nccl_unique_id, slab_select  # noqa: E402
from pic_inputs import landau_state  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    ppc = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    def fresh_id():   # one NCCL unique id per communicator
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    L, dt = 4 * np.pi, 0.05
    solver = os.environ.get("MP_SOLVER", "fft")     # "pcg": BJ config 5 (FD-PCG solve)
    pg = os.environ.get("MP_PGRID")                 # "PyxPz": pencils (default z-slabs)
    pgrid = tuple(int(v) for v in pg.split("x")) if pg else (1, world)

    def oracle_run(xv0, nsteps, phi0=None):
        if solver == "pcg":
            ref, rex, _, _, _ = O.run_pcg(n, L, dt, xv0, nsteps, phi0=phi0)
            return ref, rex
        if solver == "fem":
            ref, rex, _, _, _ = O.run_fem(n, L, dt, xv0, nsteps, phi0=phi0)
            return ref, rex
        ref, rex, _, _ = O.run(n, L, dt, xv0, nsteps)
        return ref, rex

    # ---- case 1: import the same global state, step, compare with the oracle
    xv = landau_state(n, ppc, seed=11)
    mine = slab_select(xv, n, L, rank, world, pgrid)
    sim = Simulation(n=n, ppc=ppc, half_kick=False, rank=rank, nranks=world, nccl_id=fresh_id(), solver=solver,
                     pgrid=pgrid)
    sim.set_particles(mine)
    ex = sim.step(steps)
    got = sim.get_particles()
    keys, _ = sim.keys_perm()
    mig = sim.migrated()
    gathered = sim.gather_particles()       # pic_gather_particles: rank 0, global canonical order
    transport = "peer" if sim.peer_transport() else "nccl"
    want = os.environ.get("MP_EXPECT_TRANSPORT")
    assert want is None or want == transport, f"transport {transport}, expected {want}"
    parts = [None] * world
    dist.all_gather_object(parts, (got, keys, mig, ex))
    if rank == 0:
        allx = np.concatenate([p[0] for p in parts], axis=1)
        allk = np.concatenate([p[1] for p in parts])
        order = np.argsort(allk, kind="stable")
        allx, allk = allx[:, order], allk[order]
        # the library's rank-0 gather equals the merge of the ranks' exports bit for bit
        assert gathered is not None and np.array_equal(gathered, allx)
        ref, rex = oracle_run(xv, steps)
        assert allx.shape == ref.shape, (allx.shape, ref.shape)
        assert np.all(np.diff(allk.astype(np.int64)) >= 0)
        flips = int(np.count_nonzero(allk != O.keys(n, L, ref)))
        assert flips <= 2, f"{flips} cell keys differ (near-face rounding, D#16)"
        for p in parts:
            assert np.array_equal(p[3], ex), "every rank reports the same global energies"
        rel = np.max(np.abs(ex - rex) / rex)
        dx = np.abs(allx[:3] - ref[:3])
        dx = np.max(np.minimum(dx, L - dx)) / L
        dv = np.max(np.abs(allx[3:] - ref[3:]) / np.maximum(np.abs(ref[3:]), 1.0))
        total_mig = sum(p[2] for p in parts)
        assert rel <= 1e-10, f"W_x rel err {rel}"
        assert dx <= 1e-12 and dv <= 1e-12, (dx, dv)
        assert total_mig > 0, "no particle migrated"
        msg1 = f"import: W_x rel {rel:.1e} dx/L {dx:.1e} dv {dv:.1e} migrated {total_mig} key flips {flips}"
    else:
        msg1 = ""

    # ---- case 1b (FFT solver): an injected charge grid, each rank its own block -> E blocks
    # vs the oracle's single-domain solve (1e-12 of max |E|): the pencil <-> slab
    # redistributions and the slab transposes element by element
    if solver == "fft":
        from pic_inputs import random_grid

        rho = random_grid(n, seed=17, mean=-1.0)
        y0, ny, z0, nz = sim.y0, sim.ny, sim.z0, sim.nz
        Eb, _, _ = sim.solve_injected(np.ascontiguousarray(rho[z0:z0 + nz, y0:y0 + ny, :]))
        blocks = [None] * world
        dist.all_gather_object(blocks, (y0, ny, z0, nz, Eb))
        if rank == 0:
            Eg = np.zeros((3, n, n, n))
            for (by0, bny, bz0, bnz, e) in blocks:
                Eg[:, bz0:bz0 + bnz, by0:by0 + bny, :] = e
            Eref, _ = O.solve_fft(n, L, rho)
            err = np.abs(Eg - Eref).max() / np.abs(Eref).max()
            assert err <= 1e-12, f"injected solve rel err {err}"
            msg1 += f" | injected solve rel err {err:.1e}"
    sim.close()

    # ---- case 2: the library's own sampler on P ranks
    sim = Simulation(n=n, ppc=ppc, seed=9, rank=rank, nranks=world, nccl_id=fresh_id(), solver=solver,
                     pgrid=pgrid)
    ex2 = sim.step(10)
    npl = sim.np
    counts = [None] * world
    dist.all_gather_object(counts, npl)
    if rank == 0:
        assert sum(counts) == ppc * n ** 3, counts
        if solver == "pcg":
            ref0, phi0 = O.init_state_pcg(n, ppc, seed=9)
        elif solver == "fem":
            ref0, phi0 = O.init_state_fem(n, ppc, seed=9)
        else:
            ref0, phi0 = O.init_state(n, ppc, seed=9), None
        _, rex2 = oracle_run(ref0, 10, phi0)
        rel2 = np.max(np.abs(ex2 - rex2) / rex2)
        assert rel2 <= 1e-9, rel2
        print(f"MP OK P={world} pgrid={pgrid[0]}x{pgrid[1]} n={n} ppc={ppc} steps={steps} solver={solver} "
              f"transport={transport} | {msg1} | "
              f"init: W_x rel {rel2:.1e} counts {counts}",
              flush=True)
    sim.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
