"""The multi-rank host logic with world_size 2 over gloo on CPU (no GPU): slab
geometry and particle ownership partition the box, and the bench's max-over-ranks
timing and particle-count aggregation."""
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2605_05469_b200 import default_params, slab, slab_select
        from pic_inputs import landau_state

        n, L = 32, 4 * np.pi
        p = default_params(n=n, pgrid=(1, world))
        z0, nz, cap = slab(p, rank, world)
        xv = landau_state(n, 2, seed=3)
        mine = slab_select(xv, n, L, rank, world)
        out = [None] * world
        dist.all_gather_object(out, (z0, nz, cap, mine.shape[1], mine[:, :5].tolist()))
        tmax = bench.reduce_max(10.0 + rank, world)
        tsum = bench.reduce_sum(mine.shape[1], world)
        if rank == 0:
            q.put((out, tmax, tsum, xv.shape[1]))
    finally:
        dist.destroy_process_group()


def test_two_rank_slabs_and_aggregation_gloo():
    world, port = 2, 29733
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out, tmax, tsum, npg = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    (z00, nz0, cap0, n0, _), (z01, nz1, cap1, n1, _) = out
    assert (z00, nz0, z01, nz1) == (0, 16, 16, 16)          # [0, 16) and [16, 32)
    assert n0 + n1 == npg == tsum                            # ownership partitions the particles
    assert cap0 >= n0 and cap1 >= n1
    assert tmax == 11.0                                      # job time = slowest rank
