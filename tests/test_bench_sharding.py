"""Batch sharding of bench.py for configs 2-4 (weak scaling, no collective in
the solve): rank r of world W solves the signals [rB, (r+1)B), each seeded by
its GLOBAL index, so the union over ranks is exactly the single-process batch
of W*B signals.  Checked with two gloo ranks on CPU (host generation only)."""
import os
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, cfgn, B, q):
    sys.path.insert(0, ROOT)
    import torch
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bench.CFG.clear()
    bench.CFG.update(bench.CONFIGS[cfgn])
    rows, Y, tol = bench.problem(B, rank * B)
    Yc = np.ascontiguousarray(Y.astype(np.complex128))
    yt = torch.from_numpy(Yc.view(np.float64).copy())
    tt = torch.from_numpy(np.ascontiguousarray(tol))
    ys = [torch.empty_like(yt) for _ in range(world)]
    ts = [torch.empty_like(tt) for _ in range(world)]
    dist.all_gather(ys, yt)
    dist.all_gather(ts, tt)
    if rank == 0:
        _, Yall, tall = bench.problem(world * B, 0)
        got = np.concatenate([y.numpy() for y in ys]).view(np.complex128)
        q.put(bool(np.array_equal(got, Yall.astype(np.complex128))) and
              bool(np.array_equal(np.concatenate([t.numpy() for t in ts]), tall)))
    dist.destroy_process_group()


@pytest.mark.parametrize("cfgn,B", [(2, 6), (4, 3)])
def test_bench_shards_union_is_the_global_batch(cfgn, B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + 37 * cfgn + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfgn, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True
