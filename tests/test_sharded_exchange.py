"""CPU (gloo, world size 2) test of the config-5 shard exchange: each rank
builds its identification record from its cyclic slice k = p + P k' of a
correlation vector, the records are all-gathered, and every rank merges them
with the solver's own merge rule (fmp_large_merge_records, the host twin of
the device kernel k_lg_merge).  The pick must be the reference's band
argmax over the whole vector (solvers.cpp:90-101), including exact and
in-band ties that straddle shards, an entry just outside the band, the
stagnation guard and a record that overflows."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def band_argmax(m):
    best = m.max()
    return int(np.flatnonzero(m >= best * (1 - 1e-9))[0])


def vectors(seed, n=64, steps=6):
    """fp64 |h|^2 vectors with planted ties; candidates are listed from a
    slightly perturbed working-precision copy, as the solver lists them."""
    rng = np.random.default_rng(seed)
    out = []
    for s in range(steps):
        h = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        j, k = rng.choice(n, 2, replace=False)
        peak = 10.0 + s
        h[j] = peak
        h[k] = peak * (1 - (5e-10 if s % 2 else 0.0))  # exact or in-band tie across shards
        if s == 3:
            h[k] = peak * (1 - 3e-9)                       # just outside the band
        m64 = np.abs(h) ** 2
        m32 = m64 * (1 + 1e-7 * rng.standard_normal(n))   # working precision
        out.append((m64, m32))
    return out


def record(fmp, m64, m32, p, P, band=1e-5):
    """Shard p's record: its entries within `band` of its own maximum."""
    loc64, loc32 = m64[p::P], m32[p::P]
    best32 = float(loc32.max())
    idx = np.flatnonzero(loc32 >= best32 * (1 - band))
    return fmp.make_record(best32, [(p + P * int(i), float(loc64[i])) for i in idx])


def worker(rank, world, port, result):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import paper_1205_4139_b200 as fmp
    from paper_1205_4139_b200.dist import gather_records
    ok = True
    for seed in range(5):
        for m64, m32 in vectors(seed):
            recs = gather_records(record(fmp, m64, m32, rank, world))
            pk = fmp.merge_records(recs)
            ok &= pk["flags"] == 0 and pk["atom"] == band_argmax(m64)
            ok &= pk["best64"] == float(m64.max())
    # stagnation: the pick is an atom selected before
    m64, m32 = vectors(9)[0]
    want = band_argmax(m64)
    pk = fmp.merge_records(gather_records(record(fmp, m64, m32, rank, world)), selected=[want], n=len(m64))
    ok &= pk["flags"] == 2
    # overflow: a shard with more candidates than a record carries
    many = fmp.make_record(1.0, [(rank + world * i, 1.0) for i in range(fmp.RECORD_CANDIDATES + 1)])
    ok &= fmp.merge_records(gather_records(many))["flags"] == 4
    result[rank] = bool(ok)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_distributed_record_merge_matches_global():
    pytest.importorskip("torch.distributed")
    # the package imports its CUDA library (host-loadable, no GPU needed)
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    result = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, result)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert result[0] and result[1]


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_record_merge_any_shard_count(P):
    sys.path.insert(0, ROOT)
    import paper_1205_4139_b200 as fmp
    for seed in range(4):
        for m64, m32 in vectors(seed):
            pk = fmp.merge_records([record(fmp, m64, m32, p, P) for p in range(P)])
            assert pk["flags"] == 0 and pk["atom"] == band_argmax(m64)
    # all-zero correlations: the zero stop
    z = np.zeros(16)
    assert fmp.merge_records([record(fmp, z, z, p, P) for p in range(P)])["flags"] == 1
