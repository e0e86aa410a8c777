"""CPU (gloo, world size 2) test of the config-5 shard exchange: the
distributed band argmax over cyclic shards equals the reference's band argmax
over the whole vector (solvers.cpp:90-101), including exact and near ties
that straddle shards."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def band_argmax(h):
    m = np.abs(h) ** 2
    best = m.max()
    return int(np.flatnonzero(m >= best * (1 - 1e-9))[0])


class FakeShard:
    """Stands in for LargeShard: holds the cyclic slice k = p + P k' of a
    sequence of global correlation vectors and h0."""

    def __init__(self, hs, h0, p, P):
        self.hs, self.h0, self.p, self.P, self.t = hs, h0, p, P, 0

    def local(self):
        return self.hs[self.t][self.p::self.P]

    def begin(self):
        return float(np.max(np.abs(self.local()) ** 2))

    def first(self, best):
        m = np.abs(self.local()) ** 2
        idx = np.flatnonzero(m >= best * (1 - 1e-9))
        if not len(idx):
            return 0, 0j
        k = self.p + self.P * int(idx[0])
        return k + 1, complex(self.h0[k])

    def advance(self):
        self.t += 1
        return float(np.max(np.abs(self.local()) ** 2)) if self.t < len(self.hs) else -1.0


def vectors(seed, n=64, steps=6):
    rng = np.random.default_rng(seed)
    hs = []
    for s in range(steps):
        h = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        j, k = rng.choice(n, 2, replace=False)
        peak = 10.0 + s
        h[j] = peak
        h[k] = peak * (1 - (5e-10 if s % 2 else 0.0))  # exact or in-band tie across shards
        if s == 3:
            h[k] = peak * (1 - 3e-9)                       # just outside the band
        hs.append(h)
    h0 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return hs, h0


def worker(rank, world, port, result):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from paper_1205_4139_b200.dist import TorchExchange
    ex = TorchExchange()
    ok = True
    for seed in range(5):
        hs, h0 = vectors(seed)
        sh = FakeShard(hs, h0, rank, world)
        best = ex.max([sh.begin()])
        for t in range(len(hs)):
            atom, h = ex.first([sh.first(best)])
            want = band_argmax(hs[t])
            ok &= atom == want + 1 and h == complex(h0[want])
            nb = sh.advance()
            if nb < 0:
                break
            best = ex.max([nb])
    result[rank] = ok
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_distributed_band_argmax_matches_global():
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


def test_local_exchange_emulation_matches_global():
    import sys
    sys.path.insert(0, ROOT)
    from paper_1205_4139_b200 import LocalExchange
    ex = LocalExchange()
    for P in (1, 2, 4, 8):
        for seed in range(4):
            hs, h0 = vectors(seed)
            shards = [FakeShard(hs, h0, p, P) for p in range(P)]
            best = ex.max([s.begin() for s in shards])
            for t in range(len(hs)):
                atom, h = ex.first([s.first(best) for s in shards])
                want = band_argmax(hs[t])
                assert atom == want + 1 and h == complex(h0[want])
                nbs = [s.advance() for s in shards]
                if nbs[0] < 0:
                    break
                best = ex.max(nbs)
