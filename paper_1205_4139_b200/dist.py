"""Cross-process exchange for the sharded single-signal solver (config 5).

One process per GPU, each holding one `LargeShard`; per OMP iteration the
shards agree on the picked atom with two tiny collectives over
torch.distributed (NCCL on the GPUs, gloo in the CPU tests):

  1. all-reduce MAX of the local best |h|^2            -> global best B
  2. all-gather of (first in-band atom, h0 there)       -> smallest atom wins

which is exactly the reference's band argmax over the whole vector
(solvers.cpp:90-101): every in-band entry satisfies |h|^2 >= B(1 - 1e-9), and
the smallest such global index is the minimum of the per-shard minima.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class TorchExchange:
    def __init__(self, group=None, device: str | None = None):
        self.group = group
        backend = dist.get_backend(group)
        self.device = device or ("cuda" if backend == "nccl" else "cpu")

    def max(self, values) -> float:
        t = torch.tensor([max(values)], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def first(self, atoms):
        cands = [(a, h) for a, h in atoms if a > 0]
        a, h = min(cands, key=lambda ah: ah[0]) if cands else (0, 0j)
        mine = torch.tensor([float(a), h.real, h.imag], dtype=torch.float64, device=self.device)
        out = [torch.empty_like(mine) for _ in range(dist.get_world_size(self.group))]
        dist.all_gather(out, mine, group=self.group)
        best = (0, 0j)
        for t in out:
            at = int(t[0].item())
            if at > 0 and (best[0] == 0 or at < best[0]):
                best = (at, complex(t[1].item(), t[2].item()))
        return best
