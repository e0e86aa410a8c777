"""Profiling driver for the config-5 sharded solver on one GPU (P = 1):
one signal N = 2^24, M = 2^21, K = 1024, c64, truncated to --iters iterations.

    python tools/prof_large.py --iters 200 [--mode adaptive]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--iters", type=int, default=200)
    p.add_argument("--mode", default="adaptive")
    p.add_argument("--log2n", type=int, default=24)
    p.add_argument("--reps", type=int, default=1)
    p.add_argument("--python-loop", action="store_true",
                   help="drive the shard through sharded_solve (the multi-GPU protocol)")
    a = p.parse_args()
    import torch
    import paper_1205_4139_b200 as fmp
    n, m, k = 1 << a.log2n, 1 << (a.log2n - 3), 1024
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(5, 1 << 40))
    Y, _, _ = fmp.make_batch("fourier", n, rows, k, 1, base_seed=5)
    y = Y[0].astype(np.complex64)
    ctx = fmp.Context(0)
    op = fmp.SensingOperator("fourier", n, rows, ctx)
    tol = 1e-5 * float(np.linalg.norm(Y[0]))
    fu = fmp.crossover_iteration("fourier", n) if a.mode == "adaptive" else (
        1 << 40 if a.mode == "fast" else 0)
    cfg = fmp.SolveConfig(a.iters, tol, "custom", fast_until=fu)
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if a.python_loop:
            shard = fmp.LargeShard(op, cfg, 0, 1, dtype=np.complex64)
            sup, co, it, rn, ab = fmp.sharded_solve([shard], y, tol, None)
            shard.close()
        else:
            sup, co, it, rn, ab = fmp.large_solve(op, y, cfg, dtype=np.complex64)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{it} iterations in {dt * 1e3:.1f} ms = {dt * 1e3 / max(it, 1):.3f} ms/iteration",
              flush=True)


if __name__ == "__main__":
    main()
