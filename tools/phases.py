"""Per-phase cycle breakdown of the fused OMP solver (profiling aid).

usage: python tools/phases.py [batch] [--kind fourier|hadamard --n N --m M --k K --iters T
                                        --dtype c128|c64|f64 --modes fast,custom:32]
(defaults: config 2, batch 1184, modes fast / conventional / custom:32)"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("batch", nargs="?", type=int, default=1184)
    p.add_argument("--n", type=int, default=4096)
    p.add_argument("--m", type=int, default=1024)
    p.add_argument("--k", type=int, default=64)
    p.add_argument("--iters", type=int, default=0)
    p.add_argument("--dtype", default="c128")
    p.add_argument("--kind", default="fourier")
    p.add_argument("--modes", default="fast,conventional,custom:32")
    a = p.parse_args()
    import paper_1205_4139_b200 as fmp
    n, m, k, B = a.n, a.m, a.k, a.batch
    T = a.iters or k
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(2, 1 << 40))
    Y, _, _ = fmp.make_batch(a.kind, n, rows, k, B, base_seed=2, real=a.dtype == "f64")
    Y = Y.astype({"c64": np.complex64, "c128": np.complex128, "f64": np.float64}[a.dtype]) \
        if a.dtype != "f64" else Y.real.copy()
    ctx = fmp.Context(0)
    op = fmp.SensingOperator(a.kind, n, rows, ctx)
    tol = 1e-9 * np.linalg.norm(Y.astype(np.complex128), axis=1) if a.dtype in ("c128", "f64") else \
        1e-5 * np.linalg.norm(Y.astype(np.complex128), axis=1)
    fmp.set_phase_profiling(True)
    for md in a.modes.split(","):
        mode, fu = (md.split(":")[0], int(md.split(":")[1])) if ":" in md else (md, 0)
        cfg = fmp.SolveConfig(T, 0.0, mode, fast_until=fu)
        r = fmp.omp_solve_batch(op, Y, cfg, tolerances=tol)
        ph = ctx.phase_cycles()
        tot = sum(ph.values())
        it = float(r.iterations.mean())
        per = {kk: round(v / B / 1e3, 1) for kk, v in ph.items()}
        print(md, f"{it:.0f} iterations, kcycles/problem total {tot / B / 1e3:.0f}", per, flush=True)


if __name__ == "__main__":
    main()
