"""Per-phase cycle breakdown of the fused solver on config 2 (profiling aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1205_4139_b200 as fmp
    n, m, k, B = 4096, 1024, 64, int(sys.argv[1]) if len(sys.argv) > 1 else 1184
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(2, 1 << 40))
    Y, _, _ = fmp.make_batch("fourier", n, rows, k, B, base_seed=2)
    ctx = fmp.Context(0)
    op = fmp.SensingOperator("fourier", n, rows, ctx)
    tol = 1e-9 * np.linalg.norm(Y, axis=1)
    fmp.set_phase_profiling(True)
    for mode, fu in (("fast", 0), ("conventional", 0), ("custom", 32)):
        cfg = fmp.SolveConfig(k, 0.0, mode, fast_until=fu)
        fmp.omp_solve_batch(op, Y, cfg, tolerances=tol)
        ph = ctx.phase_cycles()
        tot = sum(ph.values())
        per = {kk: round(v / B / 1e3, 1) for kk, v in ph.items()}
        print(mode, fu, f"kcycles/problem total {tot / B / 1e3:.0f}", per)


if __name__ == "__main__":
    main()
