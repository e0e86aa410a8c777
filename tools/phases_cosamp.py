"""Per-phase cycle breakdown of the fused CoSaMP solver (profiling aid).

Phases: correlation (conventional / fast), identify (top-2K select + merge +
prune select), least squares (Cholesky + triangular solves), residual, other.
usage: python tools/phases_cosamp.py [config 1|2] [batch]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_1205_4139_b200 as fmp
    cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 1184
    kind, n, m, k = ("fourier", 4096, 1024, 64) if cfgn == 2 else ("hadamard", 1024, 256, 16)
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(cfgn, 1 << 40))
    Y, _, _ = fmp.make_batch(kind, n, rows, k, B, base_seed=cfgn)
    ctx = fmp.Context(0)
    op = fmp.SensingOperator(kind, n, rows, ctx)
    tol = 1e-9 * np.linalg.norm(Y, axis=1)
    fmp.set_phase_profiling(True)
    for mode in ("fast", "conventional"):
        r = fmp.cosamp_solve_batch(op, Y, k, fmp.SolveConfig(k, 0.0, mode), tolerances=tol,
                                   want_history=False)
        ph = ctx.phase_cycles()
        it = float(r.iterations.mean())
        names = ["conventional", "fast", "identify", "least_squares", "residual", "other"]
        per = {nm: round(ph[nm] / B / it / 1e3, 1) for nm in names}
        print(f"config {cfgn} {mode}: {it:.2f} iterations, kcycles/iteration "
              f"{sum(ph.values()) / B / it / 1e3:.0f}", per)


if __name__ == "__main__":
    main()
