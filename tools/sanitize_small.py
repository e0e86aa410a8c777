"""Small-case driver for compute-sanitizer (memcheck / racecheck /
synccheck): exercises every kernel family once at small sizes — the fused
OMP solver in every dtype (incl. the fp32 refinement and the two-CTA
configuration), CoSaMP, the fast update (quad-lane f32 / f64 tiles), the
transforms (one CTA, cluster / job queue, one-pass fold, two-pass), the
sharded large solver and the streamed host path.

    compute-sanitizer --tool racecheck python tools/sanitize_small.py [quick]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1205_4139_b200 as fmp  # noqa: E402


def main():
    for kind, n, m, k in (("fourier", 256, 64, 6), ("hadamard", 256, 64, 6), ("fourier", 8192, 2048, 8)):
        rows = fmp.make_row_selection(n, m, 3)
        op = fmp.SensingOperator(kind, n, rows)
        Y, X, _ = fmp.make_batch(kind, n, rows, k, 3, base_seed=1, want_x=True)
        h, idx = op.apply_adjoint(Y, argmax=True)
        op.apply(X)
        fmp.fast_update(h, op, np.array([[1, 5, 9]] * 3), np.ones((3, 3), complex), argmax=True)
        for mode in ("fast", "conventional", "gpu"):
            fmp.omp_solve_batch(op, Y, fmp.SolveConfig(k, 1e-12, mode, record_correlations=True))
        fmp.least_squares(op, [1, 2, 3], Y[0])
        if kind == "fourier":
            fmp.large_solve(op, Y[0], fmp.SolveConfig(k, 1e-12, "gpu"))
            sh = [fmp.LargeShard(op, fmp.SolveConfig(k, 1e-12, "fast"), p, 2) for p in range(2)]
            fmp.sharded_solve(sh, Y[0].astype(np.complex64), 1e-12)
        # fp32 data (refined identification), CoSaMP
        Y32 = Y.astype(np.complex64)
        fmp.omp_solve_batch(op, Y32, fmp.SolveConfig(k, 1e-12, "gpu"))
        fmp.cosamp_solve_batch(op, Y, k, fmp.SolveConfig(4, 1e-12, "fast"))
        fmp.cosamp_solve_batch(op, Y32, k, fmp.SolveConfig(4, 1e-12, "conventional"))
        if kind == "hadamard":
            fmp.omp_solve_batch(op, Y.real.copy(), fmp.SolveConfig(k, 1e-12, "fast"), dtype=np.float64)
            fmp.omp_solve_batch(op, Y.real.astype(np.float32), fmp.SolveConfig(k, 1e-12, "fast"),
                                dtype=np.float32)
    rows = fmp.make_row_selection(65536, 8192, 3)
    op = fmp.SensingOperator("hadamard", 65536, rows)
    rng = np.random.default_rng(0)
    for dt in (np.float64, np.float32, np.complex64):
        r = rng.standard_normal((2, 8192)).astype(dt)
        op.apply_adjoint(r, argmax=True)
        h0 = rng.standard_normal((2, 65536)).astype(dt)
        sup = np.array([rng.choice(65536, 40, replace=False) + 1 for _ in range(2)])
        fmp.fast_update(h0, op, sup, rng.standard_normal((2, 40)).astype(dt), argmax=True)
    if len(sys.argv) < 2:
        # two CTAs per SM (batch >= 2 x SMs) and the streamed host path (batch >= 8 x grid)
        n, m, k = 2048, 512, 8
        rows = fmp.make_row_selection(n, m, 5)
        op = fmp.SensingOperator("fourier", n, rows)
        Y, _, _ = fmp.make_batch("fourier", n, rows, k, 2400, base_seed=5)
        fmp.omp_solve_batch(op, Y, fmp.SolveConfig(k, 1e-12, "gpu"))
    print("sanitize driver done")


if __name__ == "__main__":
    main()
