"""Small-case driver for compute-sanitizer (memcheck): exercises every kernel
family once at small sizes."""
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
    rows = fmp.make_row_selection(65536, 8192, 3)
    op = fmp.SensingOperator("hadamard", 65536, rows)
    r = np.random.default_rng(0).standard_normal((2, 8192))
    op.apply_adjoint(r, argmax=True)
    print("sanitize driver done")


if __name__ == "__main__":
    main()
