"""One config-4 c64 batched OMP solve (N = 16384, M = 4096, K = 128, batch 592) for ncu captures."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_1205_4139_b200 as fmp
    n, m, k, B = 16384, 4096, 128, int(sys.argv[1]) if len(sys.argv) > 1 else 592
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(4, 1 << 40))
    Y, _, _ = fmp.make_batch("fourier", n, rows, k, B, base_seed=4)
    Y = Y.astype(np.complex64)
    op = fmp.SensingOperator("fourier", n, rows, fmp.Context(0))
    tol = 1e-5 * np.linalg.norm(Y.astype(np.complex128), axis=1)
    r = fmp.omp_solve_batch(op, Y, fmp.SolveConfig(2 * k, 0.0, "adaptive"), tolerances=tol)
    print("iterations", float(r.iterations.mean()))


if __name__ == "__main__":
    main()
