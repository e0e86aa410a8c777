"""A/B of the two host-buffer OMP paths (config 2, wrapper with fresh
page-locked outputs, as bench.py's e2e): streamed (one launch fed by
per-chunk ready flags) vs chunked (FMP_HOST_PATH=chunked)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1205_4139_b200 as fmp
    n, m, k, B = 4096, 1024, 64, 4096
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(2, 1 << 40))
    Y, _, _ = fmp.make_batch("fourier", n, rows, k, B, base_seed=2)
    tol = 1e-9 * np.linalg.norm(Y, axis=1)
    op = fmp.SensingOperator("fourier", n, rows)
    Yp = torch.from_numpy(Y).pin_memory().numpy()
    cfg = fmp.SolveConfig(k, 0.0, sys.argv[1] if len(sys.argv) > 1 else "gpu")
    res = {"streamed": [], "chunked": []}
    for rnd in range(6):
        for path in ("streamed", "chunked"):
            os.environ["FMP_HOST_PATH"] = path
            fmp.omp_solve_batch(op, Yp, cfg, tolerances=tol)
            t0 = time.perf_counter()
            for _ in range(3):
                fmp.omp_solve_batch(op, Yp, cfg, tolerances=tol)
            res[path].append((time.perf_counter() - t0) / 3 * 1e3)
    for p, v in res.items():
        print(f"{p}: median {np.median(v):.2f} ms, min {min(v):.2f} ms -> {B / np.median(v) * 1e3:.0f} recoveries/s")


if __name__ == "__main__":
    main()
