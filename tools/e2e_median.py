"""Median wall time of the host-buffer config-2 solve through the Python
wrapper (bench.py's e2e protocol) for the package under sys.argv[1]
(A/B of builds: the repo root or a copy under _variants/)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.abspath(sys.argv[1]))


def main():
    import torch
    import paper_1205_4139_b200 as fmp
    print("package", fmp.__file__)
    n, m, k, B = 4096, 1024, 64, 4096
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(2, 1 << 40))
    Y, _, _ = fmp.make_batch("fourier", n, rows, k, B, base_seed=2)
    tol = 1e-9 * np.linalg.norm(Y, axis=1)
    op = fmp.SensingOperator("fourier", n, rows)
    Yp = torch.from_numpy(Y).pin_memory().numpy()
    fu = fmp.gpu_crossover_for(op, np.complex128, B, k)
    cfg = fmp.SolveConfig(k, 0.0, "custom", fast_until=fu)
    for _ in range(2):
        fmp.omp_solve_batch(op, Yp, cfg, tolerances=tol)
    t = []
    for _ in range(15):
        t0 = time.perf_counter()
        fmp.omp_solve_batch(op, Yp, cfg, tolerances=tol)
        t.append(time.perf_counter() - t0)
    print(f"e2e median {1e3 * np.median(t):.3f} ms -> {B / np.median(t):.0f} recoveries/s "
          f"(min {1e3 * min(t):.3f} ms) path {os.environ.get('FMP_HOST_PATH', 'default')}")
    # device-resident solve, CUDA events
    y = torch.from_numpy(Y).cuda()
    td = torch.from_numpy(tol).cuda()
    out = fmp.alloc_dev_result(B, k)
    st = torch.cuda.current_stream()
    for _ in range(2):
        fmp.omp_solve_dev(op, y, cfg, out, tolerances=td, stream=st.cuda_stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
    for a, b in ev:
        a.record(st)
        fmp.omp_solve_dev(op, y, cfg, out, tolerances=td, stream=st.cuda_stream)
        b.record(st)
    torch.cuda.synchronize()
    print(f"device {np.median([a.elapsed_time(b) for a, b in ev]):.3f} ms")


if __name__ == "__main__":
    main()
