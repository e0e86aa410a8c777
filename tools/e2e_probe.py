"""Where the host-buffer solve's time goes (config 2): the C call with fresh
pageable outputs (the Python wrapper), with reused pageable outputs, and with
reused pinned outputs."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import ctypes as C
    import torch
    import paper_1205_4139_b200 as fmp
    n, m, k, B = 4096, 1024, 64, 4096
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(2, 1 << 40))
    Y, _, _ = fmp.make_batch("fourier", n, rows, k, B, base_seed=2)
    tol = 1e-9 * np.linalg.norm(Y, axis=1)
    op = fmp.SensingOperator("fourier", n, rows)
    Yp = torch.from_numpy(Y).pin_memory().numpy()
    mode = sys.argv[1] if len(sys.argv) > 1 else "gpu"
    cfg = fmp.SolveConfig(k, 0.0, mode)
    print("mode", mode)

    def timed(fn, reps=5):
        fn()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        return (time.perf_counter() - t0) / reps * 1e3

    print(flush=True); print("wrapper (fresh outputs):", round(timed(lambda: fmp.omp_solve_batch(op, Yp, cfg, tolerances=tol)), 2), "ms")
    T = k

    def raw(pinned):
        mk = (lambda shape, dt: torch.zeros(shape, dtype=dt).pin_memory().numpy()) if pinned else \
             (lambda shape, dt: np.zeros(shape, dt))
        sup = mk((B, T), torch.int64 if pinned else np.uint64)
        co = mk((B, T), torch.complex128 if pinned else np.complex128)
        sz = mk(B, torch.int64 if pinned else np.uint64)
        it = mk(B, torch.int64 if pinned else np.uint64)
        rn = mk(B, torch.float64 if pinned else np.float64)
        ab = mk(B, torch.int32 if pinned else np.int32)
        tarr = np.ascontiguousarray(tol)
        res = fmp.OmpResult(sup.ctypes.data, co.ctypes.data, sz.ctypes.data, it.ctypes.data, rn.ctypes.data,
                            ab.ctypes.data, None, None, None)
        c = fmp._config(cfg, tarr.ctypes.data_as(C.POINTER(C.c_double)))
        keep = (sup, co, sz, it, rn, ab, tarr, res, c)  # the C call writes into these

        def call():
            assert keep
            st = fmp._lib.fmp_omp_solve(op.handle, fmp.DTYPES[np.dtype(np.complex128)], Yp.ctypes.data, B,
                                        C.byref(c), C.byref(res))
            assert st == 0, st
        return call

    print("C call, reused pageable outputs:", round(timed(raw(False)), 2), "ms")
    print("C call, reused pinned outputs:", round(timed(raw(True)), 2), "ms")


if __name__ == "__main__":
    main()
