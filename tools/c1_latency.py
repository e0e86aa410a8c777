"""Config-1 latency (batch 1): device-resident solve (CUDA events) vs the
host-buffer call through the Python wrapper and through the raw C ABI with
reused page-locked outputs."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1205_4139_b200 as fmp
    n, m, k = 1024, 256, 16
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(1, 1 << 40))
    op = fmp.SensingOperator("hadamard", n, rows)
    Y, _, _ = fmp.make_batch("hadamard", n, rows, k, 1, base_seed=1, real=True)
    Y = np.ascontiguousarray(Y.real)
    tol = 1e-9 * np.linalg.norm(Y, axis=1)
    cfg = fmp.SolveConfig(k, 0.0, "fast")
    Yp = torch.from_numpy(Y).pin_memory().numpy()

    def timed(fn, reps=200):
        for _ in range(20):
            fn()
        t = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            t.append(time.perf_counter() - t0)
        return np.median(t) * 1e6

    print(f"wrapper omp_solve_batch: {timed(lambda: fmp.omp_solve_batch(op, Yp, cfg, tolerances=tol)):.1f} us")
    T = k
    pin = lambda shape, dt: torch.zeros(shape, dtype=dt).pin_memory().numpy()
    sup, co = pin((1, T), torch.int64), pin((1, T), torch.complex128)
    sz, it, rn, ab = pin(1, torch.int64), pin(1, torch.int64), pin(1, torch.float64), pin(1, torch.int32)
    res = fmp.OmpResult(sup.ctypes.data, co.ctypes.data, sz.ctypes.data, it.ctypes.data, rn.ctypes.data,
                        ab.ctypes.data, None, None, None)
    tl = np.ascontiguousarray(tol)
    c = fmp._config(cfg, tl.ctypes.data_as(C.POINTER(C.c_double)))
    raw = lambda: fmp._lib.fmp_omp_solve(op.handle, fmp.DTYPES[Yp.dtype], Yp.ctypes.data, 1, C.byref(c), C.byref(res))
    print(f"raw C call, reused pinned outputs: {timed(raw):.1f} us")
    out = fmp.alloc_dev_result(1, k)
    yd = torch.from_numpy(Y).cuda()
    td = torch.from_numpy(tol).cuda()
    def dev():
        fmp.omp_solve_dev(op, yd, cfg, out, tolerances=td)
        torch.cuda.synchronize()
    print(f"device call + synchronize: {timed(dev):.1f} us")
    st = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
    for a, b in evs:
        a.record(st)
        fmp.omp_solve_dev(op, yd, cfg, out, tolerances=td)
        b.record(st)
        torch.cuda.synchronize()
    print(f"device events (warm L2): {np.median([a.elapsed_time(b) for a, b in evs]) * 1e3:.1f} us")
    def floor():
        torch.cuda._sleep(0)
        torch.cuda.synchronize()
    print(f"empty launch + synchronize: {timed(floor):.1f} us")


if __name__ == "__main__":
    main()


def pieces():
    import torch
    import paper_1205_4139_b200 as fmp
    T, B = 16, 1
    specs = [((B, T), np.uint64, False), ((B, T), np.complex128, False), ((B,), np.uint64, False),
             ((B,), np.uint64, False), ((B,), np.float64, False), ((B,), np.int32, False),
             ((B, T), np.uint8, True), ((B,), np.uint64, False)]
    for _ in range(50):
        fmp._host_outs(specs)
    t0 = time.perf_counter()
    for _ in range(200):
        fmp._host_outs(specs)
    print(f"_host_outs: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us")
    t0 = time.perf_counter()
    for _ in range(200):
        torch.empty(1024, dtype=torch.uint8, pin_memory=True)
    print(f"torch pinned empty: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us")


if __name__ == "__main__" and len(sys.argv) > 1:
    pieces()
