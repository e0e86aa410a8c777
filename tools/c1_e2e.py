"""Config-1 end-to-end anatomy (batch 1, Hadamard N=1024 M=256 K=16 f64):
device time of the solve (CUDA events, warm L2), the host-buffer call
fmp_omp_solve (wall clock, plus CUDA events bracketing its GPU work on the
context stream), the Python wrapper, and the floor of an empty launch."""
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
    ctx = fmp.Context(0)
    op = fmp.SensingOperator("hadamard", n, rows, ctx)
    Y, _, _ = fmp.make_batch("hadamard", n, rows, k, 1, base_seed=1, real=True)
    Y = np.ascontiguousarray(Y.real)
    tol = 1e-9 * np.linalg.norm(Y, axis=1)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    reps = 200

    def wall(fn):
        for _ in range(20):
            fn()
        t = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            t.append(time.perf_counter() - t0)
        return np.median(t) * 1e6

    def events(fn):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
        for a, b in evs:
            a.record(s)
            fn()
            b.record(s)
            s.synchronize()
        return np.median([a.elapsed_time(b) for a, b in evs]) * 1e3

    for mode in ("fast", "gpu", "conventional"):
        cfg = fmp.SolveConfig(k, 0.0, mode)
        out = fmp.alloc_dev_result(1, k)
        yd = torch.from_numpy(Y).cuda()
        td = torch.from_numpy(tol).cuda()
        dev = lambda: fmp.omp_solve_dev(op, yd, cfg, out, tolerances=td, stream=s.cuda_stream)
        print(f"[{mode}] device solve, events (warm L2): {events(dev):.1f} us; "
              f"enqueue + stream sync wall: {wall(lambda: (dev(), s.synchronize())):.1f} us")
        sup = np.zeros((1, k), np.uint64); co = np.zeros((1, k), np.complex128)
        sz = np.zeros(1, np.uint64); it = np.zeros(1, np.uint64); rn = np.zeros(1); ab = np.zeros(1, np.int32)
        res = fmp.OmpResult(sup.ctypes.data, co.ctypes.data, sz.ctypes.data, it.ctypes.data, rn.ctypes.data,
                            ab.ctypes.data, None, None, None)
        tl = np.ascontiguousarray(tol)
        c = fmp._config(cfg, tl.ctypes.data_as(C.POINTER(C.c_double)))
        raw = lambda: fmp._lib.fmp_omp_solve(op.handle, fmp.DTYPES[Y.dtype], Y.ctypes.data, 1,
                                             C.byref(c), C.byref(res))
        print(f"[{mode}] raw fmp_omp_solve: wall {wall(raw):.1f} us, GPU span (events) {events(raw):.1f} us")
        print(f"[{mode}] wrapper omp_solve_batch: wall "
              f"{wall(lambda: fmp.omp_solve_batch(op, Y, cfg, tolerances=tol)):.1f} us")
    print(f"empty launch + stream sync: {wall(lambda: (torch.cuda._sleep(0), torch.cuda.synchronize())):.1f} us")
    cfg = fmp.SolveConfig(k, 0.0, "fast")
    c = fmp._config(cfg, None)
    print(f"ctypes no-op (validation failure path): "
          f"{wall(lambda: fmp._lib.fmp_omp_solve(op.handle, 99, None, 1, C.byref(c), None)):.1f} us")


if __name__ == "__main__":
    main()
