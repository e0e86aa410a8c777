"""Profiling driver: one batched config-2 OMP solve (or a config-3 kernel) on
cuda:0, for ncu / compute-sanitizer runs.  Not part of the bench contract.

    python tools/prof_omp.py --what omp --mode fast --batch 512
    python tools/prof_omp.py --what c3fast --dtype f64
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--what", default="omp")
    p.add_argument("--mode", default="fast")
    p.add_argument("--batch", type=int, default=512)
    p.add_argument("--dtype", default="f64")
    p.add_argument("--reps", type=int, default=2)
    p.add_argument("--fu", type=int, default=12)
    a = p.parse_args()
    import torch
    import paper_1205_4139_b200 as fmp
    ctx = fmp.Context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    if a.what == "omp":
        n, m, k = 4096, 1024, 64
        rows = fmp.make_row_selection(n, m, fmp.derive_seed(2, 1 << 40))
        Y, _, _ = fmp.make_batch("fourier", n, rows, k, a.batch, base_seed=2)
        op = fmp.SensingOperator("fourier", n, rows, ctx)
        y = torch.from_numpy(Y).cuda()
        tol = torch.from_numpy(1e-9 * np.linalg.norm(Y, axis=1)).cuda()
        out = fmp.alloc_dev_result(a.batch, k)
        cfg = fmp.SolveConfig(k, 0.0, a.mode, fast_until=a.fu)
        for _ in range(a.reps):
            fmp.omp_solve_dev(op, y, cfg, out, tolerances=tol, stream=st.cuda_stream)
    else:
        n, m, t, B = 65536, 8192, 256, a.batch
        rows = fmp.make_row_selection(n, m, fmp.derive_seed(3, 1 << 40))
        op = fmp.SensingOperator("hadamard", n, rows, ctx)
        dt = torch.float64 if a.dtype == "f64" else torch.float32
        h0 = torch.randn(B, n, dtype=dt, device="cuda")
        r = torch.randn(B, m, dtype=dt, device="cuda")
        co = torch.randn(B, t, dtype=dt, device="cuda")
        sup = torch.argsort(torch.rand(B, n, device="cuda"), dim=1)[:, :t].to(torch.int32).contiguous()
        h = torch.empty_like(h0)
        idx = torch.empty(B, dtype=torch.int64, device="cuda")
        for _ in range(a.reps):
            if a.what == "c3fast":
                fmp.fast_update_dev(op, h0, sup, co, h_out=h, argmax_out=idx, stream=st.cuda_stream)
            else:
                fmp.apply_adjoint_dev(op, r, h_out=h, argmax_out=idx, stream=st.cuda_stream)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
