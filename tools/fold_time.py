"""Config-3 FWHT (Omega-scattered residual, 1024 x 65536) per transform plan:
FMP_FOLD=-1 is the job-queue path, 0..3 the one-pass fold plans
(fmp_transform_fold.cu).  Prints ms, algorithmic GB/s and the deviation from
the oracle on one vector, for real and complex element types."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1205_4139_b200 as fmp
    from oracle import Oracle
    orc = Oracle("restatement")
    n, m, B = 65536, 8192, 1024
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(3, 1 << 40))
    ctx = fmp.Context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    op = fmp.SensingOperator("hadamard", n, rows, ctx)
    g = torch.Generator(device="cuda").manual_seed(3)
    plans = [int(p) for p in (sys.argv[1].split(",") if len(sys.argv) > 1 else "-1,0,1,2,3".split(","))]
    for dt, s in ((torch.float64, 8), (torch.float32, 4), (torch.complex64, 8), (torch.complex128, 16)):
        r = torch.randn(B, m, dtype=dt, device="cuda", generator=g)
        h = torch.empty(B, n, dtype=dt, device="cuda")
        want = orc.apply_adjoint("hadamard", n, rows, r[5].cpu().numpy().astype(complex))
        for plan in plans:
            os.environ["FMP_FOLD"] = str(plan)
            h.zero_()
            for _ in range(3):
                fmp.apply_adjoint_dev(op, r, h_out=h, stream=st.cuda_stream)
            torch.cuda.synchronize()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
            for a, b in ev:
                a.record(st)
                fmp.apply_adjoint_dev(op, r, h_out=h, stream=st.cuda_stream)
                b.record(st)
            torch.cuda.synchronize()
            ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
            gbs = B * (m + n) * s / (ms * 1e-3) / 1e9
            got = h[5].cpu().numpy().astype(complex)
            err = np.linalg.norm(got - want) / np.linalg.norm(want)
            print(f"{str(dt)[6:]:10s} plan {plan:2d}: {ms:.3f} ms, {gbs:6.0f} GB/s algorithmic, "
                  f"rel err {err:.1e}", flush=True)
        del r, h


if __name__ == "__main__":
    main()
