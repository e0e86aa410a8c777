"""Config-3 transform timing (FWHT of the Omega-scattered residual, 1024 x
65536, f64 and f32) with a parity spot check against the oracle.  The
transform path can be forced with FMP_TRANSFORM_PATH=queue|cluster."""
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
    # a real stream: handle 0 would mean "the context's own stream"
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    op = fmp.SensingOperator("hadamard", n, rows, ctx)
    g = torch.Generator(device="cuda").manual_seed(3)
    for dt, s in ((torch.float64, 8), (torch.float32, 4)):
        r = torch.randn(B, m, dtype=dt, device="cuda", generator=g)
        h = torch.empty(B, n, dtype=dt, device="cuda")
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
        want = orc.apply_adjoint("hadamard", n, rows, r[5].double().cpu().numpy().astype(complex))
        err = np.linalg.norm(h[5].double().cpu().numpy() - want.real) / np.linalg.norm(want)
        print(f"{str(dt)[6:]}: {ms:.3f} ms, {gbs:.0f} GB/s algorithmic, rel err {err:.1e}", flush=True)


if __name__ == "__main__":
    main()
