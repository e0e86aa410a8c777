"""One config-3 FWHT launch (f64 or f32, batch 1024) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1205_4139_b200 as fmp
    dt = {"f64": torch.float64, "f32": torch.float32}[sys.argv[1] if len(sys.argv) > 1 else "f64"]
    n, m, B = 65536, 8192, 1024
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(3, 1 << 40))
    ctx = fmp.Context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    op = fmp.SensingOperator("hadamard", n, rows, ctx)
    g = torch.Generator(device="cuda").manual_seed(3)
    r = torch.randn(B, m, dtype=dt, device="cuda", generator=g)
    h = torch.empty(B, n, dtype=dt, device="cuda")
    for _ in range(2):
        fmp.apply_adjoint_dev(op, r, h_out=h, stream=st.cuda_stream)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
