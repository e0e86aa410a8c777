"""One config-3 fast-update launch (Hadamard N=65536, |Lambda|=256, batch
1024; f64 or f32) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1205_4139_b200 as fmp
    dt = {"f64": torch.float64, "f32": torch.float32}[sys.argv[1] if len(sys.argv) > 1 else "f32"]
    n, m, t, B = 65536, 8192, 256, 1024
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(3, 1 << 40))
    ctx = fmp.Context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    op = fmp.SensingOperator("hadamard", n, rows, ctx)
    g = torch.Generator(device="cuda").manual_seed(3)
    h0 = torch.randn(B, n, dtype=dt, device="cuda", generator=g)
    co = torch.randn(B, t, dtype=dt, device="cuda", generator=g)
    sup = torch.argsort(torch.rand(B, n, device="cuda", generator=g), dim=1)[:, :t].to(torch.int32).contiguous()
    h = torch.empty_like(h0)
    for _ in range(2):
        fmp.fast_update_dev(op, h0, sup, co, h_out=h, stream=st.cuda_stream)
    torch.cuda.synchronize()
    if "--time" in sys.argv:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(5):
            fmp.fast_update_dev(op, h0, sup, co, h_out=h, stream=st.cuda_stream)
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        print(f"{sys.argv[1]}: {ms:.3f} ms, {B * n * t / (ms * 1e-3) / 1e12:.2f} T MAC/s")
    print("ok")


if __name__ == "__main__":
    main()
