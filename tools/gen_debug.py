"""Stage-by-stage comparison of the device generator with the host one."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1205_4139_b200 as fmp
    for kind, n, m, k, B, sigma, real in (("hadamard", 1024, 256, 16, 4, 0.0, True),
                                          ("fourier", 4096, 1024, 64, 4, 0.0, False),
                                          ("fourier", 256, 64, 4, 2, 0.1, False)):
        rows = fmp.make_row_selection(n, m, 5)
        op = fmp.SensingOperator(kind, n, rows, fmp.Context(0))
        Yh, Xh, nnh = fmp.make_batch(kind, n, rows, k, B, base_seed=77, noise_stddev=sigma, real=real, want_x=True)
        Yd, Xd, nnd, fix = fmp.make_batch_dev(op, k, B, base_seed=77, noise_stddev=sigma, real=real, want_x=True)
        torch.cuda.synchronize()
        Yd, Xd, nnd = Yd.cpu().numpy(), Xd.cpu().numpy(), nnd.cpu().numpy()
        print(kind, n, "fix", fix)
        for b in range(B):
            sh, sd = np.flatnonzero(Xh[b]), np.flatnonzero(Xd[b])
            print(" b", b, "support equal", np.array_equal(sh, sd), sh[:5], sd[:5])
            if np.array_equal(sh, sd):
                d = Xh[b, sh] - Xd[b, sh]
                print("   x maxdiff", np.abs(d).max(), "n differ", int(np.sum(Xh[b, sh] != Xd[b, sh])))
                for j in np.flatnonzero(Xh[b, sh] != Xd[b, sh])[:3]:
                    print("    ", Xh[b, sh[j]].real.hex(), Xd[b, sh[j]].real.hex(), Xh[b, sh[j]].imag.hex(), Xd[b, sh[j]].imag.hex())
            print("   y maxdiff", np.abs(Yh[b] - Yd[b]).max(), "n differ", int(np.sum(Yh[b] != Yd[b])), "nn", nnh[b], nnd[b])


if __name__ == "__main__":
    main()
