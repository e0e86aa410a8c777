"""Host vs device instance generation at the config-2 and
config-4 batch shapes: seconds per batch and the host-recomputed count."""
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1205_4139_b200 as fmp
    ctx = fmp.Context(0)
    for name, kind, n, m, k, B, sigma in (
            ("config2", "fourier", 4096, 1024, 64, 4096, 0.0),
            ("config4", "fourier", 16384, 4096, 128, 2048, math.sqrt(128 / (2 * 16384 * 1e3)))):
        rows = fmp.make_row_selection(n, m, fmp.derive_seed(2, 1 << 40))
        op = fmp.SensingOperator(kind, n, rows, ctx)
        fmp.make_batch_dev(op, k, 8, base_seed=2, noise_stddev=sigma)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Yd, _, nnd, fix = fmp.make_batch_dev(op, k, B, base_seed=2, noise_stddev=sigma)
        torch.cuda.synchronize()
        td = time.perf_counter() - t0
        t0 = time.perf_counter()
        Yh, _, nnh = fmp.make_batch(kind, n, rows, k, B, base_seed=2, noise_stddev=sigma)
        th = time.perf_counter() - t0
        same = np.array_equal(Yd.cpu().numpy().view(np.uint64), Yh.view(np.uint64)) and \
            np.array_equal(nnd.cpu().numpy(), nnh)
        print(f"{name}: batch {B}: device {td*1e3:.1f} ms ({fix} values recomputed on the host), "
              f"host {th*1e3:.1f} ms on {os.cpu_count()} cores, bit-identical {same}", flush=True)


if __name__ == "__main__":
    main()
