"""Support agreement of the fp32 (c64) GPU solve with the fp64 oracle on the
same fp32-rounded measurements (config 4 shape, 30 dB noise)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_1205_4139_b200 as fmp
    from oracle import Oracle
    orc = Oracle("restatement")
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    n, m, k = 16384, 4096, 128
    sigma = np.sqrt(k / (2 * n * 1e3))
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(4, 1 << 40))
    op = fmp.SensingOperator("fourier", n, rows)
    Y, X, nn = fmp.make_batch("fourier", n, rows, k, B, base_seed=4, noise_stddev=sigma, want_x=True)
    Y32 = Y.astype(np.complex64)
    res = fmp.omp_solve_batch(op, Y32, fmp.SolveConfig(2 * k, 0.0, "gpu"), tolerances=nn)

    def one(b):
        return orc.omp_solve("fourier", n, rows, Y32[b].astype(np.complex128), 2 * k, nn[b], "adaptive")
    with ThreadPoolExecutor(os.cpu_count()) as ex:
        ref = list(ex.map(one, range(B)))
    same = [list(res.support[b, :int(res.support_size[b])]) == list(ref[b].support) for b in range(B)]
    first_diff = []
    for b in range(B):
        g = list(res.support[b, :int(res.support_size[b])])
        r = list(ref[b].support)
        d = next((i for i in range(min(len(g), len(r))) if g[i] != r[i]), min(len(g), len(r)))
        first_diff.append((d, len(g), len(r)))
    print("c64 support agreement", sum(same), "/", B, first_diff)


if __name__ == "__main__":
    main()
