"""Diagnose fp32 (c64) support disagreements with the fp64 oracle at the
config-4 shape: for every signal whose GPU support differs from the oracle's,
report where (first differing position, or the halting iteration) and the
oracle's |h|^2 margin at that iteration (top-2 gap, band edge).

    python tools/fp32_diag.py [batch] [gpu_mode] [oracle_mode]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_1205_4139_b200 as fmp
    from oracle import Oracle
    orc = Oracle("restatement")
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    gmode = sys.argv[2] if len(sys.argv) > 2 else "gpu"
    omode = sys.argv[3] if len(sys.argv) > 3 else "fast"
    n, m, k = 16384, 4096, 128
    sigma = np.sqrt(k / (2 * n * 1e3))
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(4, 1 << 40))
    op = fmp.SensingOperator("fourier", n, rows)
    Y, X, nn = fmp.make_batch("fourier", n, rows, k, B, base_seed=4, noise_stddev=sigma, want_x=True)
    Y32 = Y.astype(np.complex64)
    res = fmp.omp_solve_batch(op, Y32, fmp.SolveConfig(2 * k, 0.0, gmode), tolerances=nn)
    Yo = Y32.astype(np.complex128)
    bad = 0
    from concurrent.futures import ThreadPoolExecutor

    def one(b):
        return orc.omp_solve("fourier", n, rows, Yo[b], 2 * k, float(nn[b]), omode)
    with ThreadPoolExecutor(os.cpu_count()) as ex:
        refs = list(ex.map(one, range(B)))
    for b in range(B):
        r = refs[b]
        s = int(res.support_size[b])
        g = list(res.support[b, :s])
        rs = list(r.support)
        if g == rs:
            continue
        bad += 1
        d = next((i for i in range(min(len(g), len(rs))) if g[i] != rs[i]), min(len(g), len(rs)))
        info = f"signal {b}: first diff at {d} (gpu {len(g)} atoms it {int(res.iterations[b])} " \
               f"rn {res.residual[b]:.9e}; oracle {len(rs)} atoms it {r.iterations_run} " \
               f"rn {r.residual_norm:.9e}; tol {nn[b]:.9e})"
        rr = orc.omp_solve("fourier", n, rows, Yo[b], d + 1, 0.0, omode, record=True)
        if len(rr.correlation_history) > d:
            h = rr.correlation_history[d]
            a2 = np.abs(h) ** 2
            o = np.argsort(-a2)
            best = a2[o[0]]
            info += f"\n   oracle iteration {d + 1}: top |h|^2 {best:.12e} at {o[0] + 1}, " \
                    f"2nd {a2[o[1]]:.12e} at {o[1] + 1} (rel gap {(best - a2[o[1]]) / best:.3e})"
            if d < len(g):
                gp = g[d] - 1
                info += f"; gpu pick {g[d]} has rel {(best - a2[gp]) / best:.3e}"
        print(info, flush=True)
    print(f"c64 support agreement {B - bad} / {B} (gpu mode {gmode}, oracle mode {omode})")


if __name__ == "__main__":
    main()
