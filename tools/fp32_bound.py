"""Check the fp32 solver's rounding bound against measured errors.

For a few config-4-shape c64 signals whose GPU support equals the oracle's,
compares the recorded fp32 correlation vectors h32 (record_correlations) with
the oracle's fp64 ones, per iteration: max_j |h32_j - h64_j| against the
bound the solver assumes, 2^-24 (log2 N + 2) (hy + goff sum|x| + gamma max|x|)
(fmp_omp_impl.cuh, REFINE; the kernel multiplies it by 8).  Also prints the
refinement statistics of a full 2048-signal solve.

    python tools/fp32_bound.py [signals]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_1205_4139_b200 as fmp
    from oracle import Oracle
    orc = Oracle("restatement")
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    n, m, k = 16384, 4096, 128
    sigma = np.sqrt(k / (2 * n * 1e3))
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(4, 1 << 40))
    ctx = fmp.Context(0)
    op = fmp.SensingOperator("fourier", n, rows, ctx)
    c, _, _ = orc.compute_kernel("fourier", n, rows)
    gamma = float(np.abs(c[0]))
    goff = float(np.abs(c[1:]).max())
    Y, X, nn = fmp.make_batch("fourier", n, rows, k, B, base_seed=4, noise_stddev=sigma, want_x=True)
    Y32 = Y.astype(np.complex64)
    res = fmp.omp_solve_batch(op, Y32, fmp.SolveConfig(2 * k, 0.0, "adaptive", record_correlations=True),
                              tolerances=nn)
    unit = 2.0 ** -24 * (np.log2(n) + 2)
    worst = 0.0
    for b in range(B):
        Yo = Y32[b].astype(np.complex128)
        r = orc.omp_solve("fourier", n, rows, Yo, 2 * k, float(nn[b]), "adaptive", record=True)
        s = int(res.support_size[b])
        if list(res.support[b, :s]) != list(r.support):
            print(f"signal {b}: support differs, skipped")
            continue
        hy = np.sqrt(m / n) * np.linalg.norm(Yo)
        xa = np.abs(r.coeffs)
        E = unit * (hy + goff * xa.sum() + gamma * xa.max())
        H = res.history[b]
        ratios = []
        for t, h64 in enumerate(r.correlation_history):
            d = np.abs(H[t].astype(np.complex128) - h64).max()
            ratios.append(d / E)
        ratios = np.array(ratios)
        worst = max(worst, ratios.max())
        print(f"signal {b}: {len(ratios)} iterations, max |h32-h64| / E_unit = {ratios.max():.3f} "
              f"(median {np.median(ratios):.3f}); E_unit = {E:.3e}, final best |h| = "
              f"{np.sqrt((np.abs(r.correlation_history[-1]) ** 2).max()):.3e}")
    print(f"worst ratio {worst:.3f} (the kernel's candidate band uses 8 x E_unit)")

    fmp.set_phase_profiling(True)
    Bf = 2048
    Y, _, nn = fmp.make_batch("fourier", n, rows, k, Bf, base_seed=4, noise_stddev=sigma)
    fmp.omp_solve_batch(op, Y.astype(np.complex64), fmp.SolveConfig(2 * k, 0.0, "gpu"), tolerances=nn)
    st = ctx.refine_stats()
    fmp.set_phase_profiling(False)
    print(f"refinement over {Bf} signals: {st['identifications']:.0f} identifications, "
          f"{st['candidates'] / max(st['identifications'], 1):.2f} candidates each, "
          f"{st['overflows']:.0f} overflows")


if __name__ == "__main__":
    main()
