"""GPU parity for CoSaMP (solvers.cpp:413-544) through the C ABI.

Bars: identical support after every iteration (support_history), identical
iteration counts and rank-deficient aborts; coefficients, residual norms and
correlation vectors within 1e-10 relative in fp64 (1e-4 in fp32).  The
oracle is the C restatement, pinned bitwise to the reference by
tests/test_oracle.py (test_cosamp_*), plus the reference's golden vectors.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")
KN = {0: "fourier", 1: "hadamard"}
TOL64 = 1e-10


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def _same(g, r, sh, tol=TOL64):
    assert g.support_history == [[int(v) for v in row] for row in sh]
    assert g.support == [int(v) for v in r.support]
    assert g.iterations_run == r.iterations_run
    assert g.rank_deficient_abort == r.rank_deficient_abort
    assert rel(g.coeffs, r.coeffs) < tol
    assert abs(g.residual_norm - r.residual_norm) <= tol * max(r.residual_norm, 1e-300) + 1e-12


def test_cosamp_golden(fmp):
    gold = np.load(GOLD)
    for i in range(int(gold["cos_count"][0])):
        kind, n, m, k, T = (int(v) for v in gold[f"cos{i}_meta"])
        tol = float(gold[f"cos{i}_tol"][0])
        op = fmp.SensingOperator(KN[kind], n, gold[f"cos{i}_omega"])
        for mode in ("conventional", "fast"):
            g = fmp.cosamp_solve(op, gold[f"cos{i}_y"], k, fmp.SolveConfig(T, tol, mode))
            hist = gold[f"cos{i}_{mode}_history"]
            assert g.support == [int(v) for v in gold[f"cos{i}_{mode}_support"]], (i, mode)
            assert g.support_history == [[int(v) for v in row[row > 0]]
                                         for row in hist[: g.iterations_run]], (i, mode)
            it, rn, ab = gold[f"cos{i}_{mode}_scalars"]
            assert g.iterations_run == int(it) and g.rank_deficient_abort == bool(ab)
            assert rel(g.coeffs, gold[f"cos{i}_{mode}_coeffs"]) < TOL64


@pytest.mark.parametrize("kind", ["fourier", "hadamard"])
@pytest.mark.parametrize("mode", ["conventional", "fast", "adaptive"])
@pytest.mark.parametrize("n,m,k", [(64, 32, 4), (128, 64, 4), (256, 96, 8), (1024, 256, 16),
                                   (4096, 1024, 32), (512, 128, 40), (64, 64, 40), (256, 16, 8),
                                   (4096, 1024, 64)])
def test_cosamp_matches_oracle(fmp, oracle, kind, mode, n, m, k):
    # k = 64 at n = 4096 (config-2 shape): merged sets of up to 3k = 192 atoms
    # exceed the shared-memory Cholesky (~166) and take the global-memory path
    op = None
    for seed in range(3):
        om = oracle.make_row_selection(n, m, oracle.derive_seed(seed + 7 * n, 1))
        if op is None or seed:
            op = fmp.SensingOperator(kind, n, om)
        x, y, e = oracle.make_instance(kind, n, om, k, 0.05 if seed == 1 else 0.0, seed + 100 * k)
        tol = 0.0 if seed == 2 else 1e-9 * np.linalg.norm(y)
        T = max(6, k // 2)
        cfg = fmp.SolveConfig(T, tol, mode, record_correlations=True)
        g = fmp.cosamp_solve(op, y, k, cfg)
        r, sh = oracle.cosamp_solve(kind, n, om, y, k, T, tol, mode, record=True)
        _same(g, r, sh)
        assert len(g.correlation_history) == len(r.correlation_history)
        # after exact recovery with tol = 0 the correlation is rounding noise
        # (|h| ~ 1e-16..1e-14 |y|, larger for near-square merged Grams):
        # relative 1e-10, floored at an absolute 1e-12 |y|
        ny = np.linalg.norm(y)
        for p, q in zip(g.correlation_history, r.correlation_history):
            assert np.linalg.norm(p - q) <= TOL64 * max(np.linalg.norm(q), 1e-2 * ny)


def test_cosamp_edge_cases(fmp, oracle):
    # test_solvers.cpp:236-277
    for kind in ("fourier", "hadamard"):
        om = oracle.make_row_selection(64, 32, 51)
        x, y, e = oracle.make_instance(kind, 64, om, 4, 0.0, 52)
        op = fmp.SensingOperator(kind, 64, om)
        g = fmp.cosamp_solve(op, y, 4, fmp.SolveConfig(8, 1e-9 * np.linalg.norm(y), "fast"))
        assert g.support == [j + 1 for j in np.flatnonzero(x)]
        assert g.residual_norm < 1e-9 * np.linalg.norm(y)
        assert np.linalg.norm(g.x_hat - x) < 1e-8 * np.linalg.norm(x)
    om = oracle.make_row_selection(64, 8, 61)
    x, y, e = oracle.make_instance("fourier", 64, om, 4, 0.0, 62)
    op = fmp.SensingOperator("fourier", 64, om)
    g0 = fmp.cosamp_solve(op, y, 0, fmp.SolveConfig(1, np.linalg.norm(y), "fast"))
    assert g0.iterations_run == 0 and g0.support == []
    gc = fmp.cosamp_solve(op, y, 4, fmp.SolveConfig(6, 0.0, "conventional"))
    gf = fmp.cosamp_solve(op, y, 4, fmp.SolveConfig(6, 0.0, "fast"))
    assert gc.rank_deficient_abort and gf.rank_deficient_abort
    assert gc.support_history == gf.support_history
    assert gc.iterations_run == gf.iterations_run
    # tolerance already met: no iterations
    g = fmp.cosamp_solve(op, y, 4, fmp.SolveConfig(6, 2 * np.linalg.norm(y), "fast"))
    assert g.iterations_run == 0 and g.support == []
    with pytest.raises(fmp.InvalidArgument):
        fmp.cosamp_solve(op, y, 4, fmp.SolveConfig(0, 0.0, "fast"))
    with pytest.raises(fmp.InvalidArgument):
        fmp.cosamp_solve(op, y[:-1], 4, fmp.SolveConfig(6, 0.0, "fast"))


def test_cosamp_fast_equals_conventional_campaign(fmp, oracle):
    # test_solvers.cpp:279-305: both modes walk identical supports
    for kind in ("fourier", "hadamard"):
        for trial in range(20):
            seed = oracle.derive_seed(80, trial)
            om = oracle.make_row_selection(128, 64, oracle.derive_seed(seed, 1))
            op = fmp.SensingOperator(kind, 128, om)
            x, y, e = oracle.make_instance(kind, 128, om, 4, 0.05, seed)
            tol = 1e-9 * np.linalg.norm(y)
            gc = fmp.cosamp_solve(op, y, 4, fmp.SolveConfig(6, tol, "conventional",
                                                            record_correlations=True))
            gf = fmp.cosamp_solve(op, y, 4, fmp.SolveConfig(6, tol, "fast", record_correlations=True))
            assert gc.support_history == gf.support_history
            for p, q in zip(gc.correlation_history, gf.correlation_history):
                assert rel(q, p) < TOL64


@pytest.mark.parametrize("kind", ["fourier", "hadamard"])
def test_cosamp_batch_matches_per_problem_oracle(fmp, oracle, kind):
    n, m, k, B = 1024, 256, 16, 300
    om = oracle.make_row_selection(n, m, 4242)
    op = fmp.SensingOperator(kind, n, om)
    Y, _, _ = fmp.make_batch(kind, n, om, k, B, base_seed=99, noise_stddev=0.01)
    tols = 1e-9 * np.linalg.norm(Y, axis=1)
    r = fmp.cosamp_solve_batch(op, Y, k, fmp.SolveConfig(10, 0.0, "fast"), tolerances=tols)
    for b in range(0, B, 23):
        o, sh = oracle.cosamp_solve(kind, n, om, Y[b], k, 10, tols[b], "fast")
        s = int(r.support_size[b])
        assert [int(v) for v in r.support[b, :s]] == [int(v) for v in o.support]
        assert int(r.iterations[b]) == o.iterations_run
        assert rel(r.coeffs[b, :s], o.coeffs) < TOL64
        assert [[int(v) for v in row if v] for row in r.support_history[b, : o.iterations_run]] == \
            [[int(v) for v in row] for row in sh]


def test_cosamp_real_and_single_precision(fmp, oracle):
    n, m, k = 1024, 256, 16
    om = oracle.make_row_selection(n, m, oracle.derive_seed(1, 1 << 40))
    op = fmp.SensingOperator("hadamard", n, om)
    for b in range(4):
        x, y = oracle.make_real_instance("hadamard", n, om, k, oracle.derive_seed(1, b))
        tol = 1e-9 * np.linalg.norm(y)
        r, sh = oracle.cosamp_solve("hadamard", n, om, y, k, 8, tol, "fast")
        g = fmp.cosamp_solve(op, y.real, k, fmp.SolveConfig(8, tol, "fast"), dtype=np.float64)
        _same(g, r, sh)
        g32 = fmp.cosamp_solve(op, y.real, k, fmp.SolveConfig(8, 1e-5 * np.linalg.norm(y), "fast"),
                               dtype=np.float32)
        assert g32.support == [j + 1 for j in np.flatnonzero(x)]
        assert rel(g32.coeffs, r.coeffs) < 1e-4
    om = oracle.make_row_selection(4096, 1024, 5)
    op = fmp.SensingOperator("fourier", 4096, om)
    x, y, e = oracle.make_instance("fourier", 4096, om, 32, 0.0, 6)
    g = fmp.cosamp_solve(op, y, 32, fmp.SolveConfig(8, 1e-5 * np.linalg.norm(y), "fast"),
                         dtype=np.complex64)
    assert g.support == [j + 1 for j in np.flatnonzero(x)]
    assert rel(g.coeffs, x[np.flatnonzero(x)]) < 1e-4


def test_cosamp_host_streamed_equals_pageable_path(fmp, oracle):
    # batches >= 8 x grid with page-locked results (the wrapper) take the
    # one-launch streamed path (per-chunk ready flags, results stored into
    # the page-locked buffers); pageable results take the plain copy path:
    # both must agree bitwise, and with the oracle on sampled problems
    import ctypes as C
    n, m, k, B = 1024, 256, 16, 2400
    om = oracle.make_row_selection(n, m, 77)
    op = fmp.SensingOperator("fourier", n, om)
    Y, _, _ = fmp.make_batch("fourier", n, om, k, B, base_seed=77, noise_stddev=0.01)
    tol = np.ascontiguousarray(1e-9 * np.linalg.norm(Y, axis=1))
    cfg = fmp.SolveConfig(10, 0.0, "fast")
    r = fmp.cosamp_solve_batch(op, Y, k, cfg, tolerances=tol, want_history=True)
    sup = np.zeros((B, k), np.uint64)
    co = np.zeros((B, k), np.complex128)
    sz, it = np.zeros(B, np.uint64), np.zeros(B, np.uint64)
    rn, ab = np.zeros(B), np.zeros(B, np.int32)
    sh = np.zeros((B, 10, k), np.uint64)
    res = fmp.CosampResult(sup.ctypes.data, co.ctypes.data, sz.ctypes.data, it.ctypes.data,
                           rn.ctypes.data, ab.ctypes.data, sh.ctypes.data, None)
    c = fmp._config(cfg, tol.ctypes.data_as(C.POINTER(C.c_double)))
    assert fmp._lib.fmp_cosamp_solve(op.handle, fmp.DTYPES[Y.dtype], Y.ctypes.data, B, k,
                                     C.byref(c), C.byref(res)) == 0
    assert np.array_equal(sup, r.support) and np.array_equal(co, r.coeffs)
    assert np.array_equal(sz, r.support_size) and np.array_equal(it, r.iterations)
    assert np.array_equal(rn, r.residual) and np.array_equal(ab.astype(bool), r.aborted)
    assert np.array_equal(sh, r.support_history)
    for b in range(0, B, 599):
        o, _ = oracle.cosamp_solve("fourier", n, om, Y[b], k, 10, tol[b], "fast")
        s = int(r.support_size[b])
        assert [int(v) for v in r.support[b, :s]] == [int(v) for v in o.support]
