"""GPU parity of the sharded single-signal solver (config 5 path):
fmp_large_solve against the oracle, shards emulated on one GPU against the
unsharded solve, and a config-5-shaped prefix (N = 2^24, M = 2^21)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("mode", ["fast", "adaptive", "conventional", "gpu"])
@pytest.mark.parametrize("dtype,tol", [(np.complex128, 1e-10), (np.complex64, 1e-4)])
def test_large_solve_matches_oracle(fmp, oracle, mode, dtype, tol):
    n, m, k = 4096, 1024, 48
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(5, 1 << 40))
    op = fmp.SensingOperator("fourier", n, rows)
    Y, X, _ = fmp.make_batch("fourier", n, rows, k, 2, base_seed=5, want_x=True)
    for b in range(2):
        y = Y[b].astype(dtype)
        t = 1e-9 * np.linalg.norm(y.astype(np.complex128))
        cfg = fmp.SolveConfig(k, t, mode)
        sup, co, it, rn, ab = fmp.large_solve(op, y, cfg, dtype=dtype)
        r = oracle.omp_solve("fourier", n, rows, y.astype(np.complex128), k, t,
                             "adaptive" if mode == "gpu" else mode)
        assert list(sup) == list(r.support)
        assert rel(co, r.coeffs) < tol
        assert it == r.iterations_run and not ab
        assert sorted(sup) == list(np.flatnonzero(X[b]) + 1)


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("mode", ["fast", "gpu"])
def test_emulated_shards_equal_unsharded(fmp, P, mode):
    n, m, k = 4096, 1024, 40
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(6, 1 << 40))
    op = fmp.SensingOperator("fourier", n, rows)
    Y, _, _ = fmp.make_batch("fourier", n, rows, k, 1, base_seed=6)
    y = Y[0].astype(np.complex64)
    t = 1e-9 * np.linalg.norm(Y[0])
    cfg = fmp.SolveConfig(k, t, mode)
    one = fmp.large_solve(op, y, cfg)
    shards = [fmp.LargeShard(op, cfg, p, P) for p in range(P)]
    many = fmp.sharded_solve(shards, y, t)
    assert list(many[0]) == list(one[0])
    assert np.array_equal(many[1], one[1])  # replicated LS: bit-identical
    assert many[2] == one[2]


@pytest.mark.slow
def test_config5_prefix(fmp, oracle):
    # config 5 shape: N = 2^24, M = 2^21, K = 1024 nonzeros, c64; first iterations
    n, m, k, T = 1 << 24, 1 << 21, 1024, 4
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(5, 1 << 40))
    op = fmp.SensingOperator("fourier", n, rows)
    Y, _, _ = fmp.make_batch("fourier", n, rows, k, 1, base_seed=5)
    y = Y[0].astype(np.complex64)
    cfg = fmp.SolveConfig(T, 0.0, "fast")
    sup, co, it, rn, ab = fmp.large_solve(op, y, cfg)
    r = oracle.omp_solve("fourier", n, rows, y.astype(np.complex128), T, 0.0, "fast")
    assert list(sup) == list(r.support)
    assert rel(co, r.coeffs) < 1e-4


@pytest.mark.parametrize("mode,noise", [("gpu", 0.0), ("conventional", 0.02), ("fast", 0.02)])
def test_single_round_trip_equals_two_round_trips(fmp, mode, noise):
    # fmp_large_solve's one-synchronisation iteration (speculative next
    # correlation, fmp_capi.cu lg_advance_fused) against the two-round-trip
    # protocol: bitwise the same supports, coefficients, counters, residual
    # (noisy signals halt on the tolerance, exercising the discarded
    # speculation and the explicit-residual branches)
    import os
    n, m, k = 4096, 1024, 40
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(8, 1 << 40))
    op = fmp.SensingOperator("fourier", n, rows)
    Y, _, nn = fmp.make_batch("fourier", n, rows, k, 1, base_seed=8, noise_stddev=noise)
    y = Y[0]
    t = float(nn[0]) if noise else 1e-9 * np.linalg.norm(y)
    cfg = fmp.SolveConfig(2 * k, t, mode)
    one = fmp.large_solve(op, y, cfg, dtype=np.complex128)
    os.environ["FMP_LARGE_TWO_TRIPS"] = "1"
    try:
        two = fmp.large_solve(op, y, cfg, dtype=np.complex128)
    finally:
        del os.environ["FMP_LARGE_TWO_TRIPS"]
    assert np.array_equal(one[0], two[0]) and np.array_equal(one[1], two[1])
    assert one[2:] == two[2:]
