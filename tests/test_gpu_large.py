"""GPU parity of the sharded single-signal solver (config 5 path,
fmp_large_*): one shard against the oracle; P shards emulated on one GPU
(class-major fast rows, folded np-point conventional rows, residual summed
over shards, records merged) against one shard — picks and coefficients do
not depend on P; and a config-5 prefix (N = 2^24, M = 2^21) of 32
iterations against the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("mode", ["fast", "adaptive", "conventional", "gpu"])
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_large_solve_matches_oracle(fmp, oracle, mode, dtype):
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
        # decisions and least squares in fp64 for both dtypes
        assert rel(co, r.coeffs) < 1e-10
        assert it == r.iterations_run and not ab
        assert abs(rn - r.residual_norm) <= 1e-6 * r.residual_norm + 1e-13 * np.linalg.norm(y)
        assert sorted(sup) == list(np.flatnonzero(X[b]) + 1)


@pytest.mark.parametrize("n,m,k", [(4096, 1024, 40), (1 << 19, 1 << 16, 40)])
@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("mode", ["fast", "adaptive", "conventional"])
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_emulated_shards_equal_one_shard(fmp, n, m, k, P, mode, dtype):
    """P shards on one GPU (the exchanges as copies and fixed-order sums)
    against one shard: bitwise the same supports, coefficients and counters;
    the residual norm (a sum of P partial transforms) to rounding."""
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(6, 1 << 40))
    op = fmp.SensingOperator("fourier", n, rows)
    Y, _, _ = fmp.make_batch("fourier", n, rows, k, 1, base_seed=6)
    y = Y[0].astype(dtype)
    t = 1e-9 * np.linalg.norm(Y[0])
    cfg = fmp.SolveConfig(k, t, mode)
    one = fmp.large_solve(op, y, cfg, dtype=dtype)
    shards = [fmp.LargeShard(op, cfg, p, P, dtype=dtype) for p in range(P)]
    many = fmp.sharded_solve(shards, y, t)
    for sh in shards:
        sh.close()
    assert list(many[0]) == list(one[0])
    assert np.array_equal(many[1], one[1])
    assert many[2] == one[2] and many[4] == one[4]
    assert abs(many[3] - one[3]) <= 1e-9 * one[3] + 1e-14 * np.linalg.norm(Y[0])


@pytest.mark.parametrize("mode,noise", [("conventional", 0.02), ("fast", 0.02), ("gpu", 0.02)])
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_large_noisy_halting(fmp, oracle, mode, noise, dtype):
    # halting on ||r|| <= ||noise|| before 2K iterations (solvers.cpp:388-402)
    n, m, k = 4096, 1024, 40
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(8, 1 << 40))
    op = fmp.SensingOperator("fourier", n, rows)
    Y, _, nn = fmp.make_batch("fourier", n, rows, k, 2, base_seed=8, noise_stddev=noise)
    for b in range(2):
        y = Y[b].astype(dtype)
        cfg = fmp.SolveConfig(2 * k, float(nn[b]), mode)
        sup, co, it, rn, ab = fmp.large_solve(op, y, cfg, dtype=dtype)
        r = oracle.omp_solve("fourier", n, rows, y.astype(np.complex128), 2 * k, float(nn[b]),
                             "adaptive" if mode == "gpu" else mode)
        assert list(sup) == list(r.support) and it == r.iterations_run
        assert rel(co, r.coeffs) < 1e-10
        assert abs(rn - r.residual_norm) <= 1e-9 * r.residual_norm


def test_large_validation(fmp):
    n, m = 4096, 1024
    rows = fmp.make_row_selection(n, m, 3)
    op = fmp.SensingOperator("fourier", n, rows)
    cfg = fmp.SolveConfig(8, 0.0, "fast")
    with pytest.raises(Exception):
        fmp.LargeShard(op, cfg, 0, 3)          # not a power of two
    with pytest.raises(Exception):
        fmp.LargeShard(op, cfg, 2, 2)          # shard out of range
    sh = [fmp.LargeShard(op, cfg, p, 2) for p in range(2)]
    with pytest.raises(Exception):
        fmp.sharded_solve(sh[:1], np.zeros(m, np.complex64), 0.0)  # emulation needs every shard


@pytest.mark.slow
@pytest.mark.parametrize("P", [1, 2])
def test_config5_prefix(fmp, oracle, P):
    """config 5 shape: N = 2^24, M = 2^21, K = 1024 nonzeros, c64; the first
    32 iterations on one shard and on two emulated shards."""
    n, m, k, T = 1 << 24, 1 << 21, 1024, 32
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(5, 1 << 40))
    op = fmp.SensingOperator("fourier", n, rows)
    Y, _, _ = fmp.make_batch("fourier", n, rows, k, 1, base_seed=5)
    y = Y[0].astype(np.complex64)
    cfg = fmp.SolveConfig(T, 0.0, "fast")
    if P == 1:
        sup, co, it, rn, ab = fmp.large_solve(op, y, cfg)
    else:
        shards = [fmp.LargeShard(op, cfg, p, P) for p in range(P)]
        sup, co, it, rn, ab = fmp.sharded_solve(shards, y, 0.0)
    r = oracle.omp_solve("fourier", n, rows, y.astype(np.complex128), T, 0.0, "fast")
    assert list(sup) == list(r.support)
    assert rel(co, r.coeffs) < 1e-10
    assert it == r.iterations_run == T
    assert abs(rn - r.residual_norm) <= 1e-9 * r.residual_norm
