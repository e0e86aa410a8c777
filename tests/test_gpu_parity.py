"""GPU parity: the CUDA path through the C ABI against the CPU oracle.

Bars (BASELINE.json north_star): identical selected supports at every
iteration; h and x within 1e-10 relative in fp64, 1e-4 relative in fp32.
The oracle is the C restatement (oracle/fmp_oracle.c), itself pinned
bit-for-bit to the reference by tests/test_oracle.py; a few cases are also
checked against the reference's own golden vectors.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")
KN = {0: "fourier", 1: "hadamard"}


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


# ----------------------------------------------------------------- kernel
@pytest.mark.parametrize("kind", ["fourier", "hadamard"])
@pytest.mark.parametrize("n,m", [(4, 2), (16, 4), (64, 16), (1024, 256), (4096, 1024),
                                 (16384, 4096), (65536, 8192)])
def test_kernel_matches_oracle(fmp, oracle, kind, n, m):
    om = oracle.make_row_selection(n, m, 1000 + n + m)
    op = fmp.SensingOperator(kind, n, om)
    ker = fmp.compute_kernel(op)
    c, vals, vidx = oracle.compute_kernel(kind, n, om)
    if kind == "hadamard":
        assert np.array_equal(ker.c, c)  # lattice snap is exact
        assert np.array_equal(ker.values, vals) and np.array_equal(ker.value_index, vidx)
    else:
        assert np.abs(ker.c - c).max() < 1e-12
        assert ker.c[0].imag == 0 and all(ker.c[1:] == np.conj(ker.c[1:][::-1]))


def test_kernel_golden(fmp, gold):
    for i in range(int(gold["ker_count"][0])):
        kind, n, m, seed = (int(v) for v in gold[f"ker{i}_meta"])
        op = fmp.SensingOperator(KN[kind], n, gold[f"ker{i}_omega"])
        ker = op.kernel()
        if kind == 1:
            assert np.array_equal(ker.c, gold[f"ker{i}_c"])
            assert np.array_equal(ker.values, gold[f"ker{i}_values"])
        else:
            assert np.abs(ker.c - gold[f"ker{i}_c"]).max() < 1e-12


# ------------------------------------------------------------- transforms
@pytest.mark.parametrize("kind", ["fourier", "hadamard"])
@pytest.mark.parametrize("n,m", [(1, 1), (2, 1), (8, 3), (64, 16), (1024, 256), (4096, 1024),
                                 (8192, 2048), (16384, 4096), (65536, 8192), (1 << 18, 1 << 15),
                                 (1 << 20, 1 << 17), (1 << 22, 1 << 19)])
def test_apply_adjoint_matches_oracle(fmp, oracle, kind, n, m):
    # n >= 2^18 runs the two-pass transform (fmp_transform_4s.cu)
    om = oracle.make_row_selection(n, m, 7 + n)
    op = fmp.SensingOperator(kind, n, om)
    B = 3 if n <= 65536 else (2 if n <= (1 << 20) else 1)  # batch > 1 through the two-pass tiles too
    R = np.stack([oracle.rng_complex_gaussian(oracle.derive_seed(n, b), m) for b in range(B)])
    H, idx = op.apply_adjoint(R, argmax=True)
    for b in range(B):
        want = oracle.apply_adjoint(kind, n, om, R[b])
        assert rel(H[b], want) < 1e-13
        assert idx[b] == oracle.argmax_magnitude(want) + 1
    if kind == "fourier" or n <= 4096:
        X = np.stack([oracle.rng_complex_gaussian(oracle.derive_seed(n, 100 + b), n) for b in range(B)])
        Y = op.apply(X)
        for b in range(B):
            assert rel(Y[b], oracle.apply(kind, n, om, X[b])) < 1e-13
        F = op.forward(X)
        A = op.adjoint(X)
        for b in range(B):
            assert rel(F[b], oracle.forward(kind, X[b])) < 1e-13
            assert rel(A[b], oracle.adjoint(kind, X[b])) < 1e-13


@pytest.mark.parametrize("dtype,tol", [(np.complex64, 1e-5), (np.float64, 1e-13), (np.float32, 1e-5)])
def test_apply_adjoint_other_dtypes(fmp, oracle, dtype, tol):
    n, m = 65536, 8192
    om = oracle.make_row_selection(n, m, 3)
    kind = "fourier" if dtype == np.complex64 else "hadamard"
    for n_, m_ in ((1024, 256), (n, m), (1 << 20, 1 << 17)):
        om = oracle.make_row_selection(n_, m_, 3)
        op = fmp.SensingOperator(kind, n_, om)
        r = oracle.rng_complex_gaussian(5, m_)
        if dtype in (np.float64, np.float32):
            r = r.real.copy()
        r = r.astype(dtype)
        h = op.apply_adjoint(r[None])[0]
        want = oracle.apply_adjoint(kind, n_, om, r.astype(np.complex128))
        assert rel(h, want) < tol


@pytest.mark.parametrize("dt", [np.float32, np.float64, np.complex64, np.complex128])
@pytest.mark.parametrize("n,m", [(65536, 8192), (65536, 8191), (1 << 17, 12345), (1 << 15, 4000)])
def test_apply_adjoint_fold_path(fmp, oracle, n, m, dt):
    """Batched Hadamard adjoint beyond one CTA (batch >= 64): the one-pass
    fold kernel (fmp_transform_fold.cu; f32: the register fold for 2, 4 or 8
    input blocks, two output blocks per walk with r staged
    by a bulk copy, 8-byte elements with r read through L1), or the job queue
    (c128); m * 4 bytes not a multiple of 16 takes the plain-load staging."""
    om = oracle.make_row_selection(n, m, 11 + m)
    op = fmp.SensingOperator("hadamard", n, om)
    B = 70
    R = np.stack([oracle.rng_complex_gaussian(oracle.derive_seed(m, b), m) for b in range(B)])
    R = (R.real if dt in (np.float32, np.float64) else R).astype(dt)
    H, idx = op.apply_adjoint(R, argmax=True)
    tol = 1e-6 if dt in (np.float32, np.complex64) else 1e-13
    for b in (0, 1, 37, B - 1):
        want = oracle.apply_adjoint("hadamard", n, om, R[b].astype(np.complex128))
        assert rel(H[b], want) < tol
        assert idx[b] == oracle.argmax_magnitude(H[b].astype(np.complex128)) + 1


# ------------------------------------------------------------ fast update
def test_fast_update_campaign(fmp, oracle):
    # test_kernel.cpp:178-219 recipe: fast = Phi^H (y - Phi_Lambda x) within 1e-10
    cases = 0
    for kind in ("fourier", "hadamard"):
        for n in (8, 16, 32, 64, 128, 256, 512, 4096):
            for trial in range(12):
                seed = oracle.derive_seed(61, n * 1000 + trial + (500000 if kind == "hadamard" else 0))
                s = oracle.rng_u64(seed, 2)
                m = 2 + int(s[0] % (n - 2))
                k = 1 + int(s[1] % min(40, m))
                om = oracle.make_row_selection(n, m, oracle.derive_seed(seed, 1))
                y = oracle.rng_complex_gaussian(oracle.derive_seed(seed, 2), m)
                sup = oracle.rng_sample(oracle.derive_seed(seed, 3), n, k)
                perm = np.argsort(oracle.rng_u64(oracle.derive_seed(seed, 5), k))
                sup = sup[perm]  # OMP keeps selection order, not sorted
                co = oracle.rng_complex_gaussian(oracle.derive_seed(seed, 4), k)
                xs = np.zeros(n, complex)
                xs[sup.astype(int) - 1] = co
                want = oracle.apply_adjoint(kind, n, om, y - oracle.apply(kind, n, om, xs))
                h0 = oracle.apply_adjoint(kind, n, om, y)
                op = fmp.SensingOperator(kind, n, om)
                got, idx = fmp.fast_update(h0, op, sup, co, argmax=True)
                assert rel(got, want) <= 1e-10
                assert rel(got, oracle.fast_update(kind, n, om, h0, sup, co)) <= 1e-13
                assert idx == oracle.argmax_magnitude(got) + 1
                cases += 1
    assert cases >= 190


def test_fast_update_batched_and_chunked(fmp, oracle):
    n, m = 2048, 512
    om = oracle.make_row_selection(n, m, 9)
    op = fmp.SensingOperator("fourier", n, om)
    B, t = 4, 1500  # t above the 1024-atom chunk
    H0 = np.stack([oracle.rng_complex_gaussian(100 + b, n) for b in range(B)])
    S = np.stack([oracle.rng_sample(200 + b, n, t)[np.argsort(oracle.rng_u64(300 + b, t))] for b in range(B)])
    X = np.stack([oracle.rng_complex_gaussian(400 + b, t) for b in range(B)]) * 1e-2
    got, idx = fmp.fast_update(H0, op, S, X, argmax=True)
    _, idx2 = fmp.fast_update(H0, op, S, X, argmax=True, want_h=False)
    for b in range(B):
        want = oracle.fast_update("fourier", n, om, H0[b], S[b], X[b])
        assert rel(got[b], want) < 1e-12
        assert idx[b] == idx2[b] == oracle.argmax_magnitude(want) + 1


@pytest.mark.parametrize("kind,dtype,tol", [("fourier", np.complex64, 1e-4),
                                            ("hadamard", np.float64, 1e-12),
                                            ("hadamard", np.float32, 1e-4),
                                            ("hadamard", np.complex128, 1e-12)])
def test_fast_update_dtypes_config3_shape(fmp, oracle, kind, dtype, tol):
    # config 3 shape: N=65536, M=8192, |Lambda| = 256, N(0,1) x and residual
    n, m, t = (65536, 8192, 256) if kind == "hadamard" else (16384, 4096, 128)
    om = oracle.make_row_selection(n, m, 21)
    op = fmp.SensingOperator(kind, n, om)
    real = dtype in (np.float64, np.float32)
    r = oracle.rng_complex_gaussian(22, m)
    x = oracle.rng_complex_gaussian(23, t)
    if real:
        r, x = np.sqrt(2) * r.real, np.sqrt(2) * x.real
    r = r.astype(dtype)
    x = x.astype(dtype)
    sup = oracle.rng_sample(24, n, t)
    h0 = op.apply_adjoint(r[None])[0]
    got = fmp.fast_update(h0[None], op, sup[None], x[None])[0]
    want = oracle.fast_update(kind, n, om, h0.astype(np.complex128), sup, x.astype(np.complex128))
    assert rel(got, want) < tol
    # size-independent property: fast update of (h0(y)) equals Phi^H(y - Phi x)
    xs = np.zeros(n, complex)
    xs[sup.astype(int) - 1] = x
    conv = oracle.apply_adjoint(kind, n, om, r.astype(np.complex128) - oracle.apply(kind, n, om, xs))
    assert rel(got, conv) < max(tol, 1e-10)


def test_fast_update_validation(fmp, oracle):
    om = oracle.make_row_selection(16, 4, 1)
    op = fmp.SensingOperator("hadamard", 16, om)
    h0 = np.ones(16, complex)
    assert np.array_equal(fmp.fast_update(h0, op, [], []), h0)
    for sup, co in (([1, 1], [1, 1]), ([0], [1]), ([17], [1])):
        with pytest.raises(fmp.InvalidArgument):
            fmp.fast_update(h0, op, sup, co)
    with pytest.raises(fmp.InvalidArgument):
        fmp.fast_update(np.ones(15, complex), op, [], [])


def test_operator_validation(fmp):
    with pytest.raises(fmp.InvalidArgument):
        fmp.SensingOperator("hadamard", 12, [1, 2])
    with pytest.raises(fmp.InvalidArgument):
        fmp.SensingOperator("fourier", 16, [3, 3, 5])
    with pytest.raises(fmp.InvalidArgument):
        fmp.SensingOperator("fourier", 16, [0, 4])
    with pytest.raises(fmp.InvalidArgument):
        fmp.SensingOperator("fourier", 16, [4, 17])
    with pytest.raises(fmp.InvalidArgument):
        fmp.SensingOperator("fourier", 16, [])
    op = fmp.SensingOperator("fourier", 16, [9, 2, 5])
    assert list(op.omega) == [2, 5, 9]


def test_argmax_band_ties(fmp, oracle):
    h = np.array([[1.0, 3.0, 3.0 * (1 - 2e-10), 3.0],
                  [1.0, 3.0 * (1 - 2e-10), 3.0, 0.5],
                  [1.0, 3.0 * (1 - 2e-9), 3.0, 0.5],
                  [0.0, 0.0, 0.0, 0.0]], complex)
    got = fmp.argmax_magnitude(h)
    assert list(got) == [oracle.argmax_magnitude(r) + 1 for r in h] == [2, 2, 3, 1]
    big = oracle.rng_complex_gaussian(5, 1 << 20)
    big[777777] = 10.0
    big[12345] = 10.0 * (1 - 1e-10)
    assert fmp.argmax_magnitude(big) == oracle.argmax_magnitude(big) + 1 == 12346


# --------------------------------------------------------------------- OMP
def _solve_both(fmp, oracle, kind, n, om, y, T, tol, mode, dtype=np.complex128, record=False):
    op = fmp.SensingOperator(kind, n, om)
    cfg = fmp.SolveConfig(max_iterations=T, residual_tolerance=tol, correlation_mode=mode,
                          record_correlations=record)
    g = fmp.omp_solve(op, np.asarray(y).astype(dtype), cfg)
    r = oracle.omp_solve(kind, n, om, np.asarray(y).astype(dtype).astype(np.complex128), T, tol, mode,
                         record=record)
    return g, r


def _assert_same(g, r, tol=1e-10, hist=False):
    assert g.support == [int(v) for v in r.support]
    assert g.iterations_run == r.iterations_run
    assert g.rank_deficient_abort == r.rank_deficient_abort
    if len(r.coeffs):
        assert rel(g.coeffs, r.coeffs) < tol
    assert abs(g.residual_norm - r.residual_norm) <= tol * max(r.residual_norm, 1e-300) + 1e-13
    if hist:
        assert len(g.correlation_history) == len(r.correlation_history)
        for p, q in zip(g.correlation_history, r.correlation_history):
            assert rel(p, q) < tol


def test_omp_modes_identical_supports(fmp, oracle):
    # test_solvers.cpp:157-186, plus correlation histories against the oracle
    for kind in ("fourier", "hadamard"):
        for trial in range(20):
            seed = oracle.derive_seed(70, trial)
            om = oracle.make_row_selection(128, 32, oracle.derive_seed(seed, 1))
            x, y, e = oracle.make_instance(kind, 128, om, 5, 0.05, seed)
            tol = 1e-9 * np.linalg.norm(y)
            for mode in ("conventional", "fast", "adaptive"):
                g, r = _solve_both(fmp, oracle, kind, 128, om, y, 5, tol, mode, record=True)
                _assert_same(g, r, hist=True)
                assert g.modes_used == r.mode_used


def test_omp_tie_seeds(fmp, oracle):
    # test_solvers.cpp:188-208: exact Hadamard magnitude ties
    for seed in (4898724841501167528, 14945121902286664584):
        om = oracle.make_row_selection(256, 16, oracle.derive_seed(seed, 1))
        x, y, e = oracle.make_instance("hadamard", 256, om, 8, 0.05, seed)
        tol = 1e-9 * np.linalg.norm(y)
        for mode in ("conventional", "fast"):
            g, r = _solve_both(fmp, oracle, "hadamard", 256, om, y, 8, tol, mode)
            _assert_same(g, r)


def test_omp_adaptive_switch(fmp, oracle):
    om = oracle.make_row_selection(64, 32, 41)
    x, y, e = oracle.make_instance("fourier", 64, om, 10, 0.0, 42)
    g, r = _solve_both(fmp, oracle, "fourier", 64, om, y, 10, 0.0, "adaptive", record=True)
    assert g.modes_used == [1] * 6 + [0] * 4
    _assert_same(g, r, hist=True)


def test_omp_noiseless_recovery_and_edges(fmp, oracle):
    # test_solvers.cpp:88-141
    for kind in ("fourier", "hadamard"):
        om = oracle.make_row_selection(64, 32, 11)
        x, y, e = oracle.make_instance(kind, 64, om, 3, 0.0, 12)
        g, r = _solve_both(fmp, oracle, kind, 64, om, y, 3, 1e-9 * np.linalg.norm(y), "fast")
        _assert_same(g, r)
        assert sorted(g.support) == list(np.flatnonzero(x) + 1)
        assert np.linalg.norm(g.x_hat - x) < 1e-8 * np.linalg.norm(x)
    op = fmp.SensingOperator("fourier", 32, oracle.make_row_selection(32, 8, 21))
    z = fmp.omp_solve(op, np.zeros(8, complex), fmp.default_config(2, 0.0))
    assert z.iterations_run == 0 and z.support == [] and z.residual_norm == 0.0
    with pytest.raises(fmp.InvalidArgument):
        fmp.omp_solve(op, np.zeros(7, complex), fmp.default_config(1, 1.0))
    with pytest.raises(fmp.InvalidArgument):
        fmp.omp_solve(op, np.ones(8, complex), fmp.SolveConfig(max_iterations=0))
    om = oracle.make_row_selection(32, 8, 21)
    x, y, e = oracle.make_instance("fourier", 32, om, 4, 0.0, 22)
    g, r = _solve_both(fmp, oracle, "fourier", 32, om, y, 8, 0.0, "conventional")
    assert g.iterations_run >= 4
    assert g.support[:4] == [int(v) for v in r.support[:4]]


def test_omp_golden(fmp, gold):
    for i in range(int(gold["omp_count"][0])):
        kind, n, m, T = (int(v) for v in gold[f"omp{i}_meta"])
        tol = float(gold[f"omp{i}_tol"][0])
        y = gold[f"omp{i}_y"]
        op = fmp.SensingOperator(KN[kind], n, gold[f"omp{i}_omega"])
        for mode in ("conventional", "fast", "adaptive"):
            dt = np.float64 if (kind == 1 and not np.iscomplex(y).any()) else np.complex128
            g = fmp.omp_solve(op, y.real if dt == np.float64 else y,
                              fmp.SolveConfig(T, tol, mode), dtype=dt)
            assert g.support == [int(v) for v in gold[f"omp{i}_{mode}_support"]], (i, mode)
            assert rel(g.coeffs, gold[f"omp{i}_{mode}_coeffs"]) < 1e-10
            it, rn, ab = gold[f"omp{i}_{mode}_scalars"]
            assert g.iterations_run == int(it)


@pytest.mark.parametrize("mode", ["conventional", "fast", "adaptive", "custom"])
def test_omp_config1(fmp, oracle, mode):
    # config 1: Hadamard N=1024, M=256, K=16, float64 real N(0,1), noiseless, K iterations
    n, m, k = 1024, 256, 16
    om = oracle.make_row_selection(n, m, oracle.derive_seed(1, 1 << 40))
    op = fmp.SensingOperator("hadamard", n, om)
    for b in range(8):
        x, y = oracle.make_real_instance("hadamard", n, om, k, oracle.derive_seed(1, b))
        tol = 1e-9 * np.linalg.norm(y)
        cfg = fmp.SolveConfig(k, tol, mode, fast_until=5)
        g = fmp.omp_solve(op, y.real, cfg, dtype=np.float64)
        r = oracle.omp_solve("hadamard", n, om, y, k, tol, "fast" if mode == "custom" else mode)
        _assert_same(g, r)
        assert sorted(g.support) == list(np.flatnonzero(x) + 1)


@pytest.mark.parametrize("mode", ["fast", "adaptive", "conventional"])
def test_omp_config2_shape(fmp, oracle, mode):
    # config 2 shape: Fourier N=4096, M=1024, K=64, c128, shared Omega, CN(0,1)
    n, m, k, B = 4096, 1024, 64, 6
    om = oracle.make_row_selection(n, m, oracle.derive_seed(2, 1 << 40))
    op = fmp.SensingOperator("fourier", n, om)
    Y, X, _ = fmp.make_batch("fourier", n, om, k, B, base_seed=2, want_x=True)
    tol = 1e-9 * np.linalg.norm(Y, axis=1)
    res = fmp.omp_solve_batch(op, Y, fmp.SolveConfig(k, 0.0, mode), tolerances=tol)
    for b in range(B):
        r = oracle.omp_solve("fourier", n, om, Y[b], k, tol[b], mode)
        s = int(res.support_size[b])
        assert list(res.support[b, :s]) == list(r.support)
        assert rel(res.coeffs[b, :s], r.coeffs) < 1e-10
        assert int(res.iterations[b]) == r.iterations_run
        assert sorted(res.support[b, :s]) == list(np.flatnonzero(X[b]) + 1)


@pytest.mark.parametrize("mode,dtype", [("gpu", np.complex128), ("fast", np.complex128),
                                        ("conventional", np.complex128), ("gpu", np.complex64)])
def test_omp_two_ctas_per_sm_batch(fmp, oracle, mode, dtype):
    """Batches of at least two problems per SM run the two-CTA-per-SM solver
    (256 threads each, kernel table through L1): every problem of a 320-signal
    batch against the oracle, and the same supports as the one-CTA solver."""
    n, m, k, B = 2048, 512, 24, 320
    om = oracle.make_row_selection(n, m, oracle.derive_seed(7, 1 << 40))
    op = fmp.SensingOperator("fourier", n, om)
    Y, X, _ = fmp.make_batch("fourier", n, om, k, B, base_seed=7, want_x=True)
    tol = 1e-9 * np.linalg.norm(Y, axis=1)
    Yd = Y.astype(dtype)
    res = fmp.omp_solve_batch(op, Yd, fmp.SolveConfig(k, 0.0, mode), tolerances=tol)
    os.environ["FMP_OMP_CTAS"] = "1"
    try:
        one = fmp.omp_solve_batch(op, Yd, fmp.SolveConfig(k, 0.0, mode), tolerances=tol)
    finally:
        del os.environ["FMP_OMP_CTAS"]
    assert np.array_equal(res.support, one.support)
    assert np.array_equal(res.iterations, one.iterations)
    omode = "fast" if mode == "gpu" else mode
    Yo = Yd.astype(np.complex128)
    for b in range(B):
        s = int(res.support_size[b])
        assert sorted(res.support[b, :s]) == list(np.flatnonzero(X[b]) + 1)
        if dtype == np.complex128 and (mode != "gpu" or b % 8 == 0):
            r = oracle.omp_solve("fourier", n, om, Yo[b], k, tol[b], omode)
            assert list(res.support[b, :s]) == list(r.support)
            assert rel(res.coeffs[b, :s], r.coeffs) < 1e-10


@pytest.mark.parametrize("dtype,tol", [(np.complex64, 1e-4), (np.complex128, 1e-10)])
def test_omp_config4_shape(fmp, oracle, dtype, tol):
    # config 4 shape (reduced batch): Fourier N=16384, M=4096, K=128, c64 and c128,
    # 30 dB noise, halt at ||r|| <= ||noise|| or 2K iterations
    n, m, k, B = 16384, 4096, 128, 2
    sigma = np.sqrt(k / (2 * n * 1e3))
    om = oracle.make_row_selection(n, m, oracle.derive_seed(4, 1 << 40))
    op = fmp.SensingOperator("fourier", n, om)
    Y, X, nn = fmp.make_batch("fourier", n, om, k, B, base_seed=4, noise_stddev=sigma, want_x=True)
    Y32 = Y.astype(dtype)
    res = fmp.omp_solve_batch(op, Y32, fmp.SolveConfig(2 * k, 0.0, "adaptive"), tolerances=nn)
    agree = 0
    for b in range(B):
        r = oracle.omp_solve("fourier", n, om, Y32[b].astype(np.complex128), 2 * k, nn[b], "adaptive")
        s = int(res.support_size[b])
        same = list(res.support[b, :s]) == list(r.support)
        agree += same
        if same:
            assert rel(res.coeffs[b, :s], r.coeffs) < tol
            assert int(res.iterations[b]) == r.iterations_run
        truth = set((np.flatnonzero(X[b]) + 1).tolist())
        assert len(truth & set(res.support[b, :s].tolist())) >= 0.9 * len(truth)
    assert agree == B


def test_omp_host_chunked_equals_device(fmp, oracle):
    # batches >= 8 x grid take a copy/compute-overlapped host path (with the
    # wrapper's page-locked results: fmp_capi.cu omp_host_streamed, one launch
    # fed by per-chunk ready flags): results must equal the device path bitwise
    import torch
    n, m, k, B = 1024, 256, 16, 1600
    rows = fmp.make_row_selection(n, m, 31)
    op = fmp.SensingOperator("fourier", n, rows)
    Y, _, _ = fmp.make_batch("fourier", n, rows, k, B, base_seed=31)
    tol = 1e-9 * np.linalg.norm(Y, axis=1)
    cfg = fmp.SolveConfig(k, 0.0, "fast")
    host = fmp.omp_solve_batch(op, Y, cfg, tolerances=tol)
    out = fmp.alloc_dev_result(B, k)
    fmp.omp_solve_dev(op, torch.from_numpy(Y).cuda(), cfg, out,
                      tolerances=torch.from_numpy(tol).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(host.support.astype(np.int64), out["support"].cpu().numpy())
    assert np.array_equal(host.coeffs, out["coeffs"].cpu().numpy())
    assert np.array_equal(host.iterations.astype(np.int64), out["iterations"].cpu().numpy())
    # page-locked measurements: the streamed path without its staging copy
    pinned = fmp.omp_solve_batch(op, torch.from_numpy(Y).pin_memory().numpy(), cfg, tolerances=tol)
    assert np.array_equal(pinned.support, host.support) and np.array_equal(pinned.coeffs, host.coeffs)
    for b in range(0, B, 397):
        r = oracle.omp_solve("fourier", n, rows, Y[b], k, tol[b], "fast")
        assert [int(v) for v in host.support[b, :int(host.support_size[b])]] == \
            [int(v) for v in r.support]


def test_omp_config1_shape_f32(fmp, oracle):
    # config-1 shape in f32 (Hadamard lattice fast tile, FP32 path): identical
    # supports to the oracle on the fp32-rounded measurements, x within 1e-4
    n, m, k = 1024, 256, 16
    om = oracle.make_row_selection(n, m, oracle.derive_seed(1, 1 << 40))
    op = fmp.SensingOperator("hadamard", n, om)
    for b in range(6):
        x, y = oracle.make_real_instance("hadamard", n, om, k, oracle.derive_seed(1, b))
        y32 = y.real.astype(np.float32)
        tol = 1e-5 * np.linalg.norm(y32)
        for mode in ("fast", "conventional"):
            g = fmp.omp_solve(op, y32, fmp.SolveConfig(k, tol, mode), dtype=np.float32)
            r = oracle.omp_solve("hadamard", n, om, y32.astype(np.complex128), k, tol, mode)
            assert g.support == [int(v) for v in r.support]
            assert rel(g.coeffs, r.coeffs) < 1e-4
            assert sorted(g.support) == list(np.flatnonzero(x) + 1)


def test_omp_host_chunked_pageable_buffers(fmp):
    # pageable (non-page-locked) input and result buffers take the staging
    # path of the chunked host call; results must equal the wrapper's bitwise
    import ctypes as C
    n, m, k, B = 1024, 256, 16, 1600
    rows = fmp.make_row_selection(n, m, 32)
    op = fmp.SensingOperator("hadamard", n, rows)
    Y, _, _ = fmp.make_batch("hadamard", n, rows, k, B, base_seed=32)
    Y = np.ascontiguousarray(Y.real)
    tol = np.ascontiguousarray(1e-9 * np.linalg.norm(Y, axis=1))
    cfg = fmp.SolveConfig(k, 0.0, "fast")
    ref = fmp.omp_solve_batch(op, Y, cfg, tolerances=tol)
    sup = np.zeros((B, k), np.uint64)
    co = np.zeros((B, k), np.complex128)
    sz = np.zeros(B, np.uint64)
    it = np.zeros(B, np.uint64)
    rn = np.zeros(B)
    ab = np.zeros(B, np.int32)
    res = fmp.OmpResult(sup.ctypes.data, co.ctypes.data, sz.ctypes.data, it.ctypes.data,
                        rn.ctypes.data, ab.ctypes.data, None, None, None)
    c = fmp._config(cfg, tol.ctypes.data_as(C.POINTER(C.c_double)))
    assert fmp._lib.fmp_omp_solve(op.handle, fmp.DTYPES[Y.dtype], Y.ctypes.data, B, C.byref(c),
                                  C.byref(res)) == 0
    assert np.array_equal(sup, ref.support) and np.array_equal(co, ref.coeffs)
    assert np.array_equal(sz, ref.support_size) and np.array_equal(it, ref.iterations)
    assert np.array_equal(rn, ref.residual) and np.array_equal(ab.astype(bool), ref.aborted)


@pytest.mark.parametrize("solver", ["omp", "cosamp"])
def test_streamed_input_failure_leaves_context_usable(fmp, oracle, solver):
    """The host-buffer solve that streams its input into a running kernel:
    when the host side fails mid-stream (test hook), the abort word releases
    the kernel (no trap, no hang), the call reports the error, and the same
    context solves correctly afterwards."""
    n, m, k, B = 1024, 256, 12, 1600  # >= 8 x grid: the streamed path
    rows = fmp.make_row_selection(n, m, 41)
    op = fmp.SensingOperator("fourier", n, rows)
    Y, _, _ = fmp.make_batch("fourier", n, rows, k, B, base_seed=41)
    tol = 1e-9 * np.linalg.norm(Y, axis=1)
    cfg = fmp.SolveConfig(k, 0.0, "fast")

    def solve():
        if solver == "omp":
            return fmp.omp_solve_batch(op, Y, cfg, tolerances=tol)
        return fmp.cosamp_solve_batch(op, Y, k, cfg, tolerances=tol, want_history=False)
    os.environ["FMP_TEST_STALL_INPUT"] = "1"
    try:
        with pytest.raises(Exception):
            solve()
    finally:
        del os.environ["FMP_TEST_STALL_INPUT"]
    res = solve()
    for b in (0, B // 2, B - 1):
        s = int(res.support_size[b])
        if solver == "omp":
            r = oracle.omp_solve("fourier", n, rows, Y[b], k, tol[b], "fast")
            assert [int(v) for v in res.support[b, :s]] == [int(v) for v in r.support]
        else:
            r, _ = oracle.cosamp_solve("fourier", n, rows, Y[b], k, k, tol[b], "fast")
            assert [int(v) for v in res.support[b, :s]] == [int(v) for v in r.support]
