"""CPU tests: pin the oracle restatement to the reference.

* against the golden fixtures the reference itself produced
  (tests/golden/reference_golden.npz, made by tests/golden/make_golden.py);
* against the live reference library (oracle/_ref) when it is built;
* the reference's own test recipes (proj/tests/test_kernel.cpp,
  test_solvers.cpp, test_transform.cpp, test_random.cpp) restated as
  properties of the restatement.
"""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")
KN = {0: "fourier", 1: "hadamard"}


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


# ------------------------------------------------------------ golden pins
def test_rng_matches_golden(oracle, gold):
    for s in (0, 1, 5, 42, 5489):
        assert np.array_equal(oracle.rng_u64(s, 32), gold[f"rng_u64_{s}"])
        assert np.array_equal(oracle.rng_complex_gaussian(s, 16), gold[f"rng_cg_{s}"])
        assert np.array_equal(oracle.rng_sample(s, 100, 13), gold[f"rng_sample_{s}"])
    for b, i, d in gold["derive_seed"]:
        assert oracle.derive_seed(int(b), int(i)) == int(d)


def test_kernels_match_golden_bitwise(oracle, gold):
    for i in range(int(gold["ker_count"][0])):
        kind, n, m, seed = (int(v) for v in gold[f"ker{i}_meta"])
        om = oracle.make_row_selection(n, m, seed)
        assert np.array_equal(om, gold[f"ker{i}_omega"])
        c, vals, vidx = oracle.compute_kernel(KN[kind], n, om)
        assert np.array_equal(c, gold[f"ker{i}_c"])
        assert np.array_equal(vals, gold[f"ker{i}_values"])
        assert np.array_equal(vidx, gold[f"ker{i}_vidx"])


def test_fast_update_matches_golden_bitwise(oracle, gold):
    for i in range(int(gold["fu_count"][0])):
        kind, n, m = (int(v) for v in gold[f"fu{i}_meta"])
        om = gold[f"fu{i}_omega"]
        h0 = oracle.apply_adjoint(KN[kind], n, om, gold[f"fu{i}_y"])
        assert np.array_equal(h0, gold[f"fu{i}_h0"])
        h = oracle.fast_update(KN[kind], n, om, h0, gold[f"fu{i}_support"], gold[f"fu{i}_coeffs"])
        assert np.array_equal(h, gold[f"fu{i}_h"])


def test_omp_matches_golden_bitwise(oracle, gold):
    for i in range(int(gold["omp_count"][0])):
        kind, n, m, T = (int(v) for v in gold[f"omp{i}_meta"])
        tol = float(gold[f"omp{i}_tol"][0])
        for mode in ("conventional", "fast", "adaptive"):
            r = oracle.omp_solve(KN[kind], n, gold[f"omp{i}_omega"], gold[f"omp{i}_y"], T, tol,
                                 mode=mode)
            assert np.array_equal(r.support, gold[f"omp{i}_{mode}_support"]), (i, mode)
            assert np.array_equal(r.coeffs, gold[f"omp{i}_{mode}_coeffs"]), (i, mode)
            it, rn, ab = gold[f"omp{i}_{mode}_scalars"]
            assert r.iterations_run == int(it) and r.residual_norm == rn and r.rank_deficient_abort == bool(ab)
            assert r.mode_used[: r.iterations_run] == list(gold[f"omp{i}_{mode}_modes"][: r.iterations_run])


def test_cosamp_matches_golden_bitwise(oracle, gold):
    # CoSaMP (solvers.cpp:413-544) against the reference's own outputs
    for i in range(int(gold["cos_count"][0])):
        kind, n, m, k, T = (int(v) for v in gold[f"cos{i}_meta"])
        tol = float(gold[f"cos{i}_tol"][0])
        for mode in ("conventional", "fast"):
            r, sh = oracle.cosamp_solve(KN[kind], n, gold[f"cos{i}_omega"], gold[f"cos{i}_y"], k, T,
                                        tol, mode=mode)
            assert np.array_equal(r.support, gold[f"cos{i}_{mode}_support"]), (i, mode)
            assert np.array_equal(r.coeffs, gold[f"cos{i}_{mode}_coeffs"]), (i, mode)
            it, rn, ab = gold[f"cos{i}_{mode}_scalars"]
            assert r.iterations_run == int(it) and r.residual_norm == rn
            assert r.rank_deficient_abort == bool(ab)
            hist = gold[f"cos{i}_{mode}_history"]
            assert [list(row) for row in sh] == [list(row[row > 0]) for row in hist[: r.iterations_run]]


def test_cosamp_edge_cases(oracle):
    # test_solvers.cpp:236-277: noiseless recovery, k = 0, rank-deficient abort
    for kind in ("fourier", "hadamard"):
        om = oracle.make_row_selection(64, 32, 51)
        x, y, e = oracle.make_instance(kind, 64, om, 4, 0.0, 52)
        r, _ = oracle.cosamp_solve(kind, 64, om, y, 4, 8, 1e-9 * np.linalg.norm(y))
        assert list(r.support) == [j + 1 for j in np.flatnonzero(x)]
        assert r.residual_norm < 1e-9 * np.linalg.norm(y)
    om = oracle.make_row_selection(64, 8, 61)
    x, y, e = oracle.make_instance("fourier", 64, om, 4, 0.0, 62)
    r, _ = oracle.cosamp_solve("fourier", 64, om, y, 0, 1, np.linalg.norm(y))
    assert r.iterations_run == 0 and len(r.support) == 0
    a, sa = oracle.cosamp_solve("fourier", 64, om, y, 4, 6, 0.0, "conventional")
    b, sb = oracle.cosamp_solve("fourier", 64, om, y, 4, 6, 0.0, "fast")
    assert a.rank_deficient_abort and b.rank_deficient_abort
    assert a.iterations_run == b.iterations_run
    assert [list(v) for v in sa] == [list(v) for v in sb]


# ------------------------------------------------- live reference agreement
def test_restatement_bitwise_equals_reference(oracle, reference):
    for kind in ("fourier", "hadamard"):
        for n, m, k in ((32, 8, 3), (128, 32, 5), (512, 128, 12)):
            for seed in range(4):
                om = oracle.make_row_selection(n, m, oracle.derive_seed(seed, 1))
                x, y, e = oracle.make_instance(kind, n, om, k, 0.05, seed)
                x2, y2, e2 = reference.make_instance(kind, n, om, k, 0.05, seed)
                assert np.array_equal(y, y2) and np.array_equal(x, x2)
                for mode in ("conventional", "fast", "adaptive"):
                    for ls in ("qr", "normal"):
                        a = oracle.omp_solve(kind, n, om, y, k, 1e-9 * np.linalg.norm(y), mode, ls,
                                             symmetry=seed % 2 == 0, record=True)
                        b = reference.omp_solve(kind, n, om, y, k, 1e-9 * np.linalg.norm(y), mode, ls,
                                                symmetry=seed % 2 == 0, record=True)
                        assert np.array_equal(a.support, b.support)
                        assert np.array_equal(a.coeffs, b.coeffs)
                        assert a.residual_norm == b.residual_norm
                        for p, q in zip(a.correlation_history, b.correlation_history):
                            assert np.array_equal(p, q)


def test_cosamp_restatement_equals_reference(oracle, reference):
    # all modes, both kinds, noisy and noiseless, 3k > n and 3k > m shapes
    for kind in ("fourier", "hadamard"):
        for (n, m, k) in ((64, 32, 4), (256, 96, 8), (512, 128, 16), (64, 64, 40), (256, 16, 8)):
            for seed in range(3):
                om = oracle.make_row_selection(n, m, oracle.derive_seed(seed, 1))
                y = oracle.make_instance(kind, n, om, k, 0.05 if seed % 2 else 0.0, seed)[1]
                tol = 1e-9 * np.linalg.norm(y) if seed else 0.0
                for mode in ("conventional", "fast", "adaptive"):
                    a, sa = oracle.cosamp_solve(kind, n, om, y, k, max(k, 6), tol, mode, record=True)
                    b, sb = reference.cosamp_solve(kind, n, om, y, k, max(k, 6), tol, mode, record=True)
                    assert np.array_equal(a.support, b.support) and np.array_equal(a.coeffs, b.coeffs)
                    assert (a.iterations_run, a.residual_norm, a.rank_deficient_abort) == \
                        (b.iterations_run, b.residual_norm, b.rank_deficient_abort)
                    assert [list(v) for v in sa] == [list(v) for v in sb]
                    assert a.mode_used == b.mode_used
                    for p, q in zip(a.correlation_history, b.correlation_history):
                        assert np.array_equal(p, q)


def test_least_squares_and_rank_errors(oracle, reference):
    # test_solvers.cpp:39-86
    om = oracle.make_row_selection(64, 16, 3)
    x, y, e = oracle.make_instance("fourier", 64, om, 5, 0.1, 4)
    sup = [3, 17, 29, 40, 61]
    a = oracle.least_squares("fourier", 64, om, sup, y, "qr")
    b = oracle.least_squares("fourier", 64, om, sup, y, "normal")
    assert np.abs(a - b).max() < 1e-8
    assert np.array_equal(a, reference.least_squares("fourier", 64, om, sup, y, "qr"))
    om = oracle.make_row_selection(32, 8, 5)
    x, y, e = oracle.make_instance("hadamard", 32, om, 2, 0.0, 6)
    from oracle import OracleError
    for impl in (oracle, reference):
        for meth in ("qr", "normal"):
            with pytest.raises(OracleError) as ex:
                impl.least_squares("hadamard", 32, om, [7, 7], y, meth)
            assert ex.value.status == 2 and ex.value.aux == 1


# ------------------------------------------- reference test recipes (restated)
def _dense(kind, n):
    if kind == "fourier":
        r = np.arange(n)
        return np.exp(-2j * np.pi * ((r[:, None] * r[None, :]) % n) / n) / np.sqrt(n)
    h = np.array([[1.0]])
    while h.shape[0] < n:
        h = np.block([[h, h], [h, -h]])
    return h / np.sqrt(n)


def test_kernel_vs_dense_definition(oracle):
    # test_kernel.cpp:41-63
    for kind in ("fourier", "hadamard"):
        for n in (4, 16, 64):
            d = _dense(kind, n)
            for trial in range(0, 100, 7):
                m = 1 + trial % (n - 1)
                om = oracle.make_row_selection(n, m, oracle.derive_seed(50, n * 100 + trial))
                c, vals, vidx = oracle.compute_kernel(kind, n, om)
                rows = d[om.astype(int) - 1]
                ref = rows.conj().T @ rows[:, 0]
                assert np.abs(c - ref).max() < 1e-12


def test_kernel_conditioning_exact(oracle):
    # test_kernel.cpp:65-107
    om = oracle.make_row_selection(64, 16, 3)
    c, vals, vidx = oracle.compute_kernel("fourier", 64, om)
    assert c[0].imag == 0.0 and c[32].imag == 0.0
    assert all(c[j] == np.conj(c[64 - j]) for j in range(1, 64))
    assert len(vals) == 0
    c, vals, vidx = oracle.compute_kernel("hadamard", 64, om)
    assert 0 < len(vals) <= 17 and np.all(np.diff(vals) > 0)
    assert np.array_equal(c.real, vals[vidx]) and np.all(c.imag == 0)
    assert np.all(c.real * 64 == np.round(c.real * 64)) and c[0].real == 16 / 64
    for kind in ("fourier", "hadamard"):
        c, _, _ = oracle.compute_kernel(kind, 32, np.arange(1, 33))
        assert abs(c[0] - 1) < 1e-12 and np.abs(c[1:]).max() < 1e-12


def test_fast_update_equals_conventional_campaign(oracle):
    # test_kernel.cpp:178-219: >= 1000 cases within 1e-10 relative
    cases = 0
    for kind in ("fourier", "hadamard"):
        for n in (8, 16, 32, 64, 128, 256):
            for trial in range(60):
                seed = oracle.derive_seed(60, n * 1000 + trial + (500000 if kind == "hadamard" else 0))
                s = oracle.rng_u64(seed, 2)
                m = 2 + int(s[0] % (n - 2))
                k = 1 + int(s[1] % min(8, m))
                om = oracle.make_row_selection(n, m, oracle.derive_seed(seed, 1))
                y = oracle.rng_complex_gaussian(oracle.derive_seed(seed, 2), m)
                sup = oracle.rng_sample(oracle.derive_seed(seed, 3), n, k)
                co = oracle.rng_complex_gaussian(oracle.derive_seed(seed, 4), k)
                xs = np.zeros(n, complex)
                xs[sup.astype(int) - 1] = co
                want = oracle.apply_adjoint(kind, n, om, y - oracle.apply(kind, n, om, xs))
                h0 = oracle.apply_adjoint(kind, n, om, y)
                for sym in ((False, True) if kind == "fourier" else (False,)):
                    got = oracle.fast_update(kind, n, om, h0, sup, co, symmetry=sym)
                    assert np.linalg.norm(got - want) <= 1e-10 * max(np.linalg.norm(want), 1e-300)
                    cases += 1
    assert cases >= 1000


def test_fast_update_validation(oracle):
    # test_kernel.cpp:221-236
    from oracle import OracleError
    om = oracle.make_row_selection(16, 4, 1)
    h0 = np.ones(16, complex)
    assert np.array_equal(oracle.fast_update("hadamard", 16, om, h0, [], []), h0)
    for sup, co in (([1, 1], [1, 1]), ([0], [1]), ([17], [1])):
        with pytest.raises(OracleError):
            oracle.fast_update("hadamard", 16, om, h0, sup, co)


def test_modes_walk_identical_supports(oracle):
    # test_solvers.cpp:157-186
    for kind in ("fourier", "hadamard"):
        for trial in range(50):
            seed = oracle.derive_seed(70, trial)
            om = oracle.make_row_selection(128, 32, oracle.derive_seed(seed, 1))
            x, y, e = oracle.make_instance(kind, 128, om, 5, 0.05, seed)
            tol = 1e-9 * np.linalg.norm(y)
            rs = [oracle.omp_solve(kind, 128, om, y, 5, tol, mode, record=True,
                                   symmetry=trial % 2 == 0)
                  for mode in ("conventional", "fast", "adaptive")]
            assert rs[0].support_history == rs[1].support_history == rs[2].support_history
            for p, q in zip(rs[0].correlation_history, rs[1].correlation_history):
                assert np.linalg.norm(p - q) <= 1e-10 * max(np.linalg.norm(p), 1e-300)


def test_tie_seeds(oracle):
    # test_solvers.cpp:188-208
    for seed in (4898724841501167528, 14945121902286664584):
        om = oracle.make_row_selection(256, 16, oracle.derive_seed(seed, 1))
        x, y, e = oracle.make_instance("hadamard", 256, om, 8, 0.05, seed)
        tol = 1e-9 * np.linalg.norm(y)
        a = oracle.omp_solve("hadamard", 256, om, y, 8, tol, "conventional")
        b = oracle.omp_solve("hadamard", 256, om, y, 8, tol, "fast")
        assert list(a.support) == list(b.support)


def test_adaptive_switch_and_crossover(oracle):
    # test_solvers.cpp:210-234, acceptance.cpp:166-188
    assert oracle.crossover_iteration("fourier", 64) == 6
    assert oracle.crossover_iteration("fourier", 4096) == 11
    assert oracle.crossover_iteration("hadamard", 1024) == 11
    om = oracle.make_row_selection(64, 32, 41)
    x, y, e = oracle.make_instance("fourier", 64, om, 10, 0.0, 42)
    r = oracle.omp_solve("fourier", 64, om, y, 10, 0.0, "adaptive")
    assert r.mode_used == [1] * 6 + [0] * 4  # t = 1 is booked under the plan (solvers.cpp:336-340)


def test_transform_small_known_values(oracle):
    # test_transform.cpp:34-101
    for kind in ("fourier", "hadamard"):
        for n in (1, 2, 4, 8, 16, 32, 64):
            d = _dense(kind, n)
            v = oracle.rng_complex_gaussian(oracle.derive_seed(11, n), n)
            assert np.linalg.norm(oracle.forward(kind, v) - d @ v) < 1e-10 * np.linalg.norm(v)
            assert np.linalg.norm(oracle.adjoint(kind, v) - d.conj().T @ v) < 1e-10 * np.linalg.norm(v)
    assert abs(oracle.entry("fourier", 4, 2, 2) - (-0.5j)) < 1e-15
    t = oracle.forward("hadamard", np.ones(2, complex))
    assert abs(t[0] - np.sqrt(2)) < 1e-15 and abs(t[1]) < 1e-15


def test_argmax_band(oracle):
    # solvers.cpp:90-101: first index within 1e-9 of the max wins
    h = np.array([1.0, 3.0, 3.0 * (1 - 2e-10), 3.0], complex)
    assert oracle.argmax_magnitude(h) == 1
    h = np.array([1.0, 3.0 * (1 - 2e-10), 3.0], complex)
    assert oracle.argmax_magnitude(h) == 1
    h = np.array([1.0, 3.0 * (1 - 2e-9), 3.0], complex)
    assert oracle.argmax_magnitude(h) == 2
