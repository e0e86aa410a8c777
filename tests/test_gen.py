"""GPU-side instance generation (csrc/fmp_gen.cu).

The device generator must reproduce fmp_make_batch bit for bit (which
tests/test_abi.py pins to the reference's make_instance draws).  Its
transcendentals are correctly rounded double-double evaluations with a
host (glibc) recomputation near rounding midpoints; the CPU tests check the
double-double code against 200-bit mpmath and that every glibc disagreement
falls inside the recomputed band.
"""
import math

import numpy as np
import pytest

ARGS_SEED = 17


def _args(n):
    rng = np.random.default_rng(ARGS_SEED)
    u1 = (rng.integers(0, 2**53, n, dtype=np.uint64).astype(np.float64) + 1.0) * 2.0**-53
    ang = 2.0 * np.pi * (rng.integers(0, 2**53, n, dtype=np.uint64).astype(np.float64) * 2.0**-53)
    th = -2.0 * np.pi * np.arange(n, dtype=np.float64) / n
    return u1, ang, th


def test_dd_functions_correctly_rounded(fmp):
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.prec = 200
    u1, ang, th = _args(1500)
    edge_log = np.array([1.0, 2.0**-53, 0.5, 0.7071067811865476, 1 - 2.0**-53, 0.75])
    edge_trig = np.array([0.0, -0.0, 1e-20, math.pi, math.pi / 2, 2 * math.pi, -2 * math.pi,
                          3 * math.pi / 2, 7.9, -7.9])
    for name, xs in (("log", np.concatenate([u1, edge_log])),
                     ("cos", np.concatenate([ang, th, edge_trig])),
                     ("sin", np.concatenate([ang, th, edge_trig]))):
        out, frac = fmp.dd_eval(name, xs)
        f = getattr(mpmath, name)
        for v, o, fr in zip(xs, out, frac):
            cr = float(f(mpmath.mpf(float(v))))
            assert o == cr or (o == 0.0 and cr == 0.0), (name, v, o, cr)
            assert 0.0 <= fr <= 0.5
    # glibc's own sign of zero
    assert math.copysign(1.0, fmp.dd_eval("sin", [-0.0])[0][0]) == -1.0


def test_glibc_disagreements_fall_in_the_recomputed_band(fmp):
    # a value is recomputed on the host when frac > 0.5 - 0.025 (fmp_gen.cu
    # kBand); outside that band glibc must agree with the rounded value
    u1, ang, th = _args(200000)
    for name, xs in (("log", u1), ("cos", ang), ("sin", ang), ("cos", th), ("sin", th)):
        out, frac = fmp.dd_eval(name, xs)
        ref = np.array([getattr(math, name)(v) for v in xs])
        differ = ref != out
        assert not np.any(differ & (frac <= 0.475)), name
        assert 0.03 < np.mean(frac > 0.475) < 0.07  # ~5 % listed


def test_make_batch_dev_rejects_like_make_instance(fmp):
    # argument checks of make_instance (sensing.cpp:121-124) come before any
    # device work, so they are testable without a GPU only through the C ABI
    assert fmp._lib.fmp_make_batch_dev(None, 4, 0.0, 0, 1, 0, 1, None, None, None, None, None) == 1


# ------------------------------------------------------------------ GPU
CASES = [
    # kind, n, m, k, batch, sigma, real, first
    ("fourier", 4096, 1024, 64, 48, 0.0, False, 0),          # config-2 shape
    ("fourier", 16384, 4096, 128, 6, math.sqrt(128 / (2 * 16384 * 1e3)), False, 5),  # config-4 shape, 30 dB
    ("hadamard", 1024, 256, 16, 40, 0.0, True, 0),           # config-1 shape, real N(0,1)
    ("hadamard", 2048, 512, 20, 12, 0.05, False, 3),         # complex, noisy
    ("fourier", 256, 64, 0, 4, 0.1, False, 0),               # empty support, noise only
    ("fourier", 64, 40, 39, 9, 0.0, False, 1),               # k = m - 1, dense sample
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[1]}-k{c[3]}" for c in CASES])
def test_make_batch_dev_bit_identical(fmp, case):
    import torch
    kind, n, m, k, B, sigma, real, first = case
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(77, 1 << 40))
    op = fmp.SensingOperator(kind, n, rows, fmp.Context(0))
    Yh, Xh, nnh = fmp.make_batch(kind, n, rows, k, B, base_seed=77, first=first,
                                 noise_stddev=sigma, real=real, want_x=True)
    Yd, Xd, nnd, fix = fmp.make_batch_dev(op, k, B, base_seed=77, first=first, noise_stddev=sigma,
                                          real=real, want_x=True)
    torch.cuda.synchronize()
    assert np.array_equal(Yd.cpu().numpy().view(np.uint64), Yh.view(np.uint64))
    assert np.array_equal(Xd.cpu().numpy().view(np.uint64), Xh.view(np.uint64))
    assert np.array_equal(nnd.cpu().numpy().view(np.uint64), nnh.view(np.uint64))
    assert fix >= 0


@pytest.mark.gpu
def test_make_batch_dev_errors(fmp):
    rows = fmp.make_row_selection(256, 64, 3)
    op = fmp.SensingOperator("fourier", 256, rows, fmp.Context(0))
    with pytest.raises(fmp.FmpError):
        fmp.make_batch_dev(op, 64, 2, base_seed=1)            # k >= m
    with pytest.raises(fmp.FmpError):
        fmp.make_batch_dev(op, 4, 2, base_seed=1, real=True)  # real needs Hadamard
    with pytest.raises(fmp.FmpError):
        fmp.make_batch_dev(op, 4, 2, base_seed=1, noise_stddev=-1.0)


@pytest.mark.gpu
def test_dd_functions_same_on_device(fmp):
    u1, ang, th = _args(50000)
    for name, xs in (("log", u1), ("cos", ang), ("sin", ang), ("cos", th), ("sin", th)):
        oh, fh = fmp.dd_eval(name, xs)
        od, fd = fmp.dd_eval(name, xs, device=True)
        assert np.array_equal(oh.view(np.uint64), od.view(np.uint64)), name
        assert np.array_equal(fh, fd), name
