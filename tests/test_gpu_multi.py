"""The multi-device batch path: fmp_omp_solve_multi (one operator per GPU,
contiguous blocks of the batch, one host thread per device, no collective)
and the seeded C++ driver fmp_driver over it.  One GPU is visible on the
test box, so the several "devices" are several contexts on cuda:0: the
blocks then run on one GPU through independent contexts — the same host
code path as on eight GPUs (the block split, the per-block offsets of every
input and output array, the per-thread error propagation)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "paper_1205_4139_b200", "fmp_driver")


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def test_driver_built():
    assert os.path.exists(DRIVER), "fmp_driver missing: run python -m paper_1205_4139_b200.build"


@pytest.mark.gpu
@pytest.mark.parametrize("nops,B", [(2, 37), (3, 600), (4, 5)])
def test_multi_blocks_match_one_call(fmp, oracle, nops, B):
    n, m, k = 1024, 256, 12
    rows = fmp.make_row_selection(n, m, fmp.derive_seed(31, 1 << 40))
    Y, X, _ = fmp.make_batch("fourier", n, rows, k, B, base_seed=31, want_x=True)
    tol = 1e-9 * np.linalg.norm(Y, axis=1)
    cfg = fmp.SolveConfig(k, 0.0, "fast")
    ops = [fmp.SensingOperator("fourier", n, rows, fmp.Context(0)) for _ in range(nops)]
    multi = fmp.omp_solve_multi(ops, Y, cfg, tolerances=tol)
    one = fmp.omp_solve_batch(ops[0], Y, cfg, tolerances=tol)
    assert np.array_equal(multi.support, one.support)
    assert np.array_equal(multi.support_size, one.support_size)
    assert np.array_equal(multi.iterations, one.iterations)
    assert rel(multi.coeffs, one.coeffs) < 1e-12
    # every block against the oracle on its first signal
    per = -(-B // nops)
    for b in range(0, B, per):
        r = oracle.omp_solve("fourier", n, rows, Y[b], k, float(tol[b]), "fast")
        s = int(multi.support_size[b])
        assert [int(v) for v in multi.support[b, :s]] == [int(v) for v in r.support]
        assert rel(multi.coeffs[b, :s], r.coeffs) < 1e-10


@pytest.mark.gpu
def test_multi_rejects_mismatched_operators(fmp):
    n, m = 1024, 256
    a = fmp.SensingOperator("fourier", n, fmp.make_row_selection(n, m, 1))
    b = fmp.SensingOperator("fourier", n, fmp.make_row_selection(n, m, 2))
    Y, _, _ = fmp.make_batch("fourier", n, fmp.make_row_selection(n, m, 1), 4, 4, base_seed=1)
    with pytest.raises(fmp.InvalidArgument):
        fmp.omp_solve_multi([a, b], Y, fmp.SolveConfig(4, 0.0, "fast"))


@pytest.mark.gpu
@pytest.mark.parametrize("args", [["--config", "2", "--batch", "512"], ["--config", "1"],
                                  ["--config", "4", "--batch", "256", "--dtype", "c64", "--mode", "adaptive"]])
def test_driver_runs_and_recovers(args):
    r = subprocess.run([DRIVER, "--gpus", "1", "--steps", "2", "--warmup", "1"] + args,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0
    # noiseless configs recover every true support; the 30 dB config most
    assert line["true_support_recovered"] >= (0.5 if "4" in args[1] else 1.0)
