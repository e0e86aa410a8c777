"""TEST INFRASTRUCTURE ONLY — numpy front end for the CPU oracles.

Two interchangeable backends export ``oracle/oracle_abi.h``:

* ``restatement`` — ``oracle/_build/libfmp_oracle.so``, the plain-C restatement
  of the reference algorithm (``oracle/fmp_oracle.c``);
* ``reference``   — ``oracle/_ref/libfmp_ref.so``, the unmodified reference
  sources (``/root/reference/proj/src``) compiled by ``oracle/Makefile``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline /
``--impl reference``) may import this module, and only as the checker or the
CPU baseline; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "restatement": os.path.join(HERE, "_build", "libfmp_oracle.so"),
    "reference": os.path.join(HERE, "_ref", "libfmp_ref.so"),
}

KIND = {"fourier": 0, "hadamard": 1}
MODE = {"conventional": 0, "fast": 1, "adaptive": 2}
LS = {"qr": 0, "normal": 1}

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")


class SolveConfig(C.Structure):
    _fields_ = [
        ("max_iterations", C.c_uint64),
        ("residual_tolerance", C.c_double),
        ("mode", C.c_int),
        ("ls_method", C.c_int),
        ("fourier_symmetry", C.c_int),
        ("record_correlations", C.c_int),
    ]


class SolveResult(C.Structure):
    _fields_ = [
        ("support", C.POINTER(C.c_uint64)),
        ("coeffs", C.POINTER(C.c_double)),
        ("support_size", C.c_uint64),
        ("iterations_run", C.c_uint64),
        ("residual_norm", C.c_double),
        ("rank_deficient_abort", C.c_int),
        ("history_len", C.c_uint64),
        ("correlation_history", C.POINTER(C.c_double)),
        ("mode_used", C.POINTER(C.c_int)),
    ]


class OracleError(RuntimeError):
    def __init__(self, status: int, aux: int = 0):
        super().__init__(f"oracle status {status}")
        self.status = status
        self.aux = aux


@dataclass
class Recovery:
    support: np.ndarray
    coeffs: np.ndarray
    iterations_run: int
    residual_norm: float
    rank_deficient_abort: bool
    correlation_history: list = field(default_factory=list)
    mode_used: list = field(default_factory=list)

    @property
    def support_history(self):
        return [list(self.support[: i + 1]) for i in range(self.iterations_run)]


def build(which: str = "all") -> None:
    """Compile the oracle(s) with oracle/Makefile (reference needs /root/reference)."""
    subprocess.run(["make", "-s", "-C", HERE, which], check=True)


def _c(z) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(z, dtype=np.complex128)).view(np.float64)


def _u(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.uint64))


class Oracle:
    def __init__(self, which: str = "restatement"):
        path = PATHS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.which = which
        L = self.lib = C.CDLL(path)
        L.fmpo_derive_seed.restype = C.c_uint64
        L.fmpo_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.fmpo_splitmix64.restype = C.c_uint64
        L.fmpo_splitmix64.argtypes = [C.c_uint64]
        L.fmpo_rng_u64.argtypes = [C.c_uint64, C.c_uint64, u64p]
        L.fmpo_rng_complex_gaussian.argtypes = [C.c_uint64, C.c_uint64, f64p]
        L.fmpo_rng_sample.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        L.fmpo_make_row_selection.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        L.fmpo_make_instance.argtypes = [C.c_int, C.c_uint64, u64p, C.c_uint64, C.c_uint64,
                                         C.c_double, C.c_uint64, f64p, f64p, f64p]
        L.fmpo_make_real_instance.argtypes = [C.c_int, C.c_uint64, u64p, C.c_uint64,
                                              C.c_uint64, C.c_uint64, f64p, f64p]
        for nm in ("fmpo_forward", "fmpo_adjoint"):
            getattr(L, nm).argtypes = [C.c_int, C.c_uint64, f64p, f64p]
        for nm in ("fmpo_apply", "fmpo_apply_adjoint"):
            getattr(L, nm).argtypes = [C.c_int, C.c_uint64, u64p, C.c_uint64, f64p, f64p]
        L.fmpo_column.argtypes = [C.c_int, C.c_uint64, u64p, C.c_uint64, C.c_uint64, f64p]
        L.fmpo_entry.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, f64p]
        L.fmpo_compute_kernel.argtypes = [C.c_int, C.c_uint64, u64p, C.c_uint64, f64p, f64p,
                                          u32p, C.POINTER(C.c_uint64)]
        L.fmpo_fast_update.argtypes = [C.c_int, C.c_uint64, u64p, C.c_uint64, f64p, u64p, f64p,
                                       C.c_uint64, C.c_int, f64p]
        L.fmpo_crossover_iteration.restype = C.c_uint64
        L.fmpo_crossover_iteration.argtypes = [C.c_int, C.c_uint64]
        L.fmpo_argmax_magnitude.restype = C.c_uint64
        L.fmpo_argmax_magnitude.argtypes = [f64p, C.c_uint64]
        L.fmpo_least_squares.argtypes = [C.c_int, C.c_uint64, u64p, C.c_uint64, u64p, C.c_uint64,
                                         f64p, C.c_int, f64p, C.POINTER(C.c_uint64)]
        L.fmpo_omp_solve.argtypes = [C.c_int, C.c_uint64, u64p, C.c_uint64, f64p,
                                     C.POINTER(SolveConfig), C.POINTER(SolveResult)]
        L.fmpo_omp_solve_batch.argtypes = [C.c_int, C.c_uint64, u64p, C.c_uint64, f64p,
                                           C.c_uint64, C.POINTER(SolveConfig), C.c_int,
                                           u64p, f64p, u64p, f64p,
                                           np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")]
        L.fmpo_cosamp_solve.argtypes = [C.c_int, C.c_uint64, u64p, C.c_uint64, f64p, C.c_uint64,
                                        C.POINTER(SolveConfig), C.POINTER(SolveResult), u64p]
        L.fmpo_impl.restype = C.c_char_p

    # -- helpers ------------------------------------------------------------
    @staticmethod
    def _check(st, aux=0):
        if st:
            raise OracleError(st, aux)

    def impl(self) -> str:
        return self.lib.fmpo_impl().decode()

    def derive_seed(self, base: int, index: int) -> int:
        return int(self.lib.fmpo_derive_seed(base, index))

    def splitmix64(self, x: int) -> int:
        return int(self.lib.fmpo_splitmix64(x))

    def rng_u64(self, seed: int, count: int) -> np.ndarray:
        out = np.zeros(count, np.uint64)
        self.lib.fmpo_rng_u64(seed, count, out)
        return out

    def rng_complex_gaussian(self, seed: int, count: int) -> np.ndarray:
        out = np.zeros(2 * count, np.float64)
        self.lib.fmpo_rng_complex_gaussian(seed, count, out)
        return out.view(np.complex128)

    def rng_sample(self, seed: int, n: int, m: int) -> np.ndarray:
        out = np.zeros(max(m, 1), np.uint64)
        self._check(self.lib.fmpo_rng_sample(seed, n, m, out))
        return out[:m]

    def make_row_selection(self, n: int, m: int, seed: int) -> np.ndarray:
        out = np.zeros(max(m, 1), np.uint64)
        self._check(self.lib.fmpo_make_row_selection(n, m, seed, out))
        return out[:m]

    def make_instance(self, kind: str, n: int, omega, k: int, noise: float, seed: int):
        omega = _u(omega)
        m = len(omega)
        x = np.zeros(2 * n)
        y = np.zeros(2 * m)
        e = np.zeros(2 * m)
        self._check(self.lib.fmpo_make_instance(KIND[kind], n, omega, m, k, noise, seed, x, y, e))
        return x.view(np.complex128), y.view(np.complex128), e.view(np.complex128)

    def make_real_instance(self, kind: str, n: int, omega, k: int, seed: int):
        omega = _u(omega)
        m = len(omega)
        x = np.zeros(2 * n)
        y = np.zeros(2 * m)
        self._check(self.lib.fmpo_make_real_instance(KIND[kind], n, omega, m, k, seed, x, y))
        return x.view(np.complex128), y.view(np.complex128)

    def forward(self, kind: str, v) -> np.ndarray:
        v = _c(v)
        out = np.zeros_like(v)
        self._check(self.lib.fmpo_forward(KIND[kind], len(v) // 2, v, out))
        return out.view(np.complex128)

    def adjoint(self, kind: str, v) -> np.ndarray:
        v = _c(v)
        out = np.zeros_like(v)
        self._check(self.lib.fmpo_adjoint(KIND[kind], len(v) // 2, v, out))
        return out.view(np.complex128)

    def apply(self, kind: str, n: int, omega, x) -> np.ndarray:
        omega = _u(omega)
        out = np.zeros(2 * len(omega))
        self._check(self.lib.fmpo_apply(KIND[kind], n, omega, len(omega), _c(x), out))
        return out.view(np.complex128)

    def apply_adjoint(self, kind: str, n: int, omega, r) -> np.ndarray:
        omega = _u(omega)
        out = np.zeros(2 * n)
        self._check(self.lib.fmpo_apply_adjoint(KIND[kind], n, omega, len(omega), _c(r), out))
        return out.view(np.complex128)

    def column(self, kind: str, n: int, omega, j: int) -> np.ndarray:
        omega = _u(omega)
        out = np.zeros(2 * len(omega))
        self._check(self.lib.fmpo_column(KIND[kind], n, omega, len(omega), j, out))
        return out.view(np.complex128)

    def entry(self, kind: str, n: int, row: int, col: int) -> complex:
        out = np.zeros(2)
        self._check(self.lib.fmpo_entry(KIND[kind], n, row, col, out))
        return complex(out[0], out[1])

    def compute_kernel(self, kind: str, n: int, omega):
        omega = _u(omega)
        c = np.zeros(2 * n)
        vals = np.zeros(n)
        vidx = np.zeros(n, np.uint32)
        nv = C.c_uint64(0)
        self._check(self.lib.fmpo_compute_kernel(KIND[kind], n, omega, len(omega), c, vals, vidx,
                                                 C.byref(nv)))
        nv = nv.value
        return c.view(np.complex128), vals[:nv], (vidx if nv else np.zeros(0, np.uint32))

    def fast_update(self, kind: str, n: int, omega, h0, support, coeffs, symmetry=False):
        omega = _u(omega)
        support = _u(support)
        out = np.zeros(2 * n)
        self._check(self.lib.fmpo_fast_update(KIND[kind], n, omega, len(omega), _c(h0),
                                              support if len(support) else np.zeros(1, np.uint64),
                                              _c(coeffs) if len(support) else np.zeros(2),
                                              len(support), int(symmetry), out))
        return out.view(np.complex128)

    def crossover_iteration(self, kind: str, n: int) -> int:
        return int(self.lib.fmpo_crossover_iteration(KIND[kind], n))

    def argmax_magnitude(self, h) -> int:
        h = _c(h)
        return int(self.lib.fmpo_argmax_magnitude(h, len(h) // 2))

    def least_squares(self, kind: str, n: int, omega, support, y, method="normal"):
        omega = _u(omega)
        support = _u(support)
        out = np.zeros(2 * max(len(support), 1))
        aux = C.c_uint64(0)
        st = self.lib.fmpo_least_squares(KIND[kind], n, omega, len(omega), support, len(support),
                                         _c(y), LS[method], out, C.byref(aux))
        self._check(st, aux.value)
        return out.view(np.complex128)[: len(support)]

    def omp_solve(self, kind: str, n: int, omega, y, max_iterations: int, tol: float,
                  mode="conventional", ls="qr", symmetry=False, record=False) -> Recovery:
        omega = _u(omega)
        T = int(max_iterations)
        cfg = SolveConfig(T, tol, MODE[mode], LS[ls], int(symmetry), int(record))
        sup = np.zeros(T, np.uint64)
        co = np.zeros(2 * T)
        hist = np.zeros(2 * n * T) if record else None
        modes = np.zeros(T, np.int32)
        res = SolveResult()
        res.support = sup.ctypes.data_as(C.POINTER(C.c_uint64))
        res.coeffs = co.ctypes.data_as(C.POINTER(C.c_double))
        res.correlation_history = (hist.ctypes.data_as(C.POINTER(C.c_double))
                                   if record else C.POINTER(C.c_double)())
        res.mode_used = modes.ctypes.data_as(C.POINTER(C.c_int))
        self._check(self.lib.fmpo_omp_solve(KIND[kind], n, omega, len(omega), _c(y),
                                            C.byref(cfg), C.byref(res)))
        s = res.support_size
        H = []
        if record:
            hv = hist.view(np.complex128).reshape(T, n)
            H = [hv[i].copy() for i in range(res.history_len)]
        return Recovery(sup[:s].copy(), co.view(np.complex128)[:s].copy(), int(res.iterations_run),
                        float(res.residual_norm), bool(res.rank_deficient_abort), H,
                        [int(v) for v in modes[: res.history_len if record else T]])

    def cosamp_solve(self, kind: str, n: int, omega, y, k: int, max_iterations: int, tol: float,
                     mode="conventional", symmetry=False, record=False):
        """solvers.cpp:413-544.  Returns (Recovery, support_history list of arrays)."""
        omega = _u(omega)
        T, K = int(max_iterations), int(k)
        cfg = SolveConfig(T, tol, MODE[mode], 1, int(symmetry), int(record))
        sup = np.zeros(max(K, 1), np.uint64)
        co = np.zeros(2 * max(K, 1))
        hist = np.zeros(2 * n * T) if record else None
        sh = np.zeros(T * max(K, 1), np.uint64)
        modes = np.zeros(T, np.int32)
        res = SolveResult()
        res.support = sup.ctypes.data_as(C.POINTER(C.c_uint64))
        res.coeffs = co.ctypes.data_as(C.POINTER(C.c_double))
        res.correlation_history = (hist.ctypes.data_as(C.POINTER(C.c_double))
                                   if record else C.POINTER(C.c_double)())
        res.mode_used = modes.ctypes.data_as(C.POINTER(C.c_int))
        self._check(self.lib.fmpo_cosamp_solve(KIND[kind], n, omega, len(omega), _c(y), K,
                                               C.byref(cfg), C.byref(res), sh))
        s, it = res.support_size, int(res.iterations_run)
        H = []
        if record:
            hv = hist.view(np.complex128).reshape(T, n)
            H = [hv[i].copy() for i in range(res.history_len)]
        shv = sh.reshape(T, max(K, 1))
        SH = [row[row > 0].copy() for row in shv[:it]]
        rec = Recovery(sup[:s].copy(), co.view(np.complex128)[:s].copy(), it,
                       float(res.residual_norm), bool(res.rank_deficient_abort), H,
                       [int(v) for v in modes[: res.history_len if record else it]])
        return rec, SH

    def omp_solve_batch(self, kind: str, n: int, omega, Y, max_iterations: int, tol: float,
                        mode="fast", threads=0):
        """Y: (batch, m) complex; tol scalar (absolute) applied to every signal."""
        omega = _u(omega)
        Y = np.ascontiguousarray(Y, dtype=np.complex128)
        B = Y.shape[0]
        T = int(max_iterations)
        cfg = SolveConfig(T, tol, MODE[mode], 0, 0, 0)
        sup = np.zeros(B * T, np.uint64)
        co = np.zeros(2 * B * T)
        it = np.zeros(B, np.uint64)
        rn = np.zeros(B)
        ab = np.zeros(B, np.int32)
        self._check(self.lib.fmpo_omp_solve_batch(KIND[kind], n, omega, len(omega),
                                                  Y.view(np.float64).reshape(-1), B,
                                                  C.byref(cfg), threads, sup, co, it, rn, ab))
        return (sup.reshape(B, T), co.view(np.complex128).reshape(B, T), it, rn, ab)
