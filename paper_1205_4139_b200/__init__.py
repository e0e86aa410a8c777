"""paper_1205_4139_b200 — B200-native OMP correlation path.

Python host side of the drop-in for the reference library ``fastmp``
(/root/reference/proj/include/fastmp).  Every call goes through the C ABI of
``libfmp_cuda.so`` (``include/fmp.h``); there is no CPU fallback: importing
this package without the built library raises immediately.

Names and argument meaning follow the reference:

==========================  ===============================================
this module                 reference (proj/include/fastmp)
==========================  ===============================================
SensingOperator             sensing.hpp:39-66  (apply / apply_adjoint / column)
compute_kernel              kernel.hpp:42-43   -> CorrelationKernel
fast_update                 kernel.hpp:95-98
argmax_magnitude            solvers.cpp:90-101 (tie band 1e-9)
SolveConfig/default_config  solvers.hpp:26-37
omp_solve                   solvers.hpp:70-71  -> RecoveryResult
crossover_iteration         cost_model.hpp:76
make_row_selection          sensing.hpp:31-33
==========================  ===============================================

Atom / row indices are 1-based as in the reference.  Batched variants take a
leading batch dimension.  ``*_dev`` helpers take torch CUDA tensors.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfmp_cuda.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_1205_4139_b200.build` "
        "(the GPU path has no fallback)")

_lib = C.CDLL(LIB_PATH)

FOURIER, HADAMARD = 0, 1
KINDS = {"fourier": FOURIER, "hadamard": HADAMARD}
C128, C64, F64, F32 = 0, 1, 2, 3
DTYPES = {np.dtype(np.complex128): C128, np.dtype(np.complex64): C64,
          np.dtype(np.float64): F64, np.dtype(np.float32): F32}
NP_OF = {C128: np.complex128, C64: np.complex64, F64: np.float64, F32: np.float32}
MODES = {"conventional": 0, "fast": 1, "adaptive": 2, "custom": 3, "gpu": 4}

_vp = C.c_void_p
_u64 = C.c_uint64


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_DP = C.POINTER(C.c_double)


class OmpConfig(C.Structure):
    _fields_ = [("max_iterations", _u64), ("tolerance", C.c_double),
                ("tolerances", C.POINTER(C.c_double)), ("mode", C.c_int),
                ("fast_until", _u64), ("record_correlations", C.c_int)]


class OmpResult(C.Structure):
    _fields_ = [("support", _vp), ("coeffs", _vp), ("support_size", _vp), ("iterations", _vp),
                ("residual", _vp), ("aborted", _vp), ("modes", _vp), ("history_len", _vp),
                ("history", _vp)]


class CosampResult(C.Structure):
    _fields_ = [("support", _vp), ("coeffs", _vp), ("support_size", _vp), ("iterations", _vp),
                ("residual", _vp), ("aborted", _vp), ("support_history", _vp), ("history", _vp)]


_sig("fmp_version", C.c_int)
_sig("fmp_fma_peak", C.c_int, _vp, C.c_int, C.POINTER(C.c_double))
_sig("fmp_last_error", C.c_char_p)
_sig("fmp_set_phase_profiling", C.c_int, C.c_int)
_sig("fmp_phase_cycles", C.c_int, _vp, _vp)
_sig("fmp_refine_stats", C.c_int, _vp, _vp)
_sig("fmp_last_launch_count", C.c_int)
_sig("fmp_ctx_create", C.c_int, C.c_int, C.POINTER(_vp))
_sig("fmp_ctx_destroy", C.c_int, _vp)
_sig("fmp_ctx_set_stream", C.c_int, _vp, _vp)
_sig("fmp_ctx_stream", _vp, _vp)
_sig("fmp_ctx_synchronize", C.c_int, _vp)
_sig("fmp_operator_create", C.c_int, _vp, C.c_int, _u64, _vp, _u64, C.POINTER(_vp))
_sig("fmp_operator_destroy", C.c_int, _vp)
_sig("fmp_operator_info", C.c_int, _vp, C.POINTER(C.c_int), C.POINTER(_u64), C.POINTER(_u64))
_sig("fmp_operator_kernel", C.c_int, _vp, _vp, _vp, _vp, C.POINTER(_u64))
_sig("fmp_crossover_iteration", _u64, C.c_int, _u64)
_sig("fmp_gpu_crossover", _u64, C.c_int, _u64)
_sig("fmp_gpu_crossover_for", _u64, _vp, C.c_int, _u64, _u64)
_sig("fmp_omp_plan_info", C.c_int, _vp, C.c_int, _u64, _u64, _vp)
_sig("fmp_apply", C.c_int, _vp, C.c_int, _vp, _u64, _vp)
_sig("fmp_apply_dev", C.c_int, _vp, C.c_int, _vp, _u64, _vp, _vp)
_sig("fmp_apply_adjoint", C.c_int, _vp, C.c_int, _vp, _u64, _vp, _vp)
_sig("fmp_apply_adjoint_dev", C.c_int, _vp, C.c_int, _vp, _u64, _vp, _vp, _vp)
_sig("fmp_unitary_forward", C.c_int, _vp, C.c_int, _vp, _u64, _vp)
_sig("fmp_unitary_adjoint", C.c_int, _vp, C.c_int, _vp, _u64, _vp)
_sig("fmp_fast_update", C.c_int, _vp, C.c_int, _vp, _vp, _vp, _u64, _u64, _vp, _vp)
_sig("fmp_fast_update_dev", C.c_int, _vp, C.c_int, _vp, _vp, _vp, _u64, _u64, _vp, _vp, _vp)
_sig("fmp_argmax_band", C.c_int, _vp, C.c_int, _vp, _u64, _u64, _vp)
_sig("fmp_omp_solve", C.c_int, _vp, C.c_int, _vp, _u64, C.POINTER(OmpConfig), C.POINTER(OmpResult))
_sig("fmp_omp_solve_multi", C.c_int, _vp, C.c_int, C.c_int, _vp, _u64, C.POINTER(OmpConfig),
     C.POINTER(OmpResult))
_sig("fmp_device_count", C.c_int, C.POINTER(C.c_int))
_sig("fmp_host_alloc", C.c_int, C.c_size_t, C.POINTER(_vp))
_sig("fmp_host_free", C.c_int, _vp)
_sig("fmp_omp_solve_dev", C.c_int, _vp, C.c_int, _vp, _u64, C.POINTER(OmpConfig),
     C.POINTER(OmpResult), _vp)
_sig("fmp_cosamp_solve", C.c_int, _vp, C.c_int, _vp, _u64, _u64, C.POINTER(OmpConfig),
     C.POINTER(CosampResult))
_sig("fmp_cosamp_solve_dev", C.c_int, _vp, C.c_int, _vp, _u64, _u64, C.POINTER(OmpConfig),
     C.POINTER(CosampResult), _vp)
_sig("fmp_qr_create", C.c_int, _vp, _u64, _u64, C.POINTER(_vp))
_sig("fmp_qr_destroy", C.c_int, _vp)
_sig("fmp_qr_push_column", C.c_int, _vp, _vp, C.POINTER(C.c_int))
_sig("fmp_qr_solve", C.c_int, _vp, _vp, _vp)
_sig("fmp_qr_cols", _u64, _vp)
_sig("fmp_comm_unique_id", C.c_int, _vp)
_sig("fmp_comm_init_rank", C.c_int, C.c_int, C.c_int, C.c_int, _vp, C.POINTER(_vp))
_sig("fmp_comm_init_all", C.c_int, _vp, C.c_int, _vp)
_sig("fmp_comm_destroy", C.c_int, _vp)
_sig("fmp_large_create", C.c_int, _vp, C.c_int, _u64, _u64, C.POINTER(OmpConfig), _vp, C.POINTER(_vp))
_sig("fmp_large_destroy", C.c_int, _vp)
_sig("fmp_large_group_solve", C.c_int, _vp, C.c_int, _vp, C.c_double)
_sig("fmp_large_result", C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp)
_sig("fmp_large_record_size", C.c_int)
_sig("fmp_large_merge_records", C.c_int, _vp, C.c_int, _vp, _vp)
_sig("fmp_large_solve", C.c_int, _vp, C.c_int, _vp, C.POINTER(OmpConfig), C.POINTER(OmpResult))
_sig("fmp_least_squares", C.c_int, _vp, C.c_int, _vp, _vp, _u64, _u64, _vp, C.POINTER(C.c_int64))
_sig("fmp_make_row_selection", C.c_int, _u64, _u64, _u64, _vp)
_sig("fmp_make_batch", C.c_int, C.c_int, _u64, _vp, _u64, _u64, C.c_double, C.c_int, _u64, _u64,
     _u64, C.c_int, _vp, _vp, _vp)
_sig("fmp_derive_seed", _u64, _u64, _u64)
_sig("fmp_make_batch_dev", C.c_int, _vp, _u64, C.c_double, C.c_int, _u64, _u64, _u64, _vp, _vp, _vp,
     C.POINTER(_u64), _vp)
_sig("fmp_dd_eval", C.c_int, C.c_int, _vp, _u64, _vp, _vp)
_sig("fmp_dd_eval_dev", C.c_int, C.c_int, _vp, _u64, _vp, _vp, _vp)


# ---------------------------------------------------------------- errors
class FmpError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[fmp status {status}] {message}")
        self.status = status


class InvalidArgument(FmpError, ValueError):
    """std::invalid_argument in the reference."""


class RankDeficientError(FmpError):
    """RankDeficientError (solvers.hpp:42-51)."""


class Unsupported(FmpError):
    pass


def _check(status: int) -> None:
    if status == 0:
        return
    msg = (_lib.fmp_last_error() or b"").decode()
    cls = {1: InvalidArgument, 2: RankDeficientError, 5: Unsupported}.get(status, FmpError)
    raise cls(status, msg)


def set_phase_profiling(enabled: bool) -> None:
    _check(_lib.fmp_set_phase_profiling(int(enabled)))


def last_launch_count() -> int:
    return int(_lib.fmp_last_launch_count())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


def _dtype_code(arr) -> int:
    dt = np.dtype(arr.dtype) if not hasattr(arr, "is_cuda") else _torch_np_dtype(arr.dtype)
    if dt not in DTYPES:
        raise InvalidArgument(1, f"unsupported dtype {dt}")
    return DTYPES[dt]


def _torch_np_dtype(tdt):
    import torch
    return np.dtype({torch.complex128: np.complex128, torch.complex64: np.complex64,
                     torch.float64: np.float64, torch.float32: np.float32}[tdt])


# --------------------------------------------------------------- context
class Context:
    """A GPU, a stream and a device workspace (one per host thread)."""

    def __init__(self, device: int = 0):
        h = _vp()
        _check(_lib.fmp_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        _check(_lib.fmp_ctx_set_stream(self.handle, stream_ptr))

    @property
    def stream(self) -> int:
        return _lib.fmp_ctx_stream(self.handle) or 0

    def synchronize(self) -> None:
        _check(_lib.fmp_ctx_synchronize(self.handle))

    def fma_peak(self, double: bool = True) -> float:
        """Measured FMA-pipe throughput of this GPU (FMAs per second)."""
        v = C.c_double(0)
        _check(_lib.fmp_fma_peak(self.handle, int(double), C.byref(v)))
        return v.value

    def phase_cycles(self) -> dict:
        """Per-phase SM cycles of the last fused solve (fmp_set_phase_profiling(1))."""
        v = np.zeros(6)
        _check(_lib.fmp_phase_cycles(self.handle, _ptr(v)))
        return dict(zip(["conventional", "fast", "identify", "least_squares", "residual", "other"], v))

    def refine_stats(self) -> dict:
        """fp32 solves, last solve with phase profiling on: identifications,
        candidates re-evaluated in fp64, identifications that overflowed the
        per-CTA candidate list."""
        v = np.zeros(3)
        _check(_lib.fmp_refine_stats(self.handle, _ptr(v)))
        return dict(zip(["identifications", "candidates", "overflows"], v))

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.fmp_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: dict = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


# ---------------------------------------------------------- sensing / kernel
def crossover_iteration(kind, n: int) -> int:
    kind = KINDS.get(kind, kind)
    return int(_lib.fmp_crossover_iteration(kind, n))


def gpu_crossover(kind, n: int) -> int:
    """Switch point of the GPU-calibrated Adaptive mode ("gpu") for the
    one-CTA-per-SM solver (small batches)."""
    kind = KINDS.get(kind, kind)
    return int(_lib.fmp_gpu_crossover(kind, n))


def gpu_crossover_for(op: "SensingOperator", dtype, batch: int, max_iterations: int) -> int:
    """Switch point mode "gpu" uses for this batched solve (the solver runs two
    CTAs per SM when the batch and shared memory allow, which moves it)."""
    return int(_lib.fmp_gpu_crossover_for(op.handle, DTYPES[np.dtype(dtype)], batch, max_iterations))


def omp_plan_info(op: "SensingOperator", dtype, batch: int, max_iterations: int) -> dict:
    """The fused solver's configuration for a batched solve (tests / tools)."""
    v = np.zeros(4, np.int32)
    _check(_lib.fmp_omp_plan_info(op.handle, DTYPES[np.dtype(dtype)], batch, max_iterations, _ptr(v)))
    return {"ctas_per_sm": int(v[0]), "threads": int(v[1]),
            "kernel_table": ("global", "smem_full", "smem_conj_half")[int(v[2])],
            "buffer_in_global": bool(v[3])}


def make_row_selection(n: int, m: int, seed: int) -> np.ndarray:
    out = np.zeros(max(m, 1), np.uint64)
    _check(_lib.fmp_make_row_selection(n, m, seed, _ptr(out)))
    return out[:m]


def derive_seed(base: int, index: int) -> int:
    return int(_lib.fmp_derive_seed(base, index))


@dataclass
class CorrelationKernel:
    """kernel.hpp:31-40"""
    kind: str
    n: int
    m: int
    c: np.ndarray
    values: np.ndarray
    value_index: np.ndarray


class SensingOperator:
    """Phi = S_Omega U (sensing.hpp:39-66) resident on one GPU."""

    def __init__(self, kind, n: int, rows: Sequence[int], ctx: Optional[Context] = None):
        self.kind_name = kind if isinstance(kind, str) else ("fourier" if kind == 0 else "hadamard")
        self.kind = KINDS[self.kind_name]
        self.ctx = ctx or default_context()
        rows = np.ascontiguousarray(np.asarray(rows, dtype=np.uint64))
        h = _vp()
        _check(_lib.fmp_operator_create(self.ctx.handle, self.kind, int(n), _ptr(rows), len(rows),
                                        C.byref(h)))
        self.handle = h
        self.n = int(n)
        self.omega = np.sort(rows)
        self.m = len(rows)

    def close(self):
        if getattr(self, "handle", None):
            _lib.fmp_operator_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _default_dtype(self, a):
        return np.asarray(a).dtype if np.iscomplexobj(a) or self.kind == HADAMARD else np.complex128

    def _prep(self, a, length: int, dtype=None):
        a = np.asarray(a)
        if dtype is None:
            dtype = a.dtype if a.dtype in DTYPES else np.complex128
            if self.kind == FOURIER and not np.issubdtype(dtype, np.complexfloating):
                dtype = np.complex128
        a = np.ascontiguousarray(a, dtype=dtype)
        if a.shape[-1] != length:
            raise InvalidArgument(1, f"length mismatch: expected {length}, got {a.shape[-1]}")
        return a

    def apply(self, x, dtype=None) -> np.ndarray:
        """Phi x (sensing.cpp:93-100); x of shape (n,) or (batch, n)."""
        x = self._prep(x, self.n, dtype)
        b = 1 if x.ndim == 1 else x.shape[0]
        out = np.empty(x.shape[:-1] + (self.m,), x.dtype)
        _check(_lib.fmp_apply(self.handle, DTYPES[x.dtype], _ptr(x), b, _ptr(out)))
        return out

    def apply_adjoint(self, r, dtype=None, argmax: bool = False):
        """Phi^H r (sensing.cpp:102-109): the conventional correlation."""
        r = self._prep(r, self.m, dtype)
        b = 1 if r.ndim == 1 else r.shape[0]
        out = np.empty(r.shape[:-1] + (self.n,), r.dtype)
        idx = np.zeros(b, np.uint64)
        _check(_lib.fmp_apply_adjoint(self.handle, DTYPES[r.dtype], _ptr(r), b, _ptr(out),
                                      _ptr(idx) if argmax else None))
        if argmax:
            return out, (idx if r.ndim > 1 else int(idx[0]))
        return out

    def forward(self, v, dtype=None) -> np.ndarray:
        """StructuredUnitary::forward (transform.hpp:46)."""
        v = self._prep(v, self.n, dtype)
        out = np.empty_like(v)
        _check(_lib.fmp_unitary_forward(self.handle, DTYPES[v.dtype], _ptr(v),
                                        1 if v.ndim == 1 else v.shape[0], _ptr(out)))
        return out

    def adjoint(self, v, dtype=None) -> np.ndarray:
        """StructuredUnitary::adjoint (transform.hpp:47)."""
        v = self._prep(v, self.n, dtype)
        out = np.empty_like(v)
        _check(_lib.fmp_unitary_adjoint(self.handle, DTYPES[v.dtype], _ptr(v),
                                        1 if v.ndim == 1 else v.shape[0], _ptr(out)))
        return out

    def column(self, j: int) -> np.ndarray:
        """Column j (1-based) of Phi (sensing.cpp:111-117), as Phi e_j on the GPU."""
        if not 1 <= j <= self.n:
            raise InvalidArgument(1, "column: index out of range")
        e = np.zeros(self.n, np.complex128)
        e[j - 1] = 1.0
        return self.apply(e)

    def kernel(self) -> CorrelationKernel:
        c = np.zeros(self.n, np.complex128)
        vals = np.zeros(self.m + 1)
        vidx = np.zeros(self.n, np.uint32)
        nv = _u64(0)
        had = self.kind == HADAMARD
        _check(_lib.fmp_operator_kernel(self.handle, _ptr(c), _ptr(vals) if had else None,
                                        _ptr(vidx) if had else None, C.byref(nv)))
        return CorrelationKernel(self.kind_name, self.n, self.m, c, vals[: nv.value].copy(),
                                 vidx if had else np.zeros(0, np.uint32))


def compute_kernel(op: SensingOperator) -> CorrelationKernel:
    """compute_kernel (kernel.hpp:42-43); built on the device at operator creation."""
    return op.kernel()


def fast_update(h0, op: SensingOperator, support, coeffs, argmax: bool = False, want_h: bool = True):
    """fast_update (kernel.hpp:95-98).

    h0: (n,) or (batch, n); support: (t,) or (batch, t) 1-based; coeffs alike.
    Returns h (and the 1-based band argmax when ``argmax``)."""
    h0 = np.asarray(h0)
    dt = h0.dtype if h0.dtype in DTYPES else np.complex128
    h0 = np.ascontiguousarray(h0, dtype=dt)
    batched = h0.ndim > 1
    b = h0.shape[0] if batched else 1
    support = np.ascontiguousarray(np.asarray(support, dtype=np.uint64).reshape(b, -1))
    t = support.shape[1]
    coeffs = np.ascontiguousarray(np.asarray(coeffs).astype(dt, copy=False).reshape(b, t))
    if h0.shape[-1] != op.n:
        raise InvalidArgument(1, "fast_update: h0 length")
    out = np.empty_like(h0) if want_h else None
    idx = np.zeros(b, np.uint64)
    _check(_lib.fmp_fast_update(op.handle, DTYPES[h0.dtype], _ptr(h0), _ptr(support) if t else None,
                                _ptr(coeffs) if t else None, t, b,
                                _ptr(out) if want_h else None, _ptr(idx) if argmax else None))
    if argmax:
        return out, (idx if batched else int(idx[0]))
    return out


def argmax_magnitude(h, ctx: Optional[Context] = None):
    """1-based band argmax (solvers.cpp:90-101); h (n,) or (batch, n)."""
    h = np.asarray(h)
    dt = h.dtype if h.dtype in DTYPES else np.complex128
    h = np.ascontiguousarray(h, dtype=dt)
    b = h.shape[0] if h.ndim > 1 else 1
    out = np.zeros(b, np.uint64)
    ctx = ctx or default_context()
    _check(_lib.fmp_argmax_band(ctx.handle, DTYPES[h.dtype], _ptr(h), h.shape[-1], b, _ptr(out)))
    return out if h.ndim > 1 else int(out[0])


# ------------------------------------------------------------------- OMP
@dataclass
class SolveConfig:
    """SolveConfig (solvers.hpp:26-34); ls_method is fixed to the GPU's
    incremental Cholesky on Gram entries."""
    max_iterations: int = 1
    residual_tolerance: float = 0.0
    correlation_mode: str = "conventional"
    fast_until: int = 0                # used when correlation_mode == "custom"
    record_correlations: bool = False


def default_config(k: int, y_norm: float) -> SolveConfig:
    """solvers.cpp:216-221"""
    return SolveConfig(max_iterations=max(1, int(k)), residual_tolerance=1e-9 * float(y_norm))


@dataclass
class RecoveryResult:
    """RecoveryResult (solvers.hpp:53-64)."""
    x_hat: np.ndarray
    support: list
    coeffs: np.ndarray
    iterations_run: int
    residual_norm: float
    rank_deficient_abort: bool
    support_history: list = field(default_factory=list)
    correlation_history: list = field(default_factory=list)
    modes_used: list = field(default_factory=list)


@dataclass
class BatchResult:
    support: np.ndarray        # (batch, T) 1-based, 0 padded
    coeffs: np.ndarray         # (batch, T) complex128
    support_size: np.ndarray
    iterations: np.ndarray
    residual: np.ndarray
    aborted: np.ndarray
    modes: np.ndarray
    history_len: np.ndarray
    history: Optional[np.ndarray]


def _config(cfg: SolveConfig, tolerances=None):
    c = OmpConfig()
    c.max_iterations = int(cfg.max_iterations)
    c.tolerance = float(cfg.residual_tolerance)
    c.tolerances = tolerances
    c.mode = MODES[cfg.correlation_mode]
    c.fast_until = int(cfg.fast_until)
    c.record_correlations = int(cfg.record_correlations)
    return c



# batches below this size take the library's small-batch path, which stages
# through the context's own page-locked block: plain numpy result buffers
_PINNED_MIN_BATCH = 1024


def _host_outs(specs, pinned=True):
    """Several result buffers carved from ONE allocation — page-locked (one
    trip through torch's host allocator per call instead of one per buffer;
    each view keeps the block alive) or, pinned=False (small batches), plain
    numpy arrays.  specs: (shape, dtype, zero) tuples."""
    if not pinned:
        return [np.zeros(shape, dt) if zero else np.empty(shape, dt) for shape, dt, zero in specs]
    sizes = [int(np.prod(shape, dtype=np.int64)) * np.dtype(dt).itemsize for shape, dt, _ in specs]
    offs, tot = [], 0
    for b in sizes:
        offs.append(tot)
        tot += (b + 63) // 64 * 64
    try:
        import torch
        if torch.cuda.is_available():
            blk = torch.empty(max(tot, 64), dtype=torch.uint8, pin_memory=True).numpy()
            out = []
            for (shape, dt, zero), o, b in zip(specs, offs, sizes):
                v = blk[o:o + b].view(dt).reshape(shape)
                if zero:
                    v.fill(0)
                out.append(v)
            return out
    except (ImportError, RuntimeError):
        pass
    return [np.zeros(shape, dt) for shape, dt, _ in specs]


def omp_solve_batch(op: SensingOperator, Y, cfg: SolveConfig, tolerances=None,
                    dtype=None) -> BatchResult:
    """omp_solve over a batch of measurements Y (batch, m) sharing `op`."""
    Y = np.asarray(Y)
    if dtype is None:
        dtype = Y.dtype if Y.dtype in DTYPES else np.complex128
        if op.kind == FOURIER and not np.issubdtype(dtype, np.complexfloating):
            dtype = np.complex128
    Y = np.ascontiguousarray(Y, dtype=dtype)
    if Y.ndim == 1:
        Y = Y[None]
    if Y.shape[-1] != op.m:
        raise InvalidArgument(1, "omp_solve: measurement length mismatch")
    B, T, n = Y.shape[0], int(cfg.max_iterations), op.n
    if T < 1:
        raise InvalidArgument(1, "omp_solve: max_iterations must be >= 1")
    # every entry of these is written by the solve (support / coeffs zero
    # padded, modes 0 past the last iteration)
    specs = (((B, T), np.uint64), ((B, T), np.complex128), ((B,), np.uint64), ((B,), np.uint64),
             ((B,), np.float64), ((B,), np.int32), ((B, T), np.uint8), ((B,), np.uint64))
    if B >= _PINNED_MIN_BATCH:
        outs = _host_outs([(sh, dt, False) for sh, dt in specs])
        addr = [o.ctypes.data for o in outs]
    else:
        # small batches (the library stages them itself): one plain block,
        # its address taken once (per-array ctypes lookups cost ~1 us each)
        offs, tot = [], 0
        for sh, dt in specs:
            offs.append(tot)
            tot += (math.prod(sh) * np.dtype(dt).itemsize + 63) & ~63
        blk = np.empty(tot, np.uint8)
        base = blk.ctypes.data
        outs = [np.ndarray(sh, dt, blk, o) for (sh, dt), o in zip(specs, offs)]
        addr = [base + o for o in offs]
    sup, co, sz, it, rn, ab, md, hl = outs
    hist = np.zeros((B, T, n), Y.dtype) if cfg.record_correlations else None
    tol = None
    if tolerances is not None:
        tarr = np.asarray(tolerances, np.float64)
        if tarr.shape != (B,) or not tarr.flags.c_contiguous:
            tarr = np.ascontiguousarray(np.broadcast_to(tarr, (B,)))
        tol = C.cast(tarr.ctypes.data, _DP)
    res = OmpResult(*addr, hist.ctypes.data if hist is not None else None)
    c = _config(cfg, tol)
    _check(_lib.fmp_omp_solve(op.handle, DTYPES[Y.dtype], Y.ctypes.data, B, C.byref(c), C.byref(res)))
    return BatchResult(sup, co, sz, it, rn, ab.astype(bool), md, hl, hist)


def device_count() -> int:
    """CUDA devices visible to this process (fmp_device_count)."""
    v = C.c_int(0)
    _check(_lib.fmp_device_count(C.byref(v)))
    return int(v.value)


def omp_solve_multi(ops, Y, cfg: SolveConfig, tolerances=None) -> BatchResult:
    """omp_solve over a batch split across several GPUs (fmp_omp_solve_multi):
    ops[i] is the operator built on GPU i (same kind, n and rows); contiguous
    blocks of the batch, one host thread per device, no collective."""
    Y = np.ascontiguousarray(np.asarray(Y))
    if Y.ndim == 1:
        Y = Y[None]
    B, T = Y.shape[0], int(cfg.max_iterations)
    sup = np.zeros((B, T), np.uint64)
    co = np.zeros((B, T), np.complex128)
    sz, it = np.zeros(B, np.uint64), np.zeros(B, np.uint64)
    rn, ab = np.zeros(B), np.zeros(B, np.int32)
    md, hl = np.zeros((B, T), np.uint8), np.zeros(B, np.uint64)
    tarr = None
    if tolerances is not None:
        tarr = np.ascontiguousarray(np.broadcast_to(np.asarray(tolerances, np.float64), (B,)))
    res = OmpResult(sup.ctypes.data, co.ctypes.data, sz.ctypes.data, it.ctypes.data, rn.ctypes.data,
                    ab.ctypes.data, md.ctypes.data, hl.ctypes.data, None)
    c = _config(cfg, C.cast(tarr.ctypes.data, _DP) if tarr is not None else None)
    hs = (_vp * len(ops))(*[o.handle for o in ops])
    _check(_lib.fmp_omp_solve_multi(hs, len(ops), DTYPES[Y.dtype], Y.ctypes.data, B, C.byref(c),
                                    C.byref(res)))
    return BatchResult(sup, co, sz, it, rn, ab.astype(bool), md, hl, None)


def omp_solve(op: SensingOperator, y, cfg: SolveConfig, dtype=None) -> RecoveryResult:
    """omp_solve (solvers.hpp:70-71) for one measurement vector."""
    r = omp_solve_batch(op, np.asarray(y)[None], cfg, dtype=dtype)
    s = int(r.support_size[0])
    support = [int(v) for v in r.support[0, :s]]
    coeffs = r.coeffs[0, :s].copy()
    x = np.zeros(op.n, np.complex128)
    for a, v in zip(support, coeffs):
        x[a - 1] = v
    iters = int(r.iterations[0])
    hl = int(r.history_len[0])
    hist = [r.history[0, i].copy() for i in range(hl)] if r.history is not None else []
    return RecoveryResult(x, support, coeffs, iters, float(r.residual[0]), bool(r.aborted[0]),
                          [support[: i + 1] for i in range(iters)], hist,
                          [int(v) for v in r.modes[0, :hl]])


def make_batch(kind, n: int, rows, k: int, batch: int, base_seed: int, first: int = 0,
               noise_stddev: float = 0.0, real: bool = False, want_x: bool = False, threads: int = 0):
    """Seeded synthetic measurements (see fmp.h fmp_make_batch).

    Returns (Y (batch, m) complex128, X or None, noise_norms)."""
    rows = np.ascontiguousarray(np.asarray(rows, np.uint64))
    m = len(rows)
    Y = np.zeros((batch, m), np.complex128)
    X = np.zeros((batch, n), np.complex128) if want_x else None
    nn = np.zeros(batch)
    _check(_lib.fmp_make_batch(KINDS.get(kind, kind), n, _ptr(rows), m, k, noise_stddev, int(real),
                               base_seed, first, batch, threads, _ptr(Y),
                               _ptr(X) if want_x else None, _ptr(nn)))
    return Y, X, nn


def make_batch_dev(op: "SensingOperator", k: int, batch: int, base_seed: int, first: int = 0,
                   noise_stddev: float = 0.0, real: bool = False, want_x: bool = False,
                   stream=None):
    """make_batch generated on the operator's GPU (fmp.h fmp_make_batch_dev):
    bit-identical to make_batch for the operator's rows.

    Returns (Y (batch, m) complex128, X or None, noise_norms, fixups) as torch
    device tensors (fixups: values recomputed on the host with glibc)."""
    import torch
    dev = torch.device("cuda", op.ctx.device)
    Y = torch.empty((batch, op.m), dtype=torch.complex128, device=dev)
    X = torch.empty((batch, op.n), dtype=torch.complex128, device=dev) if want_x else None
    nn = torch.empty(batch, dtype=torch.float64, device=dev)
    fix = _u64(0)
    st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    _check(_lib.fmp_make_batch_dev(op.handle, k, noise_stddev, int(real), base_seed, first, batch,
                                   Y.data_ptr(), X.data_ptr() if want_x else None, nn.data_ptr(),
                                   C.byref(fix), C.c_void_p(st)))
    return Y, X, nn, int(fix.value)


def dd_eval(fn: str, x, device: bool = False) -> tuple:
    """The device generator's double-double log / cos / sin (fmp.h
    fmp_dd_eval[_dev]): (correctly rounded values, ulp position), evaluated
    on the host or, with device=True, by a kernel on cuda:0."""
    x = np.ascontiguousarray(np.asarray(x, np.float64))
    code = {"log": 0, "cos": 1, "sin": 2}[fn]
    if device:
        import torch
        xd = torch.from_numpy(x).cuda()
        out = torch.empty_like(xd)
        frac = torch.empty_like(xd)
        st = torch.cuda.current_stream().cuda_stream
        _check(_lib.fmp_dd_eval_dev(code, xd.data_ptr(), x.size, out.data_ptr(), frac.data_ptr(),
                                    C.c_void_p(st)))
        torch.cuda.synchronize()
        return out.cpu().numpy(), frac.cpu().numpy()
    out = np.empty_like(x)
    frac = np.empty_like(x)
    _check(_lib.fmp_dd_eval(code, _ptr(x), x.size, _ptr(out), _ptr(frac)))
    return out, frac


def least_squares(op: SensingOperator, support, y, dtype=None) -> np.ndarray:
    """least_squares (solvers.hpp:82-85), normal-equations form, on the GPU.
    Raises RankDeficientError(position) for dependent columns."""
    y = op._prep(y, op.m, dtype)
    Y = y[None] if y.ndim == 1 else y
    sup = np.ascontiguousarray(np.asarray(support, np.uint64).reshape(Y.shape[0], -1))
    s = sup.shape[1]
    out = np.zeros((Y.shape[0], s), np.complex128)
    pos = C.c_int64(-1)
    st = _lib.fmp_least_squares(op.handle, DTYPES[Y.dtype], _ptr(Y), _ptr(sup) if s else None, s,
                                Y.shape[0], _ptr(out) if s else None, C.byref(pos))
    if st == 2:
        e = RankDeficientError(2, (_lib.fmp_last_error() or b"").decode())
        e.position = int(pos.value)
        raise e
    _check(st)
    return out[0] if y.ndim == 1 else out


@dataclass
class CosampBatch:
    support: np.ndarray          # (batch, k) ascending 1-based, 0 padded
    coeffs: np.ndarray           # (batch, k) complex128
    support_size: np.ndarray
    iterations: np.ndarray
    residual: np.ndarray
    aborted: np.ndarray
    support_history: Optional[np.ndarray]  # (batch, T, k) or None
    history: Optional[np.ndarray]          # (batch, T, n) or None


def cosamp_solve_batch(op: SensingOperator, Y, k: int, cfg: SolveConfig, tolerances=None,
                       dtype=None, want_history: bool = True) -> CosampBatch:
    """cosamp_solve (solvers.hpp:73-78) over a batch of measurements (batch, m)."""
    Y = np.asarray(Y)
    if dtype is None:
        dtype = Y.dtype if Y.dtype in DTYPES else np.complex128
        if op.kind == FOURIER and not np.issubdtype(dtype, np.complexfloating):
            dtype = np.complex128
    Y = np.ascontiguousarray(Y, dtype=dtype)
    if Y.ndim == 1:
        Y = Y[None]
    if Y.shape[-1] != op.m:
        raise InvalidArgument(1, "cosamp_solve: measurement length mismatch")
    B, T, n, K = Y.shape[0], int(cfg.max_iterations), op.n, int(k)
    if T < 1:
        raise InvalidArgument(1, "cosamp_solve: max_iterations must be >= 1")
    kk = max(K, 1)
    specs = [((B, kk), np.uint64, True), ((B, kk), np.complex128, True), ((B,), np.uint64, True),
             ((B,), np.uint64, True), ((B,), np.float64, True), ((B,), np.int32, True)]
    if want_history:
        specs.append(((B, T, kk), np.uint64, True))
    outs = _host_outs(specs)  # page-locked: the device->host copies run at full speed
    sup, co, sz, it, rn, ab = outs[:6]
    sh = outs[6] if want_history else None
    hist = np.zeros((B, T, n), Y.dtype) if cfg.record_correlations else None
    tol = None
    if tolerances is not None:
        tarr = np.ascontiguousarray(np.broadcast_to(np.asarray(tolerances, np.float64), (B,)))
        tol = tarr.ctypes.data_as(C.POINTER(C.c_double))
    res = CosampResult(_ptr(sup), _ptr(co), _ptr(sz), _ptr(it), _ptr(rn), _ptr(ab),
                       _ptr(sh) if sh is not None else None, _ptr(hist) if hist is not None else None)
    c = _config(cfg, tol)
    _check(_lib.fmp_cosamp_solve(op.handle, DTYPES[Y.dtype], _ptr(Y), B, K, C.byref(c),
                                 C.byref(res)))
    return CosampBatch(sup[:, :K], co[:, :K], sz, it, rn, ab.astype(bool),
                       sh[:, :, :K] if sh is not None else None, hist)


def cosamp_solve(op: SensingOperator, y, k: int, cfg: SolveConfig, dtype=None) -> RecoveryResult:
    """cosamp_solve (solvers.hpp:73-78, solvers.cpp:413-544) for one vector."""
    r = cosamp_solve_batch(op, np.asarray(y)[None], k, cfg, dtype=dtype)
    s, iters = int(r.support_size[0]), int(r.iterations[0])
    support = [int(v) for v in r.support[0, :s]]
    coeffs = r.coeffs[0, :s].copy()
    x = np.zeros(op.n, np.complex128)
    for a, v in zip(support, coeffs):
        x[a - 1] = v
    sh = [[int(v) for v in row if v] for row in r.support_history[0, :iters]]
    hist = [r.history[0, i].copy() for i in range(T_rec(r, iters))] if r.history is not None else []
    fast = cfg.correlation_mode in ("fast", "gpu", "custom") or (
        cfg.correlation_mode == "adaptive" and adaptive_cosamp_uses_fast(op.kind, op.n, k))
    return RecoveryResult(x, support, coeffs, iters, float(r.residual[0]), bool(r.aborted[0]),
                          sh, hist, [int(fast)] * len(hist))


def T_rec(r: CosampBatch, iters: int) -> int:
    """correlation vectors computed: one per completed iteration, plus the
    one of an iteration that ended in a rank-deficient abort"""
    return iters + (1 if bool(r.aborted[0]) else 0)


def adaptive_cosamp_uses_fast(kind, n: int, k: int) -> bool:
    """cost_model.cpp:91-96 (power-of-two n)."""
    kind = KINDS.get(kind, kind)
    if k == 0:
        return True
    logn = int(n).bit_length() - 1
    return (6 if kind == FOURIER else 2) * n * k <= (5 if kind == FOURIER else 2) * n * logn


class IncrementalQR:
    """IncrementalQR (solvers.hpp:90-109): thin QR of a growing column set,
    Q resident on the device (fmp_qr_*)."""

    def __init__(self, rows: int, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.rows = int(rows)
        h = _vp()
        _check(_lib.fmp_qr_create(self.ctx.handle, self.rows, 64, C.byref(h)))
        self.handle = h

    def cols(self) -> int:
        return int(_lib.fmp_qr_cols(self.handle))

    def push_column(self, col) -> bool:
        col = np.ascontiguousarray(np.asarray(col, np.complex128))
        if col.shape != (self.rows,):
            raise InvalidArgument(1, "qr: column length mismatch")
        ok = C.c_int(0)
        _check(_lib.fmp_qr_push_column(self.handle, _ptr(col), C.byref(ok)))
        return bool(ok.value)

    def solve(self, rhs) -> np.ndarray:
        rhs = np.ascontiguousarray(np.asarray(rhs, np.complex128))
        if rhs.shape != (self.rows,):
            raise InvalidArgument(1, "qr: rhs length mismatch")
        x = np.zeros(self.cols(), np.complex128)
        _check(_lib.fmp_qr_solve(self.handle, _ptr(rhs), _ptr(x) if x.size else None))
        return x

    def __del__(self):
        if getattr(self, "handle", None):
            _lib.fmp_qr_destroy(self.handle)
            self.handle = None


# ------------------------------------------- sharded single-signal solver
class Comm:
    """An NCCL communicator for one shard (fmp_comm_*)."""

    def __init__(self, handle, nranks: int, rank: int):
        self.handle, self.nranks, self.rank = handle, nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_char * 128)()
        _check(_lib.fmp_comm_unique_id(buf))
        return bytes(buf)

    @classmethod
    def init_rank(cls, device: int, nranks: int, rank: int, uid: bytes) -> "Comm":
        h = _vp()
        buf = (C.c_char * 128).from_buffer_copy(uid)
        _check(_lib.fmp_comm_init_rank(int(device), int(nranks), int(rank), buf, C.byref(h)))
        return cls(h, nranks, rank)

    @classmethod
    def init_all(cls, devices) -> list:
        devs = (C.c_int * len(devices))(*devices)
        hs = (_vp * len(devices))()
        _check(_lib.fmp_comm_init_all(devs, len(devices), hs))
        return [cls(hs[i], len(devices), i) for i in range(len(devices))]

    def close(self):
        if getattr(self, "handle", None):
            _lib.fmp_comm_destroy(self.handle)
            self.handle = None


class LargeShard:
    """Shard p of P of the config-5 solver (fmp_large_*): correlation entries
    k = p + P k' live here; least squares is replicated.  `comm`: this shard's
    NCCL communicator (one rank per GPU), or None for P = 1 and for shards
    emulated on one GPU (all P passed to one sharded_solve call)."""

    def __init__(self, op: SensingOperator, cfg: SolveConfig, shard: int = 0, nshards: int = 1,
                 dtype=np.complex64, comm: Optional[Comm] = None):
        self.op = op
        self.dtype = np.dtype(dtype)
        self.comm = comm
        c = _config(cfg)
        h = _vp()
        _check(_lib.fmp_large_create(op.handle, DTYPES[self.dtype], shard, nshards, C.byref(c),
                                     comm.handle if comm is not None else None, C.byref(h)))
        self.handle = h
        self.T = int(cfg.max_iterations)

    def close(self):
        if getattr(self, "handle", None):
            _lib.fmp_large_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def result(self):
        sup = np.zeros(self.T, np.uint64)
        co = np.zeros(self.T, np.complex128)
        sz, it = _u64(0), _u64(0)
        rn = C.c_double(0)
        ab = C.c_int32(0)
        _check(_lib.fmp_large_result(self.handle, _ptr(sup), _ptr(co), C.byref(sz), C.byref(it),
                                     C.byref(rn), C.byref(ab)))
        s = sz.value
        return sup[:s].copy(), co[:s].copy(), int(it.value), rn.value, bool(ab.value)


def sharded_solve(shards, y, tol: float):
    """One solve over the local shards (fmp_large_group_solve): all P of them
    when emulating on one GPU, this process's shard(s) with NCCL otherwise.
    Returns (support, coeffs, iterations, residual_norm, aborted)."""
    y = np.ascontiguousarray(np.asarray(y, shards[0].dtype))
    hs = (_vp * len(shards))(*[sh.handle for sh in shards])
    _check(_lib.fmp_large_group_solve(hs, len(shards), _ptr(y), float(tol)))
    return shards[0].result()


RECORD_BYTES = int(_lib.fmp_large_record_size())
RECORD_CANDIDATES = (RECORD_BYTES - 16) // 16


def make_record(best32: float, cands) -> bytes:
    """One shard's identification record (fmp_kernels.cuh LgRec): its best
    working-precision |h|^2 and its (global atom 0-based, fp64 |h|^2)
    candidates; more than RECORD_CANDIDATES sets the overflow count."""
    buf = np.zeros(RECORD_BYTES, np.uint8)
    buf[:8] = np.frombuffer(np.float64(best32).tobytes(), np.uint8)
    buf[8:12] = np.frombuffer(np.uint32(len(cands)).tobytes(), np.uint8)
    for i, (j, m64) in enumerate(cands[:RECORD_CANDIDATES]):
        o = 16 + 16 * i
        buf[o:o + 8] = np.frombuffer(np.uint64(j).tobytes(), np.uint8)
        buf[o + 8:o + 16] = np.frombuffer(np.float64(m64).tobytes(), np.uint8)
    return buf.tobytes()


def merge_records(records, selected=None, n: int = 0) -> dict:
    """The merge every shard runs after the all-gather of records
    (fmp_large_merge_records; the device kernel's host twin)."""
    blob = np.frombuffer(b"".join(records), np.uint8).copy()
    sel = None
    if selected is not None:
        bits = np.zeros((n + 31) // 32, np.uint32)
        for a in selected:
            bits[a >> 5] |= np.uint32(1 << (a & 31))
        sel = bits
    out = np.zeros(4)
    _check(_lib.fmp_large_merge_records(_ptr(blob), len(records), _ptr(sel) if sel is not None else None,
                                        _ptr(out)))
    return {"atom": int(out[0]) if out[0] >= 0 else None, "best64": float(out[1]), "flags": int(out[2])}


def large_solve(op: SensingOperator, y, cfg: SolveConfig, dtype=np.complex64):
    """omp_solve for one large signal on one GPU (fmp_large_solve)."""
    y = np.ascontiguousarray(np.asarray(y, dtype))
    T = int(cfg.max_iterations)
    sup = np.zeros(T, np.uint64)
    co = np.zeros(T, np.complex128)
    sz = np.zeros(1, np.uint64)
    it = np.zeros(1, np.uint64)
    rn = np.zeros(1)
    ab = np.zeros(1, np.int32)
    res = OmpResult(_ptr(sup), _ptr(co), _ptr(sz), _ptr(it), _ptr(rn), _ptr(ab), None, None, None)
    c = _config(cfg)
    _check(_lib.fmp_large_solve(op.handle, DTYPES[np.dtype(dtype)], _ptr(y), C.byref(c), C.byref(res)))
    s = int(sz[0])
    return sup[:s].copy(), co[:s].copy(), int(it[0]), float(rn[0]), bool(ab[0])


# --------------------------------------------------- device (torch) variants
def omp_solve_dev(op: SensingOperator, y, cfg: SolveConfig, out: dict, tolerances=None,
                  stream: Optional[int] = None) -> None:
    """Enqueue a batched solve on device tensors (no host synchronisation).

    y: torch (batch, m) of a supported dtype; out: dict of preallocated torch
    tensors from :func:`alloc_dev_result`; tolerances: torch float64 (batch,)."""
    B = y.shape[0]
    c = _config(cfg, C.cast(C.c_void_p(tolerances.data_ptr()), C.POINTER(C.c_double))
                if tolerances is not None else None)
    res = OmpResult(out["support"].data_ptr(), out["coeffs"].data_ptr(), out["support_size"].data_ptr(),
                    out["iterations"].data_ptr(), out["residual"].data_ptr(), out["aborted"].data_ptr(),
                    out["modes"].data_ptr() if "modes" in out else None,
                    out["history_len"].data_ptr() if "history_len" in out else None,
                    out["history"].data_ptr() if "history" in out else None)
    _check(_lib.fmp_omp_solve_dev(op.handle, _dtype_code(y), y.data_ptr(), B, C.byref(c), C.byref(res),
                                  stream))


def cosamp_solve_dev(op: SensingOperator, y, k: int, cfg: SolveConfig, out: dict, tolerances=None,
                     stream: Optional[int] = None) -> None:
    """Enqueue a batched CoSaMP solve on device tensors; out from
    alloc_dev_result(batch, k) (support / coeffs hold k entries per problem)."""
    B = y.shape[0]
    c = _config(cfg, C.cast(C.c_void_p(tolerances.data_ptr()), C.POINTER(C.c_double))
                if tolerances is not None else None)
    res = CosampResult(out["support"].data_ptr(), out["coeffs"].data_ptr(),
                       out["support_size"].data_ptr(), out["iterations"].data_ptr(),
                       out["residual"].data_ptr(), out["aborted"].data_ptr(),
                       out["support_history"].data_ptr() if "support_history" in out else None,
                       out["history"].data_ptr() if "history" in out else None)
    _check(_lib.fmp_cosamp_solve_dev(op.handle, _dtype_code(y), y.data_ptr(), B, int(k), C.byref(c),
                                     C.byref(res), stream))


def alloc_dev_result(B: int, T: int, device="cuda") -> dict:
    import torch
    return {
        "support": torch.zeros((B, T), dtype=torch.int64, device=device),
        "coeffs": torch.zeros((B, T), dtype=torch.complex128, device=device),
        "support_size": torch.zeros(B, dtype=torch.int64, device=device),
        "iterations": torch.zeros(B, dtype=torch.int64, device=device),
        "residual": torch.zeros(B, dtype=torch.float64, device=device),
        "aborted": torch.zeros(B, dtype=torch.int32, device=device),
    }


def fast_update_dev(op: SensingOperator, h0, support0, coeffs, h_out=None, argmax_out=None,
                    stream: Optional[int] = None) -> None:
    """Device variant: h0 (batch, n), support0 int32 0-based (batch, t), coeffs (batch, t)."""
    B, t = support0.shape
    _check(_lib.fmp_fast_update_dev(op.handle, _dtype_code(h0), h0.data_ptr(), support0.data_ptr(),
                                    coeffs.data_ptr(), t, B,
                                    h_out.data_ptr() if h_out is not None else None,
                                    argmax_out.data_ptr() if argmax_out is not None else None, stream))


def apply_adjoint_dev(op: SensingOperator, r, h_out=None, argmax_out=None,
                      stream: Optional[int] = None) -> None:
    B = r.shape[0]
    _check(_lib.fmp_apply_adjoint_dev(op.handle, _dtype_code(r), r.data_ptr(), B,
                                      h_out.data_ptr() if h_out is not None else None,
                                      argmax_out.data_ptr() if argmax_out is not None else None,
                                      stream))


__all__ = [
    "Context", "SensingOperator", "CorrelationKernel", "compute_kernel", "fast_update",
    "argmax_magnitude", "SolveConfig", "default_config", "RecoveryResult", "omp_solve",
    "omp_solve_batch", "omp_solve_multi", "device_count", "crossover_iteration", "gpu_crossover", "gpu_crossover_for", "make_row_selection", "make_batch", "make_batch_dev", "dd_eval", "derive_seed",
    "FmpError", "InvalidArgument", "RankDeficientError", "Unsupported", "LIB_PATH",
    "least_squares", "IncrementalQR", "cosamp_solve", "cosamp_solve_batch", "cosamp_solve_dev", "adaptive_cosamp_uses_fast",
    "LargeShard", "LocalExchange", "sharded_solve", "large_solve",
]
