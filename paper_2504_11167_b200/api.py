"""Python mirror of the lrspike operations over the C-ABI (include/lrspike_capi.h).

Names, argument meaning and error behaviour follow the reference interface:
``CsrMatrix``/``spmv``/``band_metrics`` (proj/core/include/lrspike/matrix.hpp),
the exception taxonomy (proj/core/include/lrspike/errors.hpp:11-94), and the
SPEC operations make_layout / factorize / solve_block / apply_precond_T /
apply_block_jacobi / bicgstab / solve.  GMRES(m) is the one
added method.

Every call goes to liblrspike_cuda.so; there is no CPU fallback: importing this
module on a machine without the built library raises, and any operation on a
machine without a GPU fails with CudaError.

Arrays: numpy arrays are host buffers (copied by the library); torch CUDA
tensors (or any object with ``data_ptr()`` and ``is_cuda``) are used in place
on the device.  Blocks are column-major (Fortran order), shape (n, n_rhs).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.environ.get("LRS_LIB") or os.path.join(_HERE, "liblrspike_cuda.so")

LRS_OK = 0
F64, C128 = 0, 1
MEM_HOST, MEM_DEVICE = 0, 1
VARIANT_T, VARIANT_BJ, VARIANT_I, VARIANT_OTF = 0, 1, 2, 3
_VARIANTS = {"T": VARIANT_T, "BJ": VARIANT_BJ, "I": VARIANT_I, "OTF": VARIANT_OTF}
GMRES, BICGSTAB, CG = 0, 1, 2
_METHODS = {"gmres": GMRES, "bicgstab": BICGSTAB, "cg": CG}
SIDE_T, SIDE_W = 0, 1
_SPIKE_MODES = {"spike": 0, "coupling": 1}  # lrs_spike_mode
STAGES = ("reduced-matvec", "precond-apply", "recovery")
KERNEL_CLASSES = ("lu_diag", "lu_panel", "lu_update", "band_solve", "band_solve_adjoint", "spmv",
                  "iface_apply", "recovery", "krylov_vec", "setup_misc", "spike_band_solve")

i64, f64, i32, u64 = ctypes.c_int64, ctypes.c_double, ctypes.c_int32, ctypes.c_uint64
vp = ctypes.c_void_p


class SolverCfgC(ctypes.Structure):
    _fields_ = [("variant", i32), ("passes", i32), ("p", i64), ("k", i64), ("n_svd", i64),
                ("oversample", i64), ("seed", u64), ("inner_tol", f64), ("inner_max_iters", i64),
                ("otf_tol", f64), ("otf_max_iters", i64), ("otf_escalations", i32),
                ("factor_fp32", i32), ("spike_mode", i32)]


class IterCfgC(ctypes.Structure):
    _fields_ = [("method", i32), ("restart", i32), ("tol", f64), ("max_iters", i64),
                ("breakdown_eps", f64), ("x0", vp)]


class ReportC(ctypes.Structure):
    _fields_ = [("converged", i32), ("breakdown", i32), ("iterations", f64),
                ("precond_applications", i64), ("matvecs", i64), ("residual_final", f64),
                ("comm_messages", i64 * 3), ("comm_scalars", i64 * 3), ("t_solve", f64),
                ("seed", u64), ("history", ctypes.POINTER(f64)), ("history_cap", i64),
                ("history_len", i64), ("history_total", i64), ("inner_iterations", f64),
                ("inner_solves", i64), ("comm_calls", i64), ("comm_host_syncs", i64),
                ("scalar_syncs", i64)]


class FactInfoC(ctypes.Structure):
    _fields_ = [("n", i64), ("p", i64), ("k", i64), ("n_svd", i64), ("l", i64), ("kl", i64),
                ("ku", i64), ("nb", i64), ("wl", i64), ("wu", i64), ("factor_bytes", i64),
                ("lu_flops", i64), ("apply_bytes", i64), ("rank_collapsed", i32),
                ("variant", i32), ("t_factorize", f64), ("t_lu", f64), ("t_spikes", f64),
                ("t_precond", f64), ("max_interface_cond", f64), ("lu_pairs", i32),
                ("pivoted", i32), ("lu_int8", i32), ("lu_sym", i32)]


_OPFN = ctypes.CFUNCTYPE(i32, vp, vp, vp, i64, i64)


class OperatorC(ctypes.Structure):
    _fields_ = [("user", vp), ("apply", _OPFN)]


class ErrorInfoC(ctypes.Structure):
    _fields_ = [("status", i32), ("message", ctypes.c_char * 512), ("line", i64), ("row", i64),
                ("col", i64), ("column", i64), ("interface_index", i64),
                ("cond_estimate", f64)]


# ---- exceptions: errors.hpp:11-94 -------------------------------------------------------
class Error(RuntimeError):
    """lrspike::Error (errors.hpp:11)."""


class ParseError(Error):
    def __init__(self, msg, line=-1):
        super().__init__(msg)
        self.line = line


class UnsupportedFieldError(Error):
    pass


class DimensionError(Error):
    pass


class SingularScalingError(Error):
    def __init__(self, msg, row=-1):
        super().__init__(msg)
        self.row = row


class LayoutError(Error):
    pass


class NotBlockTridiagonalError(Error):
    def __init__(self, msg, row=-1, col=-1):
        super().__init__(msg)
        self.row, self.col = row, col


class SingularBlockError(Error):
    def __init__(self, msg, column=-1):
        super().__init__(msg)
        self.column = column


class ParameterError(Error):
    pass


class IllConditionedInterfaceError(Error):
    def __init__(self, msg, interface_index=-1, cond_estimate=0.0):
        super().__init__(msg)
        self.interface_index, self.cond_estimate = interface_index, cond_estimate


class BreakdownError(Error):
    """BiCGStab stagnation; carries the partial x and the report."""

    def __init__(self, msg, x=None, report=None):
        super().__init__(msg)
        self.x, self.report = x, report


class CudaError(Error):
    pass


class OutOfMemoryError(Error):
    pass


class NotImplementedOnGpu(Error):
    pass


class PreconditionerFailureError(Error):
    """LR-SPIKE-I inner reduced solve did not converge."""


_lib = None


def lib():
    """Load liblrspike_cuda.so; raise loudly if it was not built (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIBPATH):
        raise ImportError(f"{_LIBPATH} is missing: build it with `make` (__graft_entry__.build())")
    L = ctypes.CDLL(_LIBPATH)
    P = ctypes.POINTER
    sig = {
        "lrs_ctx_create": (i32, [ctypes.c_int, vp, P(vp)]),
        "lrs_ctx_destroy": (None, [vp]),
        "lrs_ctx_stream": (vp, [vp]),
        "lrs_ctx_launch_count": (i64, [vp]),
        "lrs_ctx_synchronize": (i32, [vp]),
        "lrs_last_error": (i32, [vp, P(ErrorInfoC)]),
        "lrs_status_string": (ctypes.c_char_p, [i32]),
        "lrs_mat_upload_csr": (i32, [vp, i64, i64, vp, vp, vp, i32, i32, P(vp)]),
        "lrs_mat_destroy": (None, [vp]),
        "lrs_mat_band_metrics": (i32, [vp, P(i64), P(i64), P(i64), P(f64), P(f64)]),
        "lrs_spmv": (i32, [vp, vp, i64, vp, i64, i64, i32, i32]),
        "lrs_make_layout": (i32, [i64, i64, i64, P(i64)]),
        "lrs_factorize": (i32, [vp, vp, P(SolverCfgC), P(vp)]),
        "lrs_fact_destroy": (None, [vp]),
        "lrs_fact_get_info": (i32, [vp, P(FactInfoC)]),
        "lrs_fact_get_layout": (i32, [vp, vp, vp]),
        "lrs_fact_get_spike": (i32, [vp, i64, i32, vp, vp, vp]),
        "lrs_fact_get_tiles": (i32, [vp, i64, vp, i64, P(i64)]),
        "lrs_fact_get_ledger": (i32, [vp, vp, vp]),
        "lrs_solve_block": (i32, [vp, i64, vp, i64, vp, i64, i64, i32, i32]),
        "lrs_apply_precond": (i32, [vp, vp, i64, vp, i64, i64, i32]),
        "lrs_apply_block_jacobi": (i32, [vp, vp, i64, vp, i64, i64, i32]),
        "lrs_apply_precond_T": (i32, [vp, vp, i64, vp, i64, i64, i32]),
        "lrs_reduced_apply": (i32, [vp, i32, vp, i64, vp, i64, i64, i32]),
        "lrs_solve": (i32, [vp, vp, vp, i64, vp, i64, i64, P(IterCfgC), P(ReportC), i32]),
        "lrs_bench_dmma_peak": (i32, [vp, P(f64)]),
        "lrs_bench_i8_peak": (i32, [vp, P(f64)]),
        "lrs_krylov": (i32, [vp, i64, i32, P(OperatorC), P(OperatorC), vp, i64, vp, i64, i64,
                             P(IterCfgC), P(ReportC), i32]),
        "lrs_trunc_precond_create": (i32, [vp, i32, i64, i64, i64, vp, vp, vp, vp, vp, vp, i32,
                                           P(vp)]),
        "lrs_dense_qr": (i32, [vp, i32, i64, i64, vp, i64, vp, i32]),
        "lrs_dense_svd": (i32, [vp, i32, i64, vp, vp, vp, vp, i32]),
        "lrs_dense_gemm": (i32, [vp, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, i32, i32]),
        "lrs_ctx_set_profiling": (i32, [vp, i32]),
        "lrs_ctx_kernel_times": (i32, [vp, vp, vp, i32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


_EXC = {1: ParseError, 2: UnsupportedFieldError, 3: DimensionError, 4: SingularScalingError,
        5: LayoutError, 6: NotBlockTridiagonalError, 7: SingularBlockError, 8: ParameterError,
        9: IllConditionedInterfaceError, 10: BreakdownError, 11: CudaError, 12: OutOfMemoryError,
        13: CudaError, 14: NotImplementedOnGpu, 15: PreconditionerFailureError}


def _raise(status: int, ctx_handle=None):
    info = ErrorInfoC()
    lib().lrs_last_error(ctx_handle, ctypes.byref(info))
    msg = info.message.decode(errors="replace") or lib().lrs_status_string(status).decode()
    cls = _EXC.get(status, Error)
    if cls is NotBlockTridiagonalError:
        raise cls(msg, info.row, info.col)
    if cls is SingularBlockError:
        raise cls(msg, info.column)
    if cls is IllConditionedInterfaceError:
        raise cls(msg, info.interface_index, info.cond_estimate)
    if cls is ParseError:
        raise cls(msg, info.line)
    if cls is SingularScalingError:
        raise cls(msg, info.row)
    raise cls(msg)


def _check(status, ctx_handle=None):
    if status != LRS_OK:
        _raise(status, ctx_handle)


def _is_device(a) -> bool:
    return bool(getattr(a, "is_cuda", False))


def _torch_dtype(dtype):
    import torch

    return torch.complex128 if np.dtype(dtype) == np.complex128 else torch.float64


def _buf(a, n_rows, dtype=np.float64):
    """(pointer, ld, mem, ncols) of a column-major block (numpy F-order or torch CUDA)
    of the matrix scalar type (float64, or interleaved complex128)."""
    if _is_device(a):
        if a.dtype != _torch_dtype(dtype):
            raise DimensionError(f"device block must be {np.dtype(dtype).name}")
        if a.dim() == 1:
            return a.data_ptr(), n_rows, MEM_DEVICE, 1
        # torch: column-major blocks are stored as (n_rhs, n) row-major == (n, n_rhs) F-order
        if a.stride(0) == 1:
            # a single column's stride is arbitrary (numpy / torch relaxed strides)
            ld = a.stride(1) if a.shape[1] > 1 else max(n_rows, 1)
            return a.data_ptr(), ld, MEM_DEVICE, a.shape[1]
        raise DimensionError("device block must be column-major (stride(0) == 1)")
    arr = np.asarray(a)
    if arr.ndim == 1:
        arr = arr.reshape(-1, 1)
    if not (arr.flags.f_contiguous and arr.dtype == np.dtype(dtype)):
        raise DimensionError(f"host block must be {np.dtype(dtype).name} Fortran-ordered")
    return arr.ctypes.data, arr.shape[0], MEM_HOST, arr.shape[1]


def _check_out(mem, nc, memx, ncx):
    """x_out must live where b lives (the library copies / writes through one memory
    kind per call) and hold at least b's columns."""
    if memx != mem:
        raise DimensionError("x_out must live in the same memory as the right-hand side")
    if ncx < nc:
        raise DimensionError(f"x_out has {ncx} columns, the right-hand side {nc}")


class Context:
    """One device + one stream (lrs_ctx).  ``stream`` may be a torch stream handle."""

    def __init__(self, device: int = 0, stream: int | None = None):
        h = vp()
        _check(lib().lrs_ctx_create(device, stream, ctypes.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().lrs_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return lib().lrs_ctx_stream(self.h) or 0

    @property
    def launches(self) -> int:
        return lib().lrs_ctx_launch_count(self.h)

    def synchronize(self):
        _check(lib().lrs_ctx_synchronize(self.h), self.h)

    def set_profiling(self, on: bool, classes=None):
        """Per-kernel-class CUDA-event timing; `classes` (names of KERNEL_CLASSES) limits it
        to those classes."""
        v = 1 if on else 0
        if on and classes is not None:
            v = sum(1 << (KERNEL_CLASSES.index(k) + 1) for k in classes) or 0
        _check(lib().lrs_ctx_set_profiling(self.h, v), self.h)

    def kernel_times(self, reset: bool = False) -> dict:
        """{class: (total_ms, launches)} of the CUDA-event timed launches."""
        ms, cnt = (f64 * len(KERNEL_CLASSES))(), (i64 * len(KERNEL_CLASSES))()
        _check(lib().lrs_ctx_kernel_times(self.h, ms, cnt, 1 if reset else 0), self.h)
        return {k: (ms[i], cnt[i]) for i, k in enumerate(KERNEL_CLASSES)}

    def dmma_peak_tflops(self) -> float:
        out = f64()
        _check(lib().lrs_bench_dmma_peak(self.h, ctypes.byref(out)), self.h)
        return out.value

    def i8_peak_tops(self) -> float:
        out = f64()
        _check(lib().lrs_bench_i8_peak(self.h, ctypes.byref(out)), self.h)
        return out.value


@dataclass
class BandMetrics:
    """matrix.hpp:58-70."""

    ku: int
    kl: int
    k: int
    diag_weight: float
    band_density: float


class CsrMatrix:
    """Device-resident CsrMatrix (matrix.hpp:22-48).  ``validate()`` semantics are
    enforced at upload (DimensionError, matrix.cpp:21-37)."""

    def __init__(self, ctx: Context, n, row_ptr, col_idx, values):
        self.ctx = ctx
        self.n = int(n)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int64)
        cplx = np.iscomplexobj(values)
        self.dtype = np.dtype(np.complex128 if cplx else np.float64)
        va = np.ascontiguousarray(values, dtype=self.dtype)
        if rp.shape[0] != self.n + 1:
            raise DimensionError("row_ptr length must be n_rows + 1")
        if ci.shape[0] != va.shape[0]:
            raise DimensionError("col_idx/values length mismatch")
        h = vp()
        _check(lib().lrs_mat_upload_csr(ctx.h, self.n, va.shape[0], rp.ctypes.data, ci.ctypes.data,
                                        va.ctypes.data, C128 if cplx else F64, MEM_HOST,
                                        ctypes.byref(h)), ctx.h)
        self.h = h
        self.nnz = int(va.shape[0])

    @classmethod
    def from_csr(cls, ctx, csr):
        return cls(ctx, csr.n, csr.row_ptr, csr.col_idx, csr.values)

    def __del__(self):
        # a matrix may outlive Context.close() (e.g. held by a pytest traceback past the
        # fixture's close): lrs_ctx_destroy defers the context teardown until its last
        # matrix / factorization handle is destroyed, so the handle is always freed here
        try:
            if self.h:
                lib().lrs_mat_destroy(self.h)
            self.h = None
        except Exception:
            pass

    def band_metrics(self) -> BandMetrics:
        ku, kl, k, dw, bd = i64(), i64(), i64(), f64(), f64()
        _check(lib().lrs_mat_band_metrics(self.h, ctypes.byref(ku), ctypes.byref(kl),
                                          ctypes.byref(k), ctypes.byref(dw), ctypes.byref(bd)))
        return BandMetrics(ku.value, kl.value, k.value, dw.value, bd.value)

    def spmv(self, X, out=None, accumulate=False):
        """matrix.cpp:121-136: returns A X (or out += A X)."""
        px, ldx, mem, nc = _buf(X, self.n, self.dtype)
        if out is None:
            if mem == MEM_DEVICE:
                import torch

                out = torch.zeros((nc, self.n), dtype=_torch_dtype(self.dtype),
                                  device=X.device).t()
            else:
                out = np.zeros((self.n, nc), dtype=self.dtype, order="F")
        py, ldy, memy, _ = _buf(out, self.n, self.dtype)
        if memy != mem:
            raise DimensionError("x and y must live in the same memory")
        _check(lib().lrs_spmv(self.h, px, ldx, py, ldy, nc, 1 if accumulate else 0, mem),
               self.ctx.h)
        return out


def band_metrics(A: CsrMatrix) -> BandMetrics:
    return A.band_metrics()


def make_layout(n: int, p: int, k: int) -> list:
    """SPEC.md:171-179."""
    sizes = (i64 * max(p, 1))()
    _check(lib().lrs_make_layout(n, p, k, sizes))
    return list(sizes)


@dataclass
class SolverConfig:
    """SPEC.md:470-473.  variant: "T" (LR-SPIKE-T), "I" (LR-SPIKE-I), "OTF"
    (LR-SPIKE-OTF), "BJ" (Block Jacobi); inner_*: the LR-SPIKE-I reduced solve; otf_*:
    the LR-SPIKE-OTF reduced solve and its tolerance escalations."""

    variant: str = "T"
    p: int = 4
    k: int | None = None
    n_svd: int = 8
    oversample: int | None = None
    passes: int = 2
    seed: int = 0
    inner_tol: float = 1e-12
    inner_max_iters: int = 200
    otf_tol: float = 1e-8
    otf_max_iters: int = 500
    otf_escalations: int = 4
    factor_fp32: bool = False  # FP32 off-diagonal factor tiles in the applies
    # "spike" (default) | "coupling" (truncated SVD of B_i / C_i, then
    # padded solves against its singular vectors; north_star setup (1))
    spike_mode: str = "spike"

    def c(self):
        if self.variant not in _VARIANTS:
            raise ParameterError(f"unknown variant {self.variant!r}")
        if self.spike_mode not in _SPIKE_MODES:
            raise ParameterError(f"unknown spike_mode {self.spike_mode!r}")
        return SolverCfgC(_VARIANTS[self.variant], self.passes, self.p, self.k or 0, self.n_svd,
                          -1 if self.oversample is None else self.oversample, self.seed,
                          self.inner_tol, self.inner_max_iters, self.otf_tol, self.otf_max_iters,
                          self.otf_escalations, 1 if self.factor_fp32 else 0,
                          _SPIKE_MODES[self.spike_mode])


@dataclass
class IterConfig:
    """SPEC.md:411-414 (+ method and GMRES restart)."""

    tol: float = 1e-8
    max_iters: int = 1000
    breakdown_eps: float = 1e-30
    initial_guess: object = None
    method: str = "bicgstab"
    restart: int = 30


@dataclass
class SolveReport:
    """SPEC.md:415-419 + CommLedger."""

    converged: bool
    iterations: float
    residual_history: list
    precond_applications: int
    matvecs: int
    residual_final: float
    comm: dict
    seed: int
    wall_time: float
    breakdown: bool
    inner_iterations: float = 0.0  # LR-SPIKE-I inner half-iterations (summed)
    inner_solves: int = 0
    # host round trips of the solve (lrs_report): transport calls, stream syncs forced by a
    # host-callback transport, syncs to read Krylov scalars
    round_trips: dict = None


class SpikeFactorization:
    """factorize result; immutable, reusable across solves."""

    def __init__(self, ctx: Context, A: CsrMatrix, cfg: SolverConfig):
        self.ctx, self.A, self.cfg = ctx, A, cfg
        h = vp()
        c = cfg.c()
        _check(lib().lrs_factorize(ctx.h, A.h, ctypes.byref(c), ctypes.byref(h)), ctx.h)
        self.h = h
        inf = FactInfoC()
        _check(lib().lrs_fact_get_info(h, ctypes.byref(inf)))
        self.info = {f: getattr(inf, f) for f, _ in FactInfoC._fields_}
        P = self.info["p"]
        sz, of = (i64 * P)(), (i64 * P)()
        _check(lib().lrs_fact_get_layout(h, sz, of))
        self.sizes, self.offsets = list(sz), list(of)

    def __del__(self):
        try:
            if self.h:  # see CsrMatrix.__del__
                lib().lrs_fact_destroy(self.h)
            self.h = None
        except Exception:
            pass

    @property
    def n_svd(self) -> int:
        return self.info["n_svd"]

    def _apply(self, fn, f, out):
        dt = self.A.dtype
        pin, ldi, mem, nc = _buf(f, self.A.n, dt)
        if out is None:
            if mem == MEM_DEVICE:
                import torch

                out = torch.empty((nc, self.A.n), dtype=_torch_dtype(dt), device=f.device).t()
            else:
                out = np.empty((self.A.n, nc), dtype=dt, order="F")
        po, ldo, memo, _ = _buf(out, self.A.n, dt)
        if memo != mem:
            raise DimensionError("in and out must live in the same memory")
        _check(fn(self.h, pin, ldi, po, ldo, nc, mem), self.ctx.h)
        return out

    def apply_precond_T(self, f, out=None):
        """SPEC.md:485-493 (Block Jacobi if the factorization has n_svd = 0)."""
        return self._apply(lib().lrs_apply_precond_T, f, out)

    def apply_precond_I(self, f, out=None):
        """SPEC.md:494-502 (an LR-SPIKE-I factorization)."""
        if self.cfg.variant != "I":
            raise ParameterError("apply_precond_I needs a variant 'I' factorization")
        return self._apply(lib().lrs_apply_precond, f, out)

    def apply(self, f, out=None):
        """The factorization's own preconditioner (I, T or Block Jacobi)."""
        return self._apply(lib().lrs_apply_precond, f, out)

    def apply_block_jacobi(self, f, out=None):
        """SPEC.md:512-519."""
        return self._apply(lib().lrs_apply_block_jacobi, f, out)

    def _reduced(self, kind, xr):
        xr = np.asfortranarray(np.asarray(xr, dtype=self.A.dtype))
        if xr.ndim == 1:
            xr = xr.reshape(-1, 1)
        y = np.empty_like(xr, order="F")
        _check(lib().lrs_reduced_apply(self.h, kind, xr.ctypes.data, xr.shape[0], y.ctypes.data,
                                       y.shape[0], xr.shape[1], MEM_HOST), self.ctx.h)
        return y

    def matvec_lowrank(self, xr):
        """SPEC.md:349-357 on a ReducedVector block (2 k p x n_rhs, tips [t_0; b_0; t_1; ...])."""
        return self._reduced(0, xr)

    def matvec_exact(self, xr):
        """SPEC.md:340-348 / :358-366 (exact spike tips applied on the fly)."""
        return self._reduced(1, xr)

    def apply_truncated_precond(self, gr):
        """SPEC.md:376-385 on a ReducedVector block."""
        return self._reduced(2, gr)

    def solve_block(self, i: int, R, adjoint: bool = False):
        """SPEC.md:226-241 on partition i (host arrays)."""
        if not 0 <= i < len(self.sizes):
            raise ParameterError(f"partition index {i} outside [0, {len(self.sizes)})")
        R = np.asarray(R, dtype=self.A.dtype)
        if R.ndim == 1:
            R = R.reshape(-1, 1)
        if R.ndim != 2 or R.shape[0] != self.sizes[i]:
            raise DimensionError(f"right-hand side must have {self.sizes[i]} rows (partition {i})")
        R = np.asfortranarray(R)
        X = np.empty_like(R, order="F")
        _check(lib().lrs_solve_block(self.h, i, R.ctypes.data, R.shape[0], X.ctypes.data,
                                     X.shape[0], R.shape[1], 1 if adjoint else 0, MEM_HOST),
               self.ctx.h)
        return X

    def solve_block_adjoint(self, i: int, R):
        return self.solve_block(i, R, True)

    def spike(self, i: int, side: int):
        """(u n_i x r, sigma r, v r x k) of LowRankSpike T_i / W_i."""
        r, k, ni = self.n_svd, self.info["k"], self.sizes[i]
        u = np.empty((ni, r), dtype=self.A.dtype, order="F")
        s = np.empty(r)
        v = np.empty((r, k), dtype=self.A.dtype, order="F")
        _check(lib().lrs_fact_get_spike(self.h, i, side, u.ctypes.data, s.ctypes.data,
                                        v.ctypes.data), self.ctx.h)
        return u, s, v

    def tiles(self, i: int) -> np.ndarray:
        need = i64()
        _check(lib().lrs_fact_get_tiles(self.h, i, None, 0, ctypes.byref(need)), self.ctx.h)
        nb = self.info["nb"]
        W = self.info["wl"] + self.info["wu"] + 1
        out = np.empty(need.value)
        _check(lib().lrs_fact_get_tiles(self.h, i, out.ctypes.data, need.value,
                                        ctypes.byref(need)), self.ctx.h)
        if self.A.dtype == np.complex128:
            out = out.view(np.complex128)
        return out.reshape(-1, W, nb, nb).transpose(0, 1, 3, 2)  # [I][J-slot][row][col]

    def ledger(self) -> dict:
        m, s = (i64 * 3)(), (i64 * 3)()
        _check(lib().lrs_fact_get_ledger(self.h, m, s))
        return {STAGES[i]: (m[i], s[i]) for i in range(3)}


class TruncatedPrecond:
    """build_truncated_precond from explicit spikes, on the device.

    spikes_T[i] = (u, sigma, v) of T_i (i = 0..p-2), spikes_W[i] = those of W_{i+1}; only
    the two k-row tips of u are used (spike_tips).  apply(g) = apply_truncated_precond and
    matvec_lowrank(x) on ReducedVector blocks (2 k p x n_rhs, partition
    i's top tip in rows [2ki, 2ki + k), its bottom tip in [2ki + k, 2k(i+1))).
    IllConditionedInterfaceError(interface, cond_1) above cond_1 = 1e12."""

    def __init__(self, ctx: Context, spikes_T, spikes_W, k: int):
        self.ctx, self.k = ctx, int(k)
        self.p = len(spikes_T) + 1
        r = len(spikes_T[0][1])
        cplx = any(np.iscomplexobj(s[0]) or np.iscomplexobj(s[2]) for s in spikes_T + spikes_W)
        self.dtype = np.dtype(np.complex128 if cplx else np.float64)
        cat = lambda blocks: np.ascontiguousarray(  # noqa: E731
            np.concatenate([np.asarray(b, dtype=self.dtype).ravel(order="F") for b in blocks]))
        tips = lambda u: np.concatenate([u[:self.k], u[-self.k:]])  # noqa: E731  2k x r
        uT = cat([tips(u) for u, _, _ in spikes_T])
        uW = cat([tips(u) for u, _, _ in spikes_W])
        vT = cat([v for _, _, v in spikes_T])
        vW = cat([v for _, _, v in spikes_W])
        sT = np.ascontiguousarray(np.concatenate([np.asarray(s, float) for _, s, _ in spikes_T]))
        sW = np.ascontiguousarray(np.concatenate([np.asarray(s, float) for _, s, _ in spikes_W]))
        h = vp()
        _check(lib().lrs_trunc_precond_create(ctx.h, C128 if cplx else F64, self.p, self.k, r,
                                              uT.ctypes.data, vT.ctypes.data, sT.ctypes.data,
                                              uW.ctypes.data, vW.ctypes.data, sW.ctypes.data,
                                              MEM_HOST, ctypes.byref(h)), ctx.h)
        self.h, self.n_svd = h, r

    def __del__(self):
        try:
            if self.h:
                lib().lrs_fact_destroy(self.h)
            self.h = None
        except Exception:
            pass

    def _op(self, kind, x):
        X = np.asfortranarray(np.asarray(x, dtype=self.dtype).reshape(2 * self.k * self.p, -1))
        Y = np.empty_like(X, order="F")
        _check(lib().lrs_reduced_apply(self.h, kind, X.ctypes.data, X.shape[0], Y.ctypes.data,
                                       Y.shape[0], X.shape[1], MEM_HOST), self.ctx.h)
        return Y

    def apply(self, g):
        return self._op(2, g)

    def matvec_lowrank(self, x):
        return self._op(0, x)


def build_truncated_precond(ctx: Context, spikes_T, spikes_W, k: int) -> TruncatedPrecond:
    return TruncatedPrecond(ctx, spikes_T, spikes_W, k)


def factorize(ctx: Context, A: CsrMatrix, cfg: SolverConfig) -> SpikeFactorization:
    return SpikeFactorization(ctx, A, cfg)


def solve(A: CsrMatrix, f, cfg: SolverConfig | None = None, it: IterConfig | None = None,
          F: SpikeFactorization | None = None, x_out=None, history_cap: int = 4096):
    """factorize (or reuse F) and run the outer Krylov method.
    Returns (x, SolveReport, F).  Non-convergence is reported, not raised."""
    it = it or IterConfig()
    if F is None:
        F = SpikeFactorization(A.ctx, A, cfg or SolverConfig())
    dt = A.dtype
    pb, ldb, mem, nc = _buf(f, A.n, dt)
    if x_out is None:
        if mem == MEM_DEVICE:
            import torch

            x_out = torch.empty((nc, A.n), dtype=_torch_dtype(dt), device=f.device).t()
        else:
            x_out = np.empty((A.n, nc), dtype=dt, order="F")
    px, ldx, memx, ncx = _buf(x_out, A.n, dt)
    _check_out(mem, nc, memx, ncx)
    x0p = None
    if it.initial_guess is not None:
        x0p, ldx0, mem0, nc0 = _buf(it.initial_guess, A.n, dt)
        if mem0 != mem or ldx0 != ldx or nc0 < nc:
            raise DimensionError("initial guess must match x's memory kind and layout")
    if it.method not in _METHODS:
        raise ParameterError(f"unknown Krylov method {it.method!r}")
    ic = IterCfgC(_METHODS[it.method], it.restart, it.tol, it.max_iters,
                  it.breakdown_eps, x0p)
    hist = (f64 * history_cap)()
    rep = ReportC()
    rep.history = ctypes.cast(hist, ctypes.POINTER(f64))
    rep.history_cap = history_cap
    st = lib().lrs_solve(F.h, A.h, pb, ldb, px, ldx, nc, ctypes.byref(ic), ctypes.byref(rep), mem)
    report = SolveReport(bool(rep.converged), rep.iterations, list(hist[:rep.history_len]),
                         rep.precond_applications, rep.matvecs, rep.residual_final,
                         {STAGES[i]: (rep.comm_messages[i], rep.comm_scalars[i]) for i in range(3)},
                         rep.seed, rep.t_solve, bool(rep.breakdown), rep.inner_iterations,
                         rep.inner_solves, {"comm_calls": rep.comm_calls,
                                            "comm_host_syncs": rep.comm_host_syncs,
                                            "scalar_syncs": rep.scalar_syncs})
    if st == 10:
        info = ErrorInfoC()
        lib().lrs_last_error(A.ctx.h, ctypes.byref(info))
        raise BreakdownError(info.message.decode(), x_out, report)
    _check(st, A.ctx.h)
    return x_out, report, F


class _DevBlock:
    """Zero-copy column-major device block (n x n_rhs, leading dimension ld) for torch."""

    def __init__(self, ptr, ld, nrhs, dtype):
        self.__cuda_array_interface__ = {
            "shape": (int(nrhs), int(ld)), "typestr": "<c16" if dtype == np.complex128 else "<f8",
            "data": (int(ptr), False), "version": 3, "strides": None}


def _operator(fn, n, dtype):
    """Wrap fn(x, y) (torch CUDA column-major views, y written in place) as an lrs_operator."""
    import torch

    def cb(user, pin, pout, ld, nrhs):
        try:
            xin = torch.as_tensor(_DevBlock(pin, ld, nrhs, dtype), device="cuda")[:, :n].t()
            yout = torch.as_tensor(_DevBlock(pout, ld, nrhs, dtype), device="cuda")[:, :n].t()
            fn(xin, yout)
            torch.cuda.synchronize()
            return 0
        except Exception:  # reported to the caller as a failed callback
            import traceback

            traceback.print_exc()
            return 1

    f = _OPFN(cb)
    return OperatorC(None, f), f


def krylov(ctx: Context, apply_A, b, it: IterConfig | None = None, apply_M=None, x_out=None,
           history_cap: int = 4096):
    """bicgstab / cg (it.method; "gmres" too) on caller operators.

    apply_A(x, y) and apply_M(x, y) receive column-major torch CUDA views (n x n_rhs) of
    the library's device blocks and must write y = Op(x) (e.g. ``A.spmv(x, y)`` or
    ``F.apply_precond_T(x, y)``).  apply_M None = identity.  Returns (x, SolveReport)."""
    it = it or IterConfig()
    b_arr = b
    dt = np.complex128 if (getattr(b, "dtype", None) in (np.complex128,) or
                           str(getattr(b, "dtype", "")) == "torch.complex128") else np.float64
    n = int(b.shape[0])
    pb, ldb, mem, nc = _buf(b_arr, n, dt)
    if x_out is None:
        if mem == MEM_DEVICE:
            import torch

            x_out = torch.empty((nc, n), dtype=_torch_dtype(dt), device=b.device).t()
        else:
            x_out = np.empty((n, nc), dtype=dt, order="F")
    px, ldx, memx, ncx = _buf(x_out, n, dt)
    _check_out(mem, nc, memx, ncx)
    if it.method not in _METHODS:
        raise ParameterError(f"unknown Krylov method {it.method!r}")
    x0p = None
    if it.initial_guess is not None:
        x0p, ldx0, mem0, nc0 = _buf(it.initial_guess, n, dt)
        if mem0 != mem or ldx0 != ldx or nc0 < nc:
            raise DimensionError("initial guess must match x's memory kind and layout")
    ic = IterCfgC(_METHODS[it.method], it.restart, it.tol, it.max_iters, it.breakdown_eps, x0p)
    opA, keepA = _operator(apply_A, n, dt)
    opM, keepM = (_operator(apply_M, n, dt) if apply_M is not None else (None, None))
    hist = (f64 * history_cap)()
    rep = ReportC()
    rep.history = ctypes.cast(hist, ctypes.POINTER(f64))
    rep.history_cap = history_cap
    st = lib().lrs_krylov(ctx.h, n, C128 if dt == np.complex128 else F64, ctypes.byref(opA),
                          ctypes.byref(opM) if opM is not None else None, pb, ldb, px, ldx, nc,
                          ctypes.byref(ic), ctypes.byref(rep), mem)
    del keepA, keepM
    report = SolveReport(bool(rep.converged), rep.iterations, list(hist[:rep.history_len]),
                         rep.precond_applications, rep.matvecs, rep.residual_final,
                         {STAGES[i]: (0, 0) for i in range(3)}, 0, rep.t_solve,
                         bool(rep.breakdown))
    if st == 10:
        info = ErrorInfoC()
        lib().lrs_last_error(ctx.h, ctypes.byref(info))
        raise BreakdownError(info.message.decode(), x_out, report)
    _check(st, ctx.h)
    return x_out, report
