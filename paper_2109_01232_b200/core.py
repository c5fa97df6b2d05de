"""Precision tags, the device CSR container and the L1 vector kernels.

Mirrors the reference's ``mpgmres.core`` (pkg/src/mpgmres/core.py) with the
numeric work moved to the sm_100a library:

* ``Precision`` / ``FP32`` / ``FP64``             core.py:86-120
* ``CsrMatrix`` (device-resident, int32 pattern) core.py:123-199
* ``validate_csr`` / ``coo_to_csr``             core.py:202-249 (host setup)
* ``convert_vector`` / ``convert_matrix``       core.py:252-289 -> mpg_convert
* ``gemv``                                       core.py:295-338 -> mpg_gemv
* ``norm2``                                      core.py:341-354 -> mpg_norm2

Vectors may be numpy arrays (uploaded per call, results returned as numpy —
the drop-in path for reference callers) or CUDA torch tensors (stay on the
device).  There is no CPU compute path: without the CUDA extension and a GPU
every numeric function raises.
"""

from __future__ import annotations

import ctypes as C
from contextlib import contextmanager
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib, timing

__all__ = [
    "Precision", "FP32", "FP64", "CsrMatrix", "PrecisionError", "PrecisionOverflowError",
    "ShapeError", "CsrFormatError", "convert_vector", "convert_matrix", "gemv", "norm2",
    "validate_csr", "coo_to_csr", "deterministic_kernels",
]


class PrecisionError(ValueError):
    """Operands of mixed or unsupported precision reached a uniform-precision kernel."""


class PrecisionOverflowError(OverflowError):
    """A value exceeded the finite range of the target precision."""


class ShapeError(ValueError):
    """Operand dimensions do not conform."""


class CsrFormatError(ValueError):
    """A CSR matrix violates canonical form."""


class Precision(Enum):
    """Working precision of a vector or matrix (core.py:86-114)."""

    FP32 = "fp32"
    FP64 = "fp64"

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.float32 if self is Precision.FP32 else np.float64)

    @property
    def torch_dtype(self) -> torch.dtype:
        return torch.float32 if self is Precision.FP32 else torch.float64

    @property
    def code(self) -> int:
        return _lib.FP32 if self is Precision.FP32 else _lib.FP64

    @property
    def unit_roundoff(self) -> float:
        return 2.0 ** -24 if self is Precision.FP32 else 2.0 ** -53

    @property
    def max_finite(self) -> float:
        return float(np.finfo(self.dtype).max)

    @classmethod
    def of(cls, x) -> "Precision":
        dt = getattr(x, "dtype", None)
        if dt is not None:
            if isinstance(dt, torch.dtype):
                if dt == torch.float32:
                    return FP32
                if dt == torch.float64:
                    return FP64
            else:
                try:
                    return _BY_DTYPE[np.dtype(dt)]
                except (KeyError, TypeError):
                    pass
        raise PrecisionError(f"no precision tag for dtype {dt!r}; expected float32 or float64")


FP32 = Precision.FP32
FP64 = Precision.FP64
_BY_DTYPE = {np.dtype(np.float32): FP32, np.dtype(np.float64): FP64}


@contextmanager
def deterministic_kernels():
    """API parity with core.py:51-67.  Every reduction in this library already
    uses a fixed order (per-CTA partials + fixed-order finalisation), so runs
    are bitwise reproducible without pinning anything."""
    yield


# ---------------------------------------------------------------------------
# device plumbing

def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2109_01232_b200 needs a CUDA device (sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


class _DeviceContext:
    """Per-device reduction workspace and a small scalar scratch area."""

    def __init__(self, dev: torch.device):
        lib = _lib.load()
        self.ws = torch.zeros(int(lib.mpg_workspace_bytes()), dtype=torch.uint8, device=dev)
        self.scalars = torch.zeros(64, dtype=torch.float64, device=dev)
        self.iscalars = torch.zeros(16, dtype=torch.int64, device=dev)


_CTX: dict[int, _DeviceContext] = {}


def ctx() -> _DeviceContext:
    dev = device()
    c = _CTX.get(dev.index)
    if c is None:
        c = _CTX[dev.index] = _DeviceContext(dev)
    return c


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


# elements after the S x ldv packed stencil values: the constant-coefficient
# header written by mpg_stencil_pack* (csrc/spmv.cuh kDiaTail) and its scratch
DIA_TAIL = 64
# A/B switch: False keeps the constant-coefficient SpMV path off for new packs
STENCIL_CONST = True


def padded_length(n: int) -> int:
    """Vectors the library owns are padded to a multiple of 64 elements."""
    return max(64, (n + 63) // 64 * 64)


def dvec(n: int, prec: Precision, zero: bool = True) -> torch.Tensor:
    """A padded device vector; returns the full padded buffer."""
    fn = torch.zeros if zero else torch.empty
    return fn(padded_length(n), dtype=prec.torch_dtype, device=device())


def is_device(x) -> bool:
    return isinstance(x, torch.Tensor)


def to_device(x, prec: Precision | None = None) -> torch.Tensor:
    """Contiguous CUDA tensor view/copy of a numpy array or tensor (no cast
    unless ``prec`` is given, in which case the dtype must already match)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.device.type != "cuda":
            t = t.to(device())
    else:
        a = np.ascontiguousarray(np.asarray(x))
        t = torch.from_numpy(a).to(device(), non_blocking=False)
    if not t.is_contiguous():
        t = t.contiguous()
    return t


def padded_copy(x, prec: Precision) -> torch.Tensor:
    """Copy x (host or device, already in `prec`) into a fresh padded buffer."""
    n = int(x.shape[0])
    buf = dvec(n, prec)
    if isinstance(x, torch.Tensor):
        buf[:n].copy_(x if x.device.type == "cuda" else x.to(device()))
    else:
        src = torch.from_numpy(np.ascontiguousarray(x))
        buf[:n].copy_(src.pin_memory() if src.numel() * src.element_size() > (1 << 20) else src,
                      non_blocking=False)
    return buf


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def _result(t: torch.Tensor, like) -> np.ndarray | torch.Tensor:
    return t if isinstance(like, torch.Tensor) else to_host(t)


# ---------------------------------------------------------------------------
# CSR container

def _device_index_array(a, n: int) -> torch.Tensor:
    """int32 device array with >= 16 bytes of readable slack (C-ABI contract)."""
    if isinstance(a, torch.Tensor):
        src = a.to(device=device(), dtype=torch.int32)
    else:
        src = torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=np.int32)).to(device())
    buf = torch.zeros(n + 8, dtype=torch.int32, device=device())
    buf[:n].copy_(src.reshape(-1)[:n])
    return buf[:n]


def _device_value_array(a, n: int) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        src = a.to(device())
    else:
        arr = np.ascontiguousarray(np.asarray(a))
        if arr.dtype not in _BY_DTYPE:
            raise PrecisionError(f"no precision tag for dtype {arr.dtype!r}; expected float32 or float64")
        src = torch.from_numpy(arr).to(device())
    buf = torch.zeros(n + 4, dtype=src.dtype, device=device())
    buf[:n].copy_(src.reshape(-1)[:n])
    return buf[:n]


class CsrMatrix:
    """Device-resident canonical CSR (reference CsrMatrix, core.py:123-199).

    ``row_ptr``/``col_idx`` are int32 CUDA tensors, ``values`` a float32 or
    float64 CUDA tensor; each array is 16-byte aligned with readable slack so
    the kernels can stream it with TMA bulk copies.  Matrices are treated as
    immutable; precision copies share the pattern tensors.
    """

    def __init__(self, n_rows: int, n_cols: int, row_ptr, col_idx, values, *,
                 _trusted: bool = False):
        n_rows, n_cols = int(n_rows), int(n_cols)
        if n_rows < 0 or n_cols < 0:
            raise ShapeError("matrix dimensions must be nonnegative")
        rp_len = int(row_ptr.shape[0]) if hasattr(row_ptr, "shape") else len(row_ptr)
        if rp_len != n_rows + 1:
            raise CsrFormatError("row_ptr must have length n_rows + 1")
        nnz_c = int(col_idx.shape[0]) if hasattr(col_idx, "shape") else len(col_idx)
        nnz_v = int(values.shape[0]) if hasattr(values, "shape") else len(values)
        if nnz_c != nnz_v:
            raise CsrFormatError("col_idx and values must have equal length")
        if not _trusted:
            mx = int(row_ptr.max()) if rp_len and not isinstance(row_ptr, torch.Tensor) else (
                int(row_ptr.max().item()) if rp_len else 0)
            if mx >= 2 ** 31:
                raise CsrFormatError("nnz exceeds the 32-bit index range")
        Precision.of(values)
        self.n_rows, self.n_cols = n_rows, n_cols
        self.row_ptr = row_ptr if _trusted else _device_index_array(row_ptr, n_rows + 1)
        self.col_idx = col_idx if _trusted else _device_index_array(col_idx, nnz_c)
        self.values = values if _trusted else _device_value_array(values, nnz_v)

    # --- reference-compatible surface
    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    @property
    def precision(self) -> Precision:
        return Precision.of(self.values)

    def max_row_nnz(self) -> int:
        if self.n_rows == 0:
            return 0
        return int(torch.diff(self.row_ptr).max().item())

    def row_slice(self, r: int) -> slice:
        a, b = self.row_ptr[r:r + 2].tolist()
        return slice(int(a), int(b))

    def host_arrays(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        return to_host(self.row_ptr), to_host(self.col_idx), to_host(self.values)

    def to_dense(self) -> np.ndarray:
        rp, ci, v = self.host_arrays()
        out = np.zeros((self.n_rows, self.n_cols), dtype=v.dtype)
        out[np.repeat(np.arange(self.n_rows), np.diff(rp)), ci] = v
        return out

    @classmethod
    def from_dense(cls, a) -> "CsrMatrix":
        a = np.asarray(a)
        if a.ndim != 2:
            raise ShapeError("expected a 2-D array")
        if a.dtype not in _BY_DTYPE:
            a = a.astype(np.float64)
        rows, cols = np.nonzero(a)
        ptr_ = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=a.shape[0]))])
        return cls(a.shape[0], a.shape[1], ptr_, cols, a[rows, cols])

    @classmethod
    def from_any(cls, A) -> "CsrMatrix":
        """Accept this class or any CSR-like object (e.g. the reference's
        ``mpgmres.CsrMatrix``) and return a device matrix (uploading once)."""
        if isinstance(A, CsrMatrix):
            return A
        for attr in ("n_rows", "n_cols", "row_ptr", "col_idx", "values"):
            if not hasattr(A, attr):
                raise TypeError(f"expected a CSR matrix, got {type(A).__name__}")
        return cls(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values)

    def copy(self) -> "CsrMatrix":
        return CsrMatrix(self.n_rows, self.n_cols, self.row_ptr.clone(), self.col_idx.clone(),
                         self.values.clone())

    def with_values(self, values: torch.Tensor) -> "CsrMatrix":
        out = CsrMatrix(self.n_rows, self.n_cols, self.row_ptr, self.col_idx, values, _trusted=True)
        out._stencil = getattr(self, "_stencil", None)   # same pattern, same stencil shape
        return out

    # --- stencil-specialised storage (mpg_stencil_pack)
    def stencil_shape(self) -> tuple[int, int] | None:
        """(dims, nx) if the pattern is exactly a Dirichlet 5-point (2-D) or
        7-point (3-D) stencil on an nx-grid, else None.  Decided from the
        sizes, then confirmed on the device by the packing kernel."""
        cached = getattr(self, "_stencil", None)
        if cached is not None:
            return cached or None
        shape = None
        n, nnz = self.n_rows, self.nnz
        if n == self.n_cols and n >= 8:
            c = round(n ** (1.0 / 3.0))
            s = round(n ** 0.5)
            for dims, nx, want in ((3, c, 7 * c ** 3 - 6 * c ** 2), (2, s, 5 * s ** 2 - 4 * s)):
                if nx >= 2 and nx ** dims == n and nnz == want and n < 2 ** 32:
                    if self._pack(dims, nx) is not None:
                        shape = (dims, nx)
                        break
        self._stencil = shape if shape else False
        return shape

    def _pack(self, dims: int, nx: int) -> torch.Tensor | None:
        S = 7 if dims == 3 else 5
        ldv = padded_length(self.n_rows)
        # S x ldv packed values + the constant-coefficient header / scratch tail
        dia = torch.zeros(S * ldv + DIA_TAIL, dtype=self.values.dtype, device=self.values.device)
        bad = torch.zeros(1, dtype=torch.int32, device=self.values.device)
        _lib.call("mpg_stencil_pack", self.precision.code, dims, nx, self.n_rows, ptr(self.row_ptr),
                  ptr(self.col_idx), ptr(self.values), ptr(dia), ldv, ptr(bad), stream_handle())
        if int(bad.item()) != 0:
            return None
        if not STENCIL_CONST:
            dia[S * ldv] = 0          # keep the coefficient-stream path off (A/B, tests)
        self._dia = dia
        return dia

    def stencil_const(self) -> bool:
        """True when the packed stencil has one coefficient per slot (the SpMV
        then streams x alone; csrc/spmv.cuh StencilConst)."""
        d = self.dia()
        if d is None:
            return False
        S = 7 if self.stencil_shape()[0] == 3 else 5
        return bool(d[S * padded_length(self.n_rows)].item() != 0)

    def dia(self) -> torch.Tensor | None:
        """Slot-major packed values (S x ldv) for the stencil path, or None."""
        sh = self.stencil_shape()
        if sh is None:
            return None
        d = getattr(self, "_dia", None)
        if d is None or d.dtype != self.values.dtype:
            d = self._pack(*sh)
        return d

    def __repr__(self) -> str:
        return f"CsrMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz}, {self.precision.value}, cuda)"


def validate_csr(A) -> "CsrMatrix":
    """Canonical-form check (core.py:202-226), on host copies of the arrays."""
    A = CsrMatrix.from_any(A)
    rp, ci, _ = A.host_arrays()
    if rp[0] != 0:
        raise CsrFormatError("row_ptr[0] must be 0")
    if rp[-1] != A.nnz:
        raise CsrFormatError("row_ptr[-1] must equal nnz")
    if np.any(np.diff(rp) < 0):
        raise CsrFormatError("row_ptr must be nondecreasing")
    if A.nnz:
        if ci.min() < 0 or ci.max() >= A.n_cols:
            raise CsrFormatError("column index out of range")
        rows = np.repeat(np.arange(A.n_rows), np.diff(rp))
        same_row = rows[1:] == rows[:-1]
        bad = same_row & (np.diff(ci) <= 0)
        if np.any(bad):
            raise CsrFormatError(f"column indices not strictly increasing near entry {int(np.argmax(bad))}")
    return A


def coo_to_csr(n_rows: int, n_cols: int, rows, cols, values, *,
               sum_duplicates: bool = False) -> CsrMatrix:
    """Canonical CSR from triplets (core.py:229-249); host sort, device result."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    values = np.asarray(values)
    order = np.lexsort((cols, rows))
    rows, cols, values = rows[order], cols[order], values[order]
    if sum_duplicates and rows.size:
        new = np.concatenate([[True], (np.diff(rows) != 0) | (np.diff(cols) != 0)])
        starts = np.flatnonzero(new)
        values = np.add.reduceat(values, starts)
        rows, cols = rows[starts], cols[starts]
    counts = np.bincount(rows, minlength=n_rows) if rows.size else np.zeros(n_rows, dtype=np.int64)
    return CsrMatrix(n_rows, n_cols, np.concatenate([[0], np.cumsum(counts)]), cols, values)


# ---------------------------------------------------------------------------
# kernels

def _overflow_index() -> torch.Tensor:
    t = ctx().iscalars[:1]
    t.fill_(-1)
    return t


def _cast_device(t: torch.Tensor, target: Precision) -> tuple[torch.Tensor, int]:
    """Round a contiguous device vector to `target`; returns (out, first overflow index or -1)."""
    src = Precision.of(t)
    out = torch.empty(t.shape[0], dtype=target.torch_dtype, device=t.device)
    ovf = _overflow_index()
    _lib.call("mpg_convert", src.code, target.code, int(t.shape[0]), ptr(t), ptr(out), ptr(ovf),
              stream_handle())
    i = int(ovf.item()) if target.unit_roundoff > src.unit_roundoff else -1
    return out, i


def convert_vector(x, target: Precision):
    """Round a vector to `target` (core.py:252-272); overflow raises naming the entry."""
    source = Precision.of(x)
    if source is target:
        return x.clone() if isinstance(x, torch.Tensor) else np.asarray(x).copy()
    t = to_device(x)
    out, i = _cast_device(t.reshape(-1), target)
    if i >= 0:
        v = float(t.reshape(-1)[i].item())
        raise PrecisionOverflowError(f"entry {i} ({v!r}) overflows {target.value}")
    return _result(out.reshape(t.shape), x)


def convert_matrix(A, target: Precision) -> CsrMatrix:
    """Values cast to `target`, pattern shared (core.py:275-289)."""
    A = CsrMatrix.from_any(A)
    if A.precision is target:
        return A.with_values(A.values.clone())
    vals = torch.zeros(A.nnz + 4, dtype=target.torch_dtype, device=A.values.device)
    ovf = _overflow_index()
    if A.nnz:
        _lib.call("mpg_convert", A.precision.code, target.code, A.nnz, ptr(A.values), ptr(vals),
                  ptr(ovf), stream_handle())
    if target.unit_roundoff > A.precision.unit_roundoff:
        i = int(ovf.item())
        if i >= 0:
            rp = to_host(A.row_ptr)
            row = int(np.searchsorted(rp, i, side="right")) - 1
            col = int(A.col_idx[i].item())
            raise PrecisionOverflowError(
                f"entry ({row}, {col}) = {float(A.values[i].item())!r} overflows {target.value}")
    return A.with_values(vals[:A.nnz])


def gemv(a, x, y=None, *, alpha: float = 1.0, beta: float = 0.0, transpose: bool = False):
    """y = alpha*op(a) x + beta*y in one precision (core.py:295-338)."""
    host = not isinstance(a, torch.Tensor)
    if host:
        a = np.asarray(a)
        x = np.asarray(x)
    if a.ndim != 2 or x.ndim != 1:
        raise ShapeError("gemv expects a 2-D matrix and a 1-D vector")
    prec = Precision.of(a)
    if x.dtype != a.dtype or (y is not None and y.dtype != a.dtype):
        raise PrecisionError("gemv operands must share one precision; cast explicitly")
    rows, cols = a.shape
    in_len, out_len = (rows, cols) if transpose else (cols, rows)
    if x.shape[0] != in_len:
        raise ShapeError(f"operand length {x.shape[0]} does not match {in_len}")
    if y is not None and tuple(y.shape) != (out_len,):
        raise ShapeError(f"output length {tuple(y.shape)} does not match {out_len}")
    if y is None and beta != 0.0:
        raise ValueError("beta without an output vector")
    if rows == 0 or cols == 0:
        if y is None:
            z = np.zeros(out_len, dtype=prec.dtype)
            return z if host else torch.zeros(out_len, dtype=prec.torch_dtype, device=device())
        y *= beta
        return y
    if host:
        # keep Fortran-ordered multivectors column-major on the device
        ad = to_device(a.T).t() if (a.flags.f_contiguous and not a.flags.c_contiguous) else to_device(a)
    else:
        ad = a
    # express as `nvec` vectors of length `vlen` at stride lda (column-major)
    if ad.stride(0) == 1 and ad.stride(1) >= rows:
        base, vlen, nvec, lda, tr = ad, rows, cols, ad.stride(1), transpose
    elif ad.stride(1) == 1 and ad.stride(0) >= cols:
        base, vlen, nvec, lda, tr = ad, cols, rows, ad.stride(0), not transpose
    else:
        ad = ad.t().contiguous().t()
        base, vlen, nvec, lda, tr = ad, rows, cols, ad.stride(1), transpose
    if tr and nvec > 512 and cols <= 512:
        # the multi-dot kernel handles <= 512 vectors: re-lay the matrix column-major
        ad = ad.t().contiguous().t()
        base, vlen, nvec, lda, tr = ad, rows, cols, ad.stride(1), transpose
    if tr and nvec > 512:
        raise ShapeError("transposed gemv supports at most 512 vectors")
    xd = to_device(x)
    yd = torch.zeros(out_len, dtype=prec.torch_dtype, device=device()) if y is None else to_device(y)
    t0 = timing.tick()
    _lib.call("mpg_gemv", prec.code, 1 if tr else 0, vlen, nvec, ptr(base), lda, ptr(xd), ptr(yd),
              float(alpha), float(beta), ptr(ctx().ws), stream_handle())
    timing.tock(timing.GEMV_TRANS if transpose else timing.GEMV_NOTRANS, t0)
    if host:
        out = to_host(yd)
        if y is not None:
            y[...] = out
            return y
        return out
    if y is not None and yd.data_ptr() != y.data_ptr():
        y.copy_(yd)
        return y
    return yd


def norm2(x) -> float:
    """sqrt(dot(x, x)) accumulated in x's precision (core.py:341-354)."""
    prec = Precision.of(x)
    n = int(x.shape[0]) if x.ndim else 1
    if n == 0:
        return 0.0
    xd = to_device(x).reshape(-1)
    out = ctx().scalars[:1]
    t0 = timing.tick()
    _lib.call("mpg_norm2", prec.code, xd.shape[0], ptr(xd), ptr(out), ptr(ctx().ws), stream_handle())
    v = float(out.item())
    timing.tock(timing.NORM, t0)
    return v
