"""Finite-difference stencil matrices generated directly on the device.

Mirrors the reference's ``mpgmres.gen`` (pkg/src/mpgmres/gen.py).  Where the
reference builds COO triplets and lexsorts them (gen.py:146-202 +
core.py:229-249), ``generate`` launches one kernel (csrc/misc_kernels.cu,
k_generate) that writes each row's entries in ascending column order with
the reference's fp64 coefficient expressions evaluated without FMA
contraction, and row pointers from closed-form per-offset counts.  The
result is bit-identical (pattern and value bits) to ``gen.generate``, and any
row range can be produced on its own (used for row partitions).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib
from .core import CsrMatrix, device, ptr, stream_handle

__all__ = ["StencilKind", "StencilSpec", "RhsKind", "RhsSpec", "generate", "generate_rows",
           "stencil_counts", "make_rhs", "parse_stencil_spec", "parse_rhs_spec"]


class StencilKind(Enum):
    LAPLACE2D = "laplace2d"
    LAPLACE3D = "laplace3d"
    CONVDIFF2D = "convdiff2d"
    STRETCHED2D = "stretched2d"
    BIHARMONIC2D = "biharmonic2d"
    STAR2D = "star2d"
    RECIRC2D = "recirc2d"


@dataclass(frozen=True)
class StencilSpec:
    kind: StencilKind
    nx: int
    convection: float = 1.0
    stretch: float = 1.0e4

    def __post_init__(self) -> None:
        if self.nx < 2:
            raise ValueError("nx must be at least 2")

    @property
    def name(self) -> str:
        return f"{self.kind.value}:{self.nx}"


class RhsKind(Enum):
    ONES = "ones"
    FROM_FILE = "file"
    RANDOM_UNIFORM01 = "uniform"
    RANDOM_NORMAL = "normal"


@dataclass(frozen=True)
class RhsSpec:
    kind: RhsKind
    seed: int = 0
    path: str | None = None

    def __post_init__(self) -> None:
        if self.kind is RhsKind.FROM_FILE and not self.path:
            raise ValueError("file right-hand side needs a path")


def _kind(spec) -> int:
    k = spec.kind.value if hasattr(spec.kind, "value") else str(spec.kind)
    return _lib.STENCIL_KIND[k]


def stencil_counts(spec) -> tuple[int, int]:
    """(n, nnz) from closed forms, without materialising (gen.py:111-126)."""
    n, nnz = C.c_int64(), C.c_int64()
    _lib.call("mpg_stencil_counts", _kind(spec), int(spec.nx), C.byref(n), C.byref(nnz))
    return int(n.value), int(nnz.value)


def nnz_before(spec, row: int) -> int:
    return int(_lib.load().mpg_stencil_nnz_before(_kind(spec), int(spec.nx), int(row)))


def generate_rows(spec, row_begin: int, row_end: int) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Device CSR arrays of rows [row_begin, row_end): row_ptr relative to
    row_begin, global column indices, fp64 values (16-byte aligned, padded)."""
    a = nnz_before(spec, row_begin)
    b = nnz_before(spec, row_end)
    nnz = b - a
    rows = row_end - row_begin
    dev = device()
    rp = torch.zeros(rows + 1 + 8, dtype=torch.int32, device=dev)
    ci = torch.zeros(nnz + 8, dtype=torch.int32, device=dev)
    v = torch.zeros(nnz + 4, dtype=torch.float64, device=dev)
    _lib.call("mpg_generate_stencil", _kind(spec), int(spec.nx), float(spec.convection),
              float(spec.stretch), int(row_begin), int(row_end), ptr(rp), ptr(ci), ptr(v),
              stream_handle())
    return rp[: rows + 1], ci[:nnz], v[:nnz]


def generate(spec) -> CsrMatrix:
    """The stencil matrix in fp64 canonical CSR, assembled on the device."""
    n, _ = stencil_counts(spec)
    rp, ci, v = generate_rows(spec, 0, n)
    A = CsrMatrix(n, n, rp, ci, v, _trusted=True)
    kind = spec.kind.value if hasattr(spec.kind, "value") else str(spec.kind)
    if kind == "laplace3d":
        A._stencil = (3, int(spec.nx))
    elif kind in ("laplace2d", "convdiff2d", "recirc2d", "stretched2d"):
        A._stencil = (2, int(spec.nx))
    else:
        A._stencil = False
    return A


def make_rhs(spec: RhsSpec, n: int, *, on_device: bool = False):
    """fp64 right-hand side (gen.py:205-217); ``on_device`` returns a tensor."""
    kind = RhsKind(spec.kind.value if hasattr(spec.kind, "value") else spec.kind)   # reference specs too
    if kind is RhsKind.ONES:
        if on_device:
            return torch.ones(n, dtype=torch.float64, device=device())
        return np.ones(n, dtype=np.float64)
    if kind is RhsKind.RANDOM_UNIFORM01:
        v = np.random.default_rng(spec.seed).random(n)
    elif kind is RhsKind.RANDOM_NORMAL:
        v = np.random.default_rng(spec.seed).standard_normal(n)
    else:
        vals = []
        with open(spec.path) as f:
            for line in f:
                s = line.strip()
                if s and not s.startswith("%"):
                    vals.append(float(s.split()[0]))
        v = np.asarray(vals, dtype=np.float64)
        if v.shape != (n,):
            raise ValueError(f"right-hand side length {v.shape[0]} does not match n={n}")
    return torch.from_numpy(v).to(device()) if on_device else v


def parse_stencil_spec(text: str) -> StencilSpec:
    """'kind:nx[:key=value,...]' (gen.py:220-240)."""
    parts = text.strip().split(":")
    if len(parts) < 2:
        raise ValueError(f"generator spec {text!r} must look like kind:nx")
    try:
        kind = StencilKind(parts[0].lower())
    except ValueError:
        names = ", ".join(k.value for k in StencilKind)
        raise ValueError(f"unknown generator kind {parts[0]!r}; expected one of {names}")
    kwargs = {}
    if len(parts) > 2 and parts[2]:
        for item in parts[2].split(","):
            key, _, value = item.partition("=")
            if key not in ("convection", "stretch"):
                raise ValueError(f"unknown generator parameter {key!r}")
            kwargs[key] = float(value)
    return StencilSpec(kind, int(parts[1]), **kwargs)


def parse_rhs_spec(text: str, seed: int = 0) -> RhsSpec:
    text = text.strip()
    if text.startswith("file:"):
        return RhsSpec(RhsKind.FROM_FILE, seed, text[5:])
    try:
        return RhsSpec(RhsKind(text.lower()), seed)
    except ValueError:
        raise ValueError(f"unknown right-hand-side kind {text!r}; expected ones|uniform|normal|file:PATH")
