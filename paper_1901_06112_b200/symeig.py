"""Host FP64 symmetric eigensolver (mirror of reference ``symeig.py:21-125``).

The landmark kernel is at most NYS_MAX_M0 x NYS_MAX_M0, so it stays on the
host; the cyclic Jacobi sweeps run in native C++ (``nys_jacobi_eig``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native


@dataclass(frozen=True)
class SymMatrix:
    """Square symmetric matrix; symmetrised as (M + M^T)/2 at construction."""

    entries: np.ndarray

    def __post_init__(self) -> None:
        arr = np.asarray(self.entries, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[0] != arr.shape[1] or arr.shape[0] == 0:
            raise ValueError("SymMatrix requires a non-empty square matrix")
        if not np.all(np.isfinite(arr)):
            raise ValueError("SymMatrix entries must be finite")
        arr = np.ascontiguousarray((arr + arr.T) / 2.0)
        arr.flags.writeable = False
        object.__setattr__(self, "entries", arr)

    @property
    def order(self) -> int:
        return self.entries.shape[0]


@dataclass(frozen=True)
class EigenSystem:
    """Eigenvalues sorted descending; orthonormal eigenvectors as columns."""

    values: np.ndarray
    vectors: np.ndarray

    def __post_init__(self) -> None:
        values = np.ascontiguousarray(np.asarray(self.values, dtype=np.float64))
        vectors = np.ascontiguousarray(np.asarray(self.vectors, dtype=np.float64))
        values.flags.writeable = False
        vectors.flags.writeable = False
        object.__setattr__(self, "values", values)
        object.__setattr__(self, "vectors", vectors)


def jacobi_eig(matrix: SymMatrix) -> EigenSystem:
    """Cyclic Jacobi (symeig.py:107-125) in native code."""
    a = np.ascontiguousarray(matrix.entries, dtype=np.float64)
    k = a.shape[0]
    vals = np.empty(k)
    vecs = np.empty((k, k))
    sweeps = C.c_int(0)
    _native.call("nys_jacobi_eig", a.ctypes.data, k, vals.ctypes.data, vecs.ctypes.data, C.byref(sweeps))
    return EigenSystem(values=vals, vectors=vecs)
