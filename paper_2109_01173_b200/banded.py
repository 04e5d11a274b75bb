"""Band-storage matrices for the 1D FEM factors.

The reference assembles every 1D factor as a dense q x q numpy array
(fem1d.py:7-9) although all of them are banded with half-bandwidth <= k
(SURVEY App. B).  ``Band`` keeps only the diagonals: O(q k) memory and
assembly instead of O(q^2), which is what makes q = 8192 setups take
milliseconds instead of tens of seconds and ~28 GB.

A ``Band`` behaves like the dense matrix where callers expect one:
``np.asarray(band)`` (and every numpy function) sees the dense array, and
``+ - * / @ .T`` keep the banded form.  Internally it wraps a CSR matrix.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

__all__ = ["Band", "as_band", "band_arrays"]


class Band:
    """A (possibly rectangular) banded matrix."""

    __array_priority__ = 100.0

    def __init__(self, mat, shape=None):
        if isinstance(mat, Band):
            m = mat._m
        elif sp.issparse(mat):
            m = mat
        else:
            m = sp.csr_matrix(np.asarray(mat, dtype=float))
        m = sp.csr_matrix(m, dtype=float, shape=shape)
        m.eliminate_zeros()
        m.sort_indices()
        self._m = m

    # ---- construction helpers ------------------------------------------
    @classmethod
    def from_diagonals(cls, diags: dict, shape):
        """{offset: values} where values[i] sits at (i, i + offset)."""
        rows, cols, vals = [], [], []
        n, mcols = shape
        for k, v in diags.items():
            v = np.broadcast_to(np.asarray(v, dtype=float), (n,))
            i = np.arange(n)
            ok = (i + k >= 0) & (i + k < mcols)
            rows.append(i[ok])
            cols.append(i[ok] + k)
            vals.append(v[ok])
        r = np.concatenate(rows) if rows else np.zeros(0, int)
        c = np.concatenate(cols) if cols else np.zeros(0, int)
        x = np.concatenate(vals) if vals else np.zeros(0)
        return cls(sp.coo_matrix((x, (r, c)), shape=shape))

    @classmethod
    def diag(cls, values):
        values = np.asarray(values, dtype=float)
        return cls(sp.diags(values, 0, shape=(values.size, values.size), format="csr"))

    # ---- array protocol ------------------------------------------------
    @property
    def shape(self):
        return self._m.shape

    @property
    def ndim(self):
        return 2

    @property
    def dtype(self):
        return np.dtype(float)

    @property
    def sparse(self):
        return self._m

    def toarray(self) -> np.ndarray:
        return self._m.toarray()

    def __array__(self, dtype=None, copy=None):
        a = self._m.toarray()
        return a if dtype is None else a.astype(dtype)

    def __repr__(self):
        lo, hi = self.offsets()
        return f"Band(shape={self.shape}, diagonals=[{lo}, {hi}])"

    # ---- structure -----------------------------------------------------
    def offsets(self):
        """(lowest, highest) diagonal offset carrying a nonzero."""
        c = self._m.tocoo()
        if c.nnz == 0:
            return 0, 0
        k = c.col - c.row
        return int(k.min()), int(k.max())

    def half_bandwidth(self) -> int:
        lo, hi = self.offsets()
        return max(-lo, hi, 0)

    def max_abs(self) -> float:
        return float(np.max(np.abs(self._m.data))) if self._m.nnz else 0.0

    def diagonal(self, k: int = 0) -> np.ndarray:
        return self._m.diagonal(k)

    # ---- algebra (stays banded) ---------------------------------------
    @property
    def T(self):
        return Band(self._m.T)

    def _coerce(self, other):
        if isinstance(other, Band):
            return other._m
        if sp.issparse(other):
            return other
        return None

    def __add__(self, other):
        o = self._coerce(other)
        if o is None:
            return np.asarray(self) + other
        return Band(self._m + o)

    __radd__ = __add__

    def __sub__(self, other):
        o = self._coerce(other)
        if o is None:
            return np.asarray(self) - other
        return Band(self._m - o)

    def __rsub__(self, other):
        o = self._coerce(other)
        if o is None:
            return other - np.asarray(self)
        return Band(o - self._m)

    def __neg__(self):
        return Band(-self._m)

    def __mul__(self, other):
        if np.isscalar(other):
            return Band(self._m * float(other))
        o = self._coerce(other)
        if o is not None:
            return Band(self._m.multiply(o))
        other = np.asarray(other, dtype=float)
        if other.ndim == 1 or (other.ndim == 2 and 1 in other.shape):
            return Band(self._m.multiply(other))  # row/column broadcasting
        return np.asarray(self) * other

    __rmul__ = __mul__

    def __truediv__(self, other):
        if np.isscalar(other):
            return Band(self._m / float(other))
        other = np.asarray(other, dtype=float)
        if other.ndim == 2 and other.shape[1] == 1:  # row scaling  M / d[:, None]
            return Band(sp.diags(1.0 / other[:, 0]) @ self._m)
        if other.ndim == 1 or (other.ndim == 2 and other.shape[0] == 1):  # column scaling
            return Band(self._m @ sp.diags(1.0 / other.reshape(-1)))
        return np.asarray(self) / other

    def __matmul__(self, other):
        o = self._coerce(other)
        if o is None:
            return np.asarray(self) @ np.asarray(other)
        return Band(self._m @ o)

    def __rmatmul__(self, other):
        o = self._coerce(other)
        if o is None:
            return np.asarray(other) @ np.asarray(self)
        return Band(o @ self._m)

    def scale_rows(self, v):
        return Band(sp.diags(np.asarray(v, dtype=float)) @ self._m)

    def scale_cols(self, v):
        return Band(self._m @ sp.diags(np.asarray(v, dtype=float)))

    # ---- band arrays for the device ------------------------------------
    def band_rows(self, width: int, off: int) -> np.ndarray:
        """data[i, d] = M[i, i + off + d] (zero outside the matrix)."""
        c = self._m.tocoo()
        d = c.col - c.row - off
        if c.nnz and (d.min() < 0 or d.max() >= width):
            raise ValueError("band window too narrow for this matrix")
        out = np.zeros((self.shape[0], width))
        out[c.row, d] = c.data
        return out


def as_band(m) -> Band:
    return m if isinstance(m, Band) else Band(m)


def band_arrays(mats, by_rows: bool, width: int, off: int) -> np.ndarray:
    """Stack factors into [n][rows][width].

    by_rows=True  : left factors G, rows of G (gband[i][d] = G[i][i+off+d]).
    by_rows=False : right factors H acting as U H, stored by columns
                    (hband[j][e] = H[j+off+e][j]) == rows of H^T.
    """
    out = []
    for m in mats:
        b = as_band(m)
        out.append(b.band_rows(width, off) if by_rows else b.T.band_rows(width, off))
    return np.ascontiguousarray(np.stack(out))
