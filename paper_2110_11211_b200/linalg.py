"""Direct SPD solver on the device (mirrors sfcdd.linalg).

Reference: /root/reference/pkg/src/sfcdd/linalg.py:18-91.  ``Factorization``
orders (AMD), factorizes (supernodal Cholesky, block-inverse form) on the
host once, and solves on the B200 with the same dataflow kernel as the
Schwarz local solves.  Non-SPD input raises FactorizationError like the
reference's pivot check (linalg.py:51-63).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import FactorizationError

DENSE_LIMIT = 512  # kept for API compatibility (linalg.py:18); unused on device


def as_csr(A):
    import scipy.sparse as sp

    B = sp.csr_matrix(A)
    B.sort_indices()
    return B


def matvec(A, x: np.ndarray) -> np.ndarray:
    """linalg.py:31-34."""
    if A.shape[1] != x.shape[0]:
        raise ValueError(f"dimension mismatch: {A.shape} @ {x.shape}")
    return A @ x


class Factorization:
    """Direct solver for a symmetric positive definite matrix (linalg.py:37-72)."""

    def __init__(self, A):
        n, m = A.shape
        if n != m:
            raise ValueError(f"matrix is not square: {A.shape}")
        self.n = n
        B = as_csr(A.tocsr() if hasattr(A, "tocsr") else A)
        indptr = np.ascontiguousarray(B.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(B.indices, dtype=np.int32)
        data = np.ascontiguousarray(B.data, dtype=np.float64)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().sfcdd_factor_create(n, indptr.ctypes.data, indices.ctypes.data,
                                                  data.ctypes.data, _lib.device().index, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        try:
            _lib.lib().sfcdd_factor_destroy(self._h)
        except Exception:
            pass

    def info(self) -> dict:
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().sfcdd_factor_info(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return {"nnz_l": a.value, "stored": b.value, "supernodes": c.value}

    def solve(self, b):
        import torch

        is_np = isinstance(b, np.ndarray) or not hasattr(b, "data_ptr")
        bb = np.asarray(b, dtype=np.float64) if is_np else b
        if bb.shape[0] != self.n:
            raise ValueError(f"dimension mismatch: n={self.n}, b has {bb.shape[0]}")
        dev = _lib.device()
        cols = bb.reshape(self.n, -1)
        out = []
        for j in range(cols.shape[1]):
            bt = torch.as_tensor(np.ascontiguousarray(cols[:, j]) if is_np else cols[:, j].contiguous(),
                                 dtype=torch.float64).to(dev)
            xt = torch.empty_like(bt)
            _lib.check(_lib.lib().sfcdd_factor_solve(self._h, bt.data_ptr(), xt.data_ptr(), _lib.stream_ptr()))
            out.append(xt)
        x = torch.stack(out, dim=1).reshape(bb.shape) if len(out) > 1 else out[0].reshape(bb.shape)
        return x.cpu().numpy() if is_np else x


class DeviceMatrix:
    """A general sparse matrix held on the device (C ABI ``sfcdd_csr_*``):
    the ``A @ v`` of the solvers when A is not a grid Laplacian
    (krylov.py:257-291 is duck-typed over it; test_krylov.py:154-166).
    ``@`` maps CUDA tensors to CUDA tensors and numpy to numpy; the product
    is summed in scipy's csr_matvec order, so it matches scipy bit for bit."""

    def __init__(self, A):
        B = as_csr(A.tocsr() if hasattr(A, "tocsr") else A)
        self.shape = B.shape
        self.n = B.shape[0]
        self.dtype = np.float64
        self._keep = (np.ascontiguousarray(B.indptr, np.int64), np.ascontiguousarray(B.indices, np.int32),
                      np.ascontiguousarray(B.data, np.float64))
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().sfcdd_csr_create(B.shape[0], B.shape[1], *(a.ctypes.data for a in self._keep),
                                               _lib.device().index, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        try:
            _lib.lib().sfcdd_csr_destroy(self._h)
        except Exception:
            pass

    def __matmul__(self, x):
        import torch

        is_np = isinstance(x, np.ndarray) or not hasattr(x, "data_ptr")
        xt = (torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)) if is_np else x).to(
            _lib.device(), torch.float64).contiguous()
        if xt.shape[0] != self.shape[1]:
            raise ValueError(f"dimension mismatch: {self.shape} @ {tuple(xt.shape)}")
        y = torch.empty(self.shape[0], dtype=torch.float64, device=xt.device)
        _lib.check(_lib.lib().sfcdd_csr_matvec(self._h, xt.data_ptr(), y.data_ptr(), _lib.stream_ptr()))
        return y.cpu().numpy() if is_np else y


def factorize(A) -> Factorization:
    return Factorization(A)


def solve(F: Factorization, b: np.ndarray) -> np.ndarray:
    return F.solve(b)


def triple_product(R, A):
    """Galerkin product R A R^T, symmetrized when A is symmetric (linalg.py:83-91)."""
    import scipy.sparse as sp

    if R.shape[1] != A.shape[0] or A.shape[0] != A.shape[1]:
        raise ValueError(f"dimension mismatch: R {R.shape}, A {A.shape}")
    A = A.tocsr() if hasattr(A, "tocsr") else A
    B = sp.csr_matrix(R @ A @ R.T)
    if (A != A.T).nnz == 0:
        B = sp.csr_matrix((B + B.T) * 0.5)
    B.sort_indices()
    return B
