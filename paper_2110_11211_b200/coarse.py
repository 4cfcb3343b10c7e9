"""Algebraic piecewise-constant coarse space (mirrors sfcdd.coarse).

Reference: /root/reference/pkg/src/sfcdd/coarse.py:21-88.  On the device the
restriction R0 is never materialised: aggregates are q consecutive chunks of
each disjoint SFC range, so R0 v is a segmented sum and R0^T y a broadcast
(csrc/op.cu).  The Galerkin matrix A0 = R0 Â R0^T is assembled and
factorized when the Schwarz operator is set up; ``CoarseSpace.matrix`` and
``restriction`` are materialised lazily for API compatibility.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .partition import Partition


def aggregate_sizes(subdomain_size: int, q: int) -> list[int]:
    """floor(size/q)+1 for the first size mod q chunks (coarse.py:21-24)."""
    base, extra = divmod(subdomain_size, q)
    return [base + 1 if m < extra else base for m in range(q)]


def aggregate_bounds(part: Partition, q: int) -> np.ndarray:
    """Start of every aggregate in SFC order plus N (length n0 + 1)."""
    b = [0]
    for rng in part.disjoint:
        for s in aggregate_sizes(rng.length, q):
            b.append(b[-1] + s)
    return np.asarray(b, dtype=np.int64)


@dataclass
class CoarseSpace:
    """q, n0 and the lazily materialised R0 / A0 (coarse.py:27-35)."""

    q: int
    n0: int
    partition: Partition
    A: object = None
    _matrix: object = field(default=None, repr=False)

    @property
    def restriction(self):
        import scipy.sparse as sp

        bounds = aggregate_bounds(self.partition, self.q)
        n = self.partition.n
        return sp.csr_matrix((np.ones(n), np.arange(n), bounds), shape=(self.n0, n))

    @property
    def matrix(self):
        """A0 = R0 Â R0^T, symmetrized (linalg.py:83-91)."""
        if self._matrix is None:
            import scipy.sparse as sp

            R = self.restriction
            A = self.A.tocsr() if hasattr(self.A, "tocsr") else self.A
            B = sp.csr_matrix(R @ A @ R.T)
            self._matrix = sp.csr_matrix((B + B.T) * 0.5)
            self._matrix.sort_indices()
        return self._matrix


    @property
    def factorization(self):
        """Device direct solver of A0 (linalg.Factorization, coarse.py:59-60)."""
        if getattr(self, "_fact", None) is None:
            from .linalg import Factorization

            self._fact = Factorization(self.matrix)
        return self._fact


class DeflationOperators:
    """F = R0^T A0^-1 R0, G = I - A F, G^T = I - F A (coarse.py:63-84) on the
    device: R0 / R0^T as device CSR products, A0^-1 by the device direct
    solver, A by its device matvec; numpy or CUDA tensors in and out."""

    def __init__(self, cs: CoarseSpace, A):
        if A.shape[1] != cs.restriction.shape[1]:
            raise ValueError("coarse space size does not match matrix")
        from .krylov import _matvec_fn
        from .linalg import DeviceMatrix

        self._cs = cs
        R = cs.restriction
        self._R = DeviceMatrix(R)
        self._Rt = DeviceMatrix(R.T.tocsr())
        self._A = _matvec_fn(A)

    @staticmethod
    def _io(fn, v):
        from .krylov import _to_device

        is_np = isinstance(v, np.ndarray) or not hasattr(v, "data_ptr")
        out = fn(_to_device(v))
        return out.cpu().numpy() if is_np else out

    def _F(self, v):
        return self._Rt @ self._cs.factorization.solve(self._R @ v)

    def coarse_correction(self, v):
        return self._io(self._F, v)

    def project(self, v):
        return self._io(lambda x: x - self._A(self._F(x)), v)

    def project_transpose(self, v):
        return self._io(lambda x: x - self._F(self._A(x)), v)


def deflation_ops(cs: CoarseSpace, A) -> DeflationOperators:
    """coarse.py:87-88."""
    return DeflationOperators(cs, A)


def build_coarse(part: Partition, A, q: int) -> CoarseSpace:
    """Validate and describe the coarse space (coarse.py:38-60)."""
    if not 1 <= q <= part.n // part.p:
        raise ValueError(f"need 1 <= q <= floor(N/P) = {part.n // part.p}, got q={q}")
    if A.shape != (part.n, part.n):
        raise ValueError(f"matrix shape {A.shape} does not match N = {part.n}")
    return CoarseSpace(q, q * part.p, part, A)
