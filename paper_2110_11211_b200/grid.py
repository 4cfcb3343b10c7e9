"""Grids, SFC ordering and the matrix-free Laplacian (mirrors sfcdd.grid).

Reference: /root/reference/pkg/src/sfcdd/grid.py.  ``sfc_permutation`` runs
the device key + rank kernels (csrc/sfc.cu); ``assemble_laplacian`` returns
a matrix-free operator whose ``@`` is the sm_100a stencil kernel -- no
sparse matrix is materialised on the hot path.  ``tocsr()`` exists for small
diagnostics and needs scipy.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache
from typing import Callable

import numpy as np

from . import _lib

MAX_DOFS = 2**62


@dataclass(frozen=True)
class Problem:
    """Right-hand side and optional exact solution on a grid (grid.py:26-36):
    vectorized callables mapping (m, d) points of the open unit cube to (m,)."""

    levels: tuple[int, ...]
    rhs: Callable[[np.ndarray], np.ndarray]
    exact_solution: Callable[[np.ndarray], np.ndarray] | None = None


def as_levels(levels) -> tuple[int, ...]:
    ell = tuple(int(v) for v in levels)
    if not ell or any(l < 1 for l in ell):
        raise ValueError(f"level vector must have positive entries, got {levels}")
    return ell


def interior_shape(levels) -> tuple[int, ...]:
    """grid.py:46-47."""
    return tuple((1 << l) - 1 for l in as_levels(levels))


def num_dofs(levels) -> int:
    """prod_j (2**l_j - 1) with the reference's overflow guard (grid.py:50-57)."""
    n = 1
    for l in as_levels(levels):
        n *= (1 << l) - 1
        if n > MAX_DOFS:
            raise OverflowError(f"dof count for levels {levels} exceeds {MAX_DOFS}")
    return n


def sfc_permutation_device(levels, force_radix: bool = False, curve: str = "hilbert"):
    """perm (SFC rank -> lex index) and its inverse as int64 device tensors
    (``curve="lebesgue"``: Morton order, see sfc.py)."""
    import torch

    levels = as_levels(levels)
    n = num_dofs(levels)
    dev = _lib.device()
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    rank = torch.empty(n, dtype=torch.int64, device=dev)
    lv = (ctypes.c_int32 * len(levels))(*levels)
    if curve not in _lib.CURVES:
        raise ValueError(f"unknown curve {curve!r}")
    _lib.check(_lib.lib().sfcdd_sfc_perm_curve(_lib.CURVES[curve], len(levels), ctypes.cast(lv, ctypes.c_void_p),
                                               perm.data_ptr(), rank.data_ptr(), int(force_radix),
                                               _lib.stream_ptr()))
    return perm, rank


@lru_cache(maxsize=128)
def sfc_permutation(levels: tuple[int, ...], curve: str = "hilbert") -> np.ndarray:
    """``perm[s]`` = lex index of the point with the s-th smallest key (grid.py:60-77)."""
    perm, _ = sfc_permutation_device(as_levels(levels), curve=curve)
    out = perm.cpu().numpy()
    out.setflags(write=False)
    return out


def interior_points(levels, curve: str = "hilbert") -> np.ndarray:
    """Coordinates of the interior points in SFC order, shape (N, d) (grid.py:80-88)."""
    levels = as_levels(levels)
    shape = interior_shape(levels)
    axes = [np.arange(1, s + 1, dtype=np.float64) * 2.0**-l for s, l in zip(shape, levels)]
    mesh = np.meshgrid(*axes, indexing="ij")
    pts = np.stack([m.ravel() for m in mesh], axis=1)
    return pts[sfc_permutation(levels, curve)]


def scatter_to_lex(levels, values_sfc: np.ndarray, curve: str = "hilbert") -> np.ndarray:
    """Reshape an SFC-ordered vector to the lexicographic d-dim array (grid.py:169-175)."""
    levels = as_levels(levels)
    shape = interior_shape(levels)
    out = np.empty(int(np.prod(shape)), dtype=np.float64)
    out[sfc_permutation(levels, curve)] = values_sfc
    return out.reshape(shape)


class _GridHandle:
    """Device neighbour table + stencil constants for one level vector."""

    def __init__(self, levels, curve: str = "hilbert", raw: bool = False):
        from .partition import disjoint_partition

        self.levels = levels
        self.curve = curve
        self.n = num_dofs(levels)
        if len(levels) > 8:
            raise ValueError("device grids support up to 8 dimensions")
        rng = disjoint_partition(self.n, 1)
        st = np.array([r.start for r in rng], np.int64)
        ln = np.array([r.length for r in rng], np.int64)
        om = np.ones(1)
        desc = _lib.OpDesc()
        desc.dim = len(levels)
        for j, l in enumerate(levels):
            desc.levels[j] = l
        desc.p, desc.q = 1, 0
        desc.variant, desc.weighting = _lib.VARIANT_CODES["one_level"], 0
        desc.device = _lib.device().index
        desc.ov_start = desc.dj_start = st.ctypes.data
        desc.ov_len = desc.dj_len = ln.ctypes.data
        desc.omega = om.ctypes.data
        desc.host_threads = 1
        desc.curve = _lib.CURVES[curve]
        desc.raw_laplacian = 1 if raw else 0
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().sfcdd_op_create(ctypes.byref(desc), ctypes.byref(h)))
        self.handle = h
        diag = ctypes.c_double()
        off = (ctypes.c_double * 8)()
        t = ctypes.c_double()
        _lib.check(_lib.lib().sfcdd_op_stencil(h, ctypes.byref(diag), off, ctypes.byref(t)))
        self.dhat = diag.value
        self.off = [off[j] for j in range(len(levels))]
        self.t = t.value

    def __del__(self):
        try:
            _lib.lib().sfcdd_op_destroy(self.handle)
        except Exception:
            pass

    def matvec(self, x):
        import torch

        dev = _lib.device()
        xt = torch.as_tensor(x, dtype=torch.float64).to(dev).contiguous()
        y = torch.empty_like(xt)
        _lib.check(_lib.lib().sfcdd_op_matvec(self.handle, xt.data_ptr(), y.data_ptr(), _lib.stream_ptr()))
        return y


@lru_cache(maxsize=16)
def _grid_handle(levels, curve: str = "hilbert", raw: bool = False) -> _GridHandle:
    return _GridHandle(levels, curve, raw)


class GridLaplacian:
    """Matrix-free (2d+1)-point -Laplace in SFC order (grid.py:91-114).

    ``scaled=True`` is Â = T A T with T = diag(A)^-1/2 (grid.py:117-130);
    its entries are exactly fl(fl(t a) t) as in the reference.  ``@`` accepts
    numpy arrays (returns numpy) or CUDA tensors (returns a CUDA tensor).
    """

    def __init__(self, levels, scaled: bool = False, curve: str = "hilbert"):
        if curve not in _lib.CURVES:
            raise ValueError(f"unknown curve {curve!r}")
        self.levels = as_levels(levels)
        self.curve = curve
        self.n = num_dofs(self.levels)
        self.shape = (self.n, self.n)
        self.dtype = np.float64
        self.scaled = scaled
        self.ndim = 2
        diag = 0.0
        for l in self.levels:
            diag = diag + 2.0 * float(4**l)
        self._diag_raw = diag
        self._t = 1.0 / np.sqrt(diag)

    @property
    def handle(self) -> _GridHandle:
        """Device stencil of this matrix: Â's constants, or A's exact integer
        entries 2 sum 4^l / -4^l_j when unscaled (grid.py:101-110)."""
        return _grid_handle(self.levels, self.curve, not self.scaled)

    @property
    def scale(self) -> float:
        return float(self._t)

    def diagonal(self) -> np.ndarray:
        return np.full(self.n, self.handle.dhat)

    def __matmul__(self, x):
        import torch

        is_np = isinstance(x, np.ndarray)
        x_arr = np.asarray(x, dtype=np.float64) if is_np else x
        if x_arr.shape[0] != self.n:
            raise ValueError(f"dimension mismatch: {self.shape} @ {tuple(x_arr.shape)}")
        y = self.handle.matvec(x_arr)
        return y.cpu().numpy() if is_np else y

    def tocsr(self):
        """scipy CSR copy (diagnostics / small grids only)."""
        import scipy.sparse as sp

        perm = sfc_permutation(self.levels, self.curve)
        n = self.n
        rank = np.empty(n, np.int64)
        rank[perm] = np.arange(n)
        shape = interior_shape(self.levels)
        coords = np.stack(np.unravel_index(perm, shape), axis=1)  # by SFC rank
        strides = [int(np.prod(shape[j + 1:])) for j in range(len(shape))]
        h = self.handle
        rows, cols, vals = [np.arange(n)], [np.arange(n)], [np.full(n, h.dhat)]
        for j in range(len(shape)):
            oval = h.off[j]
            for step in (-1, 1):
                ok = (coords[:, j] + step >= 0) & (coords[:, j] + step < shape[j])
                s = np.nonzero(ok)[0]
                rows.append(s)
                cols.append(rank[perm[s] + step * strides[j]])
                vals.append(np.full(s.size, oval))
        A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
        A.sort_indices()
        return A

    def toarray(self) -> np.ndarray:
        return self.tocsr().toarray()

    # scipy-matrix behaviour for diagnostics (A.T, A[idx][:, idx], A - B,
    # A != A.T ...): delegated to the materialised CSR copy, as the reference
    # returns a CSR matrix from assemble_laplacian (grid.py:91-114)
    def _csr(self):
        c = getattr(self, "_csr_cache", None)
        if c is None:
            c = self.tocsr()
            self._csr_cache = c
        return c

    def __getattr__(self, name):
        # never materialise implicitly for attribute probes on large grids
        if name.startswith("_") or self.__dict__.get("n", 0) > (1 << 22):
            raise AttributeError(name)
        return getattr(self._csr(), name)

    def __getitem__(self, key):
        return self._csr()[key]

    def __sub__(self, other):
        return self._csr() - (other._csr() if isinstance(other, GridLaplacian) else other)

    def __add__(self, other):
        return self._csr() + (other._csr() if isinstance(other, GridLaplacian) else other)

    def __ne__(self, other):
        return self._csr() != (other._csr() if isinstance(other, GridLaplacian) else other)

    def __rmatmul__(self, other):
        return other @ self._csr()


def assemble_laplacian(levels, curve: str = "hilbert") -> GridLaplacian:
    """(2d+1)-point FD matrix of -Laplace in SFC order (grid.py:91-114), matrix-free.
    ``curve="lebesgue"`` orders the unknowns along the Morton curve instead."""
    levels = as_levels(levels)
    num_dofs(levels)
    return GridLaplacian(levels, scaled=False, curve=curve)


def symmetrize_diag(A, b):
    """(Â, b̂, t) with Â = T A T, b̂ = t b, T = diag(A)^-1/2 (grid.py:117-130)."""
    if isinstance(A, GridLaplacian):
        if A.scaled:
            raise ValueError("matrix is already scaled")
        t = np.full(A.n, A.scale)
        return GridLaplacian(A.levels, scaled=True, curve=A.curve), t * np.asarray(b, dtype=np.float64), t
    # generic sparse input: boundary glue with the reference's formula
    import scipy.sparse as sp

    d = np.asarray(A.diagonal())
    if np.any(d <= 0.0):
        raise ValueError("matrix has a nonpositive diagonal entry")
    t = 1.0 / np.sqrt(d)
    T = sp.diags(t)
    A_hat = sp.csr_matrix(T @ A @ T)
    A_hat.sort_indices()
    return A_hat, t * np.asarray(b, dtype=np.float64), t


def manufactured_poisson(levels) -> Problem:
    """Poisson problem with solution u = |x|_2 prod_i sin(pi x_i) (grid.py:133-161).

    u vanishes on the cube boundary (homogeneous Dirichlet data).  With
    g = prod_i sin(pi x_i), r = |x|_2, c_i = cos(pi x_i) and G_i the product
    of the sines without factor i:
        -Lap u = -( g (d - 1) / r + 2 pi sum_i (x_i / r) c_i G_i - d pi^2 u ).
    Host numpy (setup data, not the solver's hot path)."""
    levels = as_levels(levels)
    d = len(levels)

    def exact(points: np.ndarray) -> np.ndarray:
        x = np.atleast_2d(np.asarray(points, dtype=np.float64))
        return np.linalg.norm(x, axis=1) * np.prod(np.sin(np.pi * x), axis=1)

    def rhs(points: np.ndarray) -> np.ndarray:
        x = np.atleast_2d(np.asarray(points, dtype=np.float64))
        sn = np.sin(np.pi * x)
        cs = np.cos(np.pi * x)
        g = np.prod(sn, axis=1)
        r = np.linalg.norm(x, axis=1)
        u = r * g
        mixed = np.zeros_like(r)
        for i in range(d):
            rest = np.prod(np.delete(sn, i, axis=1), axis=1)
            mixed += x[:, i] / r * cs[:, i] * rest
        return -(g * (d - 1) / r + 2.0 * np.pi * mixed - d * np.pi**2 * u)

    return Problem(levels, rhs, exact)


def sample_on_grid(func, levels, curve: str = "hilbert") -> np.ndarray:
    """Values of a vectorized callable at the interior points, SFC order (grid.py:164-166)."""
    return np.asarray(func(interior_points(levels, curve)), dtype=np.float64)
