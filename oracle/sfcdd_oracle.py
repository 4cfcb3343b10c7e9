"""CPU oracle for the SFC two-level Schwarz PCG path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference algorithm
(package ``sfcdd`` of arXiv 2110.11211, mounted read-only at
/root/reference) for the hot path named in BASELINE.json:north_star:

    Hilbert keys + sort -> cyclic gamma-overlap ranges -> balanced,
    omega-weighted two-level Schwarz -> PCG on the scaled 2d+1 Laplacian.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU arms may
import it, and only as the checker / the timed CPU baseline.  The product
package (``paper_2110_11211_b200``) never imports this file.

Parity is PINNED (Hilbert path; the Lebesgue option ``lebesgue_keys`` has no
reference code and is unpinned): ``oracle/make_fixtures.py`` runs the reference itself in
the build container and commits its outputs under ``tests/golden/``;
``tests/test_oracle_golden.py`` checks every function below against them.

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/sfcdd/).  The code is vectorised numpy (keys for all
points at once) rather than the reference's per-point Python loops, and the
local/coarse direct solves use scipy's SuperLU exactly as the reference's
third-party call sites do (linalg.py:57-61, scipy >= 1.10, here 1.18.1).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import scipy.linalg as sla

MAX_KEY_BITS = 128
DENSE_LIMIT = 512  # linalg.py:18


# ---------------------------------------------------------------- Hilbert keys
def hilbert_keys(coords: np.ndarray, bits: int) -> tuple[np.ndarray, np.ndarray]:
    """Skilling transpose-form Hilbert keys for an (n, d) coordinate array.

    Restates sfc.py:56-79 (_axes_to_transpose) and sfc.py:102-107
    (_pack_transpose); d == 1 is the identity (sfc.py:133-134).  Returns the
    key as two uint64 words (hi, lo) so keys up to 128 bits (sfc.py:21) are
    exact.
    """
    coords = np.asarray(coords, dtype=np.uint64)
    n, d = coords.shape
    if d * bits > MAX_KEY_BITS:
        raise ValueError("key width exceeds 128 bits")
    x = [coords[:, i].copy() for i in range(d)]
    if d == 1:
        return np.zeros(n, np.uint64), x[0]
    one = np.uint64(1)
    m = 1 << (bits - 1)
    q = m
    while q > 1:                                   # sfc.py:61-70
        p = np.uint64(q - 1)
        qq = np.uint64(q)
        for i in range(d):
            hit = (x[i] & qq) != 0
            if i == 0:
                x[0] = np.where(hit, x[0] ^ p, x[0])
                continue
            t = (x[0] ^ x[i]) & p
            x0 = np.where(hit, x[0] ^ p, x[0] ^ t)
            xi = np.where(hit, x[i], x[i] ^ t)
            x[0], x[i] = x0, xi
        q >>= 1
    for i in range(1, d):                          # sfc.py:71-72 (Gray encode)
        x[i] = x[i] ^ x[i - 1]
    t = np.zeros(n, np.uint64)
    q = m
    while q > 1:                                   # sfc.py:73-77
        t = np.where((x[d - 1] & np.uint64(q)) != 0, t ^ np.uint64(q - 1), t)
        q >>= 1
    for i in range(d):
        x[i] = x[i] ^ t
    return _interleave(x, bits)


def _interleave(x, bits: int) -> tuple[np.ndarray, np.ndarray]:
    """sfc.py:102-107 (_pack_transpose): MSB-first, axis 0 first."""
    d = len(x)
    n = x[0].shape[0]
    one = np.uint64(1)
    hi = np.zeros(n, np.uint64)
    lo = np.zeros(n, np.uint64)
    for level in range(bits):
        for i in range(d):
            pos = level * d + (d - 1 - i)
            bit = (x[i] >> np.uint64(level)) & one
            if pos < 64:
                lo |= bit << np.uint64(pos)
            else:
                hi |= bit << np.uint64(pos - 64)
    return hi, lo


def lebesgue_keys(coords: np.ndarray, bits: int) -> tuple[np.ndarray, np.ndarray]:
    """Lebesgue (Morton, Z-order) keys: the reference's bit interleaving
    (sfc.py:102-107) of the RAW coordinates, without the Hilbert transform.

    PARITY UNPINNED: the reference has no Lebesgue curve (north star
    subsystem (1) names it), so this restatement is the
    definition the device keys are checked against.
    """
    coords = np.asarray(coords, dtype=np.uint64)
    n, d = coords.shape
    if d * bits > MAX_KEY_BITS:
        raise ValueError("key width exceeds 128 bits")
    if d == 1:
        return np.zeros(n, np.uint64), coords[:, 0].copy()
    return _interleave([coords[:, i].copy() for i in range(d)], bits)


def encode(coords, dim: int, bits: int) -> int:
    """Scalar convenience wrapper (sfc.py:120-136), returns a Python int."""
    c = np.asarray([list(coords)], dtype=np.uint64)
    if c.shape[1] != dim:
        raise ValueError("coordinate count mismatch")
    if np.any(c >= (1 << bits)):
        raise ValueError("coordinate outside lattice")
    hi, lo = hilbert_keys(c, bits)
    return (int(hi[0]) << 64) | int(lo[0])


# ----------------------------------------------------------------- grid / perm
def interior_shape(levels) -> tuple[int, ...]:
    """grid.py:46-47: 2**l - 1 interior points per axis."""
    return tuple((1 << int(l)) - 1 for l in levels)


def lex_coords(levels) -> np.ndarray:
    """All interior multi-indices (0-based) in C order (grid.py:72-75)."""
    shape = interior_shape(levels)
    grids = np.meshgrid(*[np.arange(s, dtype=np.int64) for s in shape], indexing="ij")
    return np.stack([g.ravel() for g in grids], axis=1)


def grid_keys(levels, curve: str = "hilbert") -> tuple[np.ndarray, np.ndarray]:
    """grid_point_key for every interior point (sfc.py:150-169).

    1-based index k on axis j embeds as (k-1) << (lmax - l_j); with the
    0-based C-order index i = k-1 that is i << (lmax - l_j).
    """
    levels = tuple(int(l) for l in levels)
    lmax = max(levels)
    c = lex_coords(levels).astype(np.uint64)
    for j, l in enumerate(levels):
        c[:, j] <<= np.uint64(lmax - l)
    return lebesgue_keys(c, lmax) if curve == "lebesgue" else hilbert_keys(c, lmax)


def sfc_permutation(levels, curve: str = "hilbert") -> np.ndarray:
    """perm[s] = lex index of the point with the s-th smallest key (grid.py:60-77)."""
    levels = tuple(int(l) for l in levels)
    n = int(np.prod(interior_shape(levels)))
    if len(levels) == 1:
        return np.arange(n, dtype=np.int64)
    hi, lo = grid_keys(levels, curve)
    return np.lexsort((lo, hi)).astype(np.int64)   # keys are unique


def stencil_constants(levels):
    """Scaled-operator constants of T A T (grid.py:91-130).

    A has diagonal sum_j 2*4**l_j (kron sum, grid.py:101-110) and
    off-diagonal -4**l_j; T = diag(A)**-1/2 is constant because every point
    has the same diagonal.  Scaled entries are fl(fl(t*a)*t) as produced by
    (T @ A) @ T (grid.py:127-128).  Returns (diag_hat, [off_hat_j], t).
    """
    levels = tuple(int(l) for l in levels)
    diag = 0.0
    for l in levels:
        diag = diag + 2.0 * float(4 ** l)
    t = 1.0 / np.sqrt(diag)
    dhat = (t * diag) * t
    offs = [(t * (-float(4 ** l))) * t for l in levels]
    return float(dhat), [float(o) for o in offs], float(t)


def assemble_scaled_laplacian(levels, curve: str = "hilbert") -> sp.csr_matrix:
    """Â = T A T in SFC order, assembled from the neighbour relation.

    Restates grid.py:91-130 (assemble_laplacian + symmetrize_diag) directly
    from the stencil constants instead of kron products.
    """
    levels = tuple(int(l) for l in levels)
    shape = interior_shape(levels)
    d = len(levels)
    n = int(np.prod(shape))
    perm = sfc_permutation(levels, curve)
    rank = np.empty(n, np.int64)
    rank[perm] = np.arange(n)
    dhat, offs, _ = stencil_constants(levels)
    coords = lex_coords(levels)
    strides = [int(np.prod(shape[j + 1:])) for j in range(d)]
    rows = [np.arange(n)]
    cols = [np.arange(n)]
    vals = [np.full(n, dhat)]
    for j in range(d):
        for step in (-1, 1):
            ok = (coords[:, j] + step >= 0) & (coords[:, j] + step < shape[j])
            lex = np.nonzero(ok)[0]
            rows.append(rank[lex])
            cols.append(rank[lex + step * strides[j]])
            vals.append(np.full(lex.size, offs[j]))
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n))
    A.sort_indices()
    return A


# ------------------------------------------------------------------ partition
@dataclass(frozen=True)
class Range:
    start: int
    length: int
    modulus: int

    def indices(self) -> np.ndarray:                 # partition.py:38-43
        idx = np.arange(self.start, self.start + self.length, dtype=np.int64)
        return idx % self.modulus


def disjoint_partition(n: int, p: int) -> list[Range]:
    """partition.py:64-75: first N mod P ranges get one extra index."""
    if not 1 <= p <= n:
        raise ValueError("need 1 <= P <= N")
    base, extra = divmod(n, p)
    out, start = [], 0
    for i in range(p):
        size = base + (1 if i < extra else 0)
        out.append(Range(start, size, n))
        start += size
    return out


def enlarge(disjoint: list[Range], gamma) -> list[Range]:
    """partition.py:78-116: floor(gamma) whole neighbours, ceil/floor slices."""
    p = len(disjoint)
    n = disjoint[0].modulus
    g = Fraction(gamma).limit_denominator(10 ** 6)
    if g < 0:
        raise ValueError("gamma must be nonnegative")
    if g == 0:
        return list(disjoint)
    if p < 2:
        raise ValueError("overlap requires at least two subdomains")
    if 2 * g + 1 > p:
        raise ValueError("2*gamma+1 exceeds P")
    whole = math.floor(g)
    eta = g - whole
    sizes = [r.length for r in disjoint]
    out = []
    for i in range(p):
        left = sum(sizes[(i - k) % p] for k in range(1, whole + 1))
        right = sum(sizes[(i + k) % p] for k in range(1, whole + 1))
        if eta > 0:
            left += math.ceil(eta * sizes[(i - whole - 1) % p])
            right += math.floor(eta * sizes[(i + whole + 1) % p])
        out.append(Range((disjoint[i].start - left) % n, sizes[i] + left + right, n))
    return out


def weights(overlapped: list[Range], n: int):
    """partition.py:151-157: counts, D_i = 1/counts[idx_i], omega_i = max D_i."""
    counts = np.zeros(n, np.int64)
    for r in overlapped:
        np.add.at(counts, r.indices(), 1)
    diags = [1.0 / counts[r.indices()] for r in overlapped]
    omega = np.array([dd.max() for dd in diags])
    return counts, diags, omega


def aggregate_sizes(size: int, q: int) -> list[int]:
    """coarse.py:21-24."""
    base, extra = divmod(size, q)
    return [base + (1 if m < extra else 0) for m in range(q)]


def coarse_restriction(disjoint: list[Range], n: int, q: int) -> sp.csr_matrix:
    """coarse.py:44-58: one 0/1 row per chunk of each disjoint range."""
    if not 1 <= q <= n // len(disjoint):
        raise ValueError("need 1 <= q <= floor(N/P)")
    indptr = [0]
    for r in disjoint:
        for s in aggregate_sizes(r.length, q):
            indptr.append(indptr[-1] + s)
    indptr = np.asarray(indptr, np.int64)
    return sp.csr_matrix((np.ones(n), np.arange(n), indptr), shape=(len(indptr) - 1, n))


def galerkin(R0, A) -> sp.csr_matrix:
    """linalg.py:83-91: R A R^T symmetrised as (B + B^T)/2 for symmetric A."""
    B = sp.csr_matrix(R0 @ A @ R0.T)
    B = sp.csr_matrix((B + B.T) * 0.5)
    B.sort_indices()
    return B


class DirectSolver:
    """linalg.py:37-72: dense Cholesky for n <= 512 else SuperLU MMD(A^T+A)."""

    def __init__(self, A):
        n = A.shape[0]
        self.n = n
        if n <= DENSE_LIMIT:
            self._cho = sla.cho_factor(A.toarray(), lower=True, check_finite=False)
            self._lu = None
        else:
            self._lu = spla.splu(sp.csc_matrix(A), permc_spec="MMD_AT_PLUS_A",
                                 options={"SymmetricMode": True})
            self._cho = None

    def solve(self, b):
        if self._cho is not None:
            return sla.cho_solve(self._cho, b, check_finite=False)
        return self._lu.solve(b)


# ---------------------------------------------------------------- Schwarz/PCG
class BalancedSchwarz:
    """schwarz.py:48-118, balanced variant with omega weighting only.

    apply(g) = w - F(Â w) + F g with w = sum_i R_i^T omega_i A_i^{-1} R_i
    (g - Â F g) and F = R0^T A0^{-1} R0 (coarse.py:76-78).  ``fault`` is the
    SURVEY §8(d) config-4 semantics: in apply call number ``fault[0]`` the
    local pieces of subdomains ``fault[1]`` are zeroed.
    """

    def __init__(self, A, n: int, p: int, gamma, q: int, fault=None):
        self.A = A
        self.n = n
        self.disjoint = disjoint_partition(n, p)
        self.overlapped = enlarge(self.disjoint, gamma)
        self.counts, self.diagonals, self.omega = weights(self.overlapped, n)
        self.idx = [r.indices() for r in self.overlapped]
        self.local = [DirectSolver(A[i][:, i].tocsr()) for i in self.idx]
        self.R0 = coarse_restriction(self.disjoint, n, q)
        self.A0 = galerkin(self.R0, A)
        self.coarse = DirectSolver(self.A0)
        self.fault = fault
        self.calls = 0
        self.symmetric = True

    def F(self, v):
        return self.R0.T @ self.coarse.solve(self.R0 @ v)

    def one_level(self, g):
        out = np.zeros_like(g)
        dead = set()
        if self.fault is not None and self.calls == self.fault[0]:
            dead = set(int(i) for i in self.fault[1])
        for i, (ix, solver) in enumerate(zip(self.idx, self.local)):
            piece = self.omega[i] * solver.solve(g[ix])
            if i in dead:
                piece = np.zeros_like(piece)
            out[ix] += piece
        return out

    def apply(self, g):
        fg = self.F(g)
        w = self.one_level(g - self.A @ fg)
        self.calls += 1
        return w - self.F(self.A @ w) + fg


@dataclass
class PcgResult:
    iterations: int
    converged: bool
    residual_history: list
    solution: np.ndarray


def pcg(A, b, precond, tol=1e-8, max_iters=20000, x0=None, max_steps=None):
    """krylov.py:257-291 with relative-residual stopping (krylov.py:186-200).

    ``max_steps`` bounds the number of CG steps regardless of convergence
    (used for bounded CPU-baseline samples).
    """
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
    r = b - A @ x
    hist = [float(np.linalg.norm(r))]
    base = hist[0]
    if hist[0] <= tol * base:
        return PcgResult(0, True, hist, x)
    z = precond.apply(r) if precond is not None else r.copy()
    p = z.copy()
    rz = float(r @ z)
    it = 0
    conv = False
    for k in range(1, max_iters + 1):
        Ap = A @ p
        pAp = float(p @ Ap)
        if pAp <= 0.0:
            raise RuntimeError(f"nonpositive curvature at iteration {k}")
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        it = k
        hist.append(float(np.linalg.norm(r)))
        if hist[-1] <= tol * base:
            conv = True
            break
        if max_steps is not None and k >= max_steps:
            break
        z = precond.apply(r) if precond is not None else r.copy()
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return PcgResult(it, conv, hist, x)


def seeded_rhs(n: int, seed: int = 42) -> np.ndarray:
    """b = default_rng(seed).uniform(-1, 1, N), indexed by SFC rank."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=n)


def fault_set(p: int, seed: int = 42, frac: float = 0.1) -> np.ndarray:
    """SURVEY §8(d) config-4 fault set: rng.choice(P, round(0.1 P), replace=False)."""
    return np.random.default_rng(seed).choice(p, size=int(round(frac * p)), replace=False)


def solve_config(levels, p, gamma, q, seed=42, tol=1e-8, fault_iter=None, max_steps=None, curve="hilbert"):
    """Full oracle pipeline of SURVEY §8(d): assemble, scale, set up, PCG from 0."""
    A = assemble_scaled_laplacian(levels, curve)
    n = A.shape[0]
    _, _, t = stencil_constants(levels)
    b = t * seeded_rhs(n, seed)               # b_hat = t * b (grid.py:130)
    fault = None
    if fault_iter is not None:
        fault = (fault_iter, fault_set(p, seed))
    op = BalancedSchwarz(A, n, p, gamma, q, fault=fault)
    res = pcg(A, b, op, tol=tol, max_steps=max_steps)
    return A, b, op, res


# ------------------------------------------- other outer solvers
class Tracker:
    """krylov.py:171-213: residual (and, with an exact solution, energy-error)
    histories and the stopping test metric <= tol * metric_0."""

    def __init__(self, A, b, tol, kind, exact):
        if kind == "energy_error_reduction" and exact is None:
            raise ValueError("energy stopping needs the exact solution")
        self.A, self.b, self.tol, self.kind, self.exact = A, b, tol, kind, exact
        self.a_exact = A @ exact if exact is not None else None
        self.energy, self.residual = [], []
        self.base = None

    def record(self, x, r) -> bool:
        self.residual.append(float(np.linalg.norm(r)))
        if self.exact is not None:                       # krylov.py:189-193
            e = x - self.exact
            self.energy.append(float(np.sqrt(max(e @ (self.b - r - self.a_exact), 0.0))))
        metric = self.energy[-1] if self.kind == "energy_error_reduction" else self.residual[-1]
        if self.base is None:
            self.base = metric
        return metric <= self.tol * self.base

    def diverged(self) -> bool:                           # krylov.py:205-213
        if self.base is None or self.base == 0.0:
            return False
        hist = self.energy if self.kind == "energy_error_reduction" else self.residual
        return hist[-1] > 10.0 * self.base


@dataclass
class SolverResult:
    iterations: int
    converged: bool
    residual_history: list
    energy_history: list
    solution: np.ndarray
    lambda_min: float | None = None
    lambda_max: float | None = None
    damping: float | None = None


def pcg_tracked(A, b, precond, tol=1e-8, kind="relative_residual", exact=None, max_iters=20000):
    """krylov.py:257-291 with the full tracker (energy errors when exact is given)."""
    tr = Tracker(A, b, tol, kind, exact)
    x = np.zeros_like(b)
    r = b - A @ x
    if tr.record(x, r):
        return SolverResult(0, True, tr.residual, tr.energy, x)
    z = precond.apply(r)
    p = z.copy()
    rz = float(r @ z)
    it, conv = 0, False
    for k in range(1, max_iters + 1):
        Ap = A @ p
        pAp = float(p @ Ap)
        if pAp <= 0.0:
            raise RuntimeError(f"nonpositive curvature at iteration {k}")
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        it = k
        if tr.record(x, r):
            conv = True
            break
        z = precond.apply(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return SolverResult(it, conv, tr.residual, tr.energy, x)


def estimate_extremal_eigs(apply_ca, n, iters=None, seed=0, a_matvec=None, force_iterative=False,
                           stagnation_tol=2e-5, min_iters=40):
    """krylov.py:102-168: dense eigenvalues for n <= 300, else Lanczos in the
    a_matvec inner product with full (CGS2) reorthogonalization and
    stagnation stopping."""
    if n <= 300 and not force_iterative:
        M = np.empty((n, n))
        e = np.zeros(n)
        for j in range(n):
            e[j] = 1.0
            M[:, j] = apply_ca(e)
            e[j] = 0.0
        lam = np.real(sla.eigvals(M))
        return float(lam.min()), float(lam.max())
    if iters is None:
        iters = min(200, n)
    rng = np.random.default_rng((seed, 0xE16))
    mv = a_matvec if a_matvec is not None else (lambda v: v)
    q = rng.standard_normal(n)
    q /= np.sqrt(float(q @ mv(q)))
    basis, alphas, betas = [q], [], []
    prev, stable, lo, hi = None, 0, None, None
    for k in range(iters):
        w = apply_ca(basis[k])
        alpha = float(mv(w) @ basis[k])
        alphas.append(alpha)
        w = w - alpha * basis[k]
        if k > 0:
            w = w - betas[k - 1] * basis[k - 1]
        for _ in range(2):
            aw = mv(w)
            coeffs = [float(aw @ qj) for qj in basis]
            for c, qj in zip(coeffs, basis):
                w = w - c * qj
        lam = sla.eigvalsh_tridiagonal(alphas, betas)
        lo, hi = float(lam[0]), float(lam[-1])
        if prev is not None:
            d = max(abs(lo - prev[0]) / max(abs(lo), 1e-30), abs(hi - prev[1]) / max(abs(hi), 1e-30))
            stable = stable + 1 if d < stagnation_tol else 0
        prev = (lo, hi)
        if k + 1 >= min_iters and stable >= 5:
            break
        beta = np.sqrt(max(float(w @ mv(w)), 0.0))
        if beta <= 1e-14 * max(abs(alpha), 1.0):
            break
        betas.append(beta)
        basis.append(w / beta)
    return lo, hi


def richardson(A, b, precond, tol=1e-6, kind="relative_residual", exact=None, damping="optimal", seed=42,
               eig_iters=None, max_iters=20000):
    """krylov.py:219-254: x += xi C^-1 (b - A x); xi = 2/(lmin+lmax) for 'optimal'."""
    lam = (None, None)
    if damping == "optimal":
        lam = estimate_extremal_eigs(lambda v: precond.apply(A @ v), b.shape[0], iters=eig_iters, seed=seed,
                                     a_matvec=lambda v: A @ v)
        xi = 2.0 / (lam[0] + lam[1])
    else:
        xi = float(damping)
    tr = Tracker(A, b, tol, kind, exact)
    x = np.zeros_like(b)
    it, conv = 0, False
    for k in range(max_iters + 1):
        r = b - A @ x
        if tr.record(x, r):
            it, conv = k, True
            break
        if tr.diverged():
            raise RuntimeError(f"error grew 10x after {k} iterations")
        if k == max_iters:
            it = k
            break
        x += xi * precond.apply(r)
    return SolverResult(it, conv, tr.residual, tr.energy, x, lam[0], lam[1], xi)


def fcg(A, b, precond, tol=1e-8, kind="relative_residual", exact=None, window=None, max_iters=20000):
    """krylov.py:294-326: directions explicitly A-orthogonalized against the
    stored ones (the last `window`, or all)."""
    tr = Tracker(A, b, tol, kind, exact)
    x = np.zeros_like(b)
    r = b - A @ x
    if tr.record(x, r):
        return SolverResult(0, True, tr.residual, tr.energy, x)
    dirs = []
    it, conv = 0, False
    for k in range(1, max_iters + 1):
        p = precond.apply(r)
        for pj, Apj, pApj in dirs:
            p = p - (float(p @ Apj) / pApj) * pj
        Ap = A @ p
        pAp = float(p @ Ap)
        if pAp <= 0.0:
            raise RuntimeError(f"nonpositive curvature at iteration {k}")
        alpha = float(p @ r) / pAp
        x += alpha * p
        r -= alpha * Ap
        dirs.append((p, Ap, pAp))
        if window is not None and len(dirs) > window:
            dirs.pop(0)
        it = k
        if tr.record(x, r):
            conv = True
            break
    return SolverResult(it, conv, tr.residual, tr.energy, x)
