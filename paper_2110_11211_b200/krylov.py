"""Outer solvers on the device (mirrors sfcdd.krylov).

Reference: /root/reference/pkg/src/sfcdd/krylov.py:29-334.  Richardson with
Lanczos-optimal damping and flexible CG compose the device
apply / stencil with deterministic BLAS-1 kernels of the C ABI; their
control flow is the reference's, step for step.  ``pcg`` with a
device SchwarzOperator runs the whole iteration on the B200 (csrc/op.cu:
fused matvec + p-update + p.Ap, fused x/r update + ||r|| + R0 r, the
balanced apply, r.z), captured as a CUDA graph and replayed until the
device flags convergence; the host only polls a status word.  Stopping rule
and history are the reference's relative-residual tracker
(krylov.py:186-200): history[k] = ||r_k||_2 of the recurrence residual.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import BreakdownError, DivergenceError  # noqa: F401  (re-exported)
from .grid import GridLaplacian


_METHOD_NAMES = ("richardson", "pcg", "fcg")
_TOLERANCE_KINDS = ("energy_error_reduction", "relative_residual")


@dataclass(frozen=True)
class SolverConfig:
    """Outer-solver parameters (krylov.py:29-47)."""

    method: str = "pcg"                               # one of _METHOD_NAMES
    damping: float | str = "optimal"                  # Richardson: "optimal" or a fixed xi
    tolerance: float = 1e-8                           # reduction factor of the stopping metric
    tolerance_kind: str = "energy_error_reduction"    # or "relative_residual"
    max_iters: int = 20000                            # iteration cap
    seed: int = 42                                    # Lanczos start vector / initial iterate
    eig_iters: int | None = None                      # Lanczos steps (None: automatic)
    fcg_window: int | None = None                     # FCG: stored directions (None: all)
    force_unsymmetric: bool = False                   # PCG with a non-symmetric preconditioner

    def __post_init__(self) -> None:
        checks = ((self.method in _METHOD_NAMES, f"method {self.method!r} not in {_METHOD_NAMES}"),
                  (self.tolerance_kind in _TOLERANCE_KINDS,
                   f"tolerance_kind {self.tolerance_kind!r} not in {_TOLERANCE_KINDS}"),
                  (self.tolerance > 0, f"tolerance {self.tolerance} is not positive"))
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)


@dataclass
class SolveReport:
    """Result of one outer solve (krylov.py:50-88)."""

    method: str                          # richardson | pcg | fcg
    iterations: int                      # steps taken
    converged: bool                      # stopping test met
    energy_history: list                 # ||x_k - x*||_A per step (with an exact solution)
    residual_history: list               # ||r_k||_2 per step
    lambda_min: float | None = None      # Richardson: estimated spectrum of C^-1 A
    lambda_max: float | None = None
    damping: float | None = None         # Richardson: xi used
    wall_time: float = 0.0               # seconds
    solution: np.ndarray | None = None   # x_k at exit
    params: dict = field(default_factory=dict)  # caller's parameter record

    def iteration_rows(self):
        """(k, energy error or "", residual) per recorded step."""
        en = self.energy_history
        return [(k, en[k] if en else "", res) for k, res in enumerate(self.residual_history)]

    def write_iterations_csv(self, fh) -> None:
        """CRLF CSV of the histories, floats as repr (krylov.py:71-75)."""
        lines = ["k,energy_error,residual"]
        lines += [f"{k},{'' if e == '' else repr(e)},{res!r}" for k, e, res in self.iteration_rows()]
        fh.write("".join(line + "\r\n" for line in lines))

    def summary(self) -> dict:
        """Scalar results plus the parameter record (krylov.py:77-88)."""
        keys = ("method", "iterations", "converged", "lambda_min", "lambda_max", "damping", "wall_time")
        return {**{k: getattr(self, k) for k in keys}, **self.params}


def initial_iterate(n: int, seed: int, A) -> np.ndarray:
    """Seeded U[-1, 1] entries (numpy PCG64, so bit-reproducible) rescaled to
    unit energy norm x / sqrt(x.(A x)) (krylov.py:91-99); A x on the device."""
    x = np.random.default_rng(seed).uniform(-1.0, 1.0, size=n)
    return x / np.sqrt(x @ np.asarray(A @ x))


def pcg_device(op, b, x0=None, tol: float = 1e-8, max_iters: int = 20000, exact=None,
               tolerance_kind: str = "relative_residual"):
    """Device-resident PCG on CUDA tensors.

    Returns (x, iterations, converged, residual_history); with ``exact`` the
    energy-error history is appended as a fifth element (krylov.py:189-193).
    """
    import torch

    dev = _lib.device()
    b = b.to(dev, torch.float64).contiguous()
    x = torch.zeros_like(b) if x0 is None else x0.to(dev, torch.float64).clone().contiguous()
    ex = None if exact is None else exact.to(dev, torch.float64).contiguous()
    hist = np.zeros(max_iters + 1)
    ehist = np.zeros(max_iters + 1)
    its = ctypes.c_int32()
    conv = ctypes.c_int32()
    kind = 1 if tolerance_kind == "energy_error_reduction" else 0
    _lib.check(_lib.lib().sfcdd_op_pcg_ex(op.handle, b.data_ptr(), x.data_ptr(),
                                          None if ex is None else ex.data_ptr(), kind, float(tol),
                                          int(max_iters), hist.ctypes.data, ehist.ctypes.data,
                                          ctypes.byref(its), ctypes.byref(conv), _lib.stream_ptr()))
    k = its.value
    if ex is None:
        return x, k, bool(conv.value), hist[:k + 1].tolist()
    return x, k, bool(conv.value), hist[:k + 1].tolist(), ehist[:k + 1].tolist()


def _matvec_fn(A):
    """v -> A v on CUDA tensors: the device stencil for grid Laplacians, the
    device CSR product for scipy / numpy matrices (linalg.DeviceMatrix)."""
    from .linalg import DeviceMatrix

    if isinstance(A, (GridLaplacian, DeviceMatrix)):
        return lambda v: A @ v
    if hasattr(A, "tocsr") or isinstance(A, np.ndarray):
        D = DeviceMatrix(A)
        return lambda v: D @ v
    # any other object with @ (the reference's duck typing): host product
    return lambda v: _to_device(np.asarray(A @ v.cpu().numpy(), dtype=np.float64))


def _apply_fn(precond, vec):
    """v -> C^-1 v on CUDA tensors (identity for precond=None, krylov.py:265)."""
    from .schwarz import SchwarzOperator

    if precond is None:
        return vec.copy
    if isinstance(precond, SchwarzOperator):
        return precond.apply_device
    # a caller's own preconditioner object (e.g. a dense-inverse oracle)
    return lambda v: _to_device(np.asarray(precond.apply(v.cpu().numpy()), dtype=np.float64))


def _graph_pcg_ok(A, precond) -> bool:
    """The fully device-resident PCG (csrc/op.cu) runs the operator's own
    stencil: A must be the grid Laplacian the operator was set up on."""
    from .schwarz import SchwarzOperator

    if not isinstance(precond, SchwarzOperator) or not isinstance(A, GridLaplacian):
        return False
    B = precond.A
    return (A.levels, A.scaled, A.curve) == (B.levels, B.scaled, B.curve)


def _to_device(v):
    import torch

    if isinstance(v, np.ndarray) or not hasattr(v, "data_ptr"):
        return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(_lib.device())
    return v.to(_lib.device(), torch.float64).contiguous()


class _Vec:
    """Deterministic BLAS-1 on device vectors through the C ABI (csrc/op.cu)."""

    def __init__(self, n):
        self.n = n

    def dot(self, x, y) -> float:
        out = ctypes.c_double()
        _lib.check(_lib.lib().sfcdd_vec_dot(x.data_ptr(), y.data_ptr(), self.n, ctypes.byref(out),
                                            _lib.stream_ptr()))
        return out.value

    def axpby(self, a, x, b, y):
        """y = a x + b y (in place)."""
        _lib.check(_lib.lib().sfcdd_vec_axpby(float(a), x.data_ptr(), float(b), y.data_ptr(), self.n,
                                              _lib.stream_ptr()))
        return y

    def new(self):
        import torch

        return torch.empty(self.n, dtype=torch.float64, device=_lib.device())

    def copy(self, x):
        return self.axpby(1.0, x, 0.0, self.new())

    def lin(self, a, x, b, y):
        """a x + b y as a new vector."""
        return self.axpby(a, x, b, self.copy(y))


class _DeviceTracker:
    """krylov.py:171-213 on device vectors: ||r||, and with an exact solution
    the energy error sqrt(max(e.(b - r - A x*), 0)), e = x - x*."""

    def __init__(self, matvec, b, cfg: SolverConfig, exact, vec: _Vec):
        energy_stop = cfg.tolerance_kind == "energy_error_reduction"
        if energy_stop and exact is None:
            raise ValueError("tolerance_kind='energy_error_reduction' needs the exact solution")
        self.vec, self.b, self.cfg, self.exact = vec, b, cfg, exact
        self.a_exact = None if exact is None else matvec(exact)
        self.energy_history, self.residual_history = [], []
        self._hist = self.energy_history if energy_stop else self.residual_history  # the stopping metric
        self._ref = None  # its first value

    def record(self, x, r) -> bool:
        """Append this iterate's metrics; True once the stopping test holds."""
        v = self.vec
        self.residual_history.append(float(np.sqrt(max(v.dot(r, r), 0.0))))
        if self.exact is not None:
            e = v.lin(1.0, x, -1.0, self.exact)                                   # x - x*
            ae = v.axpby(-1.0, self.a_exact, 1.0, v.lin(1.0, self.b, -1.0, r))    # (b - r) - A x*
            self.energy_history.append(float(np.sqrt(max(v.dot(e, ae), 0.0))))
        if self._ref is None:
            self._ref = self._hist[-1]
        return self._hist[-1] <= self.cfg.tolerance * self._ref

    def diverged(self) -> bool:
        """The metric grew 10x over its first value (krylov.py:202-208)."""
        return bool(self._ref) and self._hist[-1] > 10.0 * self._ref


def _finish(rep: SolveReport, t0: float, x, tracker: _DeviceTracker, to_numpy: bool) -> SolveReport:
    rep.wall_time = time.perf_counter() - t0
    rep.solution = x.cpu().numpy() if to_numpy else x
    rep.energy_history = tracker.energy_history
    rep.residual_history = tracker.residual_history
    return rep


def pcg(A, b, precond, cfg: SolverConfig, x0, exact=None) -> SolveReport:
    """Preconditioned CG; refuses non-symmetric preconditioners (krylov.py:257-291).

    Runs entirely on the device (csrc/op.cu, CUDA-graph iteration) with the
    reference tracker: residual history always, energy-error history when
    ``exact`` is given, stopping on ``cfg.tolerance_kind``."""
    t0 = time.perf_counter()
    if (precond is not None and not getattr(precond, "symmetric", True)
            and not cfg.force_unsymmetric):
        raise ValueError("preconditioner is not symmetric; use fcg or force_unsymmetric")
    if cfg.tolerance_kind == "energy_error_reduction" and exact is None:
        raise ValueError("energy stopping needs the exact solution")
    if not _graph_pcg_ok(A, precond):
        return _pcg_composed(A, b, precond, cfg, x0, exact, t0)
    to_numpy = isinstance(b, np.ndarray)
    out = pcg_device(precond, _to_device(b), _to_device(x0), cfg.tolerance, cfg.max_iters,
                     exact=None if exact is None else _to_device(exact), tolerance_kind=cfg.tolerance_kind)
    x, k, conv, hist = out[:4]
    rep = SolveReport("pcg", k, conv, out[4] if len(out) > 4 else [], hist)
    rep.solution = x.cpu().numpy() if to_numpy else x
    rep.wall_time = time.perf_counter() - t0
    return rep


def _pcg_composed(A, b, precond, cfg: SolverConfig, x0, exact, t0) -> SolveReport:
    """PCG for any matrix / preconditioner pair (krylov.py:257-291): the
    products run on the device (stencil, CSR product, Schwarz apply or the
    identity for precond=None) and the vector algebra through the
    deterministic BLAS-1 kernels; the control flow is the reference's."""
    n = b.shape[0]
    vec = _Vec(n)
    mv = _matvec_fn(A)
    apply_c = _apply_fn(precond, vec)
    to_numpy = isinstance(b, np.ndarray)
    bd = _to_device(b)
    tracker = _DeviceTracker(mv, bd, cfg, None if exact is None else _to_device(exact), vec)
    x = vec.copy(_to_device(x0))
    r = vec.axpby(1.0, bd, -1.0, mv(x))
    report = SolveReport("pcg", 0, False, [], [])
    if tracker.record(x, r):
        report.converged = True
        return _finish(report, t0, x, tracker, to_numpy)
    z = apply_c(r)
    p = vec.copy(z)
    rz = vec.dot(r, z)
    for k in range(1, cfg.max_iters + 1):
        Ap = mv(p)
        pAp = vec.dot(p, Ap)
        if pAp <= 0.0:
            raise BreakdownError(f"nonpositive curvature at iteration {k}")
        alpha = rz / pAp
        vec.axpby(alpha, p, 1.0, x)
        vec.axpby(-alpha, Ap, 1.0, r)
        report.iterations = k
        if tracker.record(x, r):
            report.converged = True
            break
        z = apply_c(r)
        rz_new = vec.dot(r, z)
        p = vec.axpby(1.0, z, rz_new / rz, p)
        rz = rz_new
    return _finish(report, t0, x, tracker, to_numpy)


def estimate_extremal_eigs(apply_ca, n: int, *, iters: int | None = None, seed: int = 0, a_matvec=None,
                           force_iterative: bool = False, stagnation_tol: float = 2e-5, min_iters: int = 40):
    """Extremal eigenvalues of C^-1 A (krylov.py:102-168) for numpy callables
    (the reference's interface): the callables are wrapped to device vectors
    and the estimate runs in estimate_extremal_eigs_device."""

    def dev(fn):
        if fn is None:
            return None
        return lambda v: _to_device(np.asarray(fn(v.cpu().numpy()), dtype=np.float64))

    return estimate_extremal_eigs_device(dev(apply_ca), n, iters=iters, seed=seed, a_matvec=dev(a_matvec),
                                         force_iterative=force_iterative, stagnation_tol=stagnation_tol,
                                         min_iters=min_iters)


def estimate_extremal_eigs_device(apply_ca, n: int, *, iters: int | None = None, seed: int = 0, a_matvec=None,
                                  force_iterative: bool = False, stagnation_tol: float = 2e-5,
                                  min_iters: int = 40):
    """Extremal eigenvalues of a preconditioned SPD operator (krylov.py:102-168).

    ``apply_ca`` and ``a_matvec`` map CUDA tensors to CUDA tensors (device
    apply / stencil).  n <= 300: dense eigenvalues of the operator matrix built
    column by column; otherwise Lanczos in the a_matvec inner product with full
    CGS2 reorthogonalization, stopping once both Ritz values stagnate.  The
    start vector is the reference's numpy draw (default_rng((seed, 0xE16)))."""
    import torch

    vec = _Vec(n)
    if n <= 300 and not force_iterative:
        M = np.empty((n, n))
        e = torch.zeros(n, dtype=torch.float64, device=_lib.device())
        for j in range(n):
            e.zero_()
            e[j] = 1.0
            M[:, j] = apply_ca(e).cpu().numpy()
        lam = np.real(np.linalg.eigvals(M))
        return float(lam.min()), float(lam.max())
    if iters is None:
        iters = min(200, n)
    rng = np.random.default_rng((seed, 0xE16))
    mv = a_matvec if a_matvec is not None else (lambda v: v)
    q = _to_device(rng.standard_normal(n))
    vec.axpby(1.0 / np.sqrt(vec.dot(q, mv(q))), q, 0.0, q)
    basis = [q]
    alphas: list[float] = []
    betas: list[float] = []
    prev = None
    stable = 0
    lam_lo = lam_hi = None
    for k in range(iters):
        w = apply_ca(basis[k])
        alpha = vec.dot(mv(w), basis[k])
        alphas.append(alpha)
        vec.axpby(-alpha, basis[k], 1.0, w)
        if k > 0:
            vec.axpby(-betas[k - 1], basis[k - 1], 1.0, w)
        for _ in range(2):  # CGS2 against the whole basis
            aw = mv(w)
            coeffs = [vec.dot(aw, qj) for qj in basis]
            for c, qj in zip(coeffs, basis):
                vec.axpby(-c, qj, 1.0, w)
        T = np.diag(alphas) + np.diag(betas[:len(alphas) - 1], 1) + np.diag(betas[:len(alphas) - 1], -1)
        lam = np.linalg.eigvalsh(T)
        lam_lo, lam_hi = float(lam[0]), float(lam[-1])
        if prev is not None:
            d_lo = abs(lam_lo - prev[0]) / max(abs(lam_lo), 1e-30)
            d_hi = abs(lam_hi - prev[1]) / max(abs(lam_hi), 1e-30)
            stable = stable + 1 if max(d_lo, d_hi) < stagnation_tol else 0
        prev = (lam_lo, lam_hi)
        if k + 1 >= min_iters and stable >= 5:
            break
        beta = float(np.sqrt(max(vec.dot(w, mv(w)), 0.0)))
        if beta <= 1e-14 * max(abs(alpha), 1.0):
            break
        betas.append(beta)
        basis.append(vec.axpby(1.0 / beta, w, 0.0, w))
    return lam_lo, lam_hi


def richardson(A, b, precond, cfg: SolverConfig, x0, exact=None) -> SolveReport:
    """Damped preconditioned Richardson x += xi C^-1 (b - A x) (krylov.py:219-254).

    ``damping="optimal"``: xi = 2/(lambda_min + lambda_max) of C^-1 A from
    estimate_extremal_eigs.  Every product runs on the device."""
    t0 = time.perf_counter()
    n = b.shape[0]
    vec = _Vec(n)
    mv = _matvec_fn(A)
    apply_c = _apply_fn(precond, vec)
    lam = (None, None)
    if cfg.damping == "optimal":
        if precond is not None and not getattr(precond, "symmetric", True):
            raise ValueError("optimal damping requires a symmetric preconditioner")
        lam = estimate_extremal_eigs_device(lambda v: apply_c(mv(v)), n, iters=cfg.eig_iters, seed=cfg.seed,
                                            a_matvec=mv)
        xi = 2.0 / (lam[0] + lam[1])
    else:
        xi = float(cfg.damping)
    to_numpy = isinstance(b, np.ndarray)
    bd = _to_device(b)
    tracker = _DeviceTracker(mv, bd, cfg, None if exact is None else _to_device(exact), vec)
    x = vec.copy(_to_device(x0))
    report = SolveReport("richardson", 0, False, [], [], lambda_min=lam[0], lambda_max=lam[1], damping=xi)
    for k in range(cfg.max_iters + 1):
        r = vec.axpby(1.0, bd, -1.0, mv(x))  # b - A x
        if tracker.record(x, r):
            report.iterations, report.converged = k, True
            break
        if tracker.diverged():
            raise DivergenceError(f"error grew 10x after {k} iterations")
        if k == cfg.max_iters:
            report.iterations = k
            break
        vec.axpby(xi, apply_c(r), 1.0, x)
    return _finish(report, t0, x, tracker, to_numpy)


def fcg(A, b, precond, cfg: SolverConfig, x0, exact=None) -> SolveReport:
    """Flexible CG (krylov.py:294-326): each new direction is A-orthogonalized
    against the stored ones (the last ``cfg.fcg_window``, or all), so
    non-symmetric preconditioners (e.g. the deflated variant) are admissible."""
    t0 = time.perf_counter()
    n = b.shape[0]
    vec = _Vec(n)
    mv = _matvec_fn(A)
    apply_c = _apply_fn(precond, vec)
    to_numpy = isinstance(b, np.ndarray)
    bd = _to_device(b)
    tracker = _DeviceTracker(mv, bd, cfg, None if exact is None else _to_device(exact), vec)
    x = vec.copy(_to_device(x0))
    r = vec.axpby(1.0, bd, -1.0, mv(x))
    report = SolveReport("fcg", 0, False, [], [])
    if tracker.record(x, r):
        report.converged = True
        return _finish(report, t0, x, tracker, to_numpy)
    directions = []
    for k in range(1, cfg.max_iters + 1):
        p = vec.copy(apply_c(r))
        for pj, Apj, pApj in directions:
            vec.axpby(-(vec.dot(p, Apj) / pApj), pj, 1.0, p)
        Ap = mv(p)
        pAp = vec.dot(p, Ap)
        if pAp <= 0.0:
            raise BreakdownError(f"nonpositive curvature at iteration {k}")
        alpha = vec.dot(p, r) / pAp
        vec.axpby(alpha, p, 1.0, x)
        vec.axpby(-alpha, Ap, 1.0, r)
        directions.append((p, Ap, pAp))
        if cfg.fcg_window is not None and len(directions) > cfg.fcg_window:
            directions.pop(0)
        report.iterations = k
        if tracker.record(x, r):
            report.converged = True
            break
    return _finish(report, t0, x, tracker, to_numpy)


_METHODS = {"richardson": richardson, "pcg": pcg, "fcg": fcg}


def run(A, b, precond, cfg: SolverConfig, x0, exact=None) -> SolveReport:
    """Dispatch on ``cfg.method`` (krylov.py:332-334)."""
    return _METHODS[cfg.method](A, b, precond, cfg, x0, exact=exact)
