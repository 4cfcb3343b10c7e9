"""Preconditioned CG on the device (mirrors sfcdd.krylov).

Reference: /root/reference/pkg/src/sfcdd/krylov.py:29-334.  ``pcg`` with a
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


@dataclass(frozen=True)
class SolverConfig:
    method: str = "pcg"  # richardson | pcg | fcg
    damping: float | str = "optimal"
    tolerance: float = 1e-8
    tolerance_kind: str = "energy_error_reduction"  # or relative_residual
    max_iters: int = 20000
    seed: int = 42
    eig_iters: int | None = None
    fcg_window: int | None = None
    force_unsymmetric: bool = False

    def __post_init__(self) -> None:
        if self.method not in ("richardson", "pcg", "fcg"):
            raise ValueError(f"unknown method {self.method!r}")
        if self.tolerance_kind not in ("energy_error_reduction", "relative_residual"):
            raise ValueError(f"unknown tolerance kind {self.tolerance_kind!r}")
        if not self.tolerance > 0:
            raise ValueError("tolerance must be positive")


@dataclass
class SolveReport:
    method: str
    iterations: int
    converged: bool
    energy_history: list
    residual_history: list
    lambda_min: float | None = None
    lambda_max: float | None = None
    damping: float | None = None
    wall_time: float = 0.0
    solution: np.ndarray | None = None
    params: dict = field(default_factory=dict)

    def iteration_rows(self):
        rows = []
        for k, res in enumerate(self.residual_history):
            energy = self.energy_history[k] if self.energy_history else ""
            rows.append((k, energy, res))
        return rows

    def write_iterations_csv(self, fh) -> None:
        fh.write("k,energy_error,residual\r\n")
        for k, energy, res in self.iteration_rows():
            e = repr(energy) if energy != "" else ""
            fh.write(f"{k},{e},{repr(res)}\r\n")

    def summary(self) -> dict:
        out = {
            "method": self.method,
            "iterations": self.iterations,
            "converged": self.converged,
            "lambda_min": self.lambda_min,
            "lambda_max": self.lambda_max,
            "damping": self.damping,
            "wall_time": self.wall_time,
        }
        out.update(self.params)
        return out


def pcg_device(op, b, x0=None, tol: float = 1e-8, max_iters: int = 20000):
    """Device-resident PCG on CUDA tensors: returns (x, iterations, converged, history)."""
    import torch

    dev = _lib.device()
    b = b.to(dev, torch.float64).contiguous()
    x = torch.zeros_like(b) if x0 is None else x0.to(dev, torch.float64).clone().contiguous()
    hist = np.zeros(max_iters + 1)
    its = ctypes.c_int32()
    conv = ctypes.c_int32()
    _lib.check(_lib.lib().sfcdd_op_pcg(op.handle, b.data_ptr(), x.data_ptr(), float(tol), int(max_iters),
                                       hist.ctypes.data, ctypes.byref(its), ctypes.byref(conv),
                                       _lib.stream_ptr()))
    k = its.value
    return x, k, bool(conv.value), hist[:k + 1].tolist()


def pcg(A, b, precond, cfg: SolverConfig, x0, exact=None) -> SolveReport:
    """Preconditioned CG; refuses non-symmetric preconditioners (krylov.py:257-291)."""
    from .schwarz import SchwarzOperator

    t0 = time.perf_counter()
    if (precond is not None and not getattr(precond, "symmetric", True)
            and not cfg.force_unsymmetric):
        raise ValueError("preconditioner is not symmetric; use fcg or force_unsymmetric")
    if cfg.tolerance_kind == "energy_error_reduction" and exact is None:
        raise ValueError("energy stopping needs the exact solution")
    if not isinstance(precond, SchwarzOperator) or not isinstance(A, GridLaplacian) or not A.scaled:
        raise NotImplementedError("device PCG needs the scaled grid Laplacian and a device SchwarzOperator")
    if cfg.tolerance_kind != "relative_residual":
        raise NotImplementedError("device PCG implements the relative_residual stopping rule")
    import torch

    bt = torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64))
    xt = torch.from_numpy(np.ascontiguousarray(x0, dtype=np.float64))
    x, k, conv, hist = pcg_device(precond, bt, xt, cfg.tolerance, cfg.max_iters)
    rep = SolveReport("pcg", k, conv, [], hist)
    rep.solution = x.cpu().numpy()
    rep.wall_time = time.perf_counter() - t0
    return rep


def _not_on_device(name):
    def fn(*args, **kwargs):
        raise NotImplementedError(f"{name} is not part of the device hot path (SURVEY §8(f))")
    fn.__name__ = name
    return fn


richardson = _not_on_device("richardson")
fcg = _not_on_device("fcg")
estimate_extremal_eigs = _not_on_device("estimate_extremal_eigs")

_METHODS = {"richardson": richardson, "pcg": pcg, "fcg": fcg}


def run(A, b, precond, cfg: SolverConfig, x0, exact=None) -> SolveReport:
    """Dispatch on ``cfg.method`` (krylov.py:332-334)."""
    return _METHODS[cfg.method](A, b, precond, cfg, x0, exact=exact)
