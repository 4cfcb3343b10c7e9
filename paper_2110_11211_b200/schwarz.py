"""Two-level overlapping Schwarz operators on the B200 (mirrors sfcdd.schwarz).

Reference: /root/reference/pkg/src/sfcdd/schwarz.py:27-130.  Variants
one_level / additive_two_level / deflated / balanced and weightings none /
omega / d_matrix, with the reference's symmetric flag.  ``setup`` builds one
device handle (csrc/op.cu): local AMD + supernodal factorizations of every
Â_i, the coarse Galerkin problem, and the dataflow execution plan.
``apply`` takes/returns numpy (the reference protocol used by krylov.pcg);
``apply_device`` works on CUDA tensors without host copies.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .coarse import CoarseSpace
from .grid import GridLaplacian
from .partition import Partition, build_partition, compute_weights, gamma_fraction, is_half_integer

VARIANTS = ("one_level", "additive_two_level", "deflated", "balanced")
WEIGHTINGS = ("none", "omega", "d_matrix")


@dataclass(frozen=True)
class SchwarzConfig:
    variant: str = "balanced"
    weighting: str = "omega"
    gamma: float = 0.5
    q: int = 1

    def __post_init__(self) -> None:
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}")
        if self.weighting not in WEIGHTINGS:
            raise ValueError(f"unknown weighting {self.weighting!r}")


class SchwarzOperator:
    """Immutable preconditioner application on one CUDA device (schwarz.py:45-118)."""

    def __init__(self, A, part: Partition, coarse: CoarseSpace | None, config: SchwarzConfig,
                 workers: int = 1):
        if not isinstance(A, GridLaplacian):
            raise ValueError("the device Schwarz operator needs a grid Laplacian "
                             "(grid.assemble_laplacian(levels), optionally through grid.symmetrize_diag)")
        self.A = A
        self.partition = part
        self.coarse = coarse
        self.config = config
        self.workers = workers
        self.n = part.n
        self.weights = compute_weights(part)
        counts_uniform = self.weights.counts.min() == self.weights.counts.max()
        weighting_symmetric = config.weighting != "d_matrix" or (
            is_half_integer(config.gamma) and counts_uniform)
        # schwarz.py:63-69: deflated projects on one side only
        self.symmetric = weighting_symmetric and config.variant != "deflated"
        if config.variant != "one_level" and coarse is None:
            raise ValueError(f"variant {config.variant!r} needs a coarse space")
        q = coarse.q if (coarse is not None and config.variant != "one_level") else 0
        desc = _lib.OpDesc()
        # the library partitions N by gamma itself (csrc/partition.cpp); explicit
        # ranges are passed only for a partition that build_partition would not give
        num, den = gamma_fraction(part.gamma)
        desc.gamma_num, desc.gamma_den = num, den
        keep = []
        if part != build_partition(part.n, part.p, part.gamma):
            arrs = [np.array([r.start for r in part.overlapped], np.int64),
                    np.array([r.length for r in part.overlapped], np.int64),
                    np.array([r.start for r in part.disjoint], np.int64),
                    np.array([r.length for r in part.disjoint], np.int64),
                    np.ascontiguousarray(self.weights.omega, dtype=np.float64)]
            keep.extend(arrs)
            desc.ov_start, desc.ov_len, desc.dj_start, desc.dj_len, desc.omega = (a.ctypes.data for a in arrs)
        desc.raw_laplacian = 0 if A.scaled else 1
        desc.dim = len(A.levels)
        for j, l in enumerate(A.levels):
            desc.levels[j] = l
        desc.p = part.p
        desc.q = q
        desc.variant = _lib.VARIANT_CODES[config.variant]
        desc.weighting = _lib.WEIGHTING_CODES[config.weighting]
        desc.device = _lib.device().index
        desc.curve = _lib.CURVES[getattr(A, "curve", "hilbert")]
        desc.host_threads = _lib.host_threads()
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().sfcdd_op_create(ctypes.byref(desc), ctypes.byref(h)))
        self._h = h
        _lib.check(_lib.lib().sfcdd_op_setup(h, _lib.stream_ptr()))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().sfcdd_op_destroy(h)
            except Exception:
                pass

    @property
    def handle(self):
        return self._h

    def subdomain_sizes(self) -> list[int]:
        return [r.length for r in self.partition.overlapped]

    def stats(self) -> dict:
        s = _lib.Stats()
        _lib.check(_lib.lib().sfcdd_op_stats(self._h, ctypes.byref(s)))
        out = {f: getattr(s, f) for f, _ in _lib.Stats._fields_ if f != "reserved"}
        # setup phases (csrc/op.cu sfcdd_op_setup): ordering + symbolic
        # analysis, execution plan, numeric factorization (wall / device)
        out["plan_seconds"] = s.reserved[4] * 1e-6
        out["numeric_device_seconds"] = s.reserved[6] * 1e-6
        return out

    def coarse_matrix_dense(self) -> np.ndarray:
        n0 = self.stats()["n0"]
        out = np.empty((n0, n0))
        _lib.check(_lib.lib().sfcdd_op_coarse_dense(self._h, out.ctypes.data))
        return out

    def set_fault(self, apply_index: int, subdomains) -> None:
        """Config-4 fault mode: zero the local pieces of
        ``subdomains`` in apply call ``apply_index`` (0 = first apply)."""
        ids = np.ascontiguousarray(np.asarray(subdomains, dtype=np.int32).ravel())
        _lib.check(_lib.lib().sfcdd_op_set_fault(self._h, int(apply_index), ids.ctypes.data if ids.size else None,
                                                 int(ids.size)))

    def reset_calls(self) -> None:
        _lib.check(_lib.lib().sfcdd_op_reset_calls(self._h))

    def apply_device(self, g, out=None):
        import torch

        if g.shape != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got {tuple(g.shape)}")
        g = g.contiguous()
        h = torch.empty_like(g) if out is None else out
        _lib.check(_lib.lib().sfcdd_op_apply(self._h, g.data_ptr(), h.data_ptr(), _lib.stream_ptr()))
        return h

    def apply(self, g):
        """h = C^{-1} g (schwarz.py:103-118); numpy in, numpy out."""
        import torch

        if not isinstance(g, np.ndarray) and hasattr(g, "data_ptr"):
            return self.apply_device(g)
        g = np.asarray(g, dtype=np.float64)
        if g.shape != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got {g.shape}")
        gt = torch.from_numpy(np.ascontiguousarray(g)).to(_lib.device())
        return self.apply_device(gt).cpu().numpy()


def setup(A, part: Partition, coarse: CoarseSpace | None, config: SchwarzConfig,
          workers: int = 1) -> SchwarzOperator:
    """Factorize all subdomain blocks and the coarse problem (schwarz.py:121-130)."""
    if A.shape != (part.n, part.n):
        raise ValueError(f"matrix shape {A.shape} does not match N = {part.n}")
    return SchwarzOperator(A, part, coarse, config, workers=workers)
