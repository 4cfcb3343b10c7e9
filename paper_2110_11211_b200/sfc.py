"""d-dimensional Hilbert curve keys on the device (mirrors sfcdd.sfc).

``CurveConfig(dim, bits, curve="lebesgue")`` selects the Lebesgue (Morton,
Z-order) curve instead: the same MSB-first bit interleaving, axis 0 first, of
the raw coordinates (north star subsystem (1); the reference has Hilbert
only, so that option is checked against the oracle restatement).

Same API and validation as the reference module (/root/reference/pkg/src/
sfcdd/sfc.py:24-169); the key arithmetic runs in the sm_100a kernels of
csrc/sfc.cu (Skilling transpose form, 128-bit keys as two 64-bit words).
Scalar calls are batches of one; ``encode_many``/``decode_many`` are the
batched entry points.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

MAX_KEY_BITS = 128


@dataclass(frozen=True)
class CurveConfig:
    """Discrete Hilbert (or Lebesgue) curve on the lattice [0, 2**bits)**dim (sfc.py:24-47)."""

    dim: int
    bits: int
    curve: str = "hilbert"  # | "lebesgue"

    def __post_init__(self) -> None:
        if self.curve not in _lib.CURVES:
            raise ValueError(f"unknown curve {self.curve!r}")
        if self.dim < 1:
            raise ValueError(f"dimension must be positive, got {self.dim}")
        if self.bits < 1:
            raise ValueError(f"refinement must be positive, got {self.bits}")
        if self.dim * self.bits > MAX_KEY_BITS:
            raise ValueError(f"key width {self.dim * self.bits} exceeds {MAX_KEY_BITS} bits")

    @property
    def key_bits(self) -> int:
        return self.dim * self.bits

    @property
    def side(self) -> int:
        return 1 << self.bits


def _check_device_cfg(cfg: CurveConfig) -> None:
    if cfg.dim > 64 or cfg.bits > 64:
        raise ValueError("device curve kernels support dim <= 64 and bits <= 64")


def encode_many(coords, cfg: CurveConfig) -> tuple[np.ndarray, np.ndarray]:
    """Keys of an (n, dim) coordinate array as (hi, lo) uint64 words."""
    import torch

    _check_device_cfg(cfg)
    c = np.ascontiguousarray(np.asarray(coords, dtype=np.uint64).reshape(-1, cfg.dim))
    n = c.shape[0]
    if n and np.any(c >= np.uint64(cfg.side) if cfg.bits < 64 else False):
        raise ValueError(f"coordinate outside [0, {cfg.side})")
    dev = _lib.device()
    ct = torch.from_numpy(c.view(np.int64)).to(dev)
    hi = torch.empty(n, dtype=torch.int64, device=dev)
    lo = torch.empty(n, dtype=torch.int64, device=dev)
    _lib.check(_lib.lib().sfcdd_sfc_encode_curve(_lib.CURVES[cfg.curve], cfg.dim, cfg.bits, ct.data_ptr(), n,
                                                 hi.data_ptr(), lo.data_ptr(), _lib.stream_ptr()))
    return hi.cpu().numpy().view(np.uint64), lo.cpu().numpy().view(np.uint64)


def decode_many(hi, lo, cfg: CurveConfig) -> np.ndarray:
    import torch

    _check_device_cfg(cfg)
    hi = np.ascontiguousarray(np.asarray(hi, dtype=np.uint64))
    lo = np.ascontiguousarray(np.asarray(lo, dtype=np.uint64))
    n = lo.shape[0]
    dev = _lib.device()
    ht = torch.from_numpy(hi.view(np.int64)).to(dev)
    lt = torch.from_numpy(lo.view(np.int64)).to(dev)
    out = torch.empty(n * cfg.dim, dtype=torch.int64, device=dev)
    _lib.check(_lib.lib().sfcdd_sfc_decode_curve(_lib.CURVES[cfg.curve], cfg.dim, cfg.bits, ht.data_ptr(),
                                                 lt.data_ptr(), n, out.data_ptr(), _lib.stream_ptr()))
    return out.cpu().numpy().view(np.uint64).reshape(n, cfg.dim)


def encode(coords, cfg: CurveConfig) -> int:
    """Hilbert key of one lattice point (sfc.py:120-136)."""
    x = [int(c) for c in coords]
    if len(x) != cfg.dim:
        raise ValueError(f"expected {cfg.dim} coordinates, got {len(x)}")
    for c in x:
        if not 0 <= c < cfg.side:
            raise ValueError(f"coordinate {c} outside [0, {cfg.side})")
    hi, lo = encode_many(np.array([x], dtype=np.uint64), cfg)
    return (int(hi[0]) << 64) | int(lo[0])


def decode(key: int, cfg: CurveConfig) -> tuple[int, ...]:
    """Inverse of :func:`encode` (sfc.py:139-147)."""
    if not 0 <= key < (1 << cfg.key_bits):
        raise ValueError(f"key {key} outside [0, 2**{cfg.key_bits})")
    out = decode_many([key >> 64], [key & ((1 << 64) - 1)], cfg)
    return tuple(int(v) for v in out[0])


def grid_point_key(multi_index, levels, curve: str = "hilbert") -> int:
    """Key of a 1-based interior index of an anisotropic grid (sfc.py:150-169)."""
    ell = tuple(int(v) for v in levels)
    idx = tuple(int(v) for v in multi_index)
    if len(idx) != len(ell):
        raise ValueError("multi-index and level vector have different lengths")
    for k, lj in zip(idx, ell):
        if not 1 <= k <= (1 << lj) - 1:
            raise ValueError(f"index {k} outside interior range of level {lj}")
    n = max(ell)
    cfg = CurveConfig(len(ell), n, curve)
    coords = tuple((k - 1) << (n - lj) for k, lj in zip(idx, ell))
    return encode(coords, cfg)
