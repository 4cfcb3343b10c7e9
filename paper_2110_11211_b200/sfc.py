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


def holder_bound(dim: int) -> float:
    """2 sqrt(dim + 3), the bound on the curve's Holder quotient (sfc.py:172-174)."""
    return 2.0 * float(np.sqrt(dim + 3))


def _split(keys: list[int]) -> tuple[np.ndarray, np.ndarray]:
    hi = np.array([k >> 64 for k in keys], dtype=np.uint64)
    lo = np.array([k & ((1 << 64) - 1) for k in keys], dtype=np.uint64)
    return hi, lo


def holder_estimate(cfg: CurveConfig, samples: int, seed: int = 0) -> float:
    """Largest |s(x) - s(y)|_2 / |x - y|^(1/dim) over sampled curve parameter
    pairs (sfc.py:177-207).  The key pairs are the reference's seeded draws
    (little-endian default_rng bytes masked to key_bits); all points are
    decoded in one batch on the device."""
    if samples < 2:
        raise ValueError("need at least 2 samples")
    rng = np.random.default_rng(seed)
    kb = cfg.key_bits
    mask = (1 << kb) - 1
    nbytes = (kb + 7) // 8
    a, b = [], []
    for _ in range(samples):
        k1 = int.from_bytes(rng.bytes(nbytes), "little") & mask
        k2 = int.from_bytes(rng.bytes(nbytes), "little") & mask
        if k1 != k2:
            a.append(k1)
            b.append(k2)
    if not a:
        return 0.0
    pa = decode_many(*_split(a), cfg).astype(np.float64)
    pb = decode_many(*_split(b), cfg).astype(np.float64)
    dist = np.sqrt(((pa - pb) ** 2).sum(axis=1)) * (1.0 / cfg.side)
    param = np.array([abs(x - y) for x, y in zip(a, b)], dtype=np.float64) * np.ldexp(1.0, -kb)
    return float(np.max(dist / param ** (1.0 / cfg.dim)))


def curve_diagnostics(cfg: CurveConfig) -> dict:
    """Exhaustive bijectivity / unit-step check over all 2**key_bits keys
    (sfc.py:210-229): decode every key on the device, re-encode, compare."""
    total = 1 << cfg.key_bits
    keys = np.arange(total, dtype=np.uint64)
    zeros = np.zeros(total, dtype=np.uint64)
    pts = decode_many(zeros, keys, cfg)
    hi, lo = encode_many(pts, cfg)
    bijective = bool(np.all(hi == 0) and np.array_equal(lo, keys))
    steps = np.abs(np.diff(pts.astype(np.int64), axis=0)).sum(axis=1)
    return {"bijective": bijective, "adjacent": bool(np.all(steps == 1))}
