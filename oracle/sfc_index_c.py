"""TEST INFRASTRUCTURE: ctypes binding of the C restatement oracle/sfc_index.c
(the index-set checker at BASELINE configs[4] sizes).  Only
tests/ and the bench's checker legs import this; the product never does."""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libsfcdd_oracle.so"
_lib = None


def build() -> Path:
    if not LIB.exists() or LIB.stat().st_mtime < (HERE / "sfc_index.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB))
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.oracle_hilbert_keys.argtypes = [i32, i32, vp, i64, vp]
        L.oracle_sfc_perm.argtypes = [i32, vp, vp]
        L.oracle_partition.argtypes = [i64, i32, i64, i64, vp, vp, vp, vp]
        L.oracle_weights.argtypes = [i64, i32, vp, vp, vp, vp]
        L.oracle_aggregates.argtypes = [i32, vp, vp, i32, vp]
        _lib = L
    return _lib


def hilbert_keys(coords: np.ndarray, bits: int) -> np.ndarray:
    c = np.ascontiguousarray(coords, dtype=np.uint64)
    n, d = c.shape
    out = np.empty(n, np.uint64)
    rc = lib().oracle_hilbert_keys(d, bits, c.ctypes.data, n, out.ctypes.data)
    assert rc == 0, rc
    return out


def sfc_perm(levels) -> np.ndarray:
    lv = np.asarray(levels, dtype=np.int32)
    n = int(np.prod([(1 << int(l)) - 1 for l in levels]))
    out = np.empty(n, np.int64)
    rc = lib().oracle_sfc_perm(len(lv), lv.ctypes.data, out.ctypes.data)
    assert rc == 0, rc
    return out


def partition(n: int, p: int, gamma_num: int, gamma_den: int):
    a = [np.empty(p, np.int64) for _ in range(4)]
    rc = lib().oracle_partition(n, p, gamma_num, gamma_den, *(x.ctypes.data for x in a))
    if rc != 0:
        raise ValueError("infeasible partition")
    return a  # dj_start, dj_len, ov_start, ov_len


def weights(n: int, ov_start, ov_len, counts: bool = False):
    p = len(ov_start)
    st = np.ascontiguousarray(ov_start, np.int64)
    ln = np.ascontiguousarray(ov_len, np.int64)
    om = np.empty(p)
    cn = np.empty(n, np.int32) if counts else None
    rc = lib().oracle_weights(n, p, st.ctypes.data, ln.ctypes.data, cn.ctypes.data if counts else None, om.ctypes.data)
    assert rc == 0
    return (om, cn) if counts else om


def aggregates(dj_start, dj_len, q: int) -> np.ndarray:
    p = len(dj_start)
    ds = np.ascontiguousarray(dj_start, np.int64)
    dl = np.ascontiguousarray(dj_len, np.int64)
    out = np.empty(p * q + 1, np.int64)
    rc = lib().oracle_aggregates(p, ds.ctypes.data, dl.ctypes.data, q, out.ctypes.data)
    assert rc == 0
    return out


def scaled_block(levels, perm, rank, start, length):
    """Â restricted to the cyclic SFC range [start, start + length): the
    reference's Â[idx][:, idx] (schwarz.py:58-61), assembled from the C
    oracle's permutation and the stencil constants (grid.py:91-130)."""
    import scipy.sparse as sp
    import sfcdd_oracle as O

    n = perm.shape[0]
    shape = O.interior_shape(levels)
    dhat, offs, _ = O.stencil_constants(levels)
    idx = (start + np.arange(length)) % n
    lex = perm[idx]
    coords = np.stack(np.unravel_index(lex, shape), axis=1)
    strides = [int(np.prod(shape[j + 1:])) for j in range(len(shape))]
    rows, cols, vals = [np.arange(length)], [np.arange(length)], [np.full(length, dhat)]
    for j in range(len(shape)):
        for step in (-1, 1):
            ok = (coords[:, j] + step >= 0) & (coords[:, j] + step < shape[j])
            r = np.nonzero(ok)[0]
            nb = rank[lex[r] + step * strides[j]]
            loc = (nb - start) % n
            inside = loc < length
            rows.append(r[inside])
            cols.append(loc[inside])
            vals.append(np.full(int(inside.sum()), offs[j]))
    B = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(length, length))
    B.sort_indices()
    return B
