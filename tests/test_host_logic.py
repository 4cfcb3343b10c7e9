"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
the host setup logic (AMD ordering, supernodal block-inverse factor, device
execution plan via its host interpreter) is exact, and the partition mirror
reproduces the reference's known answers.  No device calls."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from paper_2110_11211_b200 import _lib
from paper_2110_11211_b200 import partition as pt
from paper_2110_11211_b200.coarse import aggregate_bounds, aggregate_sizes

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "sfcdd_b200.h").read_text()
    declared = set(re.findall(r"\b(sfcdd_[a-z0-9_]+)\s*\(", header))
    L = _lib.lib()
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= declared
    assert L.sfcdd_version() == 1


def _csr_args(A):
    A = sp.csr_matrix(A)
    A.sort_indices()
    return (A.shape[0], np.ascontiguousarray(A.indptr, np.int64), np.ascontiguousarray(A.indices, np.int32),
            np.ascontiguousarray(A.data, np.float64))


def host_amd(A):
    n, ip, ix, _ = _csr_args(A)
    out = np.empty(n, np.int32)
    _lib.check(_lib.lib().sfcdd_host_amd(n, ip.ctypes.data, ix.ctypes.data, out.ctypes.data))
    return out


def host_solve(A, b):
    n, ip, ix, dv = _csr_args(A)
    x = np.empty(n)
    nl, st = ctypes.c_int64(), ctypes.c_int64()
    b = np.ascontiguousarray(b, np.float64)
    _lib.check(_lib.lib().sfcdd_host_factor_solve(n, ip.ctypes.data, ix.ctypes.data, dv.ctypes.data,
                                                  b.ctypes.data, x.ctypes.data, ctypes.byref(nl),
                                                  ctypes.byref(st)))
    return x, nl.value, st.value


def host_plan_solve(A, ranges, rhs, blob_max=0, scratch_max=0):
    n, ip, ix, dv = _csr_args(A)
    st = np.array([r.start for r in ranges], np.int64)
    ln = np.array([r.length for r in ranges], np.int64)
    xy = np.empty(int(ln.sum()))
    nf = ctypes.c_int64()
    rhs = np.ascontiguousarray(rhs, np.float64)
    _lib.check(_lib.lib().sfcdd_host_plan_solve(n, ip.ctypes.data, ix.ctypes.data, dv.ctypes.data, len(st),
                                                st.ctypes.data, ln.ctypes.data, rhs.ctypes.data,
                                                xy.ctypes.data, blob_max, scratch_max, ctypes.byref(nf)))
    return xy, nf.value


def random_spd(n, seed, density=0.05):
    rng = np.random.default_rng(seed)
    B = sp.random(n, n, density=density, random_state=rng)
    return sp.csr_matrix(B @ B.T + n * sp.eye(n))


@pytest.mark.parametrize("levels,p", [((7, 7), 16), ((4, 4, 4), 8)])
def test_amd_is_a_permutation_with_mmd_quality_fill(oracle, levels, p, monkeypatch):
    A = oracle.assemble_scaled_laplacian(levels)
    ov = oracle.enlarge(oracle.disjoint_partition(A.shape[0], p), 0.5)
    idx = ov[1].indices()
    As = A[idx][:, idx].tocsr()
    perm = host_amd(As)
    assert sorted(perm.tolist()) == list(range(len(idx)))
    monkeypatch.setenv("SFCDD_ORDER", "amd")
    x, nnz_l, stored = host_solve(As, np.ones(len(idx)))
    lu = spla.splu(sp.csc_matrix(As), permc_spec="MMD_AT_PLUS_A", options={"SymmetricMode": True})
    assert nnz_l <= 1.10 * lu.L.nnz  # AMD within 10% of SuperLU's MMD fill
    assert stored >= nnz_l
    np.testing.assert_allclose(As @ x, np.ones(len(idx)), atol=1e-10)


@pytest.mark.parametrize("levels,p,bound", [((7, 7), 16, 1.35), ((10, 10), 64, 1.15), ((4, 4, 4), 8, 1.35)])
def test_nested_dissection_fill(oracle, levels, p, bound, monkeypatch):
    """The default ordering (hybrid nested dissection, nd.cpp) trades a little
    fill for a shallow elimination tree; its fill stays within a bound of
    SuperLU's MMD (the reference's ordering) and the factor solves exactly."""
    A = oracle.assemble_scaled_laplacian(levels)
    ov = oracle.enlarge(oracle.disjoint_partition(A.shape[0], p), 0.5)
    idx = ov[1].indices()
    As = A[idx][:, idx].tocsr()
    monkeypatch.setenv("SFCDD_ORDER", "nd")
    b = np.random.default_rng(1).standard_normal(len(idx))
    x, nnz_l, stored = host_solve(As, b)
    lu = spla.splu(sp.csc_matrix(As), permc_spec="MMD_AT_PLUS_A", options={"SymmetricMode": True})
    assert nnz_l <= bound * lu.L.nnz
    np.testing.assert_allclose(As @ x, b, atol=1e-10 * np.abs(b).max())


@pytest.mark.parametrize("n,seed", [(1, 0), (2, 1), (7, 2), (60, 3), (300, 4)])
def test_host_block_inverse_solve_random_spd(n, seed):
    A = random_spd(n, seed)
    b = np.random.default_rng(seed).standard_normal(n)
    x, _, _ = host_solve(A, b)
    np.testing.assert_allclose(x, np.linalg.solve(A.toarray(), b), rtol=1e-10, atol=1e-12)


def test_host_factor_rejects_non_spd():
    A = sp.csr_matrix(np.array([[1.0, 2.0], [2.0, 1.0]]))
    with pytest.raises(_lib.FactorizationError):
        host_solve(A, np.ones(2))


@pytest.mark.parametrize("levels,p,gamma,blob", [((7, 7), 16, 0.5, 0), ((7, 7), 16, 0.25, 4096),
                                                  ((4, 4, 4), 8, 0.5, 0), ((4, 4, 4), 8, 1.0, 2048),
                                                  ((6, 5), 6, 0.75, 0),
                                                  # separators far wider than a 2 KB blob: ROW / COL values
                                                  # never pass through the blob
                                                  ((5, 5, 5), 4, 0.5, 2048)])
@pytest.mark.parametrize("split", [False, "wide", "narrow", "direct", "direct-mrow", "direct-inline"])
def test_device_plan_host_interpreter(oracle, levels, p, gamma, blob, split, monkeypatch):
    """The fragment/blob layout the DAG kernel executes, run on the host;
    ``split`` forces the ASM / XB task path of big supernodes (plan.h), with
    the default 32-row / 16-column blocks (``wide``) or narrow, non power of
    two blocks (``narrow``: several vector phases per lane group);
    ``direct``: every dense block streams its values from HBM (the form of
    the wide separators), with ASM / XB tasks or with inline gathers;
    ``direct-mrow``: the update rows as MROW tasks (plan.h)."""
    if split:
        if split != "direct-inline":
            monkeypatch.setenv("SFCDD_SPLIT_MIN", "1")
            monkeypatch.setenv("SFCDD_ASM_RED", "1")
            monkeypatch.setenv("SFCDD_XB_MIN", "1")
        if split == "narrow":
            monkeypatch.setenv("SFCDD_ROW_MAX", "6")
            monkeypatch.setenv("SFCDD_COL_MAX", "3")
        if split.startswith("direct"):
            monkeypatch.setenv("SFCDD_DIRECT_ROWS", str(1 << 20))
            monkeypatch.setenv("SFCDD_DIRECT_COLS", str(1 << 20))
            # MROW tasks (several row blocks in one value stream) for every supernode with below rows, or none
            monkeypatch.setenv("SFCDD_MROW_MIN", "1" if split == "direct-mrow" else str(1 << 30))
            if split == "direct-mrow":
                monkeypatch.setenv("SFCDD_MROW_ROWS", "40")  # several tasks per supernode, ragged last block
    A = oracle.assemble_scaled_laplacian(levels)
    n = A.shape[0]
    ov = oracle.enlarge(oracle.disjoint_partition(n, p), gamma)
    rhs = np.random.default_rng(3).standard_normal(n)
    xy, nfrag = host_plan_solve(A, ov, rhs, blob_max=blob)
    assert nfrag >= p
    off = 0
    for r in ov:
        idx = r.indices()
        xr = spla.spsolve(A[idx][:, idx].tocsc(), rhs[idx])
        np.testing.assert_allclose(xy[off:off + r.length], xr, rtol=1e-11, atol=1e-13)
        off += r.length


@pytest.mark.parametrize("levels,p,gamma", [((5, 5, 5), 2, 0.5), ((8, 8), 2, 0.5)])
def test_default_plan_few_wide_subdomains(oracle, levels, p, gamma):
    """Default blob shape and slot budget (one budget for blob + scratch) on
    few, large subdomains: separators ~ 1000 wide whose ROW / COL tasks carry
    inline gather lists and a whole front column of scratch (the C5-sized
    proxy of tools/plan_stats.py c5p at a size that runs in seconds)."""
    A = oracle.assemble_scaled_laplacian(levels)
    n = A.shape[0]
    ov = oracle.enlarge(oracle.disjoint_partition(n, p), gamma)
    rhs = np.random.default_rng(5).standard_normal(n)
    xy, nfrag = host_plan_solve(A, ov, rhs)
    off = 0
    for r in ov:
        idx = r.indices()
        xr = spla.spsolve(A[idx][:, idx].tocsc(), rhs[idx])
        assert np.linalg.norm(xy[off:off + r.length] - xr) <= 1e-11 * np.linalg.norm(xr)  # two exact factorizations
        off += r.length


@pytest.mark.parametrize("levels,blob,slot", [((7, 7), 2048, 2816), ((8, 8), 4096, 5632)])
def test_slot_budget_column_wider_than_the_slot_cap(oracle, levels, blob, slot, monkeypatch):
    """Slot budget (one budget for blob + scratch): a COL / ROW task whose
    gathered vector leaves less room than ONE column / row of values (but more
    than half a blob, so the cap applies) falls back to the separate budgets
    instead of failing with 'column does not fit a task blob' -- the C5-shaped
    GPU test's failure mode (s + m = 1625 under 16 KB blobs), scaled to
    2 / 4 KB blobs with the same slot : blob ratio."""
    monkeypatch.setenv("SFCDD_SLOT_MAX", str(slot))
    A = oracle.assemble_scaled_laplacian(levels)
    n = A.shape[0]
    ov = oracle.enlarge(oracle.disjoint_partition(n, 2), 0.5)
    rhs = np.random.default_rng(1).standard_normal(n)
    xy, _ = host_plan_solve(A, ov, rhs, blob_max=blob)
    off = 0
    for r in ov:
        idx = r.indices()
        xr = spla.spsolve(A[idx][:, idx].tocsc(), rhs[idx])
        assert np.linalg.norm(xy[off:off + r.length] - xr) <= 1e-11 * np.linalg.norm(xr)
        off += r.length


# ---- partition mirror: known answers of the reference tests (test_partition.py:24-116)
def test_partition_known_answers():
    assert [r.length for r in pt.disjoint_partition(9, 2)] == [5, 4]
    ov = pt.enlarge(pt.disjoint_partition(16, 4), 0.5)
    assert set(ov[1].indices().tolist()) == set(range(2, 10))
    assert set(ov[0].indices().tolist()) == {14, 15, 0, 1, 2, 3, 4, 5}
    ov = pt.enlarge(pt.disjoint_partition(15, 3), 0.3)
    assert all(r.length == 8 for r in ov)
    assert set(ov[1].indices().tolist()) == set(range(3, 11))
    ov = pt.enlarge(pt.disjoint_partition(75, 5), 0.2)
    assert all(r.length == 21 for r in ov)
    with pytest.raises(ValueError):
        pt.enlarge(pt.disjoint_partition(16, 4), 2.0)
    with pytest.raises(ValueError):
        pt.enlarge(pt.disjoint_partition(8, 1), 0.5)
    with pytest.raises(ValueError):
        pt.disjoint_partition(3, 4)
    assert all(r.length == 16 for r in pt.enlarge(pt.disjoint_partition(16, 4), 1.5))


@pytest.mark.parametrize("gamma", [0.5, 1.0, 1.5, 2.0])
def test_lemma_3_1_uniform_counts(gamma):
    w = pt.compute_weights(pt.build_partition(63, 8, gamma))
    c = int(round(2 * gamma + 1))
    assert np.all(w.counts == c)
    np.testing.assert_array_equal(w.omega, np.full(8, 1.0 / c))


def test_partitions_match_reference_fixtures(golden):
    import hashlib

    for name, e in golden.json("partitions.json").items():
        part = pt.build_partition(e["n"], e["p"], e["gamma"])
        assert [[r.start, r.length] for r in part.disjoint] == e["disjoint"]
        assert [[r.start, r.length] for r in part.overlapped] == e["overlapped"]
        if "omega" in e:
            w = pt.compute_weights(part)
            assert w.omega.tolist() == e["omega"]
            assert hashlib.sha256(w.counts.astype(np.int64).tobytes()).hexdigest() == e["counts_hash"]
            b = aggregate_bounds(part, e["q"])
            assert hashlib.sha256(b.tobytes()).hexdigest() == e["aggregate_bounds_hash"]


def test_cover_counts_brute_force():
    rng = np.random.default_rng(0)
    for _ in range(50):
        n = int(rng.integers(2, 400))
        p = int(rng.integers(2, min(n, 12) + 1))
        gamma = float(rng.choice([0.0, 0.25, 0.3, 0.5, 0.75, 1.0]))
        try:
            part = pt.build_partition(n, p, gamma)
        except ValueError:
            continue
        brute = np.zeros(n, int)
        for r in part.overlapped:
            brute[r.indices()] += 1
        np.testing.assert_array_equal(pt.compute_weights(part).counts, brute)


def test_aggregate_sizes():
    assert aggregate_sizes(12, 3) == [4, 4, 4]
    assert aggregate_sizes(11, 3) == [4, 4, 3]
    assert aggregate_sizes(5, 5) == [1, 1, 1, 1, 1]


def test_library_partition_matches_oracle_property(oracle):
    """csrc/partition.cpp (ranges from N, P, gamma num/den; prefix-sum window
    sums) against the oracle's restatement of partition.py:64-157 over a
    sweep of sizes, counts and fractional overlaps, including 2 gamma + 1 = P
    and gammas with large denominators."""
    rng = np.random.default_rng(7)
    gammas = [0.0, 0.1, 0.2, 0.25, 0.3, 1 / 3, 0.5, 0.75, 1.0, 1.25, 1.5, 2.0, 2.5, 0.123457, 3.75]
    for _ in range(300):
        p = int(rng.integers(2, 40))
        n = int(rng.integers(p, 5000))
        g = gammas[int(rng.integers(len(gammas)))]
        if 2 * g + 1 > p:
            with pytest.raises(ValueError):
                pt.build_partition(n, p, g)
            continue
        part = pt.build_partition(n, p, g)
        dj = oracle.disjoint_partition(n, p)
        ov = oracle.enlarge(dj, g)
        assert [(r.start, r.length) for r in part.disjoint] == [(r.start, r.length) for r in dj]
        assert [(r.start, r.length) for r in part.overlapped] == [(r.start, r.length) for r in ov]
        counts, diags, omega = oracle.weights(ov, n)
        w = pt.compute_weights(part)
        np.testing.assert_array_equal(w.counts, counts)
        np.testing.assert_array_equal(w.omega, omega)
        for a, b in zip(w.diagonals, diags):
            np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("levels,p", [((6, 6), 8), ((4, 4, 4), 8), ((7, 7), 16)])
def test_deferred_value_plan_rebuilds_blob_image(oracle, levels, p):
    """Plans built from symbolic factors (values placed later by descriptors,
    the device-factorization path) give the identical blob image and task
    list as plans built from host values."""
    A = oracle.assemble_scaled_laplacian(levels)
    ov = oracle.enlarge(oracle.disjoint_partition(A.shape[0], p), 0.5)
    n, ip, ix, dv = _csr_args(A)
    st = np.array([r.start for r in ov], np.int64)
    ln = np.array([r.length for r in ov], np.int64)
    bad, nseg, nvd = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.lib().sfcdd_host_plan_deferred_check(n, ip.ctypes.data, ix.ctypes.data, dv.ctypes.data, p,
                                                         st.ctypes.data, ln.ctypes.data, ctypes.byref(bad),
                                                         ctypes.byref(nseg), ctypes.byref(nvd)))
    assert nseg.value > 0 and nvd.value > 0
    assert bad.value == 0
