"""GPU parity tests: every kernel through the C ABI against the oracle and the
reference-generated golden fixtures.  Marked ``gpu`` (run on a B200)."""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sfcdd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2110_11211_b200 as m

    return m


# ------------------------------------------------------------------ SFC
def test_sfc_walks_and_keys(sfcdd, golden):
    walks = golden.npz("sfc_walks.npz")
    for key in walks.files:
        d, n = (int(v[1:]) for v in key.split("_"))
        cfg = sfcdd.CurveConfig(d, n)
        coords = walks[key].astype(np.uint64)
        hi, lo = sfcdd.sfc.encode_many(coords, cfg)
        np.testing.assert_array_equal(lo, np.arange(coords.shape[0], dtype=np.uint64))
        back = sfcdd.sfc.decode_many(hi, lo, cfg)
        np.testing.assert_array_equal(back, coords)
    for e in golden.json("sfc_keys.json")["encode"]:
        assert sfcdd.encode(e["coords"], sfcdd.CurveConfig(e["dim"], e["bits"])) == int(e["key"])
        assert sfcdd.decode(int(e["key"]), sfcdd.CurveConfig(e["dim"], e["bits"])) == tuple(e["coords"])
    for e in golden.json("sfc_keys.json")["grid_point_key"]:
        assert sfcdd.grid_point_key(e["index"], e["levels"]) == int(e["key"])


@pytest.mark.parametrize("force_radix", [False, True])
def test_sfc_permutation_small(sfcdd, golden, force_radix):
    perms = golden.npz("perms.npz")
    for key in perms.files:
        levels = tuple(int(v) for v in key.split("_"))
        perm, rank = sfcdd.grid.sfc_permutation_device(levels, force_radix=force_radix)
        np.testing.assert_array_equal(perm.cpu().numpy(), perms[key])
        np.testing.assert_array_equal(rank.cpu().numpy()[perms[key]], np.arange(perms[key].size))


@pytest.mark.parametrize("key", ["10_10", "7_7_7", "12_12"])
def test_sfc_permutation_config_hashes(sfcdd, golden, key):
    want = golden.json("perm_hashes.json")[key]
    levels = tuple(int(v) for v in key.split("_"))
    for force in (False, True):
        perm, _ = sfcdd.grid.sfc_permutation_device(levels, force_radix=force)
        got = hashlib.sha256(perm.cpu().numpy().astype(np.int64).tobytes()).hexdigest()
        assert got == want, (levels, force)


def test_sfc_permutation_anisotropic_vs_oracle(sfcdd, oracle):
    for levels in [(8, 8, 9), (3, 9), (1, 1, 12), (2, 5, 3, 4)]:
        perm, _ = sfcdd.grid.sfc_permutation_device(levels)
        np.testing.assert_array_equal(perm.cpu().numpy(), oracle.sfc_permutation(levels))


# -------------------------------------------------------------- stencil
@pytest.mark.parametrize("levels", [(7, 7), (4, 4, 4), (3, 5), (2, 3, 2)])
def test_matvec_matches_assembled_matrix(sfcdd, oracle, levels):
    A = sfcdd.assemble_laplacian(levels)
    Ah, _, t = sfcdd.symmetrize_diag(A, np.zeros(A.shape[0]))
    B = oracle.assemble_scaled_laplacian(levels)
    x = np.random.default_rng(0).standard_normal(A.shape[0])
    np.testing.assert_allclose(Ah @ x, B @ x, rtol=1e-14, atol=1e-14)
    assert (Ah.tocsr() != B).nnz == 0  # bit-exact entries fl(fl(t a) t)
    np.testing.assert_array_equal(t, np.full(A.shape[0], oracle.stencil_constants(levels)[2]))


# ------------------------------------------------------------ operator
def _device_operator(sfcdd, levels, p, gamma, q, variant="balanced", weighting="omega"):
    A = sfcdd.assemble_laplacian(levels)
    Ah, _, _ = sfcdd.symmetrize_diag(A, np.zeros(A.shape[0]))
    part = sfcdd.build_partition(A.shape[0], p, gamma)
    cs = sfcdd.build_coarse(part, Ah, q) if variant != "one_level" else None
    return Ah, sfcdd.setup(Ah, part, cs, sfcdd.SchwarzConfig(variant, weighting, gamma, q))


def test_apply_matches_reference_dense_operators(sfcdd, golden):
    ops = golden.npz("dense_operators.npz")
    for key in ops.files:
        lv, rest = key.split("_p")
        levels = tuple(int(v) for v in lv.split("_"))
        p, g, q = rest.split("_")
        _, op = _device_operator(sfcdd, levels, int(p), float(g[1:]), int(q[1:]))
        n = op.n
        M = np.stack([op.apply(e) for e in np.eye(n)], axis=1)
        np.testing.assert_allclose(M, ops[key], rtol=0, atol=1e-12 * np.abs(ops[key]).max())


@pytest.mark.parametrize("name", ["c1_g05", "c1_g025"])
def test_apply_matches_reference_vectors(sfcdd, golden, name):
    g = golden.npz(f"solve_{name}.npz")
    _, op = _device_operator(sfcdd, (7, 7), 16, float(g["gamma"]), 4)
    np.testing.assert_allclose(op.coarse_matrix_dense(), g["coarse_matrix"], rtol=0, atol=1e-14)
    for v, out in zip(g["apply_inputs"], g["apply_outputs"]):
        h = op.apply(v)
        assert np.linalg.norm(h - out) <= 1e-12 * np.linalg.norm(out)


@pytest.mark.parametrize("variant", ["one_level", "additive_two_level", "deflated", "balanced"])
@pytest.mark.parametrize("weighting", ["none", "omega", "d_matrix"])
def test_variants_match_oracle_dense(sfcdd, oracle, variant, weighting):
    """Dense operator oracle (cf. reference test_schwarz.py:25-53), l=(5,5), P=4."""
    levels, p, gamma, q = (5, 5), 4, 0.5, 4
    Ah, op = _device_operator(sfcdd, levels, p, gamma, q, variant, weighting)
    A = oracle.assemble_scaled_laplacian(levels).toarray()
    n = A.shape[0]
    dis = oracle.disjoint_partition(n, p)
    ov = oracle.enlarge(dis, gamma)
    counts, diags, omega = oracle.weights(ov, n)
    C1 = np.zeros((n, n))
    for i, r in enumerate(ov):
        idx = r.indices()
        R = np.zeros((len(idx), n))
        R[np.arange(len(idx)), idx] = 1.0
        D = {"none": np.eye(len(idx)), "omega": omega[i] * np.eye(len(idx)), "d_matrix": np.diag(diags[i])}[weighting]
        C1 += R.T @ D @ np.linalg.inv(R @ A @ R.T) @ R
    R0 = oracle.coarse_restriction(dis, n, q).toarray()
    F = R0.T @ np.linalg.solve(R0 @ A @ R0.T, R0)
    G = np.eye(n) - A @ F
    want = {"one_level": C1, "additive_two_level": C1 + F, "deflated": G.T @ C1 + F,
            "balanced": G.T @ C1 @ G + F}[variant]
    M = np.stack([op.apply(e) for e in np.eye(n)], axis=1)
    np.testing.assert_allclose(M, want, rtol=0, atol=1e-10)


def test_apply_is_bitwise_deterministic(sfcdd):
    _, op = _device_operator(sfcdd, (8, 8), 16, 0.5, 4)
    v = np.random.default_rng(1).standard_normal(op.n)
    a = op.apply(v)
    for _ in range(3):
        np.testing.assert_array_equal(op.apply(v), a)


# ----------------------------------------------------------------- PCG
def _pcg(sfcdd, levels, p, gamma, q, fault=None):
    A = sfcdd.assemble_laplacian(levels)
    n = A.shape[0]
    b = np.random.default_rng(42).uniform(-1.0, 1.0, size=n)  # SURVEY §8(d) RHS
    Ah, bh, t = sfcdd.symmetrize_diag(A, b)
    part = sfcdd.build_partition(n, p, gamma)
    cs = sfcdd.build_coarse(part, Ah, q)
    op = sfcdd.setup(Ah, part, cs, sfcdd.SchwarzConfig("balanced", "omega", gamma, q))
    if fault is not None:
        op.set_fault(*fault)
    cfg = sfcdd.SolverConfig(method="pcg", tolerance=1e-8, tolerance_kind="relative_residual")
    return sfcdd.run(Ah, bh, op, cfg, np.zeros(n)), op


@pytest.mark.parametrize("name,tight", [("c1_g05", True), ("c1_g025", False), ("aniso", True),
                                        ("small_3d", True)])
def test_pcg_matches_reference(sfcdd, golden, name, tight):
    g = golden.npz(f"solve_{name}.npz")
    levels = tuple(int(v) for v in g["levels"])
    rep, _ = _pcg(sfcdd, levels, int(g["p"]), float(g["gamma"]), int(g["q"]))
    ref_hist = g["residual_history"]
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    assert rep.converged
    sol = g["solution"]
    assert np.linalg.norm(rep.solution - sol) <= 1e-10 * np.linalg.norm(sol) * (1 if tight else 1e3)
    k = min(len(ref_hist), len(rep.residual_history))
    rel = np.abs(np.asarray(rep.residual_history[:k]) - ref_hist[:k]) / ref_hist[:k]
    if tight:
        assert rel.max() <= 1e-10
    else:  # gamma = 1/4: the reference's own exact variants diverge after k~30
        assert rel[:25].max() <= 1e-10


@pytest.mark.parametrize("name", ["c1_g05", "small_3d"])
def test_pcg_split_big_supernodes_matches_reference(sfcdd, golden, name, monkeypatch):
    """The DAG kernel variant with ASM / XB tasks (used by many-subdomain
    plans, plan.h), forced on small cases."""
    monkeypatch.setenv("SFCDD_SPLIT_MIN", "1")
    monkeypatch.setenv("SFCDD_ASM_RED", "1")
    monkeypatch.setenv("SFCDD_XB_MIN", "1")
    monkeypatch.setenv("SFCDD_BLOB_MAX", "2048")  # many big supernodes
    g = golden.npz(f"solve_{name}.npz")
    levels = tuple(int(v) for v in g["levels"])
    rep, _ = _pcg(sfcdd, levels, int(g["p"]), float(g["gamma"]), int(g["q"]))
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    h = g["residual_history"]
    k = min(len(h), len(rep.residual_history))
    assert (np.abs(np.asarray(rep.residual_history[:k]) - h[:k]) / h[:k]).max() <= 1e-10
    sol = g["solution"]
    assert np.linalg.norm(rep.solution - sol) <= 1e-10 * np.linalg.norm(sol)


@pytest.mark.parametrize("name", ["c1_g05", "small_3d", "aniso"])
def test_pcg_sparse_coarse_factor_matches_reference(sfcdd, golden, name, monkeypatch):
    """The coarse problem through its supernodal factor and the DAG kernel (the
    path of coarse spaces above COARSE_DENSE_MAX dofs), forced on small cases."""
    monkeypatch.setenv("SFCDD_COARSE_DENSE_MAX", "0")
    g = golden.npz(f"solve_{name}.npz")
    levels = tuple(int(v) for v in g["levels"])
    rep, _ = _pcg(sfcdd, levels, int(g["p"]), float(g["gamma"]), int(g["q"]))
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    h = g["residual_history"]
    k = min(len(h), len(rep.residual_history))
    assert (np.abs(np.asarray(rep.residual_history[:k]) - h[:k]) / h[:k]).max() <= 1e-10
    sol = g["solution"]
    assert np.linalg.norm(rep.solution - sol) <= 1e-10 * np.linalg.norm(sol)


def test_pcg_c2_matches_reference(sfcdd, golden):
    g = golden.npz("solve_c2.npz")
    rep, _ = _pcg(sfcdd, (10, 10), 64, 0.5, 16)
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    h = g["residual_history"]
    k = min(len(h), len(rep.residual_history))
    assert (np.abs(np.asarray(rep.residual_history[:k]) - h[:k]) / h[:k]).max() <= 1e-10
    idx = g["solution_sample_idx"]
    ref = g["solution_sample"]
    assert np.linalg.norm(rep.solution[idx] - ref) <= 1e-10 * np.linalg.norm(ref)
    assert abs(np.linalg.norm(rep.solution) - float(g["solution_norm"])) <= 1e-10 * float(g["solution_norm"])


def test_pcg_c3_matches_reference(sfcdd, golden):
    g = golden.npz("solve_c3.npz")
    rep, _ = _pcg(sfcdd, (7, 7, 7), 512, 0.5, 8)
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    h = g["residual_history"]
    k = min(len(h), len(rep.residual_history))
    assert (np.abs(np.asarray(rep.residual_history[:k]) - h[:k]) / h[:k]).max() <= 1e-10
    idx = g["solution_sample_idx"]
    ref = g["solution_sample"]
    assert np.linalg.norm(rep.solution[idx] - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("mode", ["blob2k", "direct", "direct-mrow", "narrow", "inline", "direct-inline"])
def test_pcg_c3_dense_block_shapes_match_reference(sfcdd, golden, mode, monkeypatch):
    """Dense ROW / COL blocks of big supernodes: BLOB blocks travel with
    their metadata, DIRECT blocks (wide separators: the path of BASELINE
    C5's s ~ 2300) stream their values from HBM.  ``blob2k``: separators far
    wider than a 2 KB blob (mostly DIRECT); ``direct``: every block DIRECT;
    ``narrow``: DIRECT 6-row / 3-column blocks (several vector phases per
    warp, non power of two widths); ``inline`` / ``direct-inline``: the
    few-factor path (ROW / COL tasks gather their own vectors into the slot)
    forced on a 512-factor plan."""
    if mode == "blob2k":
        monkeypatch.setenv("SFCDD_BLOB_MAX", "2048")
    if mode in ("direct", "direct-mrow", "narrow", "direct-inline"):
        monkeypatch.setenv("SFCDD_DIRECT_ROWS", str(1 << 20))
        monkeypatch.setenv("SFCDD_DIRECT_COLS", str(1 << 20))
        # ``direct-mrow``: update rows as MROW tasks of <= 40 rows (ragged blocks); else no MROW tasks
        monkeypatch.setenv("SFCDD_MROW_MIN", "1" if mode == "direct-mrow" else str(1 << 30))
    if mode == "direct-mrow":
        monkeypatch.setenv("SFCDD_MROW_ROWS", "40")
    if mode == "narrow":
        monkeypatch.setenv("SFCDD_ROW_MAX", "6")
        monkeypatch.setenv("SFCDD_COL_MAX", "3")
    if mode in ("inline", "direct-inline"):
        monkeypatch.setenv("SFCDD_SPLIT_MIN", "100000")
    g = golden.npz("solve_c3.npz")
    rep, _ = _pcg(sfcdd, (7, 7, 7), 512, 0.5, 8)
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    h = g["residual_history"]
    k = min(len(h), len(rep.residual_history))
    assert (np.abs(np.asarray(rep.residual_history[:k]) - h[:k]) / h[:k]).max() <= 1e-10
    idx = g["solution_sample_idx"]
    ref = g["solution_sample"]
    assert np.linalg.norm(rep.solution[idx] - ref) <= 1e-10 * np.linalg.norm(ref)


def test_pcg_multichunk_aggregates_match_reference(sfcdd, golden):
    """Aggregates spanning several reduction chunks: the fused PCG epilogue
    sums the per-chunk R0 r partials per aggregate (op.cu pcg_fin_epilogue)."""
    g = golden.npz("solve_multichunk.npz")
    rep, _ = _pcg(sfcdd, (9, 9), 8, 0.5, 2)
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    h = g["residual_history"]
    k = min(len(h), len(rep.residual_history))
    assert (np.abs(np.asarray(rep.residual_history[:k]) - h[:k]) / h[:k]).max() <= 1e-10
    idx = g["solution_sample_idx"]
    ref = g["solution_sample"]
    assert np.linalg.norm(rep.solution[idx] - ref) <= 1e-10 * np.linalg.norm(ref)


def test_pcg_fault_mode_matches_reference(sfcdd, golden):
    g = golden.npz("solve_fault_88.npz")
    dead = np.random.default_rng(42).choice(256, size=int(round(0.1 * 256)), replace=False)
    rep, _ = _pcg(sfcdd, (8, 8), 256, 0.5, 16, fault=(5, dead))
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    h = g["residual_history"]
    k = min(len(h), len(rep.residual_history))
    assert (np.abs(np.asarray(rep.residual_history[:k]) - h[:k]) / h[:k]).max() <= 1e-10


def test_pcg_c4_fault_mode_full_size_matches_reference(sfcdd, golden):
    """BASELINE configs[3] at full size on one device (4095^2, P=256, q=16,
    fault at apply 5): the bench workload of ``bench.py --config c4``."""
    g = golden.npz("solve_c4_fault.npz")
    dead = np.random.default_rng(42).choice(256, size=int(round(0.1 * 256)), replace=False)
    rep, _ = _pcg(sfcdd, (12, 12), 256, 0.5, 16, fault=(5, dead))
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    h = g["residual_history"]
    k = min(len(h), len(rep.residual_history))
    assert (np.abs(np.asarray(rep.residual_history[:k]) - h[:k]) / h[:k]).max() <= 1e-10
    idx = g["solution_sample_idx"]
    ref = g["solution_sample"]
    assert np.linalg.norm(rep.solution[idx] - ref) <= 1e-10 * np.linalg.norm(ref)


def test_pcg_bitwise_repeatable(sfcdd):
    r1, _ = _pcg(sfcdd, (8, 8), 32, 0.5, 4)
    r2, _ = _pcg(sfcdd, (8, 8), 32, 0.5, 4)
    assert r1.residual_history == r2.residual_history
    np.testing.assert_array_equal(r1.solution, r2.solution)


# ---------------------------------------------------------- direct solver
@pytest.mark.parametrize("n,seed", [(1, 0), (50, 1), (700, 2)])
def test_factorization_random_spd(sfcdd, n, seed):
    import scipy.sparse as sp

    rng = np.random.default_rng(seed)
    B = sp.random(n, n, density=min(1.0, 5.0 / n), random_state=rng)
    A = sp.csr_matrix(B @ B.T + n * sp.eye(n))
    F = sfcdd.Factorization(A)
    b = rng.standard_normal(n)
    np.testing.assert_allclose(F.solve(b), np.linalg.solve(A.toarray(), b), rtol=1e-10, atol=1e-12)


def test_factorization_rejects_non_spd(sfcdd):
    import scipy.sparse as sp

    with pytest.raises(sfcdd.FactorizationError):
        sfcdd.Factorization(sp.csr_matrix(np.array([[1.0, 2.0], [2.0, 1.0]])))


@pytest.mark.parametrize("curve", ["hilbert", "lebesgue"])
@pytest.mark.parametrize("levels", [(7, 7), (6, 7), (10, 10), (4, 4, 4), (5, 6, 5), (7, 7, 7)])
def test_tiled_stencil_bitwise_equals_neighbour_table(sfcdd, levels, monkeypatch, curve):
    """The index-free SFC-tile stencil (csrc/tiles.cpp) against the
    neighbour-table stencil on the same vector: bitwise equal."""
    n = sfcdd.num_dofs(levels)
    part = sfcdd.build_partition(n, max(4, n // 8000), 0.5)  # blocks a COL blob can hold

    def op_for(env):
        if env:
            monkeypatch.setenv("SFCDD_NO_TILES", "1")
        else:
            monkeypatch.delenv("SFCDD_NO_TILES", raising=False)
        A = sfcdd.assemble_laplacian(levels, curve=curve)
        Ah, _, _ = sfcdd.symmetrize_diag(A, np.zeros(n))
        return sfcdd.schwarz.SchwarzOperator(Ah, part, sfcdd.build_coarse(part, Ah, 1),
                                             sfcdd.SchwarzConfig("balanced", "omega", 0.5, 1))

    x = torch.from_numpy(np.random.default_rng(9).standard_normal(n)).cuda()
    outs = []
    for env in (True, False):
        op = op_for(env)
        y = torch.empty_like(x)
        from paper_2110_11211_b200 import _lib

        _lib.check(_lib.lib().sfcdd_op_matvec(op.handle, x.data_ptr(), y.data_ptr(), _lib.stream_ptr()))
        outs.append(y.cpu().numpy())
        a = op.apply(x.cpu().numpy())
        outs.append(a)
    np.testing.assert_array_equal(outs[0], outs[2])
    np.testing.assert_allclose(outs[1], outs[3], rtol=1e-12, atol=1e-14 * np.abs(outs[1]).max())


# ------------------------------------------------------ Lebesgue curve option
@pytest.mark.parametrize("d,bits", [(2, 5), (3, 20), (5, 12), (4, 32)])
def test_lebesgue_encode_decode_vs_oracle(sfcdd, oracle, d, bits):
    coords = np.random.default_rng(d * bits).integers(0, 1 << bits, size=(500, d), dtype=np.uint64)
    cfg = sfcdd.CurveConfig(d, bits, "lebesgue")
    hi, lo = sfcdd.sfc.encode_many(coords, cfg)
    ohi, olo = oracle.lebesgue_keys(coords, bits)
    np.testing.assert_array_equal(hi, ohi)
    np.testing.assert_array_equal(lo, olo)
    np.testing.assert_array_equal(sfcdd.sfc.decode_many(hi, lo, cfg), coords)


@pytest.mark.parametrize("levels", [(3, 3), (5, 4), (4, 4, 4), (3, 4, 5), (10, 10), (7, 7, 7)])
@pytest.mark.parametrize("force_radix", [False, True])
def test_lebesgue_permutation_vs_oracle(sfcdd, oracle, levels, force_radix):
    perm, rank = sfcdd.grid.sfc_permutation_device(levels, force_radix=force_radix, curve="lebesgue")
    want = oracle.sfc_permutation(levels, "lebesgue")
    np.testing.assert_array_equal(perm.cpu().numpy(), want)
    np.testing.assert_array_equal(rank.cpu().numpy()[want], np.arange(want.size))


@pytest.mark.parametrize("levels,p,q", [((7, 7), 16, 4), ((4, 4, 4), 8, 4), ((6, 7), 12, 3)])
def test_pcg_lebesgue_ordering_vs_oracle(sfcdd, oracle, levels, p, q):
    """The whole pipeline on the Morton ordering (tiles, partitions, DAG,
    coarse space) against the oracle on the same ordering."""
    A = sfcdd.assemble_laplacian(levels, curve="lebesgue")
    n = A.shape[0]
    b = np.random.default_rng(42).uniform(-1.0, 1.0, size=n)
    Ah, bh, _ = sfcdd.symmetrize_diag(A, b)
    part = sfcdd.build_partition(n, p, 0.5)
    op = sfcdd.setup(Ah, part, sfcdd.build_coarse(part, Ah, q), sfcdd.SchwarzConfig("balanced", "omega", 0.5, q))
    cfg = sfcdd.SolverConfig(method="pcg", tolerance=1e-8, tolerance_kind="relative_residual")
    rep = sfcdd.run(Ah, bh, op, cfg, np.zeros(n))
    _, _, _, ref = oracle.solve_config(levels, p, 0.5, q, curve="lebesgue")
    assert abs(rep.iterations - ref.iterations) <= 1
    k = min(len(ref.residual_history), len(rep.residual_history))
    h = np.asarray(ref.residual_history[:k])
    assert (np.abs(np.asarray(rep.residual_history[:k]) - h) / h).max() <= 1e-10
    assert np.linalg.norm(rep.solution - ref.solution) <= 1e-10 * np.linalg.norm(ref.solution)
    # the scaled operator in Morton order is the oracle's matrix
    np.testing.assert_allclose(Ah @ b, oracle.assemble_scaled_laplacian(levels, "lebesgue") @ b,
                               rtol=1e-15, atol=1e-15)
