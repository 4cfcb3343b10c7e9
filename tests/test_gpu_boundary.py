"""Drop-in boundary semantics on the device (VERDICT r1 "what's missing" 5,
ADVICE r1): the reference's own call patterns that round 1 refused or got
wrong.  Marked ``gpu``.

* SchwarzOperator on the UNSCALED Laplacian (test_schwarz.py:56-62) against
  the dense oracle of test_schwarz.py:25-53;
* pcg with precond=None and on a general scipy matrix (test_krylov.py:147-166);
* concurrent applies on one shared operator (test_schwarz.py:208-222);
* energy history of the final iterate on a fresh operator (ADVICE: k_energy
  skipped when k_update stops);
* a second pcg with a larger max_iters on one operator (ADVICE: captured
  graph kept stale history buffers);
* one-level operators with tiny subdomains (ADVICE: > 32 ranges per chunk).
"""

import threading

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


def _dense(op):
    n = op.n
    M = np.empty((n, n))
    e = np.zeros(n)
    for j in range(n):
        e[j] = 1.0
        M[:, j] = op.apply(e)
        e[j] = 0.0
    return M


def _dense_oracle(Ad, part, cs_R0, variant, weighting, weights):
    n = part.n
    C1 = np.zeros((n, n))
    for i, rng in enumerate(part.overlapped):
        idx = rng.indices()
        R = np.zeros((len(idx), n))
        R[np.arange(len(idx)), idx] = 1.0
        inv = np.linalg.inv(R @ Ad @ R.T)
        D = {"omega": weights.omega[i] * np.eye(len(idx)), "d_matrix": np.diag(weights.diagonals[i]),
             "none": np.eye(len(idx))}[weighting]
        C1 += R.T @ D @ inv @ R
    if variant == "one_level":
        return C1
    F = cs_R0.T @ np.linalg.solve(cs_R0 @ Ad @ cs_R0.T, cs_R0)
    if variant == "additive_two_level":
        return C1 + F
    G = np.eye(n) - Ad @ F
    if variant == "deflated":
        return G.T @ C1 + F
    return G.T @ C1 @ G + F


@pytest.mark.parametrize("levels,p,gamma,q", [((7,), 4, 0.5, 4), ((3, 3), 4, 0.5, 2), ((4, 3), 5, 0.75, 2)])
@pytest.mark.parametrize("variant", ["one_level", "additive_two_level", "deflated", "balanced"])
def test_unscaled_operator_matches_dense_oracle(sfcdd, levels, p, gamma, q, variant):
    A = sfcdd.assemble_laplacian(levels)  # unscaled, as test_schwarz.make_operator
    part = sfcdd.build_partition(A.shape[0], p, gamma)
    cs = sfcdd.build_coarse(part, A, q) if variant != "one_level" else None
    op = sfcdd.setup(A, part, cs, sfcdd.SchwarzConfig(variant=variant, weighting="omega", gamma=gamma, q=q))
    Ad = A.toarray()
    assert Ad[0, 0] == 2.0 * sum(4.0**l for l in levels)  # exact integer entries (grid.py:101-110)
    M = _dense(op)
    R0 = cs.restriction.toarray() if cs is not None else None
    ref = _dense_oracle(Ad, part, R0, variant, "omega", sfcdd.compute_weights(part))
    np.testing.assert_allclose(M, ref, atol=1e-10 * np.abs(ref).max())


def test_unscaled_matvec_exact(sfcdd):
    A = sfcdd.assemble_laplacian((5, 4))
    x = np.random.default_rng(1).standard_normal(A.shape[0])
    np.testing.assert_allclose(A @ x, A.tocsr() @ x, rtol=1e-15, atol=1e-12)


def test_single_subdomain_unscaled_is_exact_inverse(sfcdd):
    # test_schwarz.py:65-69
    A = sfcdd.assemble_laplacian((5,))
    part = sfcdd.build_partition(31, 1, 0.0)
    op = sfcdd.setup(A, part, None, sfcdd.SchwarzConfig(variant="one_level", gamma=0.0, q=1))
    v = np.random.default_rng(0).standard_normal(31)
    np.testing.assert_allclose(A @ op.apply(v), v, atol=1e-10)


def test_pcg_unpreconditioned_grid(sfcdd):
    # test_krylov.py:148-155: CG finite termination without a preconditioner
    A = sfcdd.assemble_laplacian((3,))
    x_star = np.random.default_rng(2).standard_normal(7)
    b = A @ x_star
    cfg = sfcdd.SolverConfig(method="pcg", tolerance=1e-12, tolerance_kind="relative_residual")
    rep = sfcdd.pcg(A, b, None, cfg, np.zeros(7))
    assert rep.converged and rep.iterations <= 9
    np.testing.assert_allclose(rep.solution, x_star, rtol=1e-9)


def test_pcg_general_csr_matrix(sfcdd):
    # test_krylov.py:157-166: a dense-derived SPD CSR matrix, precond None
    import scipy.sparse as sp

    rng = np.random.default_rng(3)
    B = rng.standard_normal((50, 50))
    A = sp.csr_matrix(B.T @ B + 50 * np.eye(50))
    x_star = rng.standard_normal(50)
    cfg = sfcdd.SolverConfig(method="pcg", tolerance=1e-12, tolerance_kind="relative_residual", max_iters=60)
    rep = sfcdd.pcg(A, A @ x_star, None, cfg, np.zeros(50))
    assert rep.converged and rep.iterations <= 52


def test_device_csr_matches_scipy_bitwise(sfcdd):
    import scipy.sparse as sp

    from paper_2110_11211_b200.linalg import DeviceMatrix

    A = sp.random(300, 200, density=0.05, random_state=4, format="csr")
    x = np.random.default_rng(5).standard_normal(200)
    np.testing.assert_array_equal(DeviceMatrix(A) @ x, A @ x)


def test_concurrent_applies_on_shared_operator(sfcdd):
    # test_schwarz.py:208-222: 8 threads share one operator
    A = sfcdd.assemble_laplacian((5, 5))
    n = A.shape[0]
    part = sfcdd.build_partition(n, 8, 0.5)
    op = sfcdd.setup(A, part, sfcdd.build_coarse(part, A, 2), sfcdd.SchwarzConfig(gamma=0.5, q=2))
    rng = np.random.default_rng(0)
    vs = [rng.standard_normal(n) for _ in range(8)]
    expect = [op.apply(v) for v in vs]
    results = [None] * 8
    errors = []

    def work(i):
        try:
            for _ in range(10):
                out = op.apply(vs[i])
                if results[i] is None:
                    results[i] = out
                assert np.array_equal(out, expect[i])
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for i in range(8):
        np.testing.assert_array_equal(results[i], expect[i])


def _op(sfcdd, levels=(6, 6), p=8, q=4):
    A = sfcdd.assemble_laplacian(levels)
    n = A.shape[0]
    b = np.random.default_rng(42).uniform(-1.0, 1.0, size=n)
    Ah, bh, _ = sfcdd.symmetrize_diag(A, b)
    part = sfcdd.build_partition(n, p, 0.5)
    return Ah, bh, sfcdd.setup(Ah, part, sfcdd.build_coarse(part, Ah, q), sfcdd.SchwarzConfig(gamma=0.5, q=q))


def test_energy_history_final_entry_fresh_operator(sfcdd, oracle):
    # relative-residual stopping with an exact solution: the last energy entry
    # must be the final iterate's energy error (krylov.py:186-200)
    Ah, bh, op = _op(sfcdd)
    ex = np.random.default_rng(9).standard_normal(Ah.shape[0])
    b = Ah @ ex
    cfg = sfcdd.SolverConfig(method="pcg", tolerance=1e-8, tolerance_kind="relative_residual")
    rep = sfcdd.pcg(Ah, b, op, cfg, np.zeros(Ah.shape[0]), exact=ex)
    assert len(rep.energy_history) == rep.iterations + 1
    e = rep.solution - ex
    want = np.sqrt(max(e @ (Ah @ e), 0.0))
    assert abs(rep.energy_history[-1] - want) <= 1e-6 * rep.energy_history[0] + 1e-9 * want


def test_pcg_larger_max_iters_second_call(sfcdd):
    Ah, bh, op = _op(sfcdd)
    n = Ah.shape[0]
    short = sfcdd.pcg(Ah, bh, op, sfcdd.SolverConfig(method="pcg", tolerance=1e-8, tolerance_kind="relative_residual",
                                                     max_iters=3), np.zeros(n))
    assert short.iterations == 3 and not short.converged
    full = sfcdd.pcg(Ah, bh, op, sfcdd.SolverConfig(method="pcg", tolerance=1e-8, tolerance_kind="relative_residual",
                                                    max_iters=500), np.zeros(n))
    again = sfcdd.pcg(Ah, bh, op, sfcdd.SolverConfig(method="pcg", tolerance=1e-8, tolerance_kind="relative_residual",
                                                     max_iters=800), np.zeros(n))
    assert full.converged and again.converged
    assert full.residual_history == again.residual_history
    assert len(full.residual_history) == full.iterations + 1
    assert np.all(np.isfinite(full.residual_history))


def test_one_level_tiny_subdomains(sfcdd, oracle):
    # 4095 points, P = 256: ~16 points per subdomain (round 1 refused this)
    A = sfcdd.assemble_laplacian((12,))
    n = A.shape[0]
    part = sfcdd.build_partition(n, 256, 0.5)
    op = sfcdd.setup(A, part, None, sfcdd.SchwarzConfig(variant="one_level", gamma=0.5, q=1))
    g = np.random.default_rng(3).standard_normal(n)
    Ad = A.tocsr()
    w = sfcdd.compute_weights(part)
    ref = np.zeros(n)
    import scipy.sparse.linalg as spla

    for i, rng in enumerate(part.overlapped):
        idx = rng.indices()
        ref[idx] += w.omega[i] * spla.spsolve(Ad[idx][:, idx].tocsc(), g[idx])
    np.testing.assert_allclose(op.apply(g), ref, rtol=1e-10, atol=1e-12 * np.abs(ref).max())
