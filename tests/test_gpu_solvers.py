"""GPU parity of the other outer solvers against the
reference's own outputs (tests/golden/solvers.npz, oracle/make_fixtures.py):
energy-error PCG, Richardson with Lanczos-optimal and fixed damping, the
forced Lanczos estimate, and flexible CG (full / windowed, balanced and the
non-symmetric deflated variant).  Marked ``gpu``."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CASES = {"b66": ((6, 6), 8, 0.5, 4, "balanced"), "b44": ((4, 4), 4, 0.5, 2, "balanced"),
         "d55": ((5, 5), 6, 0.5, 2, "deflated")}


@pytest.fixture(scope="module")
def sfcdd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2110_11211_b200 as m

    return m


def _setup(sfcdd, tag):
    levels, p, gamma, q, variant = CASES[tag]
    A = sfcdd.assemble_laplacian(levels)
    n = A.shape[0]
    b = np.random.default_rng(42).uniform(-1.0, 1.0, size=n)
    Ah, bh, _ = sfcdd.symmetrize_diag(A, b)
    part = sfcdd.build_partition(n, p, gamma)
    op = sfcdd.setup(Ah, part, sfcdd.build_coarse(part, Ah, q), sfcdd.SchwarzConfig(variant, "omega", gamma, q))
    return Ah, bh, op


def _same(rep, g, key, tol, its_slack=0):
    assert rep.converged == bool(g[f"{key}_converged"])
    assert abs(rep.iterations - int(g[f"{key}_iterations"])) <= its_slack
    k = min(len(rep.residual_history), len(g[f"{key}_residual_history"]))
    for name in ("residual_history", "energy_history"):
        ref = g[f"{key}_{name}"][:k]
        got = np.asarray(getattr(rep, name))[:k]
        assert got.shape == ref.shape
        np.testing.assert_allclose(got, ref, rtol=tol, atol=tol * ref[0])
    sol = g[f"{key}_solution"]
    assert np.linalg.norm(rep.solution - sol) <= tol * np.linalg.norm(sol)


@pytest.mark.parametrize("tag", ["b66", "b44"])
def test_pcg_energy_tracking_matches_reference(sfcdd, golden, tag):
    g = golden.npz("solvers.npz")
    A, b, op = _setup(sfcdd, tag)
    ex = g[f"{tag}_exact"]
    # the reference default: energy_error_reduction stopping (krylov.py:33)
    rep = sfcdd.run(A, b, op, sfcdd.SolverConfig(method="pcg", tolerance=1e-8), np.zeros(A.shape[0]), ex)
    _same(rep, g, f"{tag}_pcg_energy", 1e-10, its_slack=1)
    rep = sfcdd.run(A, b, op, sfcdd.SolverConfig(method="pcg", tolerance=1e-8, tolerance_kind="relative_residual"),
                    np.zeros(A.shape[0]), ex)
    _same(rep, g, f"{tag}_pcg_rel", 1e-10, its_slack=1)
    with pytest.raises(ValueError):
        sfcdd.run(A, b, op, sfcdd.SolverConfig(method="pcg"), np.zeros(A.shape[0]))


@pytest.mark.parametrize("tag", ["b66", "b44"])
def test_richardson_matches_reference(sfcdd, golden, tag):
    g = golden.npz("solvers.npz")
    A, b, op = _setup(sfcdd, tag)
    ex = g[f"{tag}_exact"]
    n = A.shape[0]
    rep = sfcdd.run(A, b, op, sfcdd.SolverConfig(method="richardson", tolerance=1e-6,
                                                 tolerance_kind="relative_residual"), np.zeros(n), ex)
    np.testing.assert_allclose([rep.lambda_min, rep.lambda_max, rep.damping],
                               [g[f"{tag}_rich_opt_{k}"] for k in ("lambda_min", "lambda_max", "damping")],
                               rtol=1e-9)
    _same(rep, g, f"{tag}_rich_opt", 1e-9, its_slack=1)
    rep = sfcdd.run(A, b, op, sfcdd.SolverConfig(method="richardson", damping=0.5, tolerance=1e-6),
                    np.zeros(n), ex)
    assert rep.damping == 0.5 and rep.lambda_min is None
    _same(rep, g, f"{tag}_rich_fixed", 1e-9, its_slack=1)
    # the forced Lanczos path (n <= 300 would otherwise be dense)
    At = lambda v: A @ v  # noqa: E731
    lam = sfcdd.krylov.estimate_extremal_eigs_device(lambda v: op.apply_device(At(v)), n, seed=42, a_matvec=At,
                                              force_iterative=True)
    np.testing.assert_allclose(lam, g[f"{tag}_lanczos_forced"], rtol=1e-9)


@pytest.mark.parametrize("tag", ["b66", "b44", "d55"])
def test_fcg_matches_reference(sfcdd, golden, tag):
    g = golden.npz("solvers.npz")
    A, b, op = _setup(sfcdd, tag)
    ex = g[f"{tag}_exact"]
    n = A.shape[0]
    if CASES[tag][4] == "deflated":  # one-sided projection: PCG refuses it (krylov.py:260-264)
        assert not op.symmetric
        with pytest.raises(ValueError):
            sfcdd.run(A, b, op, sfcdd.SolverConfig(method="pcg", tolerance_kind="relative_residual"),
                      np.zeros(n))
    rep = sfcdd.run(A, b, op, sfcdd.SolverConfig(method="fcg", tolerance=1e-8, tolerance_kind="relative_residual"),
                    np.zeros(n), ex)
    _same(rep, g, f"{tag}_fcg", 1e-9, its_slack=1)
    rep = sfcdd.run(A, b, op, sfcdd.SolverConfig(method="fcg", tolerance=1e-8, fcg_window=2), np.zeros(n), ex)
    _same(rep, g, f"{tag}_fcg_w2", 1e-9, its_slack=1)


def test_vec_kernels_deterministic(sfcdd):
    from paper_2110_11211_b200.krylov import _Vec

    rng = np.random.default_rng(3)
    x = torch.from_numpy(rng.standard_normal(100003)).cuda()
    y = torch.from_numpy(rng.standard_normal(100003)).cuda()
    v = _Vec(x.numel())
    d = v.dot(x, y)
    assert d == v.dot(x, y)
    assert abs(d - float(x.cpu().numpy() @ y.cpu().numpy())) <= 1e-12 * abs(d) + 1e-9
    z = v.lin(2.0, x, -3.0, y)
    np.testing.assert_allclose(z.cpu().numpy(), 2.0 * x.cpu().numpy() - 3.0 * y.cpu().numpy(), rtol=1e-15,
                               atol=1e-15)
