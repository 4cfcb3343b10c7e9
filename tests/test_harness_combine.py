"""Experiment harness and combination technique.

CPU tests cover the host logic (plans, closed-form counts, interpolation,
q rules, sweep levels, config parsing, CSV layout, the manufactured
problem); ``gpu`` tests run the sweeps and combination solves through the
device solver and compare them with rows the reference produced
(tests/golden/harness.json, oracle/make_fixtures.py make_harness).
Model: reference tests test_harness.py / test_combine.py.
"""

import csv
import io
import math

import numpy as np
import pytest

from paper_2110_11211_b200 import combine, grid, harness

torch = pytest.importorskip("torch")


def _brute_layer(d, total):
    if d == 1:
        return [(total,)] if total >= 1 else []
    out = []
    for first in range(1, total):
        out.extend((first,) + rest for rest in _brute_layer(d - 1, total - first))
    return out


# ------------------------------------------------------------------ host logic
def test_plan_layers_and_coefficients():
    plan = combine.enumerate_plan(2, 3)
    assert plan.layers == (((1, 3), (2, 2), (3, 1)), ((1, 2), (2, 1)))
    assert plan.coefficients == (1, -1)
    assert combine.enumerate_plan(1, 5).layers == (((5,),),)
    assert combine.enumerate_plan(4, 6).coefficients == (1, -3, 3, -1)
    for d, level in [(2, 4), (3, 6), (4, 7), (5, 9)]:
        plan = combine.enumerate_plan(d, level)
        for i, layer in enumerate(plan.layers):
            assert list(layer) == sorted(_brute_layer(d, level + d - 1 - i))
            assert len(layer) == math.comb(level + d - 2 - i, d - 1)
    with pytest.raises(ValueError):
        combine.enumerate_plan(3, 2)
    with pytest.raises(ValueError):
        combine.enumerate_plan(2, 4, p_hat=0)
    counts = {}
    for i, _, p, _ in combine.enumerate_plan(3, 5, p_hat=2).terms():
        counts.setdefault(i, set()).add(p)
    assert counts == {0: {8}, 1: {4}, 2: {2}}


def test_subdomain_count_total_closed_form():
    # values of the reference's closed form at L = 20 (test_combine.py:66-73)
    expected = {1: 1, 2: 59, 3: 1391, 4: 20889, 5: 237706, 6: 2233216}
    for d, v in expected.items():
        assert combine.subdomain_count_total(d, 20, 1) == v
        assert combine.subdomain_count_total(d, 20, 1024) == 1024 * v
    assert combine.subdomain_count_total(6, 19) == 1754744
    for d in range(1, 7):
        for level in (8, 12, 20):
            plan = combine.enumerate_plan(d, level, p_hat=3)
            assert combine.subdomain_count_total(d, level, 3) == sum(p for _, _, p, _ in plan.terms())


def test_q_rules_and_weak_levels():
    assert combine.default_q_rule(2**12, 2**4) == 16
    assert combine.default_q_rule(100, 50) == 1
    assert combine.default_q_rule(10, 1) == 1
    spec = harness.ExperimentSpec(q_rule="fixed", q_value=8, s=8)
    assert harness.resolve_q(spec, 1000, 4) == 8
    assert harness.resolve_q(spec, 20, 4) == 5
    assert harness.resolve_q(harness.ExperimentSpec(q_rule="srel4", s=8), 10**6, 4) == 16
    assert harness.resolve_q(harness.ExperimentSpec(q_rule="auto"), 2**12, 2**4) == 16
    with pytest.raises(ValueError):
        harness.resolve_q(harness.ExperimentSpec(q_rule="bogus"), 100, 4)
    assert harness.weak_levels(1, 6, 8) == (9,)
    assert harness.weak_levels(2, 6, 16) == (5, 5)
    assert harness.weak_levels(3, 6, 4) == (2, 2, 2)
    assert harness.weak_levels(2, 6, 12) is None
    assert harness.weak_levels(6, 1, 2) is None


def test_interpolation_properties():
    levels = (2, 3)
    vals = np.random.default_rng(0).standard_normal(grid.interior_shape(levels))
    for k1 in range(1, 4):
        for k2 in range(1, 8):
            got = combine.multilinear_interpolate(levels, vals, np.array([[k1 / 4.0, k2 / 8.0]]))[0]
            assert got == pytest.approx(vals[k1 - 1, k2 - 1], abs=1e-14)
    pts = np.array([[0.0, 0.5], [1.0, 0.25], [0.5, 0.0], [0.75, 1.0]])
    np.testing.assert_allclose(combine.multilinear_interpolate((2, 2), np.ones((3, 3)), pts), 0.0, atol=1e-14)
    assert combine.multilinear_interpolate((1, 1), np.array([[2.0]]), np.array([[0.25, 0.25]]))[0] == \
        pytest.approx(0.5)
    # the combination of constants telescopes to the constant in the bulk
    for d, level in [(2, 4), (3, 5)]:
        plan = combine.enumerate_plan(d, level)
        terms = [(c, lv, np.full(grid.interior_shape(lv), 3.7))
                 for layer, c in zip(plan.layers, plan.coefficients) for lv in layer]
        pts = np.random.default_rng(1).uniform(0.25, 0.75, size=(100, d))
        np.testing.assert_allclose(combine.CombinedSolution(terms)(pts), 3.7, atol=1e-12)
    with pytest.raises(ValueError):
        combine.sampled_error(lambda x: x[:, 0], lambda x: x[:, 0], 2, 4, 0)


def test_manufactured_problem_matches_reference(golden):
    g = golden.json("harness.json")["manufactured"]
    for d in (1, 2, 3):
        prob = grid.manufactured_poisson((3,) * d)
        pts = np.asarray(g[str(d)]["points"])
        np.testing.assert_allclose(prob.rhs(pts), g[str(d)]["rhs"], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(prob.exact_solution(pts), g[str(d)]["exact"], rtol=1e-14, atol=1e-15)
    # -Lap u by central differences agrees with the closed-form right-hand side
    prob = grid.manufactured_poisson((3, 3))
    x = np.array([[0.3, 0.6]])
    h = 1e-4
    lap = sum((prob.exact_solution(x + h * e) - 2 * prob.exact_solution(x) + prob.exact_solution(x - h * e)) / h**2
              for e in np.eye(2)[:, None, :])
    assert -lap[0] == pytest.approx(prob.rhs(x)[0], rel=1e-6)


def test_plateau_config_and_csv(tmp_path):
    rows = [{"P": 16, "iterations": 20, "skipped": 0}, {"P": 32, "iterations": 25, "skipped": 0},
            {"P": 64, "iterations": 23, "skipped": 0}, {"P": 128, "iterations": "", "skipped": 1}]
    assert harness.plateau_spread(rows) == (23, 25)
    with pytest.raises(ValueError):
        harness.plateau_spread(rows[:1])
    cfg = tmp_path / "exp.cfg"
    cfg.write_text("# sweep\ndim = 2\np_values = 4, 8 16\ngamma = 0.25  # overlap\n")
    spec = harness.build_spec("weak", harness.load_config_file(cfg), {"s": 7, "gamma": None})
    assert (spec.dim, spec.p_values, spec.gamma, spec.s, spec.kind) == (2, (4, 8, 16), 0.25, 7, "weak")
    (tmp_path / "bad.cfg").write_text("dim 2\n")
    with pytest.raises(ValueError):
        harness.load_config_file(tmp_path / "bad.cfg")
    with pytest.raises(ValueError):
        harness.build_spec("weak", None, {"bogus": 1})
    row = harness._row(harness.ExperimentSpec(kind="weak"), P=4, skipped=1, reason="x")
    harness.write_rows_csv(tmp_path / "r.csv", [row])
    raw = (tmp_path / "r.csv").read_bytes()
    assert raw.startswith(b"kind,method,variant,weighting,d,levels,S,L,P,gamma,q,seed,N,iterations")
    assert raw.count(b"\r\n") == 2
    harness.write_summary_json(tmp_path / "s.json", harness.ExperimentSpec(), [row])


# ------------------------------------------------------------ device solves
def _csv_rows(text):
    return list(csv.DictReader(io.StringIO(text)))


def _compare_rows(got_rows, want_csv):
    want = _csv_rows(want_csv)
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\r\n")
    w.writerow(harness.CSV_COLUMNS)
    for r in got_rows:
        w.writerow([r.get(c, "") for c in harness.CSV_COLUMNS])
    got = _csv_rows(buf.getvalue())
    assert len(got) == len(want)
    for g, r in zip(got, want):
        for c in harness.CSV_COLUMNS:
            if c == "iterations" and r[c] != "":
                assert abs(int(g[c]) - int(r[c])) <= 1, (c, g, r)
            elif c in ("lambda_min", "lambda_max") and r[c] != "":
                assert float(g[c]) == pytest.approx(float(r[c]), rel=1e-9), (c, g, r)
            else:
                assert g[c] == r[c], (c, g, r)
    return got


@pytest.fixture(scope="module")
def device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.gpu
def test_initial_iterate_matches_reference(device, golden):
    A = grid.symmetrize_diag(grid.assemble_laplacian((4, 4)), np.zeros(225))[0]
    from paper_2110_11211_b200 import krylov

    np.testing.assert_allclose(krylov.initial_iterate(225, 42, A), golden.json("harness.json")["initial_iterate_4x4"],
                               rtol=1e-14, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["weak_d2", "gamma_d1", "dim_sweep", "strong_d1", "weak_d2_richardson",
                                  "weak_d2_fcg_deflated", "weak_d3_additive", "weak_d2_s10", "weak_d3_s9"])
def test_sweeps_match_reference_rows(device, golden, name):
    g = golden.json("harness.json")[name]
    kw = {k: tuple(v) if isinstance(v, list) else v for k, v in g["spec"].items()}
    spec = harness.ExperimentSpec(**kw)
    runner = {"weak": harness.run_weak_scaling, "strong": harness.run_strong_scaling,
              "gamma_sweep": harness.run_gamma_sweep, "dim_sweep": harness.run_dim_sweep}[spec.kind]
    _compare_rows(runner(spec), g["csv"])


@pytest.mark.gpu
def test_sweep_csv_bytes_reproducible(device, tmp_path):
    spec = harness.ExperimentSpec(kind="weak", dim=2, s=6, p_values=(4, 16))
    for name in ("a.csv", "b.csv"):
        harness.write_rows_csv(tmp_path / name, harness.run_weak_scaling(spec))
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["combine_d2_l6", "combine_d3_l4", "combine_d2_l11"])
def test_combination_matches_reference(device, golden, name):
    g = golden.json("harness.json")[name]
    spec = harness.ExperimentSpec(**g["spec"])
    rows, summary = harness.run_combine_experiment(spec)
    _compare_rows(rows, g["csv"])
    want = g["summary"]
    assert summary["subproblems"] == want["subproblems"]
    assert summary["subdomains_total"] == want["subdomains_total"]
    assert summary["clamps"] == want["clamps"]
    assert summary["max_error"] == pytest.approx(want["max_error"], rel=1e-7)
    assert summary["rms_error"] == pytest.approx(want["rms_error"], rel=1e-7)
    plan = combine.enumerate_plan(spec.dim, spec.level, spec.p_hat)
    res = combine.run_combination(plan, seed=spec.seed)
    got = res.evaluator(np.asarray(g["points"]))
    np.testing.assert_allclose(got, g["values"], rtol=1e-8, atol=1e-12 * np.abs(g["values"]).max())


@pytest.mark.gpu
def test_combination_concurrent_streams_bitwise_equal_serial(device):
    plan = combine.enumerate_plan(2, 8, p_hat=4)
    serial = combine.run_combination(plan, seed=7, jobs=1)
    threaded = combine.run_combination(plan, seed=7, jobs=4)
    pts = np.random.default_rng(2).uniform(0.1, 0.9, size=(50, 2))
    np.testing.assert_array_equal(serial.evaluator(pts), threaded.evaluator(pts))


@pytest.mark.gpu
def test_combination_failures_name_level_vectors(device):
    with pytest.raises(combine.CombinationError) as err:
        combine.run_combination(combine.enumerate_plan(2, 4), seed=7, max_iters=0)
    assert "(1, 4)" in str(err.value) and "(4, 1)" in str(err.value)


def test_sweep_assignment_lpt_deterministic():
    from paper_2110_11211_b200 import sweep

    jobs = [sweep.SolveJob((l,), 4, 0.5, 2) for l in (3, 9, 5, 9, 7, 4, 8)]
    parts = sweep.assign(jobs, 3)
    assert sorted(i for p in parts for i in p) == list(range(len(jobs)))
    assert parts == sweep.assign(jobs, 3)
    loads = [sum(jobs[i].cost() for i in p) for p in parts]
    assert max(loads) <= min(loads) + max(j.cost() for j in jobs)
    assert sweep.assign(jobs, 1) == [list(range(len(jobs)))]


@pytest.mark.gpu
def test_sweep_processes_and_streams_bitwise_equal_serial(device):
    """Sweep batches spread over worker processes (one per listed device; here
    two processes on the one GPU of the box) and streams reproduce the serial
    results bit for bit."""
    from paper_2110_11211_b200 import sweep

    jobs = [sweep.SolveJob(lv, p, 0.5, 2) for lv, p in [((7,), 4), ((4, 4), 8), ((3, 3, 3), 8), ((5, 5), 16)]]
    serial = sweep.execute(jobs)
    spread = sweep.execute(jobs, devices=[0, 0], streams=2)
    for a, b in zip(serial, spread):
        assert a.error is None and b.error is None
        assert a.report.residual_history == b.report.residual_history
        assert a.report.energy_history == b.report.energy_history
        np.testing.assert_array_equal(a.report.solution, b.report.solution)
