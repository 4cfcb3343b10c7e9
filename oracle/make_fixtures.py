"""Generate golden fixtures by running the REFERENCE itself (build container only).

    PYTHONPATH= python oracle/make_fixtures.py [--big]

Imports the read-only reference package from /root/reference/pkg/src under
the alias ``sfcdd_ref`` and writes small .npz/.json files
under tests/golden/.  Nothing here runs on the GPU box; the fixtures travel
with the repo.  ``--big`` adds the C2/C3 (and C4 perm hash) reference runs,
which take a few minutes.

Fixture contents (all produced by reference code paths, file:line relative
to /root/reference/pkg/src/sfcdd/):
  sfc_walks.npz      decode() of every key for small curves (sfc.py:139-147)
  sfc_keys.json      encode() of sample coordinates incl. 66-bit keys (sfc.py:120)
  perms.npz          sfc_permutation(levels) for small/anisotropic levels (grid.py:60)
  perm_hashes.json   sha256 of sfc_permutation for config-size levels
  partitions.json    disjoint/overlapped (start, length), omega, counts summary
                     (partition.py:64-157) and aggregate boundaries (coarse.py:44-58)
  coarse_c1.npz      A0 of config 1 (coarse.py:56-59)
  solve_*.npz        PCG residual histories / solutions (krylov.py:257-291)
  apply_c1.npz       SchwarzOperator.apply on seeded vectors (schwarz.py:103-118)
  solvers.npz        Richardson (optimal / fixed damping), Lanczos estimates, flexible
                     CG (full / windowed) and energy-error PCG (krylov.py:102-326)
"""

from __future__ import annotations

import argparse
import hashlib
import importlib.util
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "sfcdd_ref", "/root/reference/pkg/src/sfcdd/__init__.py",
        submodule_search_locations=["/root/reference/pkg/src/sfcdd"])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["sfcdd_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def perm_hash(perm: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(perm, dtype=np.int64).tobytes()).hexdigest()


SMALL_LEVELS = [(1, 1), (2, 2), (2, 3), (3, 2), (3, 3), (4, 4), (5, 5), (7, 7),
                (2, 2, 2), (2, 2, 3), (3, 3, 4), (4, 4, 4), (3, 2, 1, 2), (2, 2, 2, 2),
                (6,), (1, 4), (4, 1, 3)]
BIG_LEVELS = [(10, 10), (7, 7, 7)]
HUGE_LEVELS = [(12, 12)]

# (name, levels, P, gamma, q) -- SURVEY Appendix A mapping of BASELINE configs
CONFIGS = [
    ("c1_g025", (7, 7), 16, 0.25, 4),
    ("c1_g05", (7, 7), 16, 0.5, 4),
    ("c2", (10, 10), 64, 0.5, 16),
    ("c3", (7, 7, 7), 512, 0.5, 8),
    ("c4", (12, 12), 256, 0.5, 16),
    ("c5_g1", (8, 8, 8), 512, 0.5, 64),
    ("c5_g2", (8, 8, 9), 1024, 0.5, 64),
    ("c5_g4", (8, 9, 9), 2048, 0.5, 64),
    ("c5_g8", (9, 9, 9), 4096, 0.5, 64),
    ("small_aniso", (3, 4), 6, 0.5, 2),
    ("small_3d", (3, 3, 3), 8, 0.75, 3),
    ("frac_g03", (5, 5), 7, 0.3, 5),
    ("gamma_15", (4, 4), 8, 1.5, 2),
]


def make_sfc(ref):
    sfc = ref.sfc
    walks = {}
    for d, n in [(2, 1), (2, 2), (2, 3), (3, 2), (4, 2), (5, 2), (3, 3)]:
        cfg = sfc.CurveConfig(d, n)
        walks[f"d{d}_n{n}"] = np.array([sfc.decode(k, cfg) for k in range(1 << cfg.key_bits)],
                                       dtype=np.int64)
    np.savez_compressed(OUT / "sfc_walks.npz", **walks)
    rng = np.random.default_rng(11)
    samples = []
    for d, bits in [(2, 5), (3, 7), (4, 9), (6, 11), (2, 32), (3, 21), (5, 20), (8, 16), (2, 64)]:
        cfg = sfc.CurveConfig(d, bits)
        pts = [tuple([(1 << bits) - 1] * d), tuple([0] * d)]
        for _ in range(6):
            pts.append(tuple(int(v) for v in rng.integers(0, 1 << min(bits, 62), size=d)))
        for c in pts:
            samples.append({"dim": d, "bits": bits, "coords": list(c),
                            "key": str(sfc.encode(c, cfg))})
    grid_keys = []
    for levels in [(2, 3), (3, 3), (3, 4, 2), (1, 5)]:
        shape = [(1 << l) - 1 for l in levels]
        for flat in range(0, int(np.prod(shape)), 3):
            idx = np.unravel_index(flat, shape)
            k = tuple(int(i) + 1 for i in idx)
            grid_keys.append({"levels": list(levels), "index": list(k),
                              "key": str(sfc.grid_point_key(k, levels))})
    (OUT / "sfc_keys.json").write_text(json.dumps({"encode": samples, "grid_point_key": grid_keys}))


def make_perms(ref, big):
    perms = {}
    for lv in SMALL_LEVELS:
        perms["_".join(map(str, lv))] = ref.grid.sfc_permutation(lv)
    np.savez_compressed(OUT / "perms.npz", **perms)
    hashes = {}
    path = OUT / "perm_hashes.json"
    if path.exists():
        hashes = json.loads(path.read_text())
    for lv in SMALL_LEVELS:
        hashes["_".join(map(str, lv))] = perm_hash(perms["_".join(map(str, lv))])
    if big:
        for lv in BIG_LEVELS + HUGE_LEVELS:
            key = "_".join(map(str, lv))
            if key in hashes:
                continue
            t0 = time.time()
            p = ref.grid.sfc_permutation(lv)
            hashes[key] = perm_hash(p)
            print(f"perm {lv}: {time.time() - t0:.1f}s", flush=True)
            ref.grid.sfc_permutation.cache_clear()
    path.write_text(json.dumps(hashes, indent=1))


def make_partitions(ref):
    pt = ref.partition
    out = {}
    for name, levels, p, gamma, q in CONFIGS:
        n = ref.grid.num_dofs(levels)
        part = pt.build_partition(n, p, gamma)
        entry = {
            "levels": list(levels), "n": n, "p": p, "gamma": gamma, "q": q,
            "disjoint": [[r.start, r.length] for r in part.disjoint],
            "overlapped": [[r.start, r.length] for r in part.overlapped],
        }
        if n <= 3_000_000:
            w = pt.compute_weights(part)
            entry["omega"] = [float(v) for v in w.omega]
            entry["counts_min"] = int(w.counts.min())
            entry["counts_max"] = int(w.counts.max())
            entry["counts_hash"] = hashlib.sha256(w.counts.astype(np.int64).tobytes()).hexdigest()
            bounds = [0]
            for r in part.disjoint:
                for s in ref.coarse.aggregate_sizes(r.length, q):
                    bounds.append(bounds[-1] + s)
            entry["aggregate_bounds_hash"] = hashlib.sha256(
                np.asarray(bounds, np.int64).tobytes()).hexdigest()
        out[name] = entry
    (OUT / "partitions.json").write_text(json.dumps(out))


def reference_setup(ref, levels, p, gamma, q, seed=42):
    """SURVEY §8(d) composition (mirrors combine.py:178-189 with a random RHS)."""
    A = ref.grid.assemble_laplacian(levels)
    n = A.shape[0]
    b = np.random.default_rng(seed).uniform(-1.0, 1.0, size=n)
    Ah, bh, t = ref.grid.symmetrize_diag(A, b)
    part = ref.partition.build_partition(n, p, gamma)
    cs = ref.coarse.build_coarse(part, Ah, q)
    op = ref.schwarz.setup(Ah, part, cs, ref.schwarz.SchwarzConfig("balanced", "omega", gamma, q))
    return Ah, bh, t, part, cs, op


def install_fault(op, apply_index, dead):
    """SURVEY §8(d) fault semantics by instance monkeypatching (no reference edits)."""
    state = {"calls": 0}
    orig_local = op._local_solve
    orig_apply = op.apply
    dead = set(int(i) for i in dead)

    def local(i, g):
        piece = orig_local(i, g)
        if state["calls"] == apply_index and i in dead:
            return np.zeros_like(piece)
        return piece

    def apply(g):
        out = orig_apply(g)
        state["calls"] += 1
        return out

    op._local_solve = local
    op.apply = apply


def make_solve(ref, name, levels, p, gamma, q, full_solution, fault_iter=None):
    t0 = time.time()
    Ah, bh, t, part, cs, op = reference_setup(ref, levels, p, gamma, q)
    if fault_iter is not None:
        dead = np.random.default_rng(42).choice(p, size=int(round(0.1 * p)), replace=False)
        install_fault(op, fault_iter, dead)
    cfg = ref.krylov.SolverConfig(method="pcg", tolerance=1e-8, tolerance_kind="relative_residual")
    rep = ref.krylov.run(Ah, bh, op, cfg, np.zeros(Ah.shape[0]))
    sol = rep.solution
    data = {
        "levels": np.asarray(levels), "p": p, "gamma": gamma, "q": q,
        "iterations": rep.iterations, "converged": rep.converged,
        "residual_history": np.asarray(rep.residual_history),
        "solution_norm": np.linalg.norm(sol),
        "solution_sample_idx": np.arange(0, sol.size, max(1, sol.size // 4096)),
    }
    data["solution_sample"] = sol[data["solution_sample_idx"]]
    if full_solution:
        data["solution"] = sol
    if name.startswith("c1"):
        data["coarse_matrix"] = cs.matrix.toarray()
        rng = np.random.default_rng(5)
        vs = rng.standard_normal((3, Ah.shape[0]))
        data["apply_inputs"] = vs
        data["apply_outputs"] = np.stack([op.apply(v) for v in vs])
    np.savez_compressed(OUT / f"solve_{name}.npz", **data)
    print(f"solve {name}: {rep.iterations} its, {time.time() - t0:.1f}s", flush=True)


def make_solvers(ref):
    """the reference's Richardson (optimal damping via
    Lanczos, krylov.py:102-168, 219-254), flexible CG (krylov.py:294-326) and
    the energy-error tracker (krylov.py:171-213) on small balanced / deflated
    operators.  x* = the exact discrete solution (scipy spsolve of Â x = b̂)."""
    import scipy.sparse.linalg as spla

    K = ref.krylov
    out = {}

    def store(tag, rep, extra=None):
        out[f"{tag}_iterations"] = rep.iterations
        out[f"{tag}_converged"] = rep.converged
        out[f"{tag}_residual_history"] = np.asarray(rep.residual_history)
        out[f"{tag}_energy_history"] = np.asarray(rep.energy_history)
        out[f"{tag}_solution"] = rep.solution
        for k in ("lambda_min", "lambda_max", "damping"):
            v = getattr(rep, k)
            out[f"{tag}_{k}"] = np.nan if v is None else v
        for k, v in (extra or {}).items():
            out[f"{tag}_{k}"] = v

    for tag, levels, p, gamma, q, variant in [("b66", (6, 6), 8, 0.5, 4, "balanced"),
                                              ("b44", (4, 4), 4, 0.5, 2, "balanced"),
                                              ("d55", (5, 5), 6, 0.5, 2, "deflated")]:
        A = ref.grid.assemble_laplacian(levels)
        n = A.shape[0]
        b = np.random.default_rng(42).uniform(-1.0, 1.0, size=n)
        Ah, bh, t = ref.grid.symmetrize_diag(A, b)
        part = ref.partition.build_partition(n, p, gamma)
        cs = ref.coarse.build_coarse(part, Ah, q)
        op = ref.schwarz.setup(Ah, part, cs, ref.schwarz.SchwarzConfig(variant, "omega", gamma, q))
        exact = spla.spsolve(Ah.tocsc(), bh)
        out[f"{tag}_exact"] = exact
        x0 = np.zeros(n)
        if variant == "balanced":
            store(f"{tag}_pcg_energy", K.run(Ah, bh, op, K.SolverConfig(method="pcg", tolerance=1e-8), x0, exact))
            store(f"{tag}_pcg_rel", K.run(Ah, bh, op, K.SolverConfig(
                method="pcg", tolerance=1e-8, tolerance_kind="relative_residual"), x0, exact))
            store(f"{tag}_rich_opt", K.run(Ah, bh, op, K.SolverConfig(
                method="richardson", tolerance=1e-6, tolerance_kind="relative_residual"), x0, exact))
            store(f"{tag}_rich_fixed", K.run(Ah, bh, op, K.SolverConfig(
                method="richardson", damping=0.5, tolerance=1e-6), x0, exact))
            lam = K.estimate_extremal_eigs(lambda v: op.apply(Ah @ v), n, seed=42, a_matvec=lambda v: Ah @ v,
                                           force_iterative=True)
            out[f"{tag}_lanczos_forced"] = np.asarray(lam)
        store(f"{tag}_fcg", K.run(Ah, bh, op, K.SolverConfig(method="fcg", tolerance=1e-8,
                                                            tolerance_kind="relative_residual"), x0, exact))
        store(f"{tag}_fcg_w2", K.run(Ah, bh, op, K.SolverConfig(method="fcg", tolerance=1e-8, fcg_window=2),
                                     x0, exact))
        print(f"solvers {tag}: n={n}", flush=True)
    np.savez_compressed(OUT / "solvers.npz", **out)


def make_dense_operator(ref):
    """Small operator matrices via apply() (cf. test_schwarz.py:14-22)."""
    out = {}
    for levels, p, gamma, q in [((4, 4), 4, 0.5, 2), ((3, 3, 3), 8, 0.5, 2), ((4, 4), 5, 0.25, 3)]:
        Ah, bh, t, part, cs, op = reference_setup(ref, levels, p, gamma, q)
        n = Ah.shape[0]
        M = np.empty((n, n))
        e = np.zeros(n)
        for j in range(n):
            e[j] = 1.0
            M[:, j] = op.apply(e)
            e[j] = 0.0
        out["_".join(map(str, levels)) + f"_p{p}_g{gamma}_q{q}"] = M
    np.savez_compressed(OUT / "dense_operators.npz", **out)


# harness / combination-technique runs of the reference
HARNESS_SPECS = {
    "weak_d2": dict(kind="weak", dim=2, s=6, p_values=(1, 2, 4, 8, 16, 32, 64)),
    "gamma_d1": dict(kind="gamma_sweep", dim=1, s=6, gamma_values=(0.25, 0.5, 1.0, 2.0), p_values=(2, 4, 8, 16)),
    "dim_sweep": dict(kind="dim_sweep", dims=(1, 2, 3), s=6, p_values=(4, 8, 16)),
    "strong_d1": dict(kind="strong", dim=1, level=10, p_values=(2, 4, 8, 16, 32)),
    "weak_d2_richardson": dict(kind="weak", dim=2, s=5, p_values=(4, 16), method="richardson"),
    "weak_d2_fcg_deflated": dict(kind="weak", dim=2, s=5, p_values=(4, 16), method="fcg", variant="deflated"),
    "weak_d3_additive": dict(kind="weak", dim=3, s=6, p_values=(8, 64), variant="additive_two_level"),
    "weak_d2_s10": dict(kind="weak", dim=2, s=10, p_values=(4, 16, 64, 256)),
    "weak_d3_s9": dict(kind="weak", dim=3, s=9, p_values=(8, 64)),
}
COMBINE_SPECS = {
    "combine_d2_l6": dict(kind="combine", dim=2, level=6, p_hat=2, sample_count=500),
    "combine_d3_l4": dict(kind="combine", dim=3, level=4, p_hat=1, sample_count=500),
    "combine_d2_l11": dict(kind="combine", dim=2, level=11, p_hat=8, sample_count=2000),
}


def make_harness(ref):
    """Rows (CSV text without timings) of small sweeps and combination runs."""
    import io
    import tempfile

    out = {}
    for name, kw in HARNESS_SPECS.items():
        t0 = time.time()
        spec = ref.harness.ExperimentSpec(**kw)
        runner = {"weak": ref.harness.run_weak_scaling, "strong": ref.harness.run_strong_scaling,
                  "gamma_sweep": ref.harness.run_gamma_sweep, "dim_sweep": ref.harness.run_dim_sweep}[spec.kind]
        rows = runner(spec)
        with tempfile.TemporaryDirectory() as td:
            ref.harness.write_rows_csv(Path(td) / "rows.csv", rows)
            csv_text = (Path(td) / "rows.csv").read_text(encoding="utf-8")
        out[name] = {"spec": {k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()}, "csv": csv_text}
        print(f"harness {name}: {len(rows)} rows, {time.time() - t0:.1f}s", flush=True)
    for name, kw in COMBINE_SPECS.items():
        t0 = time.time()
        spec = ref.harness.ExperimentSpec(**kw)
        rows, summary = ref.harness.run_combine_experiment(spec)
        with tempfile.TemporaryDirectory() as td:
            ref.harness.write_rows_csv(Path(td) / "rows.csv", rows)
            csv_text = (Path(td) / "rows.csv").read_text(encoding="utf-8")
        plan = ref.combine.enumerate_plan(spec.dim, spec.level, spec.p_hat)
        res = ref.combine.run_combination(plan, seed=spec.seed)
        pts = np.random.default_rng(11).uniform(0.0, 1.0, size=(64, spec.dim))
        out[name] = {"spec": kw, "csv": csv_text, "summary": summary,
                     "points": pts.tolist(), "values": res.evaluator(pts).tolist()}
        print(f"combine {name}: {len(rows)} rows, err {summary['max_error']:.3e}, {time.time() - t0:.1f}s", flush=True)
    mp = {}
    for d in (1, 2, 3):
        prob = ref.grid.manufactured_poisson((3,) * d)
        pts = np.random.default_rng(20 + d).uniform(0.01, 0.99, size=(20, d))
        mp[str(d)] = {"points": pts.tolist(), "rhs": prob.rhs(pts).tolist(),
                      "exact": prob.exact_solution(pts).tolist()}
    out["manufactured"] = mp
    x0 = ref.krylov.initial_iterate(225, 42, ref.grid.symmetrize_diag(
        ref.grid.assemble_laplacian((4, 4)), np.zeros(225))[0])
    out["initial_iterate_4x4"] = x0.tolist()
    (OUT / "harness.json").write_text(json.dumps(out, indent=1) + "\n")


# extra solve fixtures: name -> (levels, p, gamma, q, full_solution)
SOLVES = {
    # aggregates of 16320 points = 8 reduction chunks each (the R0 r partials
    # are per chunk, not per aggregate: pins the fused PCG epilogue's sums)
    "multichunk": ((9, 9), 8, 0.5, 2, False),
    # BASELINE configs[3] at full size on one device: 4095^2, P=256, q=16,
    # fault mode at apply 5; ~25 min and ~50 GB on the CPU
    "c4_fault": ((12, 12), 256, 0.5, 16, False, 5),
    # C5-shaped reduced grid (BASELINE configs[4]): 3-D, gamma = 1/2, q = 64 and
    # C5's subdomain size (31k disjoint / 62.5k overlapped points), P = 8
    # instead of 512 so the reference's SuperLU setup fits this container
    "c5shape": ((6, 6, 6), 8, 0.5, 64, True),
}

# perm hashes of the C5 weak-scaling levels (BASELINE configs[4] at G = 1, 2,
# 4, 8), from the reference's own sfc_permutation (minutes to ~1 h each)
C5_LEVELS = [(8, 8, 8), (8, 8, 9), (8, 9, 9), (9, 9, 9)]


def make_c5_perm_hashes(ref):
    path = OUT / "perm_hashes.json"
    for lv in C5_LEVELS:
        hashes = json.loads(path.read_text()) if path.exists() else {}
        key = "_".join(map(str, lv))
        if key in hashes:
            continue
        t0 = time.time()
        p = ref.grid.sfc_permutation(lv)
        h = perm_hash(p)
        del p
        ref.grid.sfc_permutation.cache_clear()
        hashes = json.loads(path.read_text()) if path.exists() else {}
        hashes[key] = h
        path.write_text(json.dumps(hashes, indent=1))
        print(f"perm {lv}: {time.time() - t0:.1f}s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default=None, help="regenerate one solve fixture (name of SOLVES)")
    args = ap.parse_args()
    OUT.mkdir(parents=True, exist_ok=True)
    ref = load_reference()
    if args.only == "harness":
        make_harness(ref)
        return
    if args.only == "c5_perms":
        make_c5_perm_hashes(ref)
        return
    if args.only:
        make_solve(ref, args.only, *SOLVES[args.only])
        return
    make_sfc(ref)
    make_perms(ref, args.big)
    make_partitions(ref)
    make_dense_operator(ref)
    make_solvers(ref)
    make_solve(ref, "c1_g05", (7, 7), 16, 0.5, 4, True)
    make_solve(ref, "c1_g025", (7, 7), 16, 0.25, 4, True)
    make_solve(ref, "small_3d", (4, 4, 4), 8, 0.5, 4, True)
    make_solve(ref, "aniso", (6, 7), 12, 0.5, 3, True)
    make_solve(ref, "fault_88", (8, 8), 256, 0.5, 16, False, fault_iter=5)
    make_solve(ref, "nofault_88", (8, 8), 256, 0.5, 16, False)
    make_solve(ref, "multichunk", *SOLVES["multichunk"])
    make_harness(ref)
    if args.big:
        make_solve(ref, "c2", (10, 10), 64, 0.5, 16, False)
        make_solve(ref, "c3", (7, 7, 7), 512, 0.5, 8, False)


if __name__ == "__main__":
    main()
