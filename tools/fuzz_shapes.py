"""GPU robustness sweep of the plan builder: set up operators of many shapes
with the DEFAULT plan options and run PCG to 1e-8; every shape must build,
converge, and solve A x = b (true residual checked with the device matvec).

    python tools/fuzz_shapes.py            # prints one line per shape, exits 1 on any failure
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2110_11211_b200 as sf  # noqa: E402

SHAPES = [
    ((12,), 8, 0.5, 4), ((9, 9), 4, 0.5, 8), ((9, 9), 2, 0.5, 16), ((10, 10), 16, 0.25, 8), ((10, 10), 16, 1.0, 8),
    ((8, 10), 12, 0.5, 4), ((11, 11), 64, 0.5, 16), ((11, 11), 1024, 0.5, 4), ((6, 6, 6), 64, 0.5, 8),
    ((6, 6, 6), 4, 0.5, 16), ((6, 6, 6), 2, 0.5, 8), ((7, 6, 5), 16, 0.75, 8), ((7, 7, 7), 64, 0.5, 64),
    ((7, 7, 7), 1024, 0.5, 8), ((5, 5, 5, 5), 16, 0.5, 4),
]
bad = 0
for levels, p, gamma, q in SHAPES:
    t0 = time.time()
    try:
        A = sf.assemble_laplacian(levels)
        n = A.shape[0]
        b = np.random.default_rng(7).uniform(-1.0, 1.0, size=n)
        Ah, bh, _ = sf.symmetrize_diag(A, b)
        part = sf.build_partition(n, p, gamma)
        op = sf.setup(Ah, part, sf.build_coarse(part, Ah, q), sf.SchwarzConfig("balanced", "omega", gamma, q))
        rep = sf.run(Ah, bh, op, sf.SolverConfig(method="pcg", tolerance=1e-8, tolerance_kind="relative_residual",
                                                 max_iters=400), np.zeros(n))
        res = np.linalg.norm(bh - Ah @ rep.solution) / np.linalg.norm(bh)
        ok = rep.converged and res <= 5e-8
        st = op.stats()
        print(f"{'ok ' if ok else 'BAD'} levels={levels} P={p} gamma={gamma} q={q}: N={n} its={rep.iterations} "
              f"true_res={res:.2e} tasks={st.get('num_tasks')} setup={st.get('setup_seconds'):.1f}s "
              f"wall={time.time() - t0:.1f}s", flush=True)
        bad += 0 if ok else 1
        del op
    except Exception as e:  # noqa: BLE001
        print(f"BAD levels={levels} P={p} gamma={gamma} q={q}: {type(e).__name__}: {e}", flush=True)
        bad += 1
sys.exit(1 if bad else 0)
