"""Small driver for ncu: set up a config and run one short device PCG solve.

    python tools/profile_pcg.py [c2|c3] [max_iters]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2110_11211_b200 as sf  # noqa: E402
from paper_2110_11211_b200.krylov import pcg_device  # noqa: E402

CFG = {"c1": ((7, 7), 16, 0.5, 4), "c2": ((10, 10), 64, 0.5, 16), "c3": ((7, 7, 7), 512, 0.5, 8),
       "c4": ((12, 12), 256, 0.5, 16)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 4
levels, p, gamma, q = CFG[name]
A = sf.assemble_laplacian(levels)
n = A.shape[0]
b = np.random.default_rng(42).uniform(-1.0, 1.0, size=n)
Ah, bh, _ = sf.symmetrize_diag(A, b)
part = sf.build_partition(n, p, gamma)
op = sf.setup(Ah, part, sf.build_coarse(part, Ah, q), sf.SchwarzConfig("balanced", "omega", gamma, q))
x, k, conv, hist = pcg_device(op, torch.from_numpy(bh), None, 1e-8, its)
torch.cuda.synchronize()
print("ok", name, k, hist[-1])
