"""Small driver for ncu: set up a config and run a few preconditioner applies.

    python tools/profile_apply.py [c2|c3] [reps]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2110_11211_b200 as sf  # noqa: E402

CFG = {"c1": ((7, 7), 16, 0.5, 4), "c2": ((10, 10), 64, 0.5, 16), "c3": ((7, 7, 7), 512, 0.5, 8),
       "c4": ((12, 12), 256, 0.5, 16), "c5": ((8, 8, 8), 512, 0.5, 64)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
levels, p, gamma, q = CFG[name]
A = sf.assemble_laplacian(levels)
n = A.shape[0]
Ah, _, _ = sf.symmetrize_diag(A, np.zeros(n))
part = sf.build_partition(n, p, gamma)
op = sf.setup(Ah, part, sf.build_coarse(part, Ah, q), sf.SchwarzConfig("balanced", "omega", gamma, q))
g = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
for _ in range(reps):
    h = op.apply_device(g)
torch.cuda.synchronize()
print("ok", name, float(h.norm()))
