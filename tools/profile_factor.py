"""Set up one operator (default C3) so ncu can capture the device numeric
factorization kernels (k_front_*): python tools/profile_factor.py c3"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2110_11211_b200 as sf  # noqa: E402

CFG = {"c3": ((7, 7, 7), 512, 0.5, 8), "c5p": ((7, 7, 7), 64, 0.5, 64), "c2": ((10, 10), 64, 0.5, 16)}
levels, p, gamma, q = CFG[sys.argv[1] if len(sys.argv) > 1 else "c3"]
A = sf.assemble_laplacian(levels)
n = A.shape[0]
Ah, _, _ = sf.symmetrize_diag(A, np.zeros(n))
part = sf.build_partition(n, p, gamma)
op = sf.setup(Ah, part, sf.build_coarse(part, Ah, q), sf.SchwarzConfig("balanced", "omega", gamma, q))
print(op.stats())
