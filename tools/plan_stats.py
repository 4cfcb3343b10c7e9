"""CPU-only: build the local-solve plan for a config and print its statistics
(SFCDD_PLAN_DEBUG).  python tools/plan_stats.py c2"""
import sys
from pathlib import Path
import os
import time
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle")); sys.path.insert(0, str(ROOT / "tests"))
os.environ.setdefault("SFCDD_PLAN_DEBUG", "1")
import sfcdd_oracle as oracle  # noqa: E402
from test_host_logic import host_plan_solve  # noqa: E402
CFG = {"c1": ((7, 7), 16, 0.5), "c2": ((10, 10), 64, 0.5), "c3": ((7, 7, 7), 512, 0.5),
       "c4p": ((11, 11), 32, 0.5),
       "c5p": ((7, 7, 7), 64, 0.5)}  # c5p: C5-sized subdomains (32k disjoint points) on 127^3  # c4p: C4-sized subdomains (131k overlapped points) on a smaller grid
levels, p, gamma = CFG[sys.argv[1] if len(sys.argv) > 1 else "c2"]
A = oracle.assemble_scaled_laplacian(levels)
ov = oracle.enlarge(oracle.disjoint_partition(A.shape[0], p), gamma)
t = time.time()
xy, nf = host_plan_solve(A, ov, np.ones(A.shape[0]))
print("groups", nf, "time", time.time() - t)
