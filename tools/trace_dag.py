"""Trace one local-solve DAG launch (per-task timestamps) -> gpurun_out/trace_<cfg>.npz"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2110_11211_b200 as sf  # noqa: E402
from paper_2110_11211_b200 import _lib  # noqa: E402

CFG = {"c1": ((7, 7), 16, 0.5, 4), "c2": ((10, 10), 64, 0.5, 16), "c3": ((7, 7, 7), 512, 0.5, 8),
       "c4": ((12, 12), 256, 0.5, 16), "c5": ((8, 8, 8), 512, 0.5, 64)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
levels, p, gamma, q = CFG[name]
A = sf.assemble_laplacian(levels)
n = A.shape[0]
Ah, _, _ = sf.symmetrize_diag(A, np.zeros(n))
part = sf.build_partition(n, p, gamma)
op = sf.setup(Ah, part, sf.build_coarse(part, Ah, q), sf.SchwarzConfig("balanced", "omega", gamma, q))
g = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
nt = ctypes.c_int64()
_lib.check(_lib.lib().sfcdd_op_trace(op.handle, g.data_ptr(), None, ctypes.byref(nt)))
out = np.zeros(24 * nt.value, dtype=np.uint64)
_lib.check(_lib.lib().sfcdd_op_trace(op.handle, g.data_ptr(), out.ctypes.data, ctypes.byref(nt)))
(ROOT / "gpurun_out").mkdir(exist_ok=True)
tag = sys.argv[2] if len(sys.argv) > 2 else ""
np.savez_compressed(ROOT / "gpurun_out" / f"trace_{name}{tag}.npz", trace=out.reshape(-1, 24), stats=str(op.stats()))
print("traced", nt.value, "tasks")
