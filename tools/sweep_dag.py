"""Time the local-solve DAG kernel for several plan/launch settings.

    python tools/sweep_dag.py c2 "WPB=4,BLOB=12288,SCR=768" "WPB=8,BLOB=8192,SCR=512" ...

Each setting is applied through the environment (SFCDD_WPB, SFCDD_BLOB_MAX,
SFCDD_SCRATCH_MAX) before the operator is set up; prints one JSON line each.
"""
import ctypes
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2110_11211_b200 as sf  # noqa: E402
from paper_2110_11211_b200 import _lib  # noqa: E402

CFG = {"c1": ((7, 7), 16, 0.5, 4), "c2": ((10, 10), 64, 0.5, 16), "c3": ((7, 7, 7), 512, 0.5, 8),
       "c4": ((12, 12), 256, 0.5, 16), "c5": ((8, 8, 8), 512, 0.5, 64)}
KEYS = {"WPB": "SFCDD_WPB", "BLOB": "SFCDD_BLOB_MAX", "SCR": "SFCDD_SCRATCH_MAX", "MODE": "SFCDD_DAG_MODE", "Q": "SFCDD_QUEUES", "W": "SFCDD_WORKERS", "ROW": "SFCDD_ROW_MAX", "COL": "SFCDD_COL_MAX", "ORD": "SFCDD_ORDER", "LEAF": "SFCDD_ND_LEAF", "SIG": "SFCDD_SIG_NS", "CTAS": "SFCDD_CTAS_PER_SM", "RS": "SFCDD_RELAX_SMALL", "RSF": "SFCDD_RELAX_SMALL_FRAC", "RF": "SFCDD_RELAX_FRAC", "SLACK": "SFCDD_SLACK_US", "AR": "SFCDD_ASM_RED", "XM": "SFCDD_XB_MIN", "PF": "SFCDD_PF_DIST", "SLOT": "SFCDD_SLOT_MAX", "DR": "SFCDD_DIRECT_ROWS", "DC": "SFCDD_DIRECT_COLS", "SPLIT": "SFCDD_SPLIT_MIN"}
name = sys.argv[1]
levels, p, gamma, q = CFG[name]
A = sf.assemble_laplacian(levels)
n = A.shape[0]
Ah, _, _ = sf.symmetrize_diag(A, np.zeros(n))
part = sf.build_partition(n, p, gamma)
coarse = sf.build_coarse(part, Ah, q)
g = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
scratch = torch.empty(n, dtype=torch.float64, device="cuda")
for spec in sys.argv[2:]:
    for v in KEYS.values():
        os.environ.pop(v, None)
    for kv in spec.split(","):
        k, v = kv.split("=")
        os.environ[KEYS[k]] = v
    try:
        op = sf.setup(Ah, part, coarse, sf.SchwarzConfig("balanced", "omega", gamma, q))
        ms = (ctypes.c_double * 3)()
        launches = (ctypes.c_int32 * 3)()
        _lib.check(_lib.lib().sfcdd_op_profile(op.handle, g.data_ptr(), scratch.data_ptr(), 20, ms, launches,
                                               None))
        st = op.stats()
        print(json.dumps({"cfg": name, "spec": spec, "dag_ms": ms[0], "apply_ms": ms[1],
                          "tasks": st.get("num_tasks"), "device_bytes": st.get("device_bytes")}), flush=True)
        del op
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"cfg": name, "spec": spec, "error": str(e)}), flush=True)
