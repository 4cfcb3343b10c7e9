"""Sum over subdomains of nnz(L) of the reference's SuperLU factors
(linalg.py:55-61: splu, MMD on A^T+A, SymmetricMode) per BASELINE config: the
nnz_alg cap of the roofline's algorithmic bytes (extra fill of
the builder is never credited).  CPU; writes profiles/superlu_nnz.json.

    python tools/superlu_nnz.py c2 c3 c4 [c5:<samples>]
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import scipy.sparse.linalg as spla

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT))
CFG = {"c1": ((7, 7), 16, 0.5), "c2": ((10, 10), 64, 0.5), "c3": ((7, 7, 7), 512, 0.5),
       "c4": ((12, 12), 256, 0.5), "c5": ((8, 8, 8), 512, 0.5)}
OUT = ROOT / "profiles" / "superlu_nnz.json"


def main():
    import sfc_index_c as C

    res = json.loads(OUT.read_text()) if OUT.exists() else {}
    for arg in sys.argv[1:]:
        name, _, samp = arg.partition(":")
        levels, p, gamma = CFG[name]
        n = int(np.prod([(1 << l) - 1 for l in levels]))
        perm = C.sfc_perm(levels)
        rank = np.empty(n, np.int64)
        rank[perm] = np.arange(n)
        from fractions import Fraction

        g = Fraction(gamma).limit_denominator(10**6)
        _, _, os_, ol = C.partition(n, p, g.numerator, g.denominator)
        idx = range(p) if not samp else np.linspace(0, p - 1, int(samp)).astype(int)
        t0 = time.time()
        tot, cnt = 0, 0
        for i in idx:
            B = C.scaled_block(levels, perm, rank, int(os_[i]), int(ol[i]))
            lu = spla.splu(B.tocsc(), permc_spec="MMD_AT_PLUS_A", options={"SymmetricMode": True})
            tot += int(lu.L.nnz)
            cnt += 1
        entry = {"levels": list(levels), "P": p, "gamma": gamma, "subdomains": cnt,
                 "sum_nnz_L": tot if cnt == p else None, "mean_nnz_L": tot / cnt,
                 "seconds": round(time.time() - t0, 1),
                 "note": "exact sum over all subdomains" if cnt == p else f"mean over {cnt} sampled subdomains"}
        res[name] = entry
        OUT.write_text(json.dumps(res, indent=1))
        print(name, entry, flush=True)


if __name__ == "__main__":
    main()
