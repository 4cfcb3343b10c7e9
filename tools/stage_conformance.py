"""Stage the reference's own test files for a conformance run of the B200
package (VERDICT r1 "next" 3).  Copies them from /root/reference
(this container only) into oracle/_ref/conformance/ -- git-ignored, so they
never enter the repo's history, but not gpurun-ignored, so a GPU box can run
them.  The staged tests import ``sfcdd``, which tests/conformance/sfcdd
aliases to paper_2110_11211_b200.

    python tools/stage_conformance.py && gpurun -- 'bash tools/run_conformance.sh'
"""
import shutil
from pathlib import Path

SRC = Path("/root/reference/pkg/tests")
ROOT = Path(__file__).resolve().parents[1]
DST = ROOT / "oracle" / "_ref" / "conformance"
FILES = ["test_sfc.py", "test_grid.py", "test_partition.py", "test_coarse.py", "test_schwarz.py",
         "test_krylov.py", "test_linalg.py", "test_acceptance.py"]

if __name__ == "__main__":
    DST.mkdir(parents=True, exist_ok=True)
    for f in FILES:
        shutil.copy2(SRC / f, DST / f)
    (DST / "conftest.py").write_text("")
    print(f"staged {len(FILES)} reference test files in {DST}")
