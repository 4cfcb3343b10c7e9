"""``sfcdd`` alias of the B200 package, so the reference's own test files
(`from sfcdd import grid`, `from sfcdd.schwarz import setup`, ...) run
unchanged against it (SURVEY §4 conformance suite).  Used only by
tools/run_conformance.sh; the reference's test files are staged next to this
package at run time (tools/stage_conformance.py) and never committed."""

import sys

import paper_2110_11211_b200 as _pkg
from paper_2110_11211_b200 import *  # noqa: F401,F403
from paper_2110_11211_b200 import __all__, __version__  # noqa: F401

for _name in ("coarse", "combine", "grid", "harness", "krylov", "linalg", "partition", "schwarz", "sfc"):
    sys.modules[f"{__name__}.{_name}"] = getattr(_pkg, _name)
    globals()[_name] = getattr(_pkg, _name)
