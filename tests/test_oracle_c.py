"""The C restatement oracle/sfc_index.c (checker of the index sets at
BASELINE configs[4] sizes) pinned to the reference's own
outputs: permutation hashes and small permutations, partitions of every
BASELINE config (C5 at G = 1, 2, 4, 8 included), weights and aggregate
bounds; and the library's partition (csrc/partition.cpp) against both.
CPU only."""

import hashlib
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import sfc_index_c as C  # noqa: E402

from paper_2110_11211_b200 import partition as pt  # noqa: E402


def _h(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def test_small_perms_match_reference(golden):
    perms = golden.npz("perms.npz")
    for key in perms.files:
        lv = tuple(int(v) for v in key.split("_"))
        if len(lv) * max(lv) > 64:
            continue
        np.testing.assert_array_equal(C.sfc_perm(lv), perms[key], err_msg=key)


@pytest.mark.parametrize("key", ["10_10", "7_7_7", "12_12", "8_8_8", "8_8_9", "8_9_9", "9_9_9"])
def test_config_perm_hashes_match_reference(golden, key):
    hashes = golden.json("perm_hashes.json")
    if key not in hashes:
        pytest.skip(f"no reference hash for {key} (oracle/make_fixtures.py --only c5_perms)")
    lv = tuple(int(v) for v in key.split("_"))
    assert _h(C.sfc_perm(lv)) == hashes[key]


def test_keys_match_python_oracle(oracle):
    rng = np.random.default_rng(0)
    for d, bits in [(2, 7), (3, 8), (3, 9), (4, 6), (2, 31), (5, 12)]:
        x = rng.integers(0, 1 << bits, size=(2000, d), dtype=np.uint64)
        hi, lo = oracle.hilbert_keys(x, bits)
        assert np.all(hi == 0)
        np.testing.assert_array_equal(C.hilbert_keys(x, bits), lo)


def test_partitions_match_reference_fixtures(golden):
    for name, e in golden.json("partitions.json").items():
        n, p, gamma, q = e["n"], e["p"], e["gamma"], e["q"]
        num, den = pt.gamma_fraction(gamma)
        ds, dl, os_, ol = C.partition(n, p, num, den)
        assert [[int(a), int(b)] for a, b in zip(ds, dl)] == e["disjoint"], name
        assert [[int(a), int(b)] for a, b in zip(os_, ol)] == e["overlapped"], name
        # the library's own partition (what the device operator uses)
        part = pt.build_partition(n, p, gamma)
        assert [[r.start, r.length] for r in part.overlapped] == e["overlapped"], name
        if "omega" in e:
            om, cn = C.weights(n, os_, ol, counts=True)
            assert om.tolist() == e["omega"], name
            assert _h(cn) == e["counts_hash"], name
            assert _h(C.aggregates(ds, dl, q)) == e["aggregate_bounds_hash"], name
