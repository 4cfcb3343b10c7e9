#!/bin/bash
# Run the reference's own tests (staged by tools/stage_conformance.py) against
# the B200 package through the `sfcdd` alias; GPU box only.
#   bash tools/run_conformance.sh [outdir]
OUT=${1:-gpurun_out/conformance}; mkdir -p $OUT
D=oracle/_ref/conformance
if [ ! -d $D ]; then echo "no staged tests ($D): run tools/stage_conformance.py first" | tee $OUT/summary.txt; exit 0; fi
export PYTHONPATH=$PWD/tests/conformance:$PWD:$PYTHONPATH
# SURVEY §4 conformance set: everything except the combination/harness drivers;
# acceptance criteria 1/2/3/4/6a/8 (5, 6b, 7, 9, 10 are sweeps of the drivers)
timeout 2400 python -m pytest -q -p no:cacheprovider --rootdir $D $D/test_sfc.py $D/test_grid.py $D/test_partition.py \
  $D/test_coarse.py $D/test_schwarz.py $D/test_linalg.py "$D/test_krylov.py" \
  "$D/test_acceptance.py::test_criterion_1_uniform_weights_for_half_integer_gamma" \
  "$D/test_acceptance.py::test_criterion_2_partition_balance_and_tiling" \
  "$D/test_acceptance.py::test_criterion_3_sfc_bijectivity_adjacency_holder" \
  "$D/test_acceptance.py::test_criterion_4_operator_dense_oracle_equivalence" \
  "$D/test_acceptance.py::test_criterion_6a_weak_scaling_iteration_counts_d1" \
  "$D/test_acceptance.py::test_criterion_8_weighting_coincidence" \
  -rfE > $OUT/pytest.log 2>&1
echo "exit $?" >> $OUT/pytest.log
tail -40 $OUT/pytest.log > $OUT/summary.txt
