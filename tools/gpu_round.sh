#!/bin/bash
# One GPU-box session: GPU parity tests, bench lines, launch list and one ncu --set full capture.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh <tag> [what...]'
# Outputs under gpurun_out/<tag>/.
set -u
TAG=${1:-r01}; shift || true
WHAT=${*:-"tests bench ref ncu"}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
for w in $WHAT; do
  case $w in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log ;;
    bench) timeout 600 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err ;;
    c3) timeout 900 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err ;;
    c4) timeout 1500 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err ;;
    c5) timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err ;;
    ncu5)
      timeout 600 python tools/profile_apply.py c5 3 > $OUT/plain_c5.log 2>&1 &&
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_dag -s 3 -c 1 \
          -o $OUT/dag_c5 python tools/profile_apply.py c5 3 > $OUT/ncu_full_c5.log 2>&1
      echo "ncu exit $?" >> $OUT/ncu_full_c5.log ;;
    ref) timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference_c2.json 2> $OUT/bench_reference_c2.err ;;
    ncu)
      timeout 300 python tools/profile_pcg.py c2 6 > $OUT/plain.log 2>&1 &&
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
          --log-file $OUT/launches_c2.csv python tools/profile_pcg.py c2 6 > $OUT/ncu_launch.log 2>&1 &&
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dag -s 2 -c 1 \
          -o $OUT/dag_c2 python tools/profile_pcg.py c2 6 > $OUT/ncu_full.log 2>&1
      echo "ncu exit $?" >> $OUT/ncu_full.log ;;
    trace) timeout 300 python tools/trace_dag.py c2 > $OUT/trace.log 2>&1; mv gpurun_out/trace_c2.npz $OUT/ ;;
  esac
done
echo done
