# A/B of the DAG worker schedule: dynamic claims (default) vs static round-robin lists (SFCDD_DAG_MODE=16)
#   gpurun --timeout 1800 -- 'bash tools/ab_static.sh <tag>'
T=${1:-abs}; O=gpurun_out/$T; mkdir -p $O
SFCDD_DAG_MODE=16 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c2_matches or c3_matches or c4_fault or bitwise" > $O/pytest_static.log 2>&1; echo "exit $?" >> $O/pytest_static.log
for cfg in c2 c3 c4; do
  for v in "dyn:" "static:SFCDD_DAG_MODE=16" "dyn2:" "static2:SFCDD_DAG_MODE=16"; do
    n=${v%%:*}; e=${v#*:}
    env $e timeout 400 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > $O/${cfg}_$n.json 2> $O/${cfg}_$n.err
  done
done
