# A/B of the DAG signaller idle wait: mbarrier suspend (default) vs nanosleep spin (SFCDD_DAG_MODE=8)
#   gpurun --timeout 1800 -- 'bash tools/ab_sig.sh <tag>'
T=${1:-ab}; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for cfg in c2 c3; do
  for v in "def:" "old:SFCDD_DAG_MODE=8" "w300:SFCDD_SIG_WAIT_NS=300" "w5000:SFCDD_SIG_WAIT_NS=5000" "def2:"; do
    n=${v%%:*}; e=${v#*:}
    env $e timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > $O/${cfg}_$n.json 2> $O/${cfg}_$n.err
  done
done
