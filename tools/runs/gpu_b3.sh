T=${1:-b3}; shift; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "split or c3 or c2 or matches_reference or grown or sparse" > gpurun_out/$T/pytest_sel.log 2>&1
for c in "$@"; do
SFCDD_PLAN_DEBUG=1 timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$T/$c.json 2> gpurun_out/$T/$c.err
done
