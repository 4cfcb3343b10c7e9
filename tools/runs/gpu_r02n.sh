T=${1:-r02n}; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "split or c3 or c2 or matches_reference" > gpurun_out/$T/pytest_sel.log 2>&1
for c in c2 c3 c4; do
SFCDD_PLAN_DEBUG=1 timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/$c.json 2> gpurun_out/$T/$c.err
done
SFCDD_PLAN_DEBUG=1 timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c5.json 2> gpurun_out/$T/c5.err
