T=${1:-r02m}; mkdir -p gpurun_out/$T
for c in c2 c3 c4; do
SFCDD_PLAN_DEBUG=1 timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/$c.json 2> gpurun_out/$T/$c.err
done
