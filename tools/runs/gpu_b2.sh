T=${1:-b2}; shift; mkdir -p gpurun_out/$T
for c in "$@"; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$T/$c.json 2> gpurun_out/$T/$c.err
done
