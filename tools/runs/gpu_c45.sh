T=${1:-c45}; mkdir -p gpurun_out/$T
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c5.json 2> gpurun_out/$T/c5.err
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c4.json 2> gpurun_out/$T/c4.err
