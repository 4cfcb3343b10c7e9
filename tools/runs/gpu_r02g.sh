T=${1:-r02g}; mkdir -p gpurun_out/$T
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c2_graph.json 2> gpurun_out/$T/c2_graph.err
timeout 600 python bench.py --steps 5 --warmup 3 --sharded > gpurun_out/$T/c2_sharded.json 2> gpurun_out/$T/c2_sharded.err
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c3_graph.json 2> gpurun_out/$T/c3_graph.err
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --sharded > gpurun_out/$T/c3_sharded.json 2> gpurun_out/$T/c3_sharded.err
