T=${1:-r02i}; mkdir -p gpurun_out/$T
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/$T/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/$T/pytest_gpu.log
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c2.json 2> gpurun_out/$T/c2.err
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c3.json 2> gpurun_out/$T/c3.err
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c4.json 2> gpurun_out/$T/c4.err
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c5.json 2> gpurun_out/$T/c5.err
