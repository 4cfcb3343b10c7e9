T=${1:-fz}; mkdir -p gpurun_out/$T
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py -q -x -k "dense_block_shapes or c5shape" > gpurun_out/$T/pytest_direct.log 2>&1
timeout 2400 python tools/fuzz_shapes.py > gpurun_out/$T/fuzz.log 2>&1; echo "exit $?" >> gpurun_out/$T/fuzz.log
