T=${1:-r02f}; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_distributed.py tests/test_harness_combine.py -m gpu -x -q > gpurun_out/$T/pytest_dist.log 2>&1; echo "exit $?" >> gpurun_out/$T/pytest_dist.log
