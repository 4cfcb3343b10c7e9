T=${1:-r02e}; mkdir -p gpurun_out/$T
SFCDD_FACTOR_DEBUG=1 timeout 300 python tools/profile_factor.py c5p > gpurun_out/$T/factor_c5p.log 2>&1
SFCDD_FACTOR_DEBUG=1 timeout 300 python tools/profile_factor.py c3 > gpurun_out/$T/factor_c3.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/$T/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/$T/pytest_gpu.log
