# Quick GPU check: parity tests + per-kernel graph-timed profile of C2 / C3.
#   gpurun --timeout 1500 -- 'bash tools/quick_gpu.sh <tag>'   (outputs under gpurun_out/<tag>/)
T=${1:-quick}; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/$T/pytest.log 2>&1; echo "exit $?" >> gpurun_out/$T/pytest.log
SFCDD_PROFILE_KERNELS=1 timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c2.json 2> gpurun_out/$T/c2.err
SFCDD_PROFILE_KERNELS=1 timeout 400 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c3.json 2> gpurun_out/$T/c3.err
