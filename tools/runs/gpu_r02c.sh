T=${1:-r02c}; mkdir -p gpurun_out/$T
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/$T/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/$T/pytest_gpu.log
bash tools/run_conformance.sh gpurun_out/$T/conformance
bash tools/gpu_c5try.sh $T
