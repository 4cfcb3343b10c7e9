mkdir -p gpurun_out/${1:-r02a}
nvidia-smi > gpurun_out/${1:-r02a}/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${1:-r02a}/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/${1:-r02a}/pytest_gpu.log
bash tools/run_conformance.sh gpurun_out/${1:-r02a}/conformance
