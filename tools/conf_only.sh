bash tools/run_conformance.sh gpurun_out/${1:-conf}/conformance
