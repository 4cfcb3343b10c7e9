T=${1:-sw9}; mkdir -p gpurun_out/$T
timeout 900 python tools/sweep_dag.py c2 "Q=16" "Q=4" "Q=64" "Q=256" "MODE=2" > gpurun_out/$T/sweep_c2.jsonl 2> gpurun_out/$T/sweep_c2.err
timeout 900 python tools/trace_dag.py c2 > gpurun_out/$T/trace_c2_m0.log 2>&1
timeout 600 python tools/analyze_trace.py gpurun_out/trace_c2.npz > gpurun_out/$T/trace_c2_m0.txt 2>&1
SFCDD_DAG_MODE=64 timeout 900 python tools/trace_dag.py c2 > gpurun_out/$T/trace_c2_m64.log 2>&1
timeout 600 python tools/analyze_trace.py gpurun_out/trace_c2.npz > gpurun_out/$T/trace_c2_m64.txt 2>&1
rm -f gpurun_out/trace_c2.npz
