T=${1:-sw8}; mkdir -p gpurun_out/$T
timeout 900 python tools/sweep_dag.py c2 "MODE=0" "MODE=64" "MODE=0" "MODE=64" > gpurun_out/$T/sweep_c2.jsonl 2> gpurun_out/$T/sweep_c2.err
timeout 900 python tools/sweep_dag.py c3 "MODE=0" "MODE=64" > gpurun_out/$T/sweep_c3.jsonl 2> gpurun_out/$T/sweep_c3.err
