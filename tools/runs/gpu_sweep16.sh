T=${1:-sw16}; mkdir -p gpurun_out/$T
SFCDD_PLAN_DEBUG=1 timeout 2400 python tools/sweep_dag.py c5 "MODE=0" "MODE=128" > gpurun_out/$T/sweep_c5.jsonl 2> gpurun_out/$T/sweep_c5.err
