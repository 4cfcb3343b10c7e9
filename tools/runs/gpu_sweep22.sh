T=${1:-sw22}; mkdir -p gpurun_out/$T
SFCDD_PLAN_DEBUG=1 timeout 1200 python tools/sweep_dag.py c2 "MODE=0" "DR=8,DC=4" "DR=16,DC=8" "DR=32,DC=8" "DR=64,DC=16" "DR=64,DC=0" "DR=0,DC=16" > gpurun_out/$T/sweep_c2.jsonl 2> gpurun_out/$T/sweep_c2.err
timeout 1200 python tools/sweep_dag.py c4 "DR=16,DC=8" "DR=64,DC=16" > gpurun_out/$T/sweep_c4.jsonl 2> gpurun_out/$T/sweep_c4.err
