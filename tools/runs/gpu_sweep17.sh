T=${1:-sw17}; mkdir -p gpurun_out/$T
timeout 3000 python tools/sweep_dag.py c5 "DR=16,DC=8" "DR=32,DC=16" "DR=64,DC=16" "DR=128,DC=16" > gpurun_out/$T/sweep_c5.jsonl 2> gpurun_out/$T/sweep_c5.err
timeout 900 python tools/sweep_dag.py c3 "MODE=0" "DR=8,DC=4" "DR=32,DC=16" "DR=128,DC=16" > gpurun_out/$T/sweep_c3.jsonl 2> gpurun_out/$T/sweep_c3.err
