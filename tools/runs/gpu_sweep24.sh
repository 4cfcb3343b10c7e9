T=${1:-sw24}; mkdir -p gpurun_out/$T
timeout 3000 python tools/sweep_dag.py c5 "PF=0" "PF=512" "PF=1536" "PF=4096" > gpurun_out/$T/sweep_c5.jsonl 2> gpurun_out/$T/sweep_c5.err
timeout 1200 python tools/sweep_dag.py c4 "PF=0" "PF=512" "PF=1536" "PF=4096" > gpurun_out/$T/sweep_c4.jsonl 2> gpurun_out/$T/sweep_c4.err
