T=${1:-sw4}; mkdir -p gpurun_out/$T
timeout 900 python tools/sweep_dag.py c2 "PF=0" "PF=256" "PF=1024" "PF=2048" "PF=4096" "PF=8192" "PF=0" > gpurun_out/$T/sweep_c2.jsonl 2> gpurun_out/$T/sweep_c2.err
timeout 900 python tools/sweep_dag.py c3 "PF=0" "PF=1024" "PF=4096" > gpurun_out/$T/sweep_c3.jsonl 2> gpurun_out/$T/sweep_c3.err
