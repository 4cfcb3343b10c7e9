T=${1:-sw34}; mkdir -p gpurun_out/$T
timeout 900 python tools/sweep_dag.py c2 "PF=0" "PF=1536,PFB=0" "PF=512,PFB=0" "PF=4096,PFB=0" "PF=1536,PFB=1" "PF=0" > gpurun_out/$T/sweep_c2.jsonl 2> gpurun_out/$T/sweep_c2.err
timeout 1200 python tools/sweep_dag.py c4 "PF=1536,PFB=0" "PF=1536,PFB=1" > gpurun_out/$T/sweep_c4.jsonl 2> gpurun_out/$T/sweep_c4.err
timeout 900 python tools/sweep_dag.py c3 "PF=1536,PFB=0" "PF=1536,PFB=1" > gpurun_out/$T/sweep_c3.jsonl 2> gpurun_out/$T/sweep_c3.err
