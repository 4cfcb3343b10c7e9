T=${1:-sw5}; mkdir -p gpurun_out/$T
timeout 900 python tools/sweep_dag.py c2 "PF=2048" "PF=2048,MODE=8,SIG=20" "PF=2048,MODE=8,SIG=100" "PF=2048,MODE=8,SIG=250" "PF=2048,MODE=8,SIG=500" "PF=2048,MODE=8,SIG=1000" "PF=2048,MODE=2" "PF=2048" > gpurun_out/$T/sweep_c2.jsonl 2> gpurun_out/$T/sweep_c2.err
