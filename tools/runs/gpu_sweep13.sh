T=${1:-sw13}; mkdir -p gpurun_out/$T
SFCDD_PLAN_DEBUG=1 timeout 1200 python tools/sweep_dag.py c4 "MODE=0" "WPB=4,BLOB=8192,SLOT=11264" > gpurun_out/$T/sweep_c4.jsonl 2> gpurun_out/$T/sweep_c4.err
SFCDD_PLAN_DEBUG=1 timeout 900 python tools/sweep_dag.py c3 "MODE=0" "WPB=4,BLOB=8192,SLOT=11264" > gpurun_out/$T/sweep_c3.jsonl 2> gpurun_out/$T/sweep_c3.err
SFCDD_PLAN_DEBUG=1 timeout 900 python tools/sweep_dag.py c2 "MODE=0" "WPB=2,BLOB=16384,SLOT=22656" > gpurun_out/$T/sweep_c2.jsonl 2> gpurun_out/$T/sweep_c2.err
