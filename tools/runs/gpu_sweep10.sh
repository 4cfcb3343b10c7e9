T=${1:-sw10}; mkdir -p gpurun_out/$T
SFCDD_PLAN_DEBUG=1 timeout 900 python tools/sweep_dag.py c2 "WPB=4,BLOB=8192" "WPB=4,BLOB=8704,SCR=320" "WPB=4,BLOB=9216,SCR=256" "WPB=4,BLOB=9728,SCR=192" "WPB=4,BLOB=8192,SCR=384" > gpurun_out/$T/sweep_c2.jsonl 2> gpurun_out/$T/sweep_c2.err
