T=${1:-sw3}; mkdir -p gpurun_out/$T
SFCDD_PLAN_DEBUG=1 timeout 900 python tools/sweep_dag.py c2 "WPB=4,BLOB=8192" "WPB=8,BLOB=8192" "WPB=8,BLOB=6144,SCR=384" "WPB=8,BLOB=6144,SCR=320" "WPB=8,BLOB=5120,SCR=320" "WPB=8,BLOB=7168,SCR=384" "WPB=4,BLOB=6144,SCR=384" "WPB=8,BLOB=6144,SCR=384,MODE=16" "WPB=4,BLOB=8192,MODE=16" > gpurun_out/$T/sweep_c2.jsonl 2> gpurun_out/$T/sweep_c2.err
