T=${1:-sw15}; mkdir -p gpurun_out/$T
SFCDD_PLAN_DEBUG=1 timeout 900 python tools/sweep_dag.py c3 "WPB=4,BLOB=8192,SLOT=11264" > gpurun_out/$T/sweep_c3.jsonl 2> gpurun_out/$T/sweep_c3.err
SFCDD_PLAN_DEBUG=1 timeout 1500 python tools/sweep_dag.py c5 "WPB=4,BLOB=8192,SLOT=11264" > gpurun_out/$T/sweep_c5.jsonl 2> gpurun_out/$T/sweep_c5.err
