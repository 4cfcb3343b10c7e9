T=${1:-sw32}; mkdir -p gpurun_out/$T
export SFCDD_LIB=$PWD/abtest/libsfcdd_r64.so
SFCDD_PLAN_DEBUG=1 timeout 900 python tools/sweep_dag.py c2 "SLOT=9344" "SLOT=9344,PF=0" "SLOT=9216" "SLOT=11264" > gpurun_out/$T/sweep_c2_r64.jsonl 2> gpurun_out/$T/sweep_c2_r64.err
SFCDD_PLAN_DEBUG=1 timeout 900 python tools/sweep_dag.py c4 "WPB=4,BLOB=8192,SLOT=9344" > gpurun_out/$T/sweep_c4_r64.jsonl 2> gpurun_out/$T/sweep_c4_r64.err
unset SFCDD_LIB
timeout 900 python tools/sweep_dag.py c3 "MODE=0" "PF=0" > gpurun_out/$T/sweep_c3.jsonl 2> gpurun_out/$T/sweep_c3.err
timeout 900 python tools/sweep_dag.py c4 "MODE=0" "PF=0" > gpurun_out/$T/sweep_c4.jsonl 2> gpurun_out/$T/sweep_c4.err
