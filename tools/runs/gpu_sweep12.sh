T=${1:-sw12}; mkdir -p gpurun_out/$T
SFCDD_PLAN_DEBUG=1 timeout 900 python tools/sweep_dag.py c2 "MODE=0" "MODE=0" > gpurun_out/$T/sweep_c2_base.jsonl 2> gpurun_out/$T/sweep_c2_base.err
export SFCDD_LIB=$PWD/abtest/libsfcdd_r80.so
SFCDD_PLAN_DEBUG=1 timeout 900 python tools/sweep_dag.py c2 "MODE=0" "MODE=0" >> gpurun_out/$T/sweep_c2_r80.jsonl 2>> gpurun_out/$T/sweep_c2_r80.err
