T=${1:-sw11}; mkdir -p gpurun_out/$T
SFCDD_PLAN_DEBUG=1 timeout 900 python tools/sweep_dag.py c2 "MODE=0" > gpurun_out/$T/sweep_c2_base.jsonl 2> gpurun_out/$T/sweep_c2_base.err
export SFCDD_LIB=$PWD/abtest/libsfcdd_r64.so
for sm in 9344 9216 11264; do
SFCDD_SLOT_MAX=$sm SFCDD_PLAN_DEBUG=1 timeout 900 python tools/sweep_dag.py c2 "MODE=0" >> gpurun_out/$T/sweep_c2_r64.jsonl 2>> gpurun_out/$T/sweep_c2_r64.err
done
