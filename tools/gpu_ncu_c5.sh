T=${1:-ncu5}; mkdir -p gpurun_out/$T
timeout 600 python tools/profile_apply.py c5 3 > gpurun_out/$T/plain_c5.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_dag<.int.2" -s 1 -c 1 -o gpurun_out/$T/dag_c5 python tools/profile_apply.py c5 3 > gpurun_out/$T/ncu_full_c5.log 2>&1
echo "ncu exit $?" >> gpurun_out/$T/ncu_full_c5.log
