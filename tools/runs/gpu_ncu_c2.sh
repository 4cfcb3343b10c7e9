T=${1:-ncu2}; mkdir -p gpurun_out/$T
timeout 300 python tools/profile_pcg.py c2 6 > gpurun_out/$T/plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dag -s 2 -c 1 -o gpurun_out/$T/dag_c2 python tools/profile_pcg.py c2 6 > gpurun_out/$T/ncu_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/$T/ncu_full.log
