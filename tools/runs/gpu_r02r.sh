T=${1:-r02r}; mkdir -p gpurun_out/$T
SFCDD_SPLIT_MIN=1 timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c5_split1.json 2> gpurun_out/$T/c5_split1.err
bash tools/gpu_trace.sh $T c5 c3
timeout 600 python tools/profile_apply.py c5 3 > gpurun_out/$T/plain_c5.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_dag -s 4 -c 1 -o gpurun_out/$T/dag_c5 python tools/profile_apply.py c5 3 > gpurun_out/$T/ncu_full_c5.log 2>&1
