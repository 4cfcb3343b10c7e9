T=${1:-ncuf}; mkdir -p gpurun_out/$T
timeout 600 python tools/profile_factor.py c5p > gpurun_out/$T/plain.log 2>&1
timeout 1500 ncu --clock-control none --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size -k regex:k_front --csv --log-file gpurun_out/$T/front_c5p.csv python tools/profile_factor.py c5p > gpurun_out/$T/ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/$T/ncu.log
