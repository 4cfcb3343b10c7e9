T=${1:-ncuv}; mkdir -p gpurun_out/$T
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tile_pm_w|k_update|k_combine_chunk|k_tile_tvec|k_tile_agg_matvec|k_coarse_gemv|k_slot_sums' -s 14 -c 8 -o gpurun_out/$T/vec_c2 python tools/profile_pcg.py c2 8 > gpurun_out/$T/ncu_vec.log 2>&1
echo "ncu exit $?" >> gpurun_out/$T/ncu_vec.log
