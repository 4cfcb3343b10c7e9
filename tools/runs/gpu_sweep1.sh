T=${1:-sw1}; mkdir -p gpurun_out/$T
run() { # name cfg env...
  n=$1; c=$2; shift 2
  env "$@" timeout 1200 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$T/$n.json 2> gpurun_out/$T/$n.err
}
run c3_a c3 SFCDD_BLOB_MAX=16384 SFCDD_WPB=2
run c3_b c3 SFCDD_BLOB_MAX=16384 SFCDD_SCRATCH_MAX=1024 SFCDD_WPB=2
run c3_c c3 SFCDD_BLOB_MAX=8192 SFCDD_SCRATCH_MAX=1024 SFCDD_WPB=2
run c3_d c3 SFCDD_BLOB_MAX=8192 SFCDD_SCRATCH_MAX=1024 SFCDD_WPB=4
run c3_e c3 SFCDD_BLOB_MAX=16384 SFCDD_SCRATCH_MAX=2048 SFCDD_WPB=2
run c3_f c3 SFCDD_BLOB_MAX=8192 SFCDD_COL_MAX=32 SFCDD_WPB=4
run c2_f c2 SFCDD_BLOB_MAX=8192 SFCDD_COL_MAX=32 SFCDD_WPB=4
run c5_b c5 SFCDD_BLOB_MAX=16384 SFCDD_SCRATCH_MAX=1024 SFCDD_WPB=2
