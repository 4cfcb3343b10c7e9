T=${1:-sw2}; mkdir -p gpurun_out/$T
run() { n=$1; c=$2; shift 2; env "$@" timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/$n.json 2> gpurun_out/$T/$n.err; }
run c3_s1024 c3 SFCDD_SCRATCH_MAX=1024
run c3_s768 c3 SFCDD_SCRATCH_MAX=768
run c3_b24 c3 SFCDD_BLOB_MAX=24576 SFCDD_WPB=2 SFCDD_SCRATCH_MAX=768
run c3_b12 c3 SFCDD_BLOB_MAX=12288 SFCDD_WPB=2
run c3_b12w4 c3 SFCDD_BLOB_MAX=12288 SFCDD_WPB=4
run c2_b12 c2 SFCDD_BLOB_MAX=12288 SFCDD_WPB=4
run c2_b10 c2 SFCDD_BLOB_MAX=10240 SFCDD_WPB=4
run c2_b6w8 c2 SFCDD_BLOB_MAX=6144 SFCDD_WPB=8
run c5_s1024 c5 SFCDD_SCRATCH_MAX=1024
