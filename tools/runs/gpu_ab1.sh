T=${1:-ab1}; mkdir -p gpurun_out/$T
run() { n=$1; c=$2; shift 2; env "$@" timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/$n.json 2> gpurun_out/$T/$n.err; }
run c2_nodirect c2 SFCDD_DIRECT_ROWS=0 SFCDD_DIRECT_COLS=0
run c2_dir4 c2 SFCDD_DIRECT_ROWS=4 SFCDD_DIRECT_COLS=2
run c3_nodirect c3 SFCDD_DIRECT_ROWS=0 SFCDD_DIRECT_COLS=0
run c3_dir4 c3 SFCDD_DIRECT_ROWS=4 SFCDD_DIRECT_COLS=2
run c3_dir16 c3 SFCDD_DIRECT_ROWS=16 SFCDD_DIRECT_COLS=8
run c3_asm1 c3 SFCDD_ASM_RED=1 SFCDD_XB_MIN=1
