T=${1:-ab4}; mkdir -p gpurun_out/$T
run() { n=$1; c=$2; shift 2; env "$@" timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$T/$n.json 2> gpurun_out/$T/$n.err; }
run c2_old c2 SFCDD_LIB=$PWD/build/variants/libsfcdd_r02g.so
run c2_v0 c2 X=1
run c2_even c2 SFCDD_EVEN_COLS=1
run c2_v8 c2 SFCDD_LIB=$PWD/build/variants/libsfcdd_lean8.so
run c2_v15 c2 SFCDD_LIB=$PWD/build/variants/libsfcdd_lean15.so
run c2_v15e c2 SFCDD_LIB=$PWD/build/variants/libsfcdd_lean15.so SFCDD_EVEN_COLS=1
