T=${1:-ab6}; mkdir -p gpurun_out/$T
run() { n=$1; c=$2; shift 2; env "$@" timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$T/$n.json 2> gpurun_out/$T/$n.err; }
run c2_oldk c2 SFCDD_LIB=$PWD/build/variants/libsfcdd_oldk.so
run c2_sw0 c2 SFCDD_LIB=$PWD/build/variants/libsfcdd_lean0.so
run c2_sw1 c2 SFCDD_LIB=$PWD/build/variants/libsfcdd_lean1.so
