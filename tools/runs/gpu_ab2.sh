T=${1:-ab2}; mkdir -p gpurun_out/$T
run() { n=$1; c=$2; shift 2; env "$@" timeout 1200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$T/$n.json 2> gpurun_out/$T/$n.err; }
run c2_v0 c2 X=1
for v in 1 3 5 7; do
run c2_v$v c2 SFCDD_LIB=$PWD/build/variants/libsfcdd_lean$v.so
done
run c2_v0b c2 X=1
run c3_v0 c3 X=1
run c3_v7 c3 SFCDD_LIB=$PWD/build/variants/libsfcdd_lean7.so
