T=${1:-ab3}; mkdir -p gpurun_out/$T
run() { n=$1; c=$2; shift 2; env "$@" timeout 1200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$T/$n.json 2> gpurun_out/$T/$n.err; }
run c2_old c2 SFCDD_LIB=$PWD/build/variants/libsfcdd_r02g.so
run c2_v0 c2 X=1
run c3_old c3 SFCDD_LIB=$PWD/build/variants/libsfcdd_r02g.so
run c3_v0 c3 X=1
for v in 1 3 5; do
run c3_v$v c3 SFCDD_LIB=$PWD/build/variants/libsfcdd_lean$v.so
done
run c4_old c4 SFCDD_LIB=$PWD/build/variants/libsfcdd_r02g.so
run c4_v0 c4 X=1
