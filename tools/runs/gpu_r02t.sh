T=${1:-r02t}; mkdir -p gpurun_out/$T
run() { n=$1; c=$2; shift 2; env "$@" timeout 1200 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --also none > gpurun_out/$T/$n.json 2> gpurun_out/$T/$n.err; }
run c5_nomrow c5 SFCDD_MROW_ROWS=0
run c5 c5 X=1
run c3 c3 X=1
run c3_mrow c3 SFCDD_DIRECT_ROWS=8 SFCDD_DIRECT_COLS=4
run c3_dir c3 SFCDD_DIRECT_ROWS=8 SFCDD_DIRECT_COLS=4 SFCDD_MROW_ROWS=0
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c3_dense" > gpurun_out/$T/pytest_sel.log 2>&1
