T=${1:-r02s}; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "split or c3 or matches_reference" > gpurun_out/$T/pytest_sel.log 2>&1
run() { n=$1; c=$2; shift 2; env "$@" timeout 1200 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --also none > gpurun_out/$T/$n.json 2> gpurun_out/$T/$n.err; }
run c5 c5 X=1
run c5_nomrow c5 SFCDD_MROW_ROWS=0
run c5_8k c5 SFCDD_BLOB_MAX=8192 SFCDD_WPB=4
run c3_mrow c3 SFCDD_DIRECT_ROWS=8 SFCDD_DIRECT_COLS=4
run c3 c3 X=1
run c3_mrow8k c3 SFCDD_DIRECT_ROWS=8 SFCDD_DIRECT_COLS=4 SFCDD_BLOB_MAX=8192 SFCDD_WPB=4
