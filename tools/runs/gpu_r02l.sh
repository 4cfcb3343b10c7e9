T=${1:-r02l}; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "split or c3 or c2 or matches_reference" > gpurun_out/$T/pytest_sel.log 2>&1
for c in c2 c3 c4; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/$c.json 2> gpurun_out/$T/$c.err
done
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c5.json 2> gpurun_out/$T/c5.err
SFCDD_BLOB_MAX=8192 SFCDD_WPB=4 SFCDD_DIRECT_ROWS=1048576 SFCDD_DIRECT_COLS=1048576 timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c5_8kd.json 2> gpurun_out/$T/c5_8kd.err
bash tools/gpu_trace.sh $T c2
