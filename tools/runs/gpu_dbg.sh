T=${1:-dbg}; mkdir -p gpurun_out/$T
( time SFCDD_DAG_MODE=32 SFCDD_WATCHDOG_MS=3000 timeout 300 python tools/profile_apply.py c3 2 ) > gpurun_out/$T/apply_c3_diag.log 2>&1
( time SFCDD_WATCHDOG_MS=3000 timeout 300 python tools/profile_apply.py c3 2 ) > gpurun_out/$T/apply_c3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "split or c3 or c2 or matches_reference" > gpurun_out/$T/pytest_sel.log 2>&1
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c3.json 2> gpurun_out/$T/c3.err
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$T/c2.json 2> gpurun_out/$T/c2.err
