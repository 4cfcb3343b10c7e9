T=${1:-sw19}; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py -q -x -k "split or c3 or c2 or matches_reference or grown or sparse or c5shape" > gpurun_out/$T/pytest_sel.log 2>&1
timeout 900 python tools/sweep_dag.py c2 "MODE=0" "MODE=0" > gpurun_out/$T/sweep_c2.jsonl 2> gpurun_out/$T/sweep_c2.err
timeout 900 python tools/sweep_dag.py c3 "MODE=0" > gpurun_out/$T/sweep_c3.jsonl 2> gpurun_out/$T/sweep_c3.err
timeout 1200 python tools/sweep_dag.py c4 "MODE=0" > gpurun_out/$T/sweep_c4.jsonl 2> gpurun_out/$T/sweep_c4.err
bash tools/gpu_trace.sh $T c3
