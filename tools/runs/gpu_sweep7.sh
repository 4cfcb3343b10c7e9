T=${1:-sw7}; mkdir -p gpurun_out/$T
timeout 900 python tools/sweep_dag.py c3 "ROW=64" "ROW=96" "ROW=128" "ROW=64,COL=24" "ROW=64,COL=32" > gpurun_out/$T/sweep_c3.jsonl 2> gpurun_out/$T/sweep_c3.err
timeout 900 python tools/sweep_dag.py c4 "ROW=32" "ROW=64" "ROW=128" "ROW=64,COL=32" > gpurun_out/$T/sweep_c4.jsonl 2> gpurun_out/$T/sweep_c4.err
timeout 300 python tools/sweep_dag.py c2 "ROW=128" "ROW=64" > gpurun_out/$T/sweep_c2.jsonl 2> gpurun_out/$T/sweep_c2.err
