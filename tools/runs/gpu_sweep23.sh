T=${1:-sw23}; mkdir -p gpurun_out/$T
timeout 900 python tools/sweep_dag.py c2 "MODE=0" > gpurun_out/$T/sweep_c2_base.jsonl 2> gpurun_out/$T/sweep_c2_base.err
SFCDD_L2_PERSIST=1 timeout 900 python tools/sweep_dag.py c2 "MODE=0" > gpurun_out/$T/sweep_c2_p1.jsonl 2> gpurun_out/$T/sweep_c2_p1.err
SFCDD_L2_PERSIST=2 timeout 900 python tools/sweep_dag.py c2 "MODE=0" > gpurun_out/$T/sweep_c2_p2.jsonl 2> gpurun_out/$T/sweep_c2_p2.err
SFCDD_L2_PERSIST=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/bench_c2_p1.json 2> gpurun_out/$T/bench_c2_p1.err
SFCDD_L2_PERSIST=1 bash tools/gpu_trace.sh $T c2
