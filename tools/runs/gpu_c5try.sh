# C5 trial: setup phases, memory, one bench line (no CPU baseline)
T=${1:-c5try}; mkdir -p gpurun_out/$T
free -g > gpurun_out/$T/free_before.txt
( while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/$T/gpumem.txt; free -g | grep Mem >> gpurun_out/$T/hostmem.txt; sleep 5; done ) &
MON=$!
SFCDD_PLAN_DEBUG=1 timeout 1700 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$T/bench_c5.json 2> gpurun_out/$T/bench_c5.err
echo "exit $?" >> gpurun_out/$T/bench_c5.err
kill $MON
