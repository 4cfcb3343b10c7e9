T=${1:-tr}; shift; mkdir -p gpurun_out/$T
for c in "$@"; do
  timeout 900 python tools/trace_dag.py $c > gpurun_out/$T/trace_$c.log 2>&1
  timeout 600 python tools/analyze_trace.py gpurun_out/trace_$c.npz > gpurun_out/$T/trace_$c.txt 2>&1
  rm -f gpurun_out/trace_$c.npz
done
