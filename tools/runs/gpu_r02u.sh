T=${1:-r02u}; mkdir -p gpurun_out/$T
export SFCDD_DIRECT_ROWS=8 SFCDD_DIRECT_COLS=4
timeout 900 python tools/trace_dag.py c3 > gpurun_out/$T/trace_c3_mrow.log 2>&1
timeout 600 python tools/analyze_trace.py gpurun_out/trace_c3.npz > gpurun_out/$T/trace_c3_mrow.txt 2>&1
python - <<'PY' > gpurun_out/r02u/mrow_detail.txt 2>&1
import numpy as np
d = np.load("gpurun_out/trace_c3.npz")
T = d['trace'].astype(np.int64)
kind=T[:,5]; vals=T[:,8]; t0=T[:,1]; tdep=T[:,2]; tdat=T[:,3]; tend=T[:,4]
m = kind==2
v = vals[m]; dur=(tend[m]-tdat[m])/1e3
for lo,hi in [(0,512),(512,2048),(2048,8192),(8192,1<<30)]:
    s=(v>=lo)&(v<hi)
    if s.any(): print("row values [%d,%d): n=%d mean vals %.0f data->end %.2f us  => %.2f GB/s/warp"%(lo,hi,s.sum(),v[s].mean(),dur[s].mean(), 8*v[s].mean()/dur[s].mean()/1e3))
m = kind==3
v = vals[m]; dur=(tend[m]-tdat[m])/1e3
for lo,hi in [(0,512),(512,2048),(2048,8192),(8192,1<<30)]:
    s=(v>=lo)&(v<hi)
    if s.any(): print("col values [%d,%d): n=%d mean vals %.0f data->end %.2f us  => %.2f GB/s/warp"%(lo,hi,s.sum(),v[s].mean(),dur[s].mean(), 8*v[s].mean()/dur[s].mean()/1e3))
PY
rm -f gpurun_out/trace_c3.npz
