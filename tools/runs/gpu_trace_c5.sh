T=${1:-tr5}; mkdir -p gpurun_out/$T
SFCDD_PLAN_DEBUG=1 timeout 1500 python tools/trace_dag.py c5 > gpurun_out/$T/trace_c5.log 2>&1
timeout 900 python tools/analyze_trace.py gpurun_out/trace_c5.npz > gpurun_out/$T/trace_c5.txt 2>&1
python - <<'PY' > gpurun_out/$T/c5_detail.txt 2>&1
import numpy as np
d = np.load("gpurun_out/trace_c5.npz")
T = d['trace'].astype(np.int64)
kind=T[:,5]; vals=T[:,8]; t0=T[:,1]; tdep=T[:,2]; tdat=T[:,3]; tend=T[:,4]; cb=T[:,6]
tot=(tend-t0).sum()
names=["frag_f","frag_b","row","col","asm","xb"]
for k in range(6):
    m=kind==k
    if m.any(): print("%-7s n=%8d  share of worker time %.1f%%  values %.2f G  mean total %.2f us"%(names[k], m.sum(), 100*(tend[m]-t0[m]).sum()/tot, vals[m].sum()/1e9, (tend[m]-t0[m]).mean()/1e3))
for k,nm in ((2,"row"),(3,"col")):
    m=kind==k
    v=vals[m]; dur=(tend[m]-tdat[m])/1e3; full=(tend[m]-t0[m])/1e3; c=cb[m]
    inblob = c > 8*v*0.9
    for tag,sel in (("blob",inblob),("direct",~inblob)):
        if not sel.any(): continue
        print("%s %s: n=%d values %.2f G share of worker time %.1f%%"%(nm,tag,sel.sum(), v[sel].sum()/1e9, 100*(full[sel]*1e3).sum()/tot))
        for lo,hi in [(0,2048),(2048,8192),(8192,32768),(32768,1<<30)]:
            s=sel&(v>=lo)&(v<hi)
            if s.any(): print("   values [%d,%d): n=%d mean vals %.0f data->end %.2f us total %.2f us => %.2f GB/s/warp"%(lo,hi,s.sum(),v[s].mean(),dur[s].mean(),full[s].mean(), 8*v[s].mean()/full[s].mean()/1e3))
PY
rm -f gpurun_out/trace_c5.npz
