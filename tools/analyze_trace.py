import numpy as np, sys
d = np.load(sys.argv[1])
T = d['trace'].astype(np.int64)
sm, t0, tdep, tdat, tend = T[:,0] & 0xffff, T[:,1], T[:,2], T[:,3], T[:,4]
wid = T[:,0] >> 16
kind = T[:,5]; cb = T[:,6]; vals = T[:,8]; wait = T[:,9]
base = t0.min(); 
print("makespan us", (tend.max()-base)/1e3)
names = ["frag_f","frag_b","row","col","asm","xb"]
for k in range(6):
    m = kind==k
    if not m.any():
        continue
    print(f"{names[k]:7s} n={m.sum():6d} claim->deps {np.mean(tdep[m]-t0[m])/1e3:6.2f}us  deps->data {np.mean(np.maximum(tdat[m]-tdep[m],0))/1e3:6.2f}  data->end {np.mean(tend[m]-tdat[m])/1e3:6.2f}  total {np.mean(tend[m]-t0[m])/1e3:6.2f}  bytes {cb[m].mean():.0f}")
# per-warp idle: gaps between consecutive tasks of same warp unknown (no warp id); utilisation over time
edges = np.linspace(0, (tend.max()-base), 21)
act = []
for a,b in zip(edges[:-1], edges[1:]):
    s = np.clip(np.minimum(tend-base, b) - np.maximum(t0-base, a), 0, None).sum()
    act.append(s/(b-a))
print("avg busy warps per 5% window:", [int(x) for x in act])
byt = []
for a,b in zip(edges[:-1], edges[1:]):
    m = (tdat-base>=a)&(tdat-base<b)
    byt.append(cb[m].sum()/((b-a)*1e-9)/1e9)
print("GB/s of blob data arriving per window:", [int(x) for x in byt])
# FRAG phase stamps (clock64): [0] start [1] prologue done [2+2l, 3+2l] level l
# (assembly / v_B rows, then items) [10] end [11] nlev
for kind, nm in ((0, "frag_f"), (1, "frag_b")):
    m = T[:, 5] == kind
    Pp = T[m][:, 12:24]
    ok = (Pp[:, 0] > 0) & (Pp[:, 10] > 0)
    Pp = Pp[ok]
    if not len(Pp):
        continue
    nl = Pp[:, 11]
    print(f"{nm}: {len(Pp)} tasks, {nl.mean():.2f} levels, {np.mean(Pp[:, 10] - Pp[:, 0]):.0f} cycles; prologue {np.mean(Pp[:, 1] - Pp[:, 0]):.0f}")
    for l in range(4):
        sel = nl > l
        a = np.mean(Pp[sel, 2 + 2 * l] - (Pp[sel, 1] if l == 0 else Pp[sel, 1 + 2 * l]))
        r = np.mean(Pp[sel, 3 + 2 * l] - Pp[sel, 2 + 2 * l])
        print(f"   level {l}: n={sel.sum()} first phase {a:.0f} items {r:.0f}")
    last = np.array([Pp[i, min(3 + 2 * (nl[i] - 1), 9)] for i in range(len(Pp))])
    print(f"   epilogue {np.mean(Pp[:, 10] - last):.0f}")

# per-worker gaps: end of a warp's task -> top of its next task (claim atomic,
# TaskDev load, mailbox post), i.e. the per-task cost outside [t_top, t_end]
# (needs a kernel that stores the worker id in the trace's upper sm bits)
if wid.max() > 0:
    o = np.lexsort((t0, wid))
    w2, a, e = wid[o], t0[o], tend[o]
    same = w2[1:] == w2[:-1]
    gap = (a[1:] - e[:-1])[same]
    print("per-worker gap between tasks: mean %.2f us, median %.2f us, p90 %.2f us" % (gap.mean()/1e3, np.median(gap)/1e3, np.percentile(gap, 90)/1e3))
    busy = (tend - t0).sum(); span = (tend.max() - t0.min()) * (wid.max() + 1)
    print("worker time in tasks %.1f%%, in gaps %.1f%%" % (100*busy/span, 100*gap.sum()/span))

# BLOB ROW phase stamps (clock64): [0] start [1] front vector in the slot [2] products + stores issued
m = (T[:, 5] == 2) & (T[:, 12] > 0) & (T[:, 14] > 0)
if m.any():
    Pp = T[m][:, 12:24]
    tot_ns = (T[m][:, 4] - T[m][:, 3])
    print(f"row (blob): {m.sum()} tasks, data->end {tot_ns.mean()/1e3:.2f} us; front gather {np.mean(Pp[:,1]-Pp[:,0]):.0f} cycles, "
          f"products + stores {np.mean(Pp[:,2]-Pp[:,1]):.0f} cycles, mean rows {np.mean(Pp[:,11]-100):.1f}")
