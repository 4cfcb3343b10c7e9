"""Multi-GPU balanced-Schwarz PCG: SFC-segment sharding.

Rank g owns the contiguous block of subdomains S_g = [P g / G, P (g+1) / G),
i.e. one contiguous SFC segment O_g of points and the aggregates of those
subdomains; only S_g is factorized on rank g (C-ABI shard mode).  Vectors are
full length N on every rank but each step computes O_g only.  Per PCG
iteration the exchanges are exactly the ones the algorithm needs:

* stencil halo of z, p_old (p = z + beta p_old is formed on the fly at
  neighbours) and of w (for R0 Â w) -- points adjacent to O_g owned elsewhere;
* overlap extension of t = g - Â R0^T y0 (the owned subdomains' ranges
  reach half a subdomain into the neighbouring segments, cyclically: the
  wrap-around couples rank 0 and rank G-1, partition.py:115);
* foreign local solutions: the pieces of neighbours' subdomain solutions
  that cover O_g, combined in fixed subdomain order (schwarz.py:97-100);
* allgather of the owned coarse restrictions (R0 r, R0 Â w) -- every rank
  then solves the full coarse problem redundantly (Bank-Holst,
  PAPER.md:191);
* allreduce of the CG scalars (p.Ap, ||r||^2, r.z).

The algorithm is written once as an SPMD generator (`pcg_program`) that
yields its collectives; `run_torch` executes it with torch.distributed
(NCCL on GPUs, gloo on CPU) and `run_lockstep` steps several ranks in one
process (used to exercise the multi-rank path on a single GPU without any
kernel waiting on another rank).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib


def block_owner(p: int, g: int) -> np.ndarray:
    """Rank of every subdomain: contiguous blocks, first P mod G get one more."""
    base, extra = divmod(p, g)
    sizes = [base + (1 if r < extra else 0) for r in range(g)]
    return np.repeat(np.arange(g), sizes)


@dataclass
class Exchange:
    """Point-to-point value exchange: per peer, indices into the local source
    buffer to send and indices into the local destination buffer to fill."""

    send: dict = field(default_factory=dict)  # peer -> int64 indices
    recv: dict = field(default_factory=dict)  # peer -> int64 indices


@dataclass
class ShardPlan:
    rank: int
    world: int
    first: int            # first owned subdomain
    count: int            # owned subdomains
    g0: int               # owned points [g0, g1)
    g1: int
    a0: int               # owned aggregates [a0, a1)
    a1: int
    n0: int
    agg_counts: list      # owned aggregates per rank (allgather layout)
    halo: Exchange
    ext: Exchange
    xy: Exchange


def build_plans(part, q: int, world: int, nbr: np.ndarray, xy_offsets: list) -> list:
    """Exchange plans of all ranks (every rank computes all, deterministically).

    ``nbr``: int32 [2d, N] stencil neighbour table in SFC order (-1 outside);
    ``xy_offsets[g]``: per-subdomain slot offsets in rank g's xy buffer.
    """
    n, p = part.n, part.p
    owner_sub = block_owner(p, world)
    dj_start = np.array([r.start for r in part.disjoint], np.int64)
    dj_end = dj_start + np.array([r.length for r in part.disjoint], np.int64)
    ov_start = np.array([r.start for r in part.overlapped], np.int64)
    ov_len = np.array([r.length for r in part.overlapped], np.int64)
    # owner rank of every point
    seg = np.zeros(world + 1, np.int64)
    firsts = [int(np.argmax(owner_sub == g)) for g in range(world)]
    counts = [int((owner_sub == g).sum()) for g in range(world)]
    for g in range(world):
        seg[g] = dj_start[firsts[g]]
    seg[world] = n
    def owner_of(pts):
        return np.searchsorted(seg, pts, side="right") - 1

    plans = []
    for g in range(world):
        g0, g1 = int(seg[g]), int(seg[g + 1])
        own = np.arange(g0, g1, dtype=np.int64)
        plans.append(ShardPlan(g, world, firsts[g], counts[g], g0, g1, firsts[g] * q,
                               (firsts[g] + counts[g]) * q, p * q, [c * q for c in counts],
                               Exchange(), Exchange(), Exchange()))
        # stencil halo
        nb = nbr[:, g0:g1].astype(np.int64).ravel()
        nb = np.unique(nb[nb >= 0])
        halo = nb[(nb < g0) | (nb >= g1)]
        # overlap extension of the owned subdomains' ranges
        ext = []
        for i in range(firsts[g], firsts[g] + counts[g]):
            idx = (ov_start[i] + np.arange(ov_len[i])) % n
            ext.append(idx[(idx < g0) | (idx >= g1)])
        ext = np.unique(np.concatenate(ext)) if ext else np.zeros(0, np.int64)
        for name, pts in (("halo", halo), ("ext", ext)):
            own_of = owner_of(pts)
            for h in np.unique(own_of):
                sel = np.sort(pts[own_of == h])
                getattr(plans[g], name).recv[int(h)] = sel
        del own
    # senders mirror the receivers (same global indices)
    for g in range(world):
        for name in ("halo", "ext"):
            for h, idx in getattr(plans[g], name).recv.items():
                getattr(plans[h], name).send[g] = idx
    # foreign local solutions covering owned points
    for g in range(world):
        g0, g1 = plans[g].g0, plans[g].g1
        for j in range(p):
            h = int(owner_sub[j])
            if h == g:
                continue
            ro = np.arange(ov_len[j], dtype=np.int64)
            pts = (ov_start[j] + ro) % n
            sel = (pts >= g0) & (pts < g1)
            if not sel.any():
                continue
            ro = ro[sel]
            dst = xy_offsets[g][j]
            src = xy_offsets[h][j]
            assert dst >= 0 and src >= 0, "missing xy slot"
            plans[g].xy.recv.setdefault(h, []).append(dst + ro)
            plans[h].xy.send.setdefault(g, []).append(src + ro)
    for g in range(world):
        for d in (plans[g].xy.recv, plans[g].xy.send):
            for k in list(d):
                d[k] = np.concatenate(d[k]).astype(np.int64)
    return plans


# ----------------------------------------------------------- SPMD program
class Req:
    def __init__(self, kind, *args):
        self.kind = kind
        self.args = args


def pcg_program(eng, plan: ShardPlan, b, x, tol: float, max_iters: int):
    """Balanced two-level Schwarz PCG (krylov.py:257-291) on one rank.

    ``b``, ``x``: full-length vectors (owned part meaningful; x holds x0 and
    receives the solution on the owned segment).  Yields collective requests;
    returns (iterations, converged, residual_history).
    """
    r, z, w, t = eng.zeros(), eng.zeros(), eng.zeros(), eng.zeros()
    pa, pb, ap = eng.zeros(), eng.zeros(), eng.zeros()

    def apply(g, cagg):
        c = yield Req("allgather", cagg)
        y0 = eng.coarse(c)
        eng.tvec(g, y0, t)
        yield Req("exchange", "ext", t)
        eng.local_solve(t)
        yield Req("exchange", "xy", eng.xy())
        eng.combine(w)
        yield Req("exchange", "halo", w)
        c2 = yield Req("allgather", eng.stencil_restrict(w))
        y0b = eng.coarse(c2)
        rz_l = eng.finalize(w, y0, y0b, z, g)
        rz = yield Req("allreduce", rz_l)
        return rz

    yield Req("exchange", "halo", x)
    rr_l, cagg = eng.residual(b, x, r)
    rr0 = yield Req("allreduce", rr_l)
    h0 = math.sqrt(rr0)
    hist = [h0]
    if h0 <= tol * h0:
        return 0, True, hist
    rz = yield from apply(r, cagg)
    beta = 0.0
    pold, pnew = pa, pb
    for k in range(1, max_iters + 1):
        yield Req("exchange", "halo", z)
        yield Req("exchange", "halo", pold)
        pap = yield Req("allreduce", eng.pm(z, pold, beta, pnew, ap))
        if not pap > 0.0:
            raise _lib.BreakdownError(f"nonpositive curvature at iteration {k}")
        alpha = rz / pap
        rr_l, cagg = eng.update(x, r, pnew, ap, alpha)
        rr = yield Req("allreduce", rr_l)
        hist.append(math.sqrt(rr))
        if hist[-1] <= tol * h0:
            return k, True, hist
        rz_new = yield from apply(r, cagg)
        beta = rz_new / rz
        rz = rz_new
        pold, pnew = pnew, pold
    return max_iters, False, hist


# ---------------------------------------------------------------- drivers
def _drive(gen, handle):
    res = None
    try:
        while True:
            req = gen.send(res)
            res = handle(req)
    except StopIteration as stop:
        return stop.value


def run_torch(eng, plan: ShardPlan, b, x, tol=1e-8, max_iters=20000, group=None):
    """Execute one rank's program with torch.distributed collectives.  With a
    gloo group and device engines the collective buffers are staged through
    host memory (gloo has no CUDA all_to_all); the kernels stay on the GPU."""
    import torch
    import torch.distributed as dist

    stage = dist.get_backend(group) == "gloo" and getattr(eng, "dev", None) is not None and \
        getattr(eng.dev, "type", "cpu") == "cuda"

    def host(t):
        return t.cpu() if stage else t

    def back(t):
        return t.to(eng.dev) if stage else t

    def exchange(kind, buf):
        ex = getattr(plan, kind)
        world = plan.world
        send_parts, send_counts, recv_counts = [], [], []
        for h in range(world):
            idx = ex.send.get(h)
            send_counts.append(0 if idx is None else len(idx))
            if idx is not None and len(idx):
                send_parts.append(eng.pack(buf, eng.index(kind, "send", h)))
            recv_counts.append(0 if ex.recv.get(h) is None else len(ex.recv[h]))
        sendbuf = host(torch.cat(send_parts) if send_parts else eng.empty(0))
        recvbuf = host(eng.empty(sum(recv_counts)))
        dist.all_to_all_single(recvbuf, sendbuf, recv_counts, send_counts, group=group)
        recvbuf = back(recvbuf)
        off = 0
        for h in range(world):
            if recv_counts[h]:
                eng.unpack(buf, eng.index(kind, "recv", h), recvbuf[off:off + recv_counts[h]])
                off += recv_counts[h]

    def handle(req):
        if req.kind == "exchange":
            exchange(*req.args)
            return None
        if req.kind == "allreduce":
            v = host(req.args[0].clone())
            dist.all_reduce(v, group=group)
            return float(v.item())
        if req.kind == "allgather":
            part = req.args[0]
            mx = max(plan.agg_counts)
            pad = host(eng.empty(mx))
            pad[: part.numel()] = host(part)
            outs = [host(eng.empty(mx)) for _ in range(plan.world)]
            dist.all_gather(outs, pad, group=group)
            return back(torch.cat([o[: plan.agg_counts[h]] for h, o in enumerate(outs)]))
        raise ValueError(req.kind)

    return _drive(pcg_program(eng, plan, b, x, tol, max_iters), handle)


def run_lockstep(engines, plans, bs, xs, tol=1e-8, max_iters=20000):
    """All ranks in one process, stepped together at every collective.  Host
    sequenced: no kernel of one rank ever waits on another rank's kernel."""
    import torch

    world = len(engines)
    gens = [pcg_program(engines[g], plans[g], bs[g], xs[g], tol, max_iters) for g in range(world)]
    results = [None] * world
    done = [False] * world
    reqs = [None] * world
    outs = [None] * world
    while not all(done):
        for g in range(world):
            if done[g]:
                continue
            try:
                reqs[g] = gens[g].send(outs[g])
            except StopIteration as stop:
                results[g] = stop.value
                done[g] = True
        if all(done):
            break
        assert not any(done), "ranks diverged"
        kind = reqs[0].kind
        assert all(r.kind == kind for r in reqs)
        if kind == "exchange":
            name = reqs[0].args[0]
            bufs = [r.args[1] for r in reqs]
            staged = {}
            for g in range(world):
                for h, idx in getattr(plans[g], name).send.items():
                    staged[(g, h)] = engines[g].pack(bufs[g], engines[g].index(name, "send", h)).clone()
            for g in range(world):
                for h in getattr(plans[g], name).recv:
                    engines[g].unpack(bufs[g], engines[g].index(name, "recv", h), staged[(h, g)])
            outs = [None] * world
        elif kind == "allreduce":
            tot = sum(float(r.args[0].item()) for r in reqs)
            outs = [tot] * world
        elif kind == "allgather":
            full = torch.cat([r.args[0] for r in reqs])
            outs = [full.clone() for _ in range(world)]
        else:
            raise ValueError(kind)
    return results


# ------------------------------------------------------ device engine
class DeviceShardEngine:
    """One rank's shard of the Schwarz operator on its CUDA device (C ABI)."""

    def __init__(self, levels, part, q: int, omega, rank: int, world: int, device=None,
                 weighting: str = "omega"):
        import torch

        self.torch = torch
        self.dev = device if device is not None else _lib.device()
        owner = block_owner(part.p, world)
        first = int(np.argmax(owner == rank))
        count = int((owner == rank).sum())
        ov_start = np.array([r.start for r in part.overlapped], np.int64)
        ov_len = np.array([r.length for r in part.overlapped], np.int64)
        dj_start = np.array([r.start for r in part.disjoint], np.int64)
        dj_len = np.array([r.length for r in part.disjoint], np.int64)
        om = np.ascontiguousarray(omega, dtype=np.float64)
        desc = _lib.OpDesc()
        desc.dim = len(levels)
        for j, l in enumerate(levels):
            desc.levels[j] = l
        desc.p, desc.q = part.p, q
        desc.variant = _lib.VARIANT_CODES["balanced"]
        desc.weighting = _lib.WEIGHTING_CODES[weighting]
        desc.device = self.dev.index
        desc.ov_start, desc.ov_len = ov_start.ctypes.data, ov_len.ctypes.data
        desc.dj_start, desc.dj_len = dj_start.ctypes.data, dj_len.ctypes.data
        desc.omega = om.ctypes.data
        desc.host_threads = _lib.host_threads()
        desc.shard_first, desc.shard_count = first, count
        h = ctypes.c_void_p()
        L = _lib.lib()
        with torch.cuda.device(self.dev):
            _lib.check(L.sfcdd_op_create(ctypes.byref(desc), ctypes.byref(h)))
            self.h = h
            _lib.check(L.sfcdd_op_setup(h, None))
        self.n = part.n
        self.p = part.p
        info = np.zeros(8, np.int64)
        self.xy_offsets = np.zeros(part.p, np.int64)
        _lib.check(L.sfcdd_shard_info(h, info.ctypes.data, self.xy_offsets.ctypes.data))
        self.g0, self.g1, self.ch0, self.ch1, self.a0, self.a1, self.xy_len, self.n0 = (int(v) for v in info)
        ptr = ctypes.c_void_p()
        _lib.check(L.sfcdd_shard_xy(h, ctypes.byref(ptr)))
        self._xy_ptr = ptr.value
        self._xy = self._wrap(ptr.value, self.xy_len)
        self._idx = {}
        self.launches = 0  # kernels this engine launched (bench.py's gpu_launches)

    def __del__(self):
        try:
            _lib.lib().sfcdd_op_destroy(self.h)
        except Exception:
            pass

    def _wrap(self, ptr, n):
        """torch view of a device buffer owned by the C ABI (no copy)."""
        torch = self.torch

        class _Buf:
            __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}

        return torch.as_tensor(_Buf(), device=self.dev)

    def neighbors(self, d: int) -> np.ndarray:
        out = np.empty((2 * d, self.n), np.int32)
        _lib.check(_lib.lib().sfcdd_op_neighbors(self.h, out.ctypes.data))
        return out

    def attach_plan(self, plan: ShardPlan):
        torch = self.torch
        for name in ("halo", "ext", "xy"):
            ex = getattr(plan, name)
            for side in ("send", "recv"):
                for h, idx in getattr(ex, side).items():
                    self._idx[(name, side, h)] = torch.from_numpy(np.ascontiguousarray(idx)).to(self.dev)

    # -- helpers used by the drivers
    def index(self, kind, side, peer):
        return self._idx[(kind, side, peer)]

    def zeros(self):
        return self.torch.zeros(self.n, dtype=self.torch.float64, device=self.dev)

    def empty(self, n):
        return self.torch.empty(n, dtype=self.torch.float64, device=self.dev)

    def pack(self, buf, idx):
        out = self.empty(idx.numel())
        self.launches += idx.numel() > 0
        _lib.check(_lib.lib().sfcdd_pack(buf.data_ptr(), idx.data_ptr(), idx.numel(), out.data_ptr(),
                                         self._stream()))
        return out

    def unpack(self, buf, idx, vals):
        vals = vals.contiguous()
        self.launches += idx.numel() > 0
        _lib.check(_lib.lib().sfcdd_unpack(vals.data_ptr(), idx.data_ptr(), idx.numel(), buf.data_ptr(),
                                           self._stream()))

    def _stream(self):
        return self.torch.cuda.current_stream(self.dev).cuda_stream

    def xy(self):
        return self._xy

    # -- algorithm steps (owned segment only)
    def residual(self, b, x, r):
        rr = self.empty(1)
        ca = self.empty(self.a1 - self.a0)
        self.launches += 3
        _lib.check(_lib.lib().sfcdd_shard_residual(self.h, b.data_ptr(), x.data_ptr(), r.data_ptr(), rr.data_ptr(),
                                                   ca.data_ptr(), self._stream()))
        return rr, ca

    def coarse(self, c):
        y = self.empty(self.n0)
        c = c.contiguous()
        self.launches += 1
        _lib.check(_lib.lib().sfcdd_shard_coarse(self.h, c.data_ptr(), y.data_ptr(), self._stream()))
        return y

    def tvec(self, g, y0, t):
        self.launches += 1
        _lib.check(_lib.lib().sfcdd_shard_tvec(self.h, g.data_ptr(), y0.data_ptr(), t.data_ptr(), self._stream()))

    def local_solve(self, t):
        self.launches += 1
        _lib.check(_lib.lib().sfcdd_shard_local_solve(self.h, t.data_ptr(), self._stream()))

    def combine(self, w):
        self.launches += 1
        _lib.check(_lib.lib().sfcdd_shard_combine(self.h, w.data_ptr(), self._stream()))

    def stencil_restrict(self, w):
        ca = self.empty(self.a1 - self.a0)
        self.launches += 2
        _lib.check(_lib.lib().sfcdd_shard_stencil_restrict(self.h, w.data_ptr(), ca.data_ptr(), self._stream()))
        return ca

    def finalize(self, w, y0, y0b, z, r):
        rz = self.empty(1)
        self.launches += 2
        _lib.check(_lib.lib().sfcdd_shard_finalize(self.h, w.data_ptr(), y0.data_ptr(), y0b.data_ptr(), z.data_ptr(),
                                                   r.data_ptr(), rz.data_ptr(), self._stream()))
        return rz

    def pm(self, z, pold, beta, pnew, ap):
        pap = self.empty(1)
        self.launches += 2
        _lib.check(_lib.lib().sfcdd_shard_pm(self.h, z.data_ptr(), pold.data_ptr(), float(beta), pnew.data_ptr(),
                                             ap.data_ptr(), pap.data_ptr(), self._stream()))
        return pap

    def update(self, x, r, p, ap, alpha):
        rr = self.empty(1)
        ca = self.empty(self.a1 - self.a0)
        self.launches += 3
        _lib.check(_lib.lib().sfcdd_shard_update(self.h, x.data_ptr(), r.data_ptr(), p.data_ptr(), ap.data_ptr(),
                                                 float(alpha), rr.data_ptr(), ca.data_ptr(), self._stream()))
        return rr, ca


# ------------------------------------------ device-driven program (C ABI)
KINDS = {"halo": 0, "ext": 1, "xy": 2}


def nccl_unique_id() -> bytes:
    """128-byte NCCL id for rank 0 to broadcast (sfcdd_nccl_unique_id)."""
    buf = ctypes.create_string_buffer(128)
    _lib.check(_lib.lib().sfcdd_nccl_unique_id(buf))
    return buf.raw


def attach_device_program(eng: DeviceShardEngine, plan: ShardPlan, nccl_id: bytes | None = None) -> None:
    """Hand the rank's exchange plan and communicator to the C ABI so that
    ``run_device`` runs the whole sharded solve as one CUDA graph (NCCL
    send / recv and allgathers inside, conditional WHILE loop)."""
    L = _lib.lib()
    counts = np.ascontiguousarray(plan.agg_counts, np.int64)
    _lib.check(L.sfcdd_shard_attach(eng.h, nccl_id, plan.rank, plan.world, counts.ctypes.data))
    for name, kind in KINDS.items():
        ex = getattr(plan, name)
        peers = sorted(set(ex.send) | set(ex.recv))
        empty = np.zeros(0, np.int64)
        sends = [np.ascontiguousarray(ex.send.get(h, empty), np.int64) for h in peers]
        recvs = [np.ascontiguousarray(ex.recv.get(h, empty), np.int64) for h in peers]
        pa = np.asarray(peers, np.int32)
        ns = np.asarray([len(a) for a in sends], np.int64)
        nr = np.asarray([len(a) for a in recvs], np.int64)
        si = np.concatenate(sends) if sends else empty
        ri = np.concatenate(recvs) if recvs else empty
        _lib.check(L.sfcdd_shard_set_exchange(eng.h, kind, len(peers), pa.ctypes.data, ns.ctypes.data,
                                              si.ctypes.data, nr.ctypes.data, ri.ctypes.data))


def run_device(eng: DeviceShardEngine, b, x, tol=1e-8, max_iters=20000):
    """One sharded solve through sfcdd_shard_pcg: (iterations, converged,
    residual history); x receives the owned segment of the solution."""
    hist = np.zeros(max_iters + 1)
    its, conv = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(_lib.lib().sfcdd_shard_pcg(eng.h, b.data_ptr(), x.data_ptr(), float(tol), int(max_iters),
                                          hist.ctypes.data, ctypes.byref(its), ctypes.byref(conv), eng._stream()))
    return its.value, bool(conv.value), hist[:its.value + 1].tolist()


def xy_offsets_for(part, world: int, rank: int) -> np.ndarray:
    """Slot layout of rank's xy buffer, identical to the C ABI's shard setup:
    owned subdomains first, then every other subdomain whose overlapped range
    covers an owned point, in subdomain order."""
    owner = block_owner(part.p, world)
    first = int(np.argmax(owner == rank))
    count = int((owner == rank).sum())
    g0 = part.disjoint[first].start
    last = part.disjoint[first + count - 1]
    g1 = last.start + last.length
    n = part.n
    off = np.full(part.p, -1, np.int64)
    pos = 0
    for i in range(first, first + count):
        off[i] = pos
        pos += part.overlapped[i].length
    for j, r in enumerate(part.overlapped):
        if first <= j < first + count:
            continue
        if (g0 - r.start) % n < r.length or g0 <= r.start < g1:
            off[j] = pos
            pos += r.length
    return off


def make_rank_shard(levels, part, q: int, rank: int, world: int, device=None):
    """This rank's engine and exchange plan (one process per GPU, torchrun)."""
    from .partition import compute_weights

    eng = DeviceShardEngine(levels, part, q, compute_weights(part).omega, rank, world, device)
    offs = [xy_offsets_for(part, world, g) for g in range(world)]
    if not np.array_equal(offs[rank], eng.xy_offsets):
        raise RuntimeError("xy slot layout mismatch between host plan and C ABI")
    plans = build_plans(part, q, world, eng.neighbors(len(levels)), offs)
    eng.attach_plan(plans[rank])
    return eng, plans[rank]


def make_device_shards(levels, part, q: int, world: int, device=None):
    """All ranks' engines + plans in one process (lockstep emulation / tests)."""
    from .partition import compute_weights

    omega = compute_weights(part).omega
    engines = [DeviceShardEngine(levels, part, q, omega, g, world, device) for g in range(world)]
    nbr = engines[0].neighbors(len(levels))
    plans = build_plans(part, q, world, nbr, [e.xy_offsets for e in engines])
    for e, pl in zip(engines, plans):
        e.attach_plan(pl)
    return engines, plans
