#!/usr/bin/env python
"""Benchmark: PCG DOF-iterations/s of the SFC two-level Schwarz solver.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

Workload (BASELINE.json configs[1]): 2D Poisson, l=(10,10)
(1023^2 interior points), Hilbert SFC, P=64, gamma=0.5, q=16, balanced
omega-weighted Schwarz, PCG from x0=0 to relative residual 1e-8 on
b = default_rng(42).uniform(-1, 1, N).  A step = one full PCG solve.

value  = N * iterations * K / (device time of K solves), inputs resident in HBM
e2e    = same metric through the public API (krylov.run with numpy host
         buffers: H2D of b and x0, D2H of the solution and history per step)
roofline: the local-solve DAG kernel (dominant), algorithmic bytes per launch
         = 16 * sum_i nnz_alg(L_i) + 16 (1 + 2 gamma) N
cpu_baseline: the oracle port (scipy SuperLU, the reference's own third-party
         calls) on a bounded sample of PCG iterations, rank 0 only.
--impl reference: the oracle port as the timed arm (the reference is pure
         Python and cannot travel to the GPU box; oracle/ restates it and is
         pinned bit-exactly to it by tests/test_oracle_golden.py).
N > 1 (torchrun, or self-launched when --gpus N is given without it; or
       --sharded at N=1): weak scaling -- the config's member for N GPUs
       (weak_family: fixed points and subdomains per GPU), ONE solve sharded
       over the ranks by contiguous SFC segments, run by the device-driven
       program (one CUDA graph per solve, NCCL inside); "scaling": "weak";
       value = N_dof * iterations * K / (max over ranks of the device time).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (levels, P, gamma, q, description)
    "c1": ((7, 7), 16, 0.5, 4, "C1: 2D 127^2 interior (l=(7,7)), P=16, gamma=0.5, q=4"),
    "c2": ((10, 10), 64, 0.5, 16, "C2: 2D 1023^2 interior (l=(10,10)), P=64, gamma=0.5 (delta=H/4), q=16 (32x32 coarse)"),
    "c3": ((7, 7, 7), 512, 0.5, 8, "C3: 3D 127^3 interior (l=(7,7,7)), P=512, gamma=0.5, q=8 (16^3 coarse)"),
    "c4": ((12, 12), 256, 0.5, 16, "C4: 2D 4095^2 interior (l=(12,12)), P=256, gamma=0.5, q=16 (64x64 coarse); "
                                   "fault mode: apply 5 of every solve zeroes the local pieces of "
                                   "default_rng(42).choice(256, 26) (SURVEY §8(d))"),
    "c5": ((8, 8, 8), 512, 0.5, 64, "C5: 3D 255^3 interior (l=(8,8,8)), P=512, gamma=0.5, q=64 (coarse 1/8 per "
                                    "dimension: N0 = 32768), the 1-GPU point of the weak-scaling sweep"),
}
METRIC = "PCG DOF-iterations/s (SFC two-level Schwarz, Poisson)"
UNIT = "DOF-it/s"


def superlu_cap(config, p):
    """Sum over the subdomains of nnz(L) of the reference's own factorization
    (SuperLU, MMD on A^T + A), cached by tools/superlu_nnz.py from the oracle:
    the algorithmic bytes never credit the builder's extra fill.  C5: the mean
    of sampled subdomains times P."""
    f = ROOT / "profiles" / "superlu_nnz.json"
    if not f.exists():
        return None
    e = json.loads(f.read_text()).get(config)
    if not e:
        return None
    if e.get("sum_nnz_L"):
        return int(e["sum_nnz_L"])
    return int(round(e["mean_nnz_L"] * p)) if e.get("mean_nnz_L") else None


def measured_peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_oracle_sample(levels, p, gamma, q, iters, seed=42):
    """Time the oracle port's PCG on a bounded number of iterations (setup untimed)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import sfcdd_oracle as O

    t0 = time.perf_counter()
    A = O.assemble_scaled_laplacian(levels)
    n = A.shape[0]
    _, _, t = O.stencil_constants(levels)
    b = t * O.seeded_rhs(n, seed)
    op = O.BalancedSchwarz(A, n, p, gamma, q)
    t_setup = time.perf_counter() - t0
    nnz_superlu = sum(int(s._lu.L.nnz) if s._lu is not None else s.n * (s.n + 1) // 2 for s in op.local)
    O.pcg(A, b, op, max_steps=1)  # warm-up (first call in a process is slower)
    t1 = time.perf_counter()
    res = O.pcg(A, b, op, max_steps=iters)
    dt = time.perf_counter() - t1
    return {"value": n * res.iterations / dt, "iterations": res.iterations, "seconds": dt,
            "setup_seconds": t_setup, "nnz_superlu": nnz_superlu, "n": n}


def cpu_extrapolated_c5(levels, p, gamma, q, samples=(0, 301), seed=42):
    """C5 cannot be set up by the CPU port on one host (512 SuperLU factors of
    ~14 M nnz each): the CPU time per PCG iteration is
    extrapolated as P x the mean SuperLU solve time of sampled C5 subdomain
    blocks (the reference's linalg.Factorization path, 76 % of its PCG time)
    plus 3 matvecs of the full scaled operator, all measured here."""
    import scipy.sparse.linalg as spla

    sys.path.insert(0, str(ROOT / "oracle"))
    sys.path.insert(0, str(ROOT / "tests"))
    import sfc_index_c as C

    n = int(np.prod([(1 << l) - 1 for l in levels]))
    perm = C.sfc_perm(levels)
    rank = np.empty(n, np.int64)
    rank[perm] = np.arange(n)
    num, den = _gamma_fraction(gamma)
    _, _, os_, ol = C.partition(n, p, num, den)
    rng = np.random.default_rng(seed)
    t_solve, nnz = [], []
    for i in samples:
        B = C.scaled_block(levels, perm, rank, int(os_[i]), int(ol[i]))
        lu = spla.splu(B.tocsc(), permc_spec="MMD_AT_PLUS_A", options={"SymmetricMode": True})
        nnz.append(int(lu.L.nnz))
        r = rng.standard_normal(B.shape[0])
        lu.solve(r)
        t0 = time.perf_counter()
        for _ in range(3):
            lu.solve(r)
        t_solve.append((time.perf_counter() - t0) / 3)
    # one matvec of the full operator, measured on the 127^3 operator and scaled by N
    import sfcdd_oracle as O

    A3 = O.assemble_scaled_laplacian((7, 7, 7))
    x = rng.standard_normal(A3.shape[0])
    t0 = time.perf_counter()
    for _ in range(5):
        A3 @ x
    t_mv = (time.perf_counter() - t0) / 5 * n / A3.shape[0]
    t_it = p * float(np.mean(t_solve)) + 3 * t_mv
    return {"value": n / t_it, "unit": UNIT, "cores": 1, "kind": "port", "superlu_nnz_l_mean": float(np.mean(nnz)),
            "sample": f"EXTRAPOLATED: {p} x mean SuperLU solve ({1e3 * np.mean(t_solve):.1f} ms) of C5 subdomains "
                      f"{list(samples)} + 3 matvecs ({1e3 * t_mv:.1f} ms, 127^3 operator scaled by N) per PCG "
                      f"iteration, 1 of {os.cpu_count()} host threads; the port cannot set C5 up on one host"}


def _gamma_fraction(gamma):
    from fractions import Fraction

    g = Fraction(gamma).limit_denominator(10**6)
    return g.numerator, g.denominator


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    levels, p, gamma, q, desc = cfg
    sys.path.insert(0, str(ROOT / "oracle"))
    import sfcdd_oracle as O

    A = O.assemble_scaled_laplacian(levels)
    n = A.shape[0]
    _, _, t = O.stencil_constants(levels)
    b = t * O.seeded_rhs(n, 42)
    t0 = time.perf_counter()
    op = O.BalancedSchwarz(A, n, p, gamma, q)
    setup_s = time.perf_counter() - t0
    per_step = args.ref_iters
    for _ in range(args.warmup):
        O.pcg(A, b, op, max_steps=per_step)
    t1 = time.perf_counter()
    its = 0
    for _ in range(args.steps):
        its += O.pcg(A, b, op, max_steps=per_step).iterations
    dt = time.perf_counter() - t1
    value = n * its / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: b = default_rng(42).uniform(-1,1,N) (SURVEY §8(d))",
        "config": {"workload": desc, "levels": list(levels), "N": n, "P": p, "gamma": gamma, "q": q,
                   "step": f"{per_step} PCG iterations of the oracle port", "setup_seconds": setup_s},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"{args.steps} x {per_step} PCG iterations after {args.warmup} warm-up samples; "
                                   f"scipy SuperLU local solves, 1 thread of {os.cpu_count()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def weak_family(cfg, world):
    """Weak-scaling member for ``world`` GPUs (BASELINE configs[4]'s rule:
    fixed points and subdomains per GPU): one level added per doubling,
    round robin from the last axis -- C5 (8,8,8) -> (8,8,9) -> (8,9,9) ->
    (9,9,9), C2 (10,10) -> (10,11) -> (11,11) -> (11,12) -- and P x world."""
    levels, p, gamma, q, desc = cfg
    if world & (world - 1):
        raise SystemExit(f"weak scaling needs a power-of-two GPU count, got {world}")
    lv = list(levels)
    for k in range(world.bit_length() - 1):
        lv[len(lv) - 1 - (k % len(lv))] += 1
    return tuple(lv), p * world, gamma, q, f"{desc} -- weak scaling member for {world} GPU(s): levels {tuple(lv)}, " \
                                           f"P={p * world}"


def run_sharded(args, cfg):
    """N GPUs, one process per GPU: the SFC-segment-sharded solve of the
    weak-scaling member for N (weak_family), run by the device-driven program
    (distributed.attach_device_program / run_device: one CUDA graph per solve,
    NCCL send / recv and allgathers inside a conditional WHILE loop)."""
    import ctypes

    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    dist.init_process_group("nccl", device_id=dev)
    import paper_2110_11211_b200 as sf
    from paper_2110_11211_b200 import _lib
    from paper_2110_11211_b200 import distributed as D

    cfg = weak_family(cfg, world)
    levels, p, gamma, q, desc = cfg
    n = sf.num_dofs(levels)
    part = sf.build_partition(n, p, gamma)
    t0 = time.perf_counter()
    eng, plan = D.make_rank_shard(levels, part, q, rank, world, dev)
    ids = [D.nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(ids, src=0)
    D.attach_device_program(eng, plan, ids[0] if world > 1 else None)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    log(f"rank {rank}: shard setup {setup_s:.2f}s, owned points [{plan.g0}, {plan.g1})")
    A = sf.assemble_laplacian(levels)
    b = np.random.default_rng(42).uniform(-1.0, 1.0, size=n)
    _, bh, _ = sf.symmetrize_diag(A, b)
    b_dev = torch.from_numpy(bh).to(dev)
    x = torch.zeros(n, dtype=torch.float64, device=dev)

    def solve():
        x.zero_()
        its, conv, hist = D.run_device(eng, b_dev, x, 1e-8, 20000)
        return its

    for _ in range(max(args.warmup, 3)):
        its = solve()
    log(f"rank {rank}: warm-up solve {its} iterations")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    launch_total = [0]
    st_l = _lib.Stats()
    with ClockSampler(local) as clk:
        ev0.record()
        total_its = 0
        for _ in range(args.steps):
            total_its += solve()
            _lib.check(_lib.lib().sfcdd_op_stats(eng.h, ctypes.byref(st_l)))
            launch_total[0] += int(st_l.reserved[7])
        ev1.record()
        torch.cuda.synchronize()
    launches = launch_total[0]
    ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    value = n * total_its / (ms / 1e3)
    # e2e: host b in, host solution (owned segment) out, every step
    bh_pin = torch.from_numpy(bh).pin_memory()
    x_host = torch.empty(plan.g1 - plan.g0, dtype=torch.float64).pin_memory()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    e_its = 0
    for _ in range(args.steps):
        b_dev.copy_(bh_pin, non_blocking=True)
        x.zero_()
        its, _, _ = D.run_device(eng, b_dev, x, 1e-8, 20000)
        x_host.copy_(x[plan.g0:plan.g1], non_blocking=True)
        e_its += its
    e1.record()
    torch.cuda.synchronize()
    e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e2e_value = n * e_its / (float(e_ms.item()) / 1e3)
    # local-solve kernel alone on this rank's shard
    g = torch.from_numpy(np.random.default_rng(7).standard_normal(n)).to(dev)
    eng.local_solve(g)
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record()
    for _ in range(10):
        eng.local_solve(g)
    k1.record()
    torch.cuda.synchronize()
    dag_ms = k0.elapsed_time(k1) / 10
    st = _lib.Stats()
    _lib.check(_lib.lib().sfcdd_op_stats(eng.h, ctypes.byref(st)))
    if rank == 0:
        peak, peak_kind = measured_peak_gbs()
        dag_bytes = 16.0 * st.factor_nnz_l + 16.0 * (1 + 2 * gamma) * (plan.g1 - plan.g0)
        achieved = dag_bytes / (dag_ms * 1e-3) / 1e9
        its_per_solve = total_its / args.steps
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: b = default_rng(42).uniform(-1,1,N) (SURVEY §8(d)); no dataset involved",
            "config": {"workload": desc, "levels": list(levels), "N": n, "P": p, "gamma": gamma, "q": q,
                       "iterations": its_per_solve, "step": "one PCG solve to relative residual 1e-8",
                       "parallelism": f"sfc-segment sharding x{world}: device-driven program, one CUDA graph per "
                                      "solve (NCCL send/recv halo + overlap + foreign solutions, coarse and scalar "
                                      "allgathers, conditional WHILE loop)",
                       "l2": "working set > L2", "setup_seconds": setup_s},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "kernel": "k_dag (rank 0 shard)",
                         "kernel_ms": dag_ms, "peak_kind": peak_kind,
                     # the same launch under ncu --set full (cold caches, serialised; same static capture as `traffic`)
                     "kernel_ms_ncu": ncu_us / 1e3 if ncu_us else None,
                     "frac_ncu": dag_bytes / (ncu_us * 1e-6) / 1e9 / peak if ncu_us else None, "algorithmic_bytes_per_launch": dag_bytes},
            "cpu_baseline": None,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                    "d2h_bytes_per_step": 8 * (plan.g1 - plan.g0)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def run_gpu(args, cfg, config=None, emit=True, cpu_baseline=True):
    import torch

    config = config or args.config

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2110_11211_b200 as sf
    from paper_2110_11211_b200 import _lib

    levels, p, gamma, q, desc = cfg
    A = sf.assemble_laplacian(levels)
    n = A.shape[0]
    b = np.random.default_rng(42).uniform(-1.0, 1.0, size=n)
    Ah, bh, _ = sf.symmetrize_diag(A, b)
    part = sf.build_partition(n, p, gamma)
    t0 = time.perf_counter()
    op = sf.setup(Ah, part, sf.build_coarse(part, Ah, q), sf.SchwarzConfig("balanced", "omega", gamma, q))
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    if config == "c4":  # BASELINE configs[3]: fault-tolerance mode
        op.set_fault(5, np.random.default_rng(42).choice(p, size=int(round(0.1 * p)), replace=False))
    stats = op.stats()
    log(f"setup {setup_s:.2f}s stats={stats}")
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    b_dev = torch.from_numpy(bh).to(dev)
    x_dev = torch.zeros(n, dtype=torch.float64, device=dev)
    hist = np.zeros(20001)
    import ctypes

    its = ctypes.c_int32()
    conv = ctypes.c_int32()

    def solve():
        x_dev.zero_()
        _lib.check(_lib.lib().sfcdd_op_pcg(op.handle, b_dev.data_ptr(), x_dev.data_ptr(), 1e-8, 20000,
                                           hist.ctypes.data, ctypes.byref(its), ctypes.byref(conv),
                                           stream.cuda_stream))
        return its.value

    for _ in range(max(args.warmup, 3)):
        log(f"warm-up solve: {solve()} iterations")
    iters = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            iters.append(solve())
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    s_after = _lib.Stats()
    _lib.check(_lib.lib().sfcdd_op_stats(op.handle, ctypes.byref(s_after)))
    launches_per_solve = int(s_after.reserved[2])
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    total_its = sum(iters)
    value = world * n * total_its / (ms / 1e3)
    log(f"timed: {ms:.2f} ms for {args.steps} solves, {total_its} iterations")

    # e2e through the public API with host buffers (H2D b, x0; D2H x, history)
    cfgs = sf.SolverConfig(method="pcg", tolerance=1e-8, tolerance_kind="relative_residual")
    x0 = np.zeros(n)
    sf.run(Ah, bh, op, cfgs, x0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e_its = 0
    for _ in range(args.steps):
        rep = sf.run(Ah, bh, op, cfgs, x0)
        e_its += rep.iterations
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    e2e_value = world * n * e_its / (e_ms / 1e3)

    # dominant kernel: local-solve DAG, timed alone on the launching stream
    prof = np.zeros(3)
    nl = (ctypes.c_int32 * 3)()
    g_dev = torch.from_numpy(np.random.default_rng(7).standard_normal(n)).to(dev)
    scratch = torch.empty_like(g_dev)
    _lib.check(_lib.lib().sfcdd_op_profile(op.handle, g_dev.data_ptr(), scratch.data_ptr(), 10,
                                           prof.ctypes.data, nl, stream.cuda_stream))
    dag_ms, apply_ms, mv_ms = prof
    log(f"e2e {e_ms:.2f} ms; profile dag={dag_ms:.4f} apply={apply_ms:.4f} matvec={mv_ms:.4f} ms")
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_kind = measured_peak_gbs()
    cpu = None
    nnz_alg = stats["factor_nnz_l"]
    cap = superlu_cap(config, p)  # cached for every config: never credit extra fill
    nnz_src = "builder nnz(L)"
    if cap is not None and cap < nnz_alg:
        nnz_alg, nnz_src = cap, "SuperLU-MMD nnz(L) of the oracle (profiles/superlu_nnz.json)"
    do_cpu = cpu_baseline and not args.no_cpu_baseline and world == 1
    if do_cpu and config == "c5":
        cpu = cpu_extrapolated_c5(levels, p, gamma, q)
    elif do_cpu:
        cb = cpu_oracle_sample(levels, p, gamma, q, args.cpu_iters)
        if cb["nnz_superlu"] < nnz_alg:
            nnz_alg, nnz_src = cb["nnz_superlu"], "SuperLU-MMD nnz(L) of the oracle (this run)"
        cpu = {"value": cb["value"], "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"ORACLE PORT (oracle/sfcdd_oracle.py: the reference's scipy SuperLU solves and numpy "
                         f"kernels, pinned bit-exactly to the reference; not the reference package itself): "
                         f"{cb['iterations']} PCG iterations on {desc.split(':')[0]}, 1 of {os.cpu_count()} host "
                         f"threads (the reference's thread pool does not parallelise SuperLU solves), setup "
                         f"{cb['setup_seconds']:.1f}s untimed"}
    dag_bytes = 16.0 * nnz_alg + 16.0 * (1 + 2 * gamma) * n
    achieved = dag_bytes / (dag_ms * 1e-3) / 1e9
    its_per_solve = total_its / args.steps
    # whole PCG iteration: B_iter = 8 V N (V = 15 vector passes) + 16 sum nnz_alg(L_i) + 32 nnz(L0)
    iter_ms = ms / args.steps / its_per_solve
    iter_bytes = 8.0 * 15 * n + 16.0 * nnz_alg + 32.0 * stats["coarse_nnz"]
    traffic, traffic_src, ncu_us = None, None, None
    tp = ROOT / "profiles" / "dag_traffic.json"
    if tp.exists():
        try:
            tj = json.loads(tp.read_text())
            traffic = tj.get(config)
            traffic_src = tj.get("_source") if traffic is not None else None
            ncu_us = tj.get(config + "_duration_us")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: b = default_rng(42).uniform(-1,1,N) (SURVEY §8(d)); no dataset involved",
        "config": {"workload": desc, "levels": list(levels), "N": n, "P": p, "gamma": gamma, "q": q,
                   "iterations": its_per_solve, "step": "one PCG solve to relative residual 1e-8",
                   "parallelism": "replicas" if world > 1 else "single-gpu",
                   "l2": "working set > L2 (factor blobs %.2f GB per sweep)" % (8e-9 * stats["factor_nnz"]),
                   "setup_seconds": setup_s,
                   "setup_phases_s": {"order_symbolic": stats["order_seconds"], "plan": stats["plan_seconds"],
                                      "numeric_wall": stats["factor_seconds"],
                                      "numeric_device": stats["numeric_device_seconds"]},
                   "factor_nnz_stored": stats["factor_nnz"],
                   "factor_nnz_l": stats["factor_nnz_l"], "dag_tasks": stats["num_tasks"]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": traffic_src, "kernel": "k_dag (local solves)",
                     "kernel_ms": dag_ms, "peak_kind": peak_kind,
                     # the same launch under ncu --set full (cold caches, serialised; same static capture as `traffic`)
                     "kernel_ms_ncu": ncu_us / 1e3 if ncu_us else None,
                     "frac_ncu": dag_bytes / (ncu_us * 1e-6) / 1e9 / peak if ncu_us else None,
                     "algorithmic_bytes_per_launch": dag_bytes, "nnz_alg": nnz_alg, "nnz_alg_source": nnz_src},
        "breakdown_ms": {"pcg_iteration": iter_ms, "apply": apply_ms,
                         "local_solves": dag_ms, "matvec": mv_ms},
        "iteration_roofline": {"bound": "hbm", "bytes": iter_bytes, "achieved": iter_bytes / (iter_ms * 1e-3) / 1e9,
                               "peak": peak, "unit": "GB/s", "frac": iter_bytes / (iter_ms * 1e-3) / 1e9 / peak,
                               "formula": "8*15*N + 16*sum nnz_alg(L_i) + 32*nnz(L0) per PCG iteration (SURVEY 8(d))"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * 8 * n,
                "d2h_bytes_per_step": 8 * n + 8 * (int(its_per_solve) + 1)},
        "gpu_launches": launches_per_solve * args.steps,
        "clocks": clk.summary(),
    }
    if dist:
        dist.destroy_process_group()
    if emit:
        print(json.dumps(line), flush=True)
    return line


def log(msg):
    print(f"[bench] {msg}", file=sys.stderr, flush=True)


def main():
    import faulthandler

    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-iters", type=int, default=4, help="PCG iterations per reference step")
    ap.add_argument("--cpu-iters", type=int, default=30, help="PCG iterations in the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="use the multi-GPU sharded path even at N=1")
    ap.add_argument("--also", default=None,
                    help="comma-separated extra configs measured in the same run and reported under \"also\" "
                         "(default: c3,c4 when the headline config c2 runs on one GPU; \"none\" disables)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    _, world, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched without torchrun: start the N ranks ourselves, the way the
        # driver does (one process per GPU, rendezvous on 127.0.0.1)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
               *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    if world > 1 and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} does not match WORLD_SIZE {world}")
    if args.impl == "reference":
        run_reference(args, cfg)
    elif world > 1 or args.sharded:
        run_sharded(args, cfg)
    else:
        also = args.also if args.also is not None else ("c3,c4" if args.config == "c2" and world == 1 else "none")
        names = [a for a in also.split(",") if a and a != "none"]
        if not names:
            run_gpu(args, cfg)
            return
        t_start = time.perf_counter()
        line = run_gpu(args, cfg, emit=False)
        extra = []
        for nm in names:  # the other single-GPU BASELINE configs, same timing rules, fewer steps
            if time.perf_counter() - t_start > 240:
                extra.append({"config": nm, "skipped": "time budget of the default run"})
                continue
            try:
                sub = argparse.Namespace(**vars(args))
                sub.steps = min(args.steps, 2)
                l2 = run_gpu(sub, CONFIGS[nm], config=nm, emit=False, cpu_baseline=False)
                extra.append({"config": nm, "workload": l2["config"]["workload"], "value": l2["value"], "unit": UNIT,
                              "steps": l2["steps"], "ms_per_step": l2["ms_per_step"],
                              "iterations": l2["config"]["iterations"], "e2e": l2["e2e"]["value"],
                              "roofline_frac": l2["roofline"]["frac"], "kernel_ms": l2["roofline"]["kernel_ms"],
                              "iteration_roofline_frac": l2["iteration_roofline"]["frac"],
                              "setup_seconds": l2["config"]["setup_seconds"], "clocks": l2["clocks"]})
            except Exception as e:  # the headline line must survive
                extra.append({"config": nm, "error": repr(e)[:300]})
        line["also"] = extra
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
