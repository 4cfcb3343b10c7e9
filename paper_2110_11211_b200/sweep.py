"""Batched execution of many independent device solves over every GPU.

The experiment sweeps (harness.py) and the combination technique
(combine.py) are, at the solver level, long lists of independent
Poisson solves -- the paper's first level of parallelism.
The reference runs them one after the other or on a thread pool of one CPU
(harness.py:142-204, combine.py:199-248).  Here a list of ``SolveJob``s is
spread over the GPUs of the node: one worker process per device (the C ABI
handles are per device; processes avoid any GIL or context contention) and,
inside a process, ``streams`` threads each driving the device on a private
CUDA stream, so small grids that cannot fill 148 SMs alone overlap.  Jobs go
to devices longest-first onto the least loaded device (LPT on N (1 + 2 gamma),
the streamed bytes of one iteration); outcomes come back in job order and are
independent of the schedule (every device solve is bitwise deterministic).

Two problem kinds cover both callers:
  * ``model``: A x = 0 after the symmetric diagonal scaling, from a seeded
    unit-energy iterate, stopping on the energy error (harness.py:75-105);
  * ``manufactured``: the manufactured Poisson problem sampled on the grid,
    x0 = 0, relative-residual stopping, solution scaled back to the
    unscaled unknowns (combine.py:161-196).
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ProcessPoolExecutor, ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import grid, krylov, schwarz
from .coarse import build_coarse
from .partition import build_partition


@dataclass(frozen=True)
class SolveJob:
    levels: tuple[int, ...]
    p: int
    gamma: float
    q: int
    problem: str = "model"  # | "manufactured"
    method: str = "pcg"
    variant: str = "balanced"
    weighting: str = "omega"
    tolerance: float = 1e-8
    seed: int = 42
    eig_iters: int | None = None
    max_iters: int = 20000
    workers: int = 1

    def cost(self) -> float:
        """Streamed bytes of one iteration, up to a constant (LPT weight)."""
        return grid.num_dofs(self.levels) * (1.0 + 2.0 * self.gamma)


@dataclass
class SolveOutcome:
    job: SolveJob
    report: krylov.SolveReport | None = None
    values: np.ndarray | None = None  # manufactured: solution in unscaled unknowns, SFC order
    error: str | None = None
    device: int = -1
    params: dict = field(default_factory=dict)


def solve_job(job: SolveJob) -> SolveOutcome:
    """One device solve (grid, partition, coarse space, Schwarz setup and the
    outer solver of this package)."""
    levels = grid.as_levels(job.levels)
    A = grid.assemble_laplacian(levels)
    n = A.shape[0]
    if job.problem == "model":
        b = np.zeros(n)
    elif job.problem == "manufactured":
        b = grid.sample_on_grid(grid.manufactured_poisson(levels).rhs, levels)
    else:
        raise ValueError(f"unknown problem kind {job.problem!r}")
    A_hat, b_hat, t = grid.symmetrize_diag(A, b)
    part = build_partition(n, job.p, job.gamma)
    cs = build_coarse(part, A_hat, job.q) if job.variant != "one_level" else None
    op = schwarz.setup(A_hat, part, cs, schwarz.SchwarzConfig(job.variant, job.weighting, job.gamma, job.q),
                       workers=job.workers)
    if job.problem == "model":
        # energy stopping against the exact solution 0; the scaled energy
        # norm equals the unscaled one (x = T x_hat)
        x0, exact, kind = krylov.initial_iterate(n, job.seed, A_hat), np.zeros(n), "energy_error_reduction"
    else:
        x0, exact, kind = np.zeros(n), None, "relative_residual"
    cfg = krylov.SolverConfig(method=job.method, tolerance=job.tolerance, tolerance_kind=kind,
                              max_iters=job.max_iters, seed=job.seed, eig_iters=job.eig_iters)
    report = krylov.run(A_hat, b_hat, op, cfg, x0, exact=exact)
    params = {"d": len(levels), "levels": levels, "N": n, "P": job.p, "gamma": job.gamma, "q": job.q,
              "variant": job.variant, "weighting": job.weighting, "method": job.method, "seed": job.seed}
    report.params.update(params)
    values = t * np.asarray(report.solution) if job.problem == "manufactured" else None
    return SolveOutcome(job, report, values, params=params)


def _safe(job: SolveJob) -> SolveOutcome:
    try:
        return solve_job(job)
    except Exception as exc:  # noqa: BLE001 - reported per job
        return SolveOutcome(job, error=f"{type(exc).__name__}: {exc}")


def _run_on_device(device: int, jobs: list[SolveJob], streams: int) -> list[SolveOutcome]:
    """All jobs of one device: ``streams`` threads, each on a private stream."""
    import torch

    torch.cuda.set_device(device)
    local = threading.local()

    def work(job):
        if not hasattr(local, "stream"):
            local.stream = torch.cuda.Stream(device=device)
        with torch.cuda.stream(local.stream):
            out = _safe(job)
            local.stream.synchronize()
        out.device = device
        return out

    if streams <= 1:
        return [work(j) for j in jobs]
    with ThreadPoolExecutor(max_workers=streams) as pool:
        return list(pool.map(work, jobs))


def assign(jobs: list[SolveJob], ndev: int) -> list[list[int]]:
    """Longest-processing-time assignment of job indices to devices (ties:
    lower job index first, lower device first): deterministic."""
    order = sorted(range(len(jobs)), key=lambda i: (-jobs[i].cost(), i))
    load = [0.0] * ndev
    out: list[list[int]] = [[] for _ in range(ndev)]
    for i in order:
        d = min(range(ndev), key=lambda k: (load[k], k))
        out[d].append(i)
        load[d] += jobs[i].cost()
    for lst in out:
        lst.sort()
    return out


def visible_devices() -> list[int]:
    import torch

    return list(range(torch.cuda.device_count()))


def execute(jobs: list[SolveJob], devices: list[int] | None = None, streams: int = 1) -> list[SolveOutcome]:
    """Run ``jobs`` on ``devices`` (default: the current device only;
    ``devices="all"`` or a list spreads them, one process per device) with
    ``streams`` concurrent solves per device.  Outcomes in job order; a
    failed job carries ``error`` instead of a report."""
    jobs = list(jobs)
    if not jobs:
        return []
    if devices == "all":
        devices = visible_devices()
    if not devices:
        from . import _lib

        devices = [_lib.device().index]
    if len(devices) == 1:
        return _run_on_device(devices[0], jobs, streams)
    parts = assign(jobs, len(devices))
    out: list[SolveOutcome | None] = [None] * len(jobs)
    import multiprocessing as mp

    ctx = mp.get_context("spawn")  # CUDA cannot be forked
    env_path = os.pathsep.join(filter(None, [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                             os.environ.get("PYTHONPATH", "")]))
    os.environ["PYTHONPATH"] = env_path
    with ProcessPoolExecutor(max_workers=len(devices), mp_context=ctx) as pool:
        futs = [pool.submit(_run_on_device, dev, [jobs[i] for i in idx], streams)
                for dev, idx in zip(devices, parts) if idx]
        for fut, idx in zip(futs, [p for p in parts if p]):
            for i, res in zip(idx, fut.result()):
                out[i] = res
    return out  # type: ignore[return-value]
