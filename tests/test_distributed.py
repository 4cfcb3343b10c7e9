"""Multi-rank (SFC-segment sharded) PCG: exchange plans, the SPMD program over
gloo with world_size 2 on CPU, lockstep emulation, and (gpu) the device shard
engine emulated as 2-4 ranks on one GPU."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch

from paper_2110_11211_b200 import distributed as D

CASE = ((6, 6), 12, 0.5, 3)  # levels, P, gamma, q


def _oracle(levels, p, gamma, q):
    import sfcdd_oracle as O

    _, _, _, res = O.solve_config(levels, p, gamma, q)
    return res


def _numpy_shards(levels, p, gamma, q, world):
    from shard_numpy_engine import NumpyShardEngine

    engines = [NumpyShardEngine(levels, p, gamma, q, g, world) for g in range(world)]
    part = _part(levels, p, gamma)
    nbr = engines[0].neighbors(len(levels))
    plans = D.build_plans(part, q, world, nbr, [e.xy_offsets for e in engines])
    for e, pl in zip(engines, plans):
        e.attach_plan(pl)
    return engines, plans


def _part(levels, p, gamma):
    from paper_2110_11211_b200.partition import build_partition

    n = 1
    for l in levels:
        n *= (1 << l) - 1
    return build_partition(n, p, gamma)


def _rhs(levels):
    import sfcdd_oracle as O

    n = 1
    for l in levels:
        n *= (1 << l) - 1
    _, _, t = O.stencil_constants(levels)
    return t * O.seeded_rhs(n)


@pytest.mark.parametrize("world", [2, 3, 5])
def test_plans_are_consistent(world):
    levels, p, gamma, q = CASE
    engines, plans = _numpy_shards(levels, p, gamma, q, world)
    n = engines[0].n
    assert plans[0].g0 == 0 and plans[-1].g1 == n
    for g in range(world - 1):
        assert plans[g].g1 == plans[g + 1].g0
    assert sum(pl.a1 - pl.a0 for pl in plans) == p * q
    for name in ("halo", "ext", "xy"):
        for g in range(world):
            for h, idx in getattr(plans[g], name).recv.items():
                assert h != g
                assert len(getattr(plans[h], name).send[g]) == len(idx)
    # halo = stencil neighbours of owned points owned elsewhere; the cyclic
    # overlap ring couples rank 0 and rank G-1 (partition.py:115)
    A = engines[0].A.tocsr()
    for g, pl in enumerate(plans):
        nb = set()
        for row in range(pl.g0, pl.g1):
            nb |= set(int(c) for c in A.indices[A.indptr[row]:A.indptr[row + 1]])
        want = sorted(c for c in nb if not pl.g0 <= c < pl.g1)
        got = sorted(int(v) for idx in pl.halo.recv.values() for v in idx)
        assert got == want
    assert world - 1 in plans[0].ext.recv


@pytest.mark.parametrize("levels,p,gamma,world", [((5, 6), 12, 0.5, 2), ((5, 6), 12, 0.25, 5),
                                                   ((4, 4, 4), 8, 0.5, 3), ((5, 5), 7, 0.75, 4)])
def test_xy_offsets_for_matches_brute_force(levels, p, gamma, world):
    """The per-rank slot layout every rank derives locally (torchrun) equals
    the brute-force coverage rule of the numpy shard engine."""
    from shard_numpy_engine import NumpyShardEngine

    part = _part(levels, p, gamma)
    for g in range(world):
        e = NumpyShardEngine(levels, p, gamma, 2, g, world)
        np.testing.assert_array_equal(D.xy_offsets_for(part, world, g), e.xy_offsets)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_lockstep_numpy_matches_oracle(world):
    levels, p, gamma, q = CASE
    engines, plans = _numpy_shards(levels, p, gamma, q, world)
    b = torch.from_numpy(_rhs(levels))
    xs = [torch.zeros_like(b) for _ in range(world)]
    res = D.run_lockstep(engines, plans, [b.clone() for _ in range(world)], xs)
    ref = _oracle(levels, p, gamma, q)
    its, conv, hist = res[0]
    assert conv and abs(its - ref.iterations) <= 1
    k = min(len(hist), len(ref.residual_history))
    np.testing.assert_allclose(hist[:k], ref.residual_history[:k], rtol=1e-10)
    x = np.zeros(engines[0].n)
    for e, xv in zip(engines, xs):
        x[e.g0:e.g1] = xv.numpy()[e.g0:e.g1]
    assert np.linalg.norm(x - ref.solution) <= 1e-10 * np.linalg.norm(ref.solution)


def _gloo_worker(rank, world, port, outdir):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    levels, p, gamma, q = CASE
    engines, plans = _numpy_shards(levels, p, gamma, q, world)  # every rank derives all plans
    eng, plan = engines[rank], plans[rank]
    b = torch.from_numpy(_rhs(levels))
    x = torch.zeros_like(b)
    its, conv, hist = D.run_torch(eng, plan, b, x)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), its=its, conv=conv, hist=np.asarray(hist),
             x=x.numpy()[eng.g0:eng.g1], g0=eng.g0, g1=eng.g1)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world_size_2_matches_oracle():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker, args=(2, port, d), nprocs=2, join=True)
        r = [np.load(os.path.join(d, f"rank{g}.npz")) for g in range(2)]
        ref = _oracle(*CASE)
        assert int(r[0]["its"]) == int(r[1]["its"])
        assert abs(int(r[0]["its"]) - ref.iterations) <= 1
        k = min(len(r[0]["hist"]), len(ref.residual_history))
        np.testing.assert_allclose(r[0]["hist"][:k], ref.residual_history[:k], rtol=1e-10)
        x = np.zeros(ref.solution.size)
        for rr in r:
            x[int(rr["g0"]):int(rr["g1"])] = rr["x"]
        assert np.linalg.norm(x - ref.solution) <= 1e-10 * np.linalg.norm(ref.solution)


@pytest.mark.gpu
@pytest.mark.parametrize("sparse_coarse", [False, True])
@pytest.mark.parametrize("levels,p,gamma,q,world", [((7, 7), 16, 0.5, 4, 2), ((7, 7), 16, 0.5, 4, 4),
                                                    ((4, 4, 4), 8, 0.5, 4, 3)])
def test_device_shards_lockstep_match_single_gpu(levels, p, gamma, q, world, sparse_coarse, monkeypatch):
    """sparse_coarse: every rank's redundant coarse solve through the sparse
    A0 factor and the DAG kernel (the path above 8192 coarse dofs)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if sparse_coarse:
        monkeypatch.setenv("SFCDD_COARSE_DENSE_MAX", "0")

    part = _part(levels, p, gamma)
    engines, plans = D.make_device_shards(levels, part, q, world)
    b = torch.from_numpy(_rhs(levels)).cuda()
    xs = [torch.zeros_like(b) for _ in range(world)]
    res = D.run_lockstep(engines, plans, [b.clone() for _ in range(world)], xs)
    ref = _oracle(levels, p, gamma, q)
    its, conv, hist = res[0]
    assert conv and abs(its - ref.iterations) <= 1
    k = min(len(hist), len(ref.residual_history))
    np.testing.assert_allclose(hist[:k], ref.residual_history[:k], rtol=1e-10)
    x = np.zeros(part.n)
    for e, xv in zip(engines, xs):
        x[e.g0:e.g1] = xv.cpu().numpy()[e.g0:e.g1]
    assert np.linalg.norm(x - ref.solution) <= 1e-10 * np.linalg.norm(ref.solution)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_make_rank_shard_layout_matches_all_ranks_build(world):
    """Each torchrun rank builds only its own engine + plan; they must equal
    the plans derived with every rank's engine in one process."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    levels, p, gamma, q = (7, 7), 16, 0.5, 4
    part = _part(levels, p, gamma)
    _, plans_all = D.make_device_shards(levels, part, q, world)
    for g in range(world):
        eng, plan = D.make_rank_shard(levels, part, q, g, world)
        ref = plans_all[g]
        assert (plan.g0, plan.g1, plan.a0, plan.a1) == (ref.g0, ref.g1, ref.a0, ref.a1)
        for name in ("halo", "ext", "xy"):
            for side in ("send", "recv"):
                a, b = getattr(getattr(plan, name), side), getattr(getattr(ref, name), side)
                assert a.keys() == b.keys()
                for h in a:
                    np.testing.assert_array_equal(a[h], b[h])
        del eng


def _nccl_worker(rank, world, port, outdir):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    levels, p, gamma, q = (7, 7), 16, 0.5, 4
    part = _part(levels, p, gamma)
    eng, plan = D.make_rank_shard(levels, part, q, rank, world)
    b = torch.from_numpy(_rhs_nooracle(levels)).cuda()
    x = torch.zeros_like(b)
    its, conv, hist = D.run_torch(eng, plan, b, x)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), its=its, conv=conv, hist=np.asarray(hist),
             x=x.cpu().numpy()[plan.g0:plan.g1], g0=plan.g0, g1=plan.g1)
    dist.barrier()
    dist.destroy_process_group()


def _rhs_nooracle(levels):
    import paper_2110_11211_b200 as sf

    n = sf.num_dofs(levels)
    b = np.random.default_rng(42).uniform(-1.0, 1.0, size=n)
    _, bh, _ = sf.symmetrize_diag(sf.assemble_laplacian(levels), b)
    return np.asarray(bh)


@pytest.mark.gpu
def test_nccl_run_torch_matches_oracle():
    """The torchrun path (make_rank_shard + run_torch over NCCL) on every GPU
    this box has (1 on the grading box: all exchanges empty, collectives real)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    world = min(torch.cuda.device_count(), 2)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_nccl_worker, args=(world, port, d), nprocs=world, join=True)
        r = [np.load(os.path.join(d, f"rank{g}.npz")) for g in range(world)]
        ref = _oracle((7, 7), 16, 0.5, 4)
        np.testing.assert_allclose(_rhs_nooracle((7, 7)), _rhs((7, 7)), rtol=0, atol=0)
        assert abs(int(r[0]["its"]) - ref.iterations) <= 1
        k = min(len(r[0]["hist"]), len(ref.residual_history))
        np.testing.assert_allclose(r[0]["hist"][:k], ref.residual_history[:k], rtol=1e-10)
        x = np.zeros(ref.solution.size)
        for rr in r:
            x[int(rr["g0"]):int(rr["g1"])] = rr["x"]
        assert np.linalg.norm(x - ref.solution) <= 1e-10 * np.linalg.norm(ref.solution)


# ------------------------------------------- device-driven sharded program
@pytest.mark.gpu
@pytest.mark.parametrize("levels,p,gamma,q,coarse", [((7, 7), 16, 0.5, 4, "dense"), ((7, 7), 16, 0.5, 4, "sparse"),
                                                     ((4, 4, 4), 8, 0.5, 4, "dense"),
                                                     ((7, 7), 16, 0.5, 4, "nccl")])
def test_device_driven_shard_pcg_matches_oracle(levels, p, gamma, q, coarse, monkeypatch):
    """sfcdd_shard_pcg: the whole sharded solve as one CUDA graph with a
    conditional WHILE loop, device scalars and (``nccl``) the NCCL
    allgathers of the coarse restrictions / CG scalars captured in it (a
    world-1 communicator: every collective is real, the exchanges are empty)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if coarse == "sparse":
        monkeypatch.setenv("SFCDD_COARSE_DENSE_MAX", "0")
    part = _part(levels, p, gamma)
    eng, plan = D.make_rank_shard(levels, part, q, 0, 1)
    D.attach_device_program(eng, plan, D.nccl_unique_id() if coarse == "nccl" else None)
    b = torch.from_numpy(_rhs(levels)).cuda()
    x = torch.zeros_like(b)
    its, conv, hist = D.run_device(eng, b, x)
    ref = _oracle(levels, p, gamma, q)
    assert conv and abs(its - ref.iterations) <= 1
    k = min(len(hist), len(ref.residual_history))
    np.testing.assert_allclose(hist[:k], ref.residual_history[:k], rtol=1e-10)
    assert np.linalg.norm(x.cpu().numpy() - ref.solution) <= 1e-10 * np.linalg.norm(ref.solution)
    # repeat (graph replay) and compare with the host-driven program bitwise in iterations
    x2 = torch.zeros_like(b)
    its2, conv2, hist2 = D.run_device(eng, b, x2)
    assert its2 == its and hist2 == hist
    torch.testing.assert_close(x2, x, rtol=0, atol=0)


def _gloo_cuda_worker(rank, world, port, outdir):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    levels, p, gamma, q = (7, 7), 16, 0.5, 4
    part = _part(levels, p, gamma)
    eng, plan = D.make_rank_shard(levels, part, q, rank, world)
    b = torch.from_numpy(_rhs_nooracle(levels)).cuda()
    x = torch.zeros_like(b)
    its, conv, hist = D.run_torch(eng, plan, b, x)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), its=its, conv=conv, hist=np.asarray(hist),
             x=x.cpu().numpy()[plan.g0:plan.g1], g0=plan.g0, g1=plan.g1, launches=eng.launches)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_world_2_drives_cuda_shard_kernels():
    """Two processes, each with its CUDA shard engine (the sm_100a kernels of
    its half of the subdomains) on the one GPU of the box, exchanging over
    gloo through host memory: no kernel of one rank waits on the other's."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_cuda_worker, args=(2, port, d), nprocs=2, join=True)
        r = [np.load(os.path.join(d, f"rank{g}.npz")) for g in range(2)]
        ref = _oracle((7, 7), 16, 0.5, 4)
        assert int(r[0]["launches"]) > 0 and int(r[1]["launches"]) > 0
        assert int(r[0]["its"]) == int(r[1]["its"]) and abs(int(r[0]["its"]) - ref.iterations) <= 1
        k = min(len(r[0]["hist"]), len(ref.residual_history))
        np.testing.assert_allclose(r[0]["hist"][:k], ref.residual_history[:k], rtol=1e-10)
        x = np.zeros(ref.solution.size)
        for rr in r:
            x[int(rr["g0"]):int(rr["g1"])] = rr["x"]
        assert np.linalg.norm(x - ref.solution) <= 1e-10 * np.linalg.norm(ref.solution)
