"""Multi-process (gloo, CPU) check of the N>1 path's host logic: trial
sharding by global index (bench.shard_range) with the oracle standing in for
each rank's ara_run (no GPU here), bench.gather_ylt -- the exchange step
bench.run_ours runs, equal and unequal shards -- and rank-count invariance
of the YLT and the measures; bench.launch_command (the
one-process-per-GPU re-exec of `bench.py --gpus N`)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import aragen
import oracle
from oracle import measures as OM


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def small_cfg():
    cfg = aragen.load_config("cfg1")
    cfg.update(n_trials=400, n_layers=2, elts_per_layer=2,
               layer_terms=[[2e5, 5e6, 2.0e7, 3.5e7], [4e5, 5e6, 1.5e7, 3.0e7]])
    return cfg


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    cfg = small_cfg()
    lo, hi = bench.shard_range(cfg["n_trials"], rank, world)
    pf = aragen.build_portfolio(cfg)
    yet = aragen.build_yet(cfg, first_trial=lo, n_trials=hi - lo)
    part = oracle.run(pf, yet, seed=cfg["seed"], n_threads=1)["ylt"]          # [L][N/P]
    # concatenation form [P*L][N/P] == the [P][L][N/P] layout ara_risk_measures takes
    gathered = torch.empty((world * part.shape[0], part.shape[1]), dtype=torch.float64)
    dist.all_gather_into_tensor(gathered, torch.from_numpy(np.ascontiguousarray(part)))
    gathered = gathered.view(world, part.shape[0], part.shape[1])
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered.npy"), gathered.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _gather_worker(rank, world, port, out_dir, n_trials):
    # bench.run_ours's exchange step on CPU tensors: each rank's YLT shard
    # (the oracle in place of ara_run) through bench.gather_ylt
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    cfg = small_cfg()
    cfg["n_trials"] = n_trials
    lo, hi = bench.shard_range(n_trials, rank, world)
    pf = aragen.build_portfolio(cfg)
    yet = aragen.build_yet(cfg, first_trial=lo, n_trials=hi - lo)
    part = torch.from_numpy(np.ascontiguousarray(oracle.run(pf, yet, seed=cfg["seed"], n_threads=1)["ylt"]))
    table, n_shards = bench.gather_ylt(part, world, n_trials)
    if rank == 0:
        np.save(os.path.join(out_dir, "table.npy"), table.numpy())
        np.save(os.path.join(out_dir, "n_shards.npy"), np.array([n_shards]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,n_trials", [(2, 400), (2, 401), (3, 400)])
def test_bench_gather_ylt(tmp_path, world, n_trials):
    mp.spawn(_gather_worker, args=(world, _free_port(), str(tmp_path), n_trials), nprocs=world, join=True)
    table = np.load(tmp_path / "table.npy")
    n_shards = int(np.load(tmp_path / "n_shards.npy")[0])
    cfg = small_cfg()
    cfg["n_trials"] = n_trials
    pf = aragen.build_portfolio(cfg)
    full = oracle.run(pf, aragen.build_yet(cfg), seed=cfg["seed"])["ylt"]      # [L][N], one process
    L, N = full.shape
    if n_trials % world == 0:
        assert n_shards == world and table.shape == (world * L, N // world)
        flat = table.reshape(world, L, N // world).transpose(1, 0, 2).reshape(L, N)   # [P][L][N/P] -> [L][N]
    else:
        assert n_shards == 1 and table.shape == (L, N)                 # pads dropped, global trial order
        flat = table
    assert np.array_equal(flat, full)
    for li in range(L):
        for rp in (10, 50):
            assert OM.pml(flat[li], rp) == OM.pml(full[li], rp)
            assert OM.tvar_rp(flat[li], rp) == OM.tvar_rp(full[li], rp)


def test_launch_command_one_process_per_gpu():
    import bench
    cmd = bench.launch_command(8, ["--gpus", "8", "--steps", "5"], port=29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--steps", "5"] and cmd[-5].endswith("bench.py")


@pytest.mark.timeout(300)
def test_sharded_gather_equals_single(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g = np.load(tmp_path / "gathered.npy")                     # [P][L][N/P]
    cfg = small_cfg()
    pf = aragen.build_portfolio(cfg)
    full = oracle.run(pf, aragen.build_yet(cfg), seed=cfg["seed"])["ylt"]  # [L][N]
    L, N = full.shape
    # trial order inside the gathered layout is shard-major: identical values
    flat = g.transpose(1, 0, 2).reshape(L, N)
    assert np.array_equal(flat, full)
    # the measures on the gathered [P][L][N/P] layout (permutation-invariant)
    for li in range(L):
        for rp in (10, 50):
            assert OM.pml(g[:, li, :].ravel(), rp) == OM.pml(full[li], rp)
            assert OM.tvar_rp(g[:, li, :].ravel(), rp) == OM.tvar_rp(full[li], rp)
    roll = g.sum(axis=1).ravel()
    assert OM.pml(roll, 10) == OM.pml(OM.rollup(full), 10)


def test_shard_range_covers_exactly():
    import bench
    for n in (0, 1, 7, 800000, 1000000):
        for world in (1, 2, 3, 4, 8):
            spans = [bench.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def _table_shard_worker(rank, world, port, out_dir, n_tables):
    # the multi-table measures exchange of bench.run_ours: each rank fills the
    # (PML, TVaR, VaR) rows of its bench.table_shard share (the oracle's measures
    # in place of ara_risk_measures_async), zeros elsewhere, then an all_reduce SUM
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    rng = np.random.default_rng(5)
    tables = rng.lognormal(14, 1.1, (n_tables, 3000))              # the same on every rank
    rows = torch.zeros((n_tables, 2, 3), dtype=torch.float64)
    for i in bench.table_shard(n_tables, rank, world):
        for q, rp in enumerate((10, 50)):
            var, tv = OM.tvar_rp(tables[i], rp)
            rows[i, q] = torch.tensor([OM.pml(tables[i], rp), tv, var], dtype=torch.float64)
    dist.all_reduce(rows, op=dist.ReduceOp.SUM)
    if rank == 0:
        np.save(os.path.join(out_dir, "rows.npy"), rows.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,n_tables", [(2, 9), (3, 9), (8, 9), (3, 2)])
def test_table_shard_measures_exchange(tmp_path, world, n_tables):
    import bench
    covered = sorted(i for r in range(world) for i in bench.table_shard(n_tables, r, world))
    assert covered == list(range(n_tables))                  # every table exactly once
    mp.spawn(_table_shard_worker, args=(world, _free_port(), str(tmp_path), n_tables), nprocs=world, join=True)
    rows = np.load(tmp_path / "rows.npy")
    rng = np.random.default_rng(5)
    tables = rng.lognormal(14, 1.1, (n_tables, 3000))
    for i in range(n_tables):
        for q, rp in enumerate((10, 50)):
            var, tv = OM.tvar_rp(tables[i], rp)
            assert rows[i, q, 0] == OM.pml(tables[i], rp) and rows[i, q, 1] == tv and rows[i, q, 2] == var
