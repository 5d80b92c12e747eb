"""Multi-process (gloo, world size 2, CPU) check of the N>1 path's host logic:
trial sharding by global index (bench.shard_range) with the oracle standing
in for each rank's ara_run, the YLT all-gather into the [P][L][N/P] layout
that ara_risk_measures consumes, and rank-count invariance."""
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
