"""Multi-process sharding of bins on CPU: world size 2 over gloo. Each rank decodes
its contiguous shard with the CPU oracle, the grids are all-gathered, and the result must equal a
single-process decode of all bins (bins are independent: no per-step collective)."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_per_rank, out_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_2605_26580_b200 as P
    from oracle.binding import Checker
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = P.Workload(m=4, slots=12, checks=8, k=2, snr_db=6.0)
    m = P.Model.ref_exact(4, 16)
    edges = wl.code()
    first, n = P.shard(0, n_per_rank, rank, world)
    _, S = wl.bins(edges, first, n)
    w = P.weights_init(m, 1).astype(np.float64)
    r = Checker("oracle").refine(m, w, edges, wl.checks, wl.slots, S.astype(np.float64), wl.k, P.RevealSchedule(steps=3))
    mine = torch.from_numpy(r["grid"])
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    if rank == 0:
        np.save(out_path, torch.cat(parts).numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_bin_sharding_gather_matches_single_process(tmp_path):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    import paper_2605_26580_b200 as P
    from oracle.binding import Checker
    world, n_per_rank = 2, 3
    out = str(tmp_path / "grids.npy")
    mp.spawn(_worker, args=(world, _free_port(), n_per_rank, out), nprocs=world, join=True)
    gathered = np.load(out)
    wl = P.Workload(m=4, slots=12, checks=8, k=2, snr_db=6.0)
    m = P.Model.ref_exact(4, 16)
    edges = wl.code()
    _, S = wl.bins(edges, 0, world * n_per_rank)
    w = P.weights_init(m, 1).astype(np.float64)
    ref = Checker("oracle").refine(m, w, edges, wl.checks, wl.slots, S.astype(np.float64), wl.k, P.RevealSchedule(steps=3))
    assert np.array_equal(gathered, ref["grid"])


def test_shard_ranges_partition_the_bins():
    import paper_2605_26580_b200 as P
    for world in (1, 2, 4, 8):
        seen = []
        for step in range(3):
            for rank in range(world):
                a, n = P.shard(0, 5, rank, world, step)
                seen.extend(range(a, a + n))
        assert sorted(seen) == list(range(3 * world * 5))
