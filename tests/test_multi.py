"""Multi-process bin sharding on CPU: world size 2 over gloo, through libcider's host
path (the per-rank seeded shard generator cider_workload_bins, the uint8 packing of the gathered
decoded sets, cider_ser_cer summed over ranks) — the same plumbing bench.py runs around the device
decode. Bins are independent (no per-step collective), so the gathered shards and the rank-summed
SER must equal a single-process run over all bins. The device decode itself needs a B200 (-m gpu:
test_gpu_parity.py runs cider_nccl_* at world 1 and bench.py's gather)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


WL = dict(m=6, slots=16, checks=8, k=3, snr_db=4.0, p_erase=0.1, p_false=0.1)


def _fake_decode(truth, bin0):
    """A deterministic stand-in for the device's decoded sets: the truth with bin-dependent row
    permutations and symbol errors (what the gather and SER plumbing must carry unchanged)."""
    out = truth.copy()
    for i in range(out.shape[0]):
        b = bin0 + i
        out[i] = np.roll(out[i], b % out.shape[1], axis=0)
        out[i, b % out.shape[1], (3 * b) % out.shape[2]] ^= 1 + b % 7
    return out


def _worker(rank, world, port, n_per_rank, out_path):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_2605_26580_b200 as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = P.Workload(**WL)
    edges = wl.code()
    first, n = P.shard(0, n_per_rank, rank, world)
    truth, S = wl.bins(edges, first, n)
    dec = _fake_decode(truth, first)
    packed = torch.from_numpy(dec.astype(np.uint8))                 # one byte per symbol (Q <= 256)
    parts = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(parts, packed)
    ser = torch.tensor([P.ser_cer(truth, dec)[0] * n], dtype=torch.float64)
    dist.all_reduce(ser)
    if rank == 0:
        np.savez(out_path, grids=torch.cat(parts).numpy(), ser=ser.numpy(), S0=S[0])
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gather_and_ser_match_single_process(tmp_path):
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    import paper_2605_26580_b200 as P
    world, n_per_rank = 2, 5
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _free_port(), n_per_rank, out), nprocs=world, join=True)
    r = np.load(out)
    wl = P.Workload(**WL)
    truth, S = wl.bins(wl.code(), 0, world * n_per_rank)
    dec = _fake_decode(truth, 0)
    assert np.array_equal(r["grids"].astype(np.int32), dec)
    assert np.array_equal(r["S0"], S[0])
    assert abs(r["ser"][0] / (world * n_per_rank) - P.ser_cer(truth, dec)[0]) < 1e-12


def test_bench_spawns_its_ranks():
    """`bench.py --gpus 2` outside torchrun launches 2 ranks (127.0.0.1 rendezvous) and prints one JSON
    line with n_gpus = 2; the CPU reference arm makes this runnable without a GPU."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "c1", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300,
                       env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"


def test_bench_rejects_world_mismatch():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "c1"], capture_output=True, text=True, timeout=120,
                       env=dict(os.environ, WORLD_SIZE="1", RANK="0"))
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr


def test_shard_ranges_partition_the_bins():
    import paper_2605_26580_b200 as P
    for world in (1, 2, 4, 8):
        seen = []
        for step in range(3):
            for rank in range(world):
                a, n = P.shard(0, 5, rank, world, step)
                seen.extend(range(a, a + n))
        assert sorted(seen) == list(range(3 * world * 5))
