"""Multi-GPU host logic on CPU: two gloo ranks shard the FE2 macro-step by
index and gather the homogenized stresses (bench.py).

The solves themselves need the GPU; here each rank evaluates the stress of
its shard with the CPU oracle on tiny networks, which is enough to prove the
shard bookkeeping (disjoint, complete, order-preserving) and the gather."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2305_07030_b200 as frb
    from oracle import frb_oracle as orc
    idx = bench.shard_indices("c5", rank, world)[:3] if rank == 0 else bench.shard_indices("c5", rank, world)[:2]
    sig = []
    for i in idx:  # a tiny stand-in network per index, the c5 gradient of that index
        net = frb.generate_lattice(3, 3, 3, 0.3, i)
        sig.append(orc.solve(net, bench.c5_gradient(i), frb.SolverConfig()).sigma.reshape(9))
    g = bench.gather_stresses(torch.tensor(np.array(sig)), world, dist)
    ids = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(ids, torch.tensor([idx[0]]))
    if rank == 0:
        np.savez(out_path, sig=g.numpy(), first=np.array([int(t.item()) for t in ids]))
    dist.barrier()
    dist.destroy_process_group()


def test_c5_shards_are_contiguous_disjoint_and_complete():
    sys.path.insert(0, ROOT)
    import bench
    for world in (1, 2, 3, 8):
        shards = [bench.shard_indices("c5", r, world) for r in range(world)]
        flat = [i for s in shards for i in s]
        assert flat == list(range(bench.C5_TOTAL))
        assert all(s == list(range(s[0], s[-1] + 1)) for s in shards if s)
    for world in (2, 4):   # strided shards of the heterogeneous / 100k-DOF batches
        for cfg in ("c3", "c4"):
            flat = sorted(i for r in range(world) for i in bench.shard_indices(cfg, r, world))
            assert flat == list(range(1024))


def test_two_rank_stress_gather(tmp_path):
    world = 2
    out = str(tmp_path / "g.npz")
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, start_method="spawn")
    z = np.load(out)
    sys.path.insert(0, ROOT)
    import bench
    import paper_2305_07030_b200 as frb
    from oracle import frb_oracle as orc
    expect = []
    for r, k in ((0, 3), (1, 2)):
        for i in bench.shard_indices("c5", r, world)[:k]:
            net = frb.generate_lattice(3, 3, 3, 0.3, i)
            expect.append(orc.solve(net, bench.c5_gradient(i), frb.SolverConfig()).sigma.reshape(9))
    assert z["sig"].shape == (5, 9)
    assert np.array_equal(z["sig"], np.array(expect))          # rank order, uneven shards
    assert list(z["first"]) == [0, bench.C5_TOTAL // 2]
