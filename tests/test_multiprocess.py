"""Multi-GPU host logic on CPU: index shards and the result
gather of ``paper_2305_07030_b200.distributed`` with two gloo ranks.

The solves need the GPU; here every rank injects synthetic per-network
result records (the bytes the kernel writes, frb_result) for its shard and
calls the product's ``gather_results`` -- the same function ``ShardedBatch``
and ``bench.py`` use with NCCL -- which must return every network's record
in global index order on every rank, for contiguous (FE2 macro step) and
strided (heterogeneous batches) shards of uneven size."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2305_07030_b200 import _native as nat  # noqa: E402
from paper_2305_07030_b200.distributed import ShardLayout, decode_records, shard_indices  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def synthetic_records(indices: np.ndarray) -> np.ndarray:
    """A distinguishable frb_result per global network index."""
    rec = np.zeros(len(indices), dtype=nat.RESULT_DTYPE)
    rec["status"] = indices % 3
    rec["iters"] = 1000 + indices
    rec["converged"] = (indices % 3 == 0).astype(np.int32)
    rec["final_residual"] = 1e-9 * indices
    rec["r_ref"] = 0.5 + indices
    rec["avg_stress"] = indices[:, None] * 10.0 + np.arange(9)[None, :]
    return rec


def _worker(rank, world, port, n_total, mode, out_path):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2305_07030_b200.distributed import gather_results
    layout = ShardLayout(n_total, world, mode)
    mine = layout.shard(rank)
    local = torch.from_numpy(synthetic_records(mine).view(np.uint8).copy())
    out = gather_results(local, layout)
    np.save(f"{out_path}.{rank}.npy", out.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shards_are_disjoint_complete_and_ordered():
    for n in (0, 1, 7, 1024, 16384):
        for world in (1, 2, 3, 8):
            c = [shard_indices(n, r, world, "contiguous") for r in range(world)]
            assert np.array_equal(np.concatenate(c), np.arange(n))
            assert all((np.diff(s) == 1).all() for s in c if len(s))
            s = [shard_indices(n, r, world, "strided") for r in range(world)]
            assert np.array_equal(np.sort(np.concatenate(s)), np.arange(n))
            assert max(len(x) for x in s) - min(len(x) for x in s) <= 1
    with pytest.raises(ValueError):
        shard_indices(10, 2, 2)


def test_layout_rows_invert_the_shards():
    lay = ShardLayout(11, 3, "strided")
    rows = lay.global_rows()
    m = lay.max_shard
    for r in range(3):
        for k, i in enumerate(lay.shard(r)):
            assert rows[i] == r * m + k


@pytest.mark.parametrize("mode,n_total", [("contiguous", 13), ("strided", 13), ("contiguous", 16384)])
def test_two_rank_result_gather(tmp_path, mode, n_total):
    world = 2
    out = str(tmp_path / "g")
    mp.start_processes(_worker, args=(world, _free_port(), n_total, mode, out), nprocs=world, start_method="spawn")
    expect = synthetic_records(np.arange(n_total))
    for r in range(world):
        got = decode_records(np.load(f"{out}.{r}.npy"))
        assert got.shape == (n_total,)
        assert np.array_equal(got.view(np.uint8), expect.view(np.uint8)), f"rank {r}"


def test_bench_uses_the_product_shards():
    import bench
    for world in (1, 2, 8):
        for r in range(world):
            assert list(bench.shard_indices("c5", r, world)) == list(shard_indices(16384, r, world, "contiguous"))
            assert list(bench.shard_indices("c3", r, world)) == list(shard_indices(1024, r, world, "strided"))


def _gpu_worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)   # two ranks share one GPU: gloo
    torch.cuda.set_device(0)
    import paper_2305_07030_b200 as frb
    from paper_2305_07030_b200.distributed import ShardedBatch
    Fs = [np.eye(3) + 0.01 * (i + 1) * np.diag([1.0, 0.5, 0.2]) for i in range(7)]
    sb = ShardedBatch(lambda i: (frb.generate_lattice(5, 5, 6, 0.3, i), frb.AffineBC(np.eye(3))), 7,
                      mode="strided", device="cuda:0")
    sig = sb.macro_step(Fs, frb.SolverConfig())           # FE2 step: new F on the resident shards
    np.save(f"{out_path}.{rank}.npy", sig)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_macro_step_on_the_gpu(cuda_device, tmp_path):
    """The product multi-GPU API on real solves: two ranks (sharing the one GPU
    of the test box, gloo) each solve their strided shard of a 7-network FE2
    macro step on the device; every rank ends with every network's stress,
    bit-identical to solving the whole batch in one process."""
    import paper_2305_07030_b200 as frb
    out = str(tmp_path / "s")
    mp.start_processes(_gpu_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn")
    Fs = [np.eye(3) + 0.01 * (i + 1) * np.diag([1.0, 0.5, 0.2]) for i in range(7)]
    ref = frb.solve_batch(frb.pack_batch([frb.generate_lattice(5, 5, 6, 0.3, i) for i in range(7)],
                                         [frb.AffineBC(F) for F in Fs]))
    want = np.array([r.avg_stress for r in ref])
    for r in range(2):
        assert np.array_equal(np.load(f"{out}.{r}.npy"), want)
