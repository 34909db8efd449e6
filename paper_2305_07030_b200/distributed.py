"""Multi-GPU solves: independent networks sharded over the GPUs of one node.

The reference solves one network per call (``dynamic_relaxation_solve``,
microsolver.py:567-574) and the paper drives thousands of them per FE2 macro
step.  Networks never exchange data during a solve
(SURVEY.md 8e), so the B200 build shards them by index -- one process per GPU
(torchrun), each packing and solving its own shard with its own persistent
kernel -- and exchanges only the per-network result records at the end: one
``all_gather_into_tensor`` (NCCL over NVLink) of the raw 144-byte
``frb_result`` records [status, iters, converged, residual, r_ref, energy
residual, sigma(9), energy(4)], issued on the device stream with no host
synchronisation.

* ``shard_indices`` -- contiguous (FE2 macro step, config 5) or strided
  (mixed sizes / loads, configs 3-4) index shards;
* ``ShardLayout`` -- every rank's shard, known on every rank without
  communication (so the gather needs no size exchange);
* ``gather_results`` -- the collective, returning the records of all networks
  in global index order (device tensor);
* ``ShardedBatch`` -- pack + upload + solve + gather for one rank, and the
  FE2 ``macro_step`` (new deformation gradients on the resident shard).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _native as nat

RECORD_BYTES = nat.RESULT_DTYPE.itemsize  # 144


def shard_indices(n_total: int, rank: int, world: int, mode: str = "contiguous") -> np.ndarray:
    """Global network indices of `rank`'s shard.

    contiguous: [r*ceil(n/w), (r+1)*ceil(n/w)) -- the FE2 macro step's
    partition (each rank owns a block of integration points).
    strided: r, r+w, r+2w, ... -- balances batches whose iteration counts
    follow the index (heterogeneous sizes / loads)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    if mode == "contiguous":
        per = -(-n_total // world) if n_total else 0
        return np.arange(rank * per, min(n_total, (rank + 1) * per), dtype=np.int64)
    if mode == "strided":
        return np.arange(rank, n_total, world, dtype=np.int64)
    raise ValueError(f"unknown shard mode {mode!r}")


@dataclass(frozen=True)
class ShardLayout:
    """Every rank's shard of n_total networks (deterministic, so each rank
    computes all of them locally)."""
    n_total: int
    world: int
    mode: str = "contiguous"

    def shard(self, rank: int) -> np.ndarray:
        return shard_indices(self.n_total, rank, self.world, self.mode)

    @property
    def max_shard(self) -> int:
        return max((len(self.shard(r)) for r in range(self.world)), default=0)

    def global_rows(self) -> np.ndarray:
        """Row of the padded [world, max_shard] gather that holds network i,
        for i in global order."""
        rows = np.empty(self.n_total, dtype=np.int64)
        m = self.max_shard
        for r in range(self.world):
            idx = self.shard(r)
            rows[idx] = r * m + np.arange(len(idx))
        return rows


def _dist():
    import torch.distributed as dist
    return dist


def gather_results(local, layout: ShardLayout, group=None, rows=None):
    """All-gather the ranks' result records into global index order.

    local: this rank's records, a uint8 tensor of len(shard) * 144 bytes
    (``DeviceResults.results``), CUDA (NCCL) or CPU (gloo).  Returns a uint8
    tensor of n_total * 144 bytes on local's device on every rank.  Shard
    sizes come from the layout, so nothing is synchronised with the host."""
    import torch
    dist = _dist()
    world = layout.world
    m = layout.max_shard
    if rows is None:
        rows = torch.from_numpy(layout.global_rows()).to(local.device)
    send = torch.zeros(m * RECORD_BYTES, dtype=torch.uint8, device=local.device)
    send[:local.numel()].copy_(local)
    out = torch.empty(world * m * RECORD_BYTES, dtype=torch.uint8, device=local.device)
    if world == 1:
        out.copy_(send)
    elif dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, send, group=group)
    else:  # gloo (CPU tests, or several ranks sharing one GPU): a host round trip
        host = torch.empty(world * m * RECORD_BYTES, dtype=torch.uint8)
        dist.all_gather(list(host.view(world, -1).unbind(0)), send.cpu(), group=group)
        out.copy_(host)
    return out.view(world * m, RECORD_BYTES).index_select(0, rows).reshape(-1)


def decode_records(records) -> np.ndarray:
    """uint8 records (tensor or array) -> numpy RESULT_DTYPE [n]."""
    a = records.cpu().numpy() if hasattr(records, "cpu") else np.asarray(records, dtype=np.uint8)
    return a.view(nat.RESULT_DTYPE)


class ShardedBatch:
    """One rank's share of a sharded batch: its networks packed and resident
    on its GPU.

    make(i) -> (FiberNetwork, AffineBC) builds global network i; only this
    rank's indices are built (host setup is per rank).  rank /
    world default to the initialised torch.distributed group (1 / 0 without
    one)."""

    def __init__(self, make: Callable[[int], tuple], n_total: int, mode: str = "contiguous", device=None,
                 rank: int | None = None, world: int | None = None, group=None):
        import torch

        from .batch import pack_batch
        dist = _dist()
        on = dist.is_available() and dist.is_initialized()
        self.rank = rank if rank is not None else (dist.get_rank(group) if on else 0)
        self.world = world if world is not None else (dist.get_world_size(group) if on else 1)
        self.group = group
        self.layout = ShardLayout(n_total, self.world, mode)
        self.indices = self.layout.shard(self.rank)
        pairs = [make(int(i)) for i in self.indices]
        self.batch = pack_batch([p[0] for p in pairs], [p[1] for p in pairs])
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dev = self.batch.to_device(self.device)
        self._rows = torch.from_numpy(self.layout.global_rows()).to(self.device)

    def prepare(self, cfg, strategy=None):
        """Launch arguments of this rank's shard (replayable)."""
        return self.dev.prepare(cfg, strategy)

    def gather(self, local_results):
        """Records of all networks, global order, on this rank's device."""
        return gather_results(local_results, self.layout, self.group, self._rows)

    def solve(self, cfg, strategy=None, stream=None):
        """Solve this rank's shard and gather every rank's records
        (asynchronous; decode_records(...) synchronises)."""
        launch = self.prepare(cfg, strategy)
        launch.run(stream)
        return self.gather(launch.out.results)

    def macro_step(self, Fs_global: Sequence, cfg, strategy=None) -> np.ndarray:
        """FE2 macro step: new deformation gradients for this rank's networks
        (global list, indexed like the layout), solve on the resident shard,
        and return the homogenized stresses of ALL networks [n_total, 3, 3]
        on every rank."""
        self.dev.set_deformation([Fs_global[int(i)] for i in self.indices])
        rec = decode_records(self.solve(cfg, strategy))
        return np.array(rec["avg_stress"], dtype=np.float64).reshape(-1, 3, 3)
