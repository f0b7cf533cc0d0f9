"""Multi-GPU host logic: frames are independent (harness.py:212 seeds every
packet separately), so the path shards by frame batch with no collective on
the data path.  torch.distributed carries only the timing
barrier, the max-over-ranks step time and the BER totals; the scalars travel
as host tensors over a gloo group (a host-side gather, as run_packets sums its
workers' results, harness.py:228-231), never through NCCL.
"""

from __future__ import annotations

import os
from typing import Optional

import torch
import torch.distributed as dist


def world() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment (1 process: 0, 0, 1)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def shard(total: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous [start, stop) frame slice of rank (strong scaling): sizes differ by at most one."""
    if world_size < 1 or not 0 <= rank < world_size or total < 0:
        raise ValueError(f"bad shard request total={total} rank={rank} world={world_size}")
    base, extra = divmod(total, world_size)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def rank_seed(seed: int, rank: int) -> int:
    """Independent synthetic frames per rank (weak scaling)."""
    return seed + 1000 * rank


_HOST_GROUP = None


def _host_group():
    """gloo process group for host scalars (created in init(), every rank in the same order)."""
    if _HOST_GROUP is not None:
        return _HOST_GROUP
    return dist.group.WORLD


def max_over_ranks(value: float) -> float:
    """The slowest rank's time: the job's step time is the max over ranks."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=_host_group())
    return float(t.item())


def sum_over_ranks(value: int) -> int:
    """Host-side totals (bit errors, bits): an int64 sum, as run_packets sums packets."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return int(value)
    t = torch.tensor([int(value)], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=_host_group())
    return int(t.item())


def barrier(sync_cuda: bool = True) -> None:
    """Device-synchronised barrier bracketing a timed region."""
    if sync_cuda and torch.cuda.is_available():
        torch.cuda.synchronize()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
    if sync_cuda and torch.cuda.is_available():
        torch.cuda.synchronize()


def init(backend: Optional[str] = None) -> tuple[int, int, int]:
    """Join the torchrun job if there is one (nccl on GPUs, gloo otherwise)."""
    rank, local, ws = world()
    if ws > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        elif backend == "gloo" and torch.cuda.is_available():
            torch.cuda.set_device(local % torch.cuda.device_count())
            dist.init_process_group("gloo")
        else:
            dist.init_process_group(backend)
        global _HOST_GROUP
        _HOST_GROUP = dist.new_group(backend="gloo") if dist.get_backend() != "gloo" else dist.group.WORLD
    return rank, local, ws
