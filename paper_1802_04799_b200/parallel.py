"""Multi-GPU plumbing: one process per GPU, torch.distributed for
the control/exchange steps, NCCL over NVLink on B200 (gloo for the CPU tests).

The hot path shards with NO data-path collective:
  * inference is batch-sharded -- every conv / depthwise / pool op is
    independent across N (R/src/ops.cpp:136-137: n is a pure data-parallel
    axis); each rank runs its slice of the batch through its own DeviceGraph
    with replicated weights. The one exchange step is the gather of the
    [B/G, classes] logits to rank 0 (all_gather_into_tensor: NCCL, or a
    gloo all_gather in tests);
  * tuning trials are sharded -- the candidate configs of one explore batch
    (R/src/tune.cpp:183-291) are split round-robin over ranks, each measures
    its share on its own GPU, and the records are gathered to rank 0, the
    single JSONL writer.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


def world() -> Tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_batch(global_batch: int, world_size: int, rank: int) -> Tuple[int, int]:
    """(start, count) of this rank's images; ranks differ by at most one."""
    if global_batch < world_size:
        raise ValueError(f"batch {global_batch} smaller than world size {world_size}")
    base, rem = divmod(global_batch, world_size)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def gather_rows(local: torch.Tensor, global_rows: int) -> Optional[torch.Tensor]:
    """Concatenate every rank's [rows_r, ...] slice (rank order) on every
    rank; uneven slices are padded to the largest and trimmed. Returns the
    [global_rows, ...] tensor (None when torch.distributed is not set up
    and world size is 1 -> the local tensor itself)."""
    rank, ws = world()
    if ws == 1:
        return local
    counts = [shard_batch(global_rows, ws, r)[1] for r in range(ws)]
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]].copy_(local)
    out = torch.empty((mx * ws,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, pad)
    else:
        parts = list(out.chunk(ws))
        dist.all_gather(parts, pad)
    return torch.cat([out[r * mx:r * mx + counts[r]] for r in range(ws)])


def shard_configs(n_configs: int, world_size: int, rank: int) -> List[int]:
    """Round-robin trial indices of one explore batch for this rank."""
    return list(range(rank, n_configs, world_size))


def sharded_measure(configs: Sequence[dict], measure_one: Callable[[dict], object]) -> list:
    """Each rank measures its round-robin share; every rank gets all
    records back in the original order (rank 0 then appends them to the
    trial DB as the single writer)."""
    rank, ws = world()
    mine = {i: measure_one(configs[i]) for i in shard_configs(len(configs), ws, rank)}
    if ws == 1:
        return [mine[i] for i in range(len(configs))]
    parts: list = [None] * ws
    dist.all_gather_object(parts, mine)
    merged = {}
    for p in parts:
        merged.update(p)
    return [merged[i] for i in range(len(configs))]
