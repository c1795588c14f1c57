"""Multi-GPU partitioning along the hot path's two natural shards.

* Independent sample groups (config 5): group g runs on rank g mod world;
  each GPU evaluates the whole network on its groups.  There is no
  data-path collective -- only the max-over-ranks of the timed region and
  an optional gather of the decrypted logits at the end.
* Output-channel ciphertexts (config 4): rank r owns the contiguous block
  ``channel_shards(q, G)[r]`` of every conv layer's output channels; the next
  layer needs every input channel, so sharded_cnn.py passes each tile's
  input-row window around a ring of the ranks (the whole first activation map,
  16384 ciphertexts at 12 limbs, could not be replicated on one device).

One process per GPU; torch.distributed carries the collectives (NCCL on the
B200 box, gloo for the CPU tests).
"""

from __future__ import annotations

import numpy as np


def assign_groups(n_groups: int, world: int, rank: int) -> list[int]:
    """Round-robin ciphertext groups to ranks (group g -> rank g mod world)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of world {world}")
    return list(range(rank, n_groups, world))


def channel_shards(q: int, world: int) -> list[range]:
    """Contiguous output-channel blocks, sizes differing by at most one."""
    base, extra = divmod(q, world)
    out, start = [], 0
    for r in range(world):
        size = base + (1 if r < extra else 0)
        out.append(range(start, start + size))
        start += size
    return out


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a scalar over ranks (timed regions: slowest rank defines the job)."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_group_results(local: dict, world: int) -> dict:
    """Gather {group: ndarray} from every rank onto every rank (object collective)."""
    if world == 1:
        return dict(local)
    import torch.distributed as dist

    parts = [None] * world
    dist.all_gather_object(parts, {int(k): np.asarray(v) for k, v in local.items()})
    out = {}
    for p in parts:
        out.update(p)
    return out
