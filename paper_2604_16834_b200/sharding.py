"""Multi-GPU partitioning along the hot path's two natural shards.

* Independent sample groups (config 5): group g runs on rank g mod world;
  each GPU evaluates the whole network on its groups.  There is no
  data-path collective -- only the max-over-ranks of the timed region and
  an optional gather of the decrypted logits at the end.
* Output-channel ciphertexts (config 4): rank r owns a contiguous block of
  every conv layer's output channels; the next layer needs every input
  channel, so activations are exchanged with a chunked all-gather over
  input-channel blocks (``allgather_chunks``).  Chunks bound the staging
  memory: config 4's first activation map (16384 ciphertexts at >= 11 limbs)
  cannot be replicated on one 180 GB device.

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


def allgather_chunks(n_items: int, world: int, chunk: int) -> list[list[tuple[int, range]]]:
    """Schedule of a chunked all-gather of per-rank item blocks.

    Returns rounds; round k lists, for every rank r, the slice of r's block
    sent in that round.  Every item of every block appears exactly once."""
    blocks = channel_shards(n_items, world)
    rounds = []
    k = 0
    while True:
        step = []
        for r, b in enumerate(blocks):
            lo = b.start + k * chunk
            hi = min(b.stop, lo + chunk)
            if lo < hi:
                step.append((r, range(lo, hi)))
        if not step:
            return rounds
        rounds.append(step)
        k += 1


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


def allgather_tensor_blocks(block, world: int):
    """All-gather equally sized tensor blocks (e.g. one chunk of ciphertexts,
    int64 [items, n_comp, limbs, N]) -> [world * items, ...]."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return block
    out = torch.empty((world * block.shape[0],) + tuple(block.shape[1:]), dtype=block.dtype, device=block.device)
    dist.all_gather_into_tensor(out, block.contiguous())
    return out
