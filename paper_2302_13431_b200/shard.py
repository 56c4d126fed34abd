"""Multi-GPU plumbing for the sharded configurations.

Multislice 2-D (C3) is a set of independent estimate_maps problems, one per
slice: slices are split into contiguous blocks across ranks (one process per
GPU) and every rank runs the whole pipeline (its own Gram, eigensolve, G(x),
power iteration) on its block.  There is no data-path collective; the only
communication is an optional gather of the per-slice outputs to rank 0
(NCCL over NVLink on the box, gloo in the CPU tests).  Single-slice configs
(C1, C2, C5) do not shard: ranks run independent replicas.
"""
from __future__ import annotations

import numpy as np


def partition(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [start, stop) of `n_items` for `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def counts(n_items: int, world: int) -> list[int]:
    return [b - a for a, b in (partition(n_items, world, r) for r in range(world))]


def run_local(estimate_one, calibs_local):
    """Apply `estimate_one(calib) -> dict of arrays` to each local slice; stack per key."""
    outs = [estimate_one(c) for c in calibs_local]
    if not outs:
        return {}
    return {k: np.stack([o[k] for o in outs]) for k in outs[0]}


def gather_slices(local: np.ndarray, n_items: int, group=None, device=None):
    """Gather per-rank slice blocks (leading axis = slices) to every rank, in slice order.

    Uses all_gather over equal-size padded blocks (the block sizes differ by at
    most one); returns the concatenated (n_items, ...) array on every rank.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    cnt = counts(n_items, world)
    pad = max(cnt)
    shape = local.shape[1:]
    buf = np.zeros((pad,) + shape, dtype=local.dtype)
    buf[: local.shape[0]] = local
    t = torch.from_numpy(buf.view(np.uint8).reshape(pad, -1).copy())
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    rows = []
    for r, p in enumerate(parts):
        arr = p.cpu().numpy().reshape((pad,) + (-1,)).view(local.dtype).reshape((pad,) + shape)
        rows.append(arr[: cnt[r]])
    return np.concatenate(rows, axis=0)
