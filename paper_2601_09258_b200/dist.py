"""Multi-GPU plumbing: instance sharding and the final alert/summary gather.

Monitored instances are independent, so the event streams are
partitioned by instance with no data-path collective; the only collective is
the final gather of each shard's alerts + summaries to rank 0 (NCCL over
NVLink in bench.py; gloo in the CPU tests).  Plumbing only — no analysis here.
"""
from __future__ import annotations

import numpy as np


def shard_by_weight(weights, world: int):
    """Contiguous instance ranges [b, e) per rank balancing sum(weights)
    (events per instance).  Every rank gets a range (possibly empty)."""
    w = np.asarray(weights, dtype=np.float64)
    n = len(w)
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(0, world - 1)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        k = int(np.searchsorted(cum, target, side="left"))
        k = min(max(k, cuts[-1]), n)
        cuts.append(k)
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def gather_bytes(payload: np.ndarray, device=None):
    """Gather variable-size uint8 payloads from every rank to rank 0.
    Returns the list of per-rank arrays on rank 0, None elsewhere.
    Two collectives: sizes (all_gather), then padded payloads (all_gather)."""
    import torch
    import torch.distributed as dist

    payload = np.ascontiguousarray(payload, dtype=np.uint8)
    world = dist.get_world_size()
    t = torch.from_numpy(payload.copy())
    if device is not None:
        t = t.to(device)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    mx = max(1, int(max(s.item() for s in sizes)))
    buf = torch.zeros(mx, dtype=torch.uint8, device=t.device)
    buf[: t.numel()] = t
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    if dist.get_rank() != 0:
        return None
    return [b[: int(s.item())].cpu().numpy() for b, s in zip(bufs, sizes)]


def max_over_ranks(value: float, device=None) -> float:
    """Max of a timing over ranks (device timers, max-over-ranks rule)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
