"""Data-parallel plumbing for the SDNN path.

Every stage of the forward path is per sample (rank coding ranks within a
sample, conv / fire / pool / inhibit / WTA / gather are per sample), so a batch
shards by contiguous image ranges with no data-path collective.  The only
collectives are the weight broadcast before a sharded forward and an optional
gather of features/records after it.  STDP training is sample-sequential
(reading R-BATCH): training ranks run independent replicas, or — with
data-parallel mini-batch STDP (`Network.enable_dp`) — one
model whose global mini-batch is split across ranks: every rank all-gathers the
winner records and the trained layer's input latency maps and applies the same
sequential update, so the replicas stay bit-identical with no weight broadcast.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard of n items for `rank` of `world`: (start, count); sizes differ by <= 1."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def broadcast_weights(weights: list[torch.Tensor], src: int = 0) -> None:
    """Make every rank's weights bit-identical to rank `src`'s (NCCL over NVLink on GPUs, gloo on CPU)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return
    for w in weights:
        dist.broadcast(w, src=src)


def gather_rows(x: torch.Tensor, n_total: int) -> torch.Tensor | None:
    """All-gather per-rank row blocks (shard_range sizes) into the full [n_total, ...] on every rank."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return x
    world = dist.get_world_size()
    sizes = [shard_range(n_total, world, r)[1] for r in range(world)]
    m = max(sizes)
    pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    pad[: x.shape[0]] = x
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])


def allgather_equal(dst: torch.Tensor, src: torch.Tensor) -> None:
    """dst[r * n : (r + 1) * n] = rank r's src (n = src.shape[0], equal on every rank), in rank order."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        dst.copy_(src)
        return
    try:
        dist.all_gather_into_tensor(dst, src.contiguous())
    except (RuntimeError, NotImplementedError):  # backends without the fused form (older gloo)
        parts = list(dst.chunk(dist.get_world_size()))
        tmp = [torch.empty_like(p) for p in parts]
        dist.all_gather(tmp, src.contiguous())
        for p, t in zip(parts, tmp):
            p.copy_(t)
