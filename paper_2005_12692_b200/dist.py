"""Multi-GPU plumbing for batched barcodes (PAPER.md:489-496 batches of images).

Images of a batch are independent, so a batch is sharded into contiguous slices, one per rank
(one process per GPU, torch.distributed over NCCL on the GPU box); nothing is exchanged while the
barcodes are computed.  The only collective is the final gather of the variable-length barcodes
onto one rank (rank 0 by default) in input order: every rank sends its (pair count, image count)
and then its exact-size payloads point to point; the destination concatenates them.  Bytes moved
= the barcodes once (12 B per bar + 8 B per image), not N times as an all-gather would.
Single images are not sharded (replicas only).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced slice [start, stop) of n items for `rank` of `world`."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_barcodes(pairs: torch.Tensor, offsets: torch.Tensor, dst: int = 0, group=None):
    """Gather every rank's (pairs (M,3) int32, offsets (B+1,) int64 CSR) onto rank `dst`, in rank
    order (= input order for contiguous shards).  Returns (pairs_all, offsets_all) on `dst` and
    None on the other ranks.  Any backend (NCCL for CUDA tensors, gloo for CPU tensors)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    gdst = dist.get_global_rank(group, dst) if group is not None else dst
    dev = pairs.device
    m = torch.tensor([pairs.shape[0], offsets.shape[0] - 1], dtype=torch.int64, device=dev)
    if rank != dst:
        dist.send(m, gdst, group=group)
        if pairs.shape[0]:
            dist.send(pairs.contiguous(), gdst, group=group)
        dist.send(offsets.contiguous(), gdst, group=group)
        return None
    parts_p, parts_o = [], []
    for r in range(world):
        src = dist.get_global_rank(group, r) if group is not None else r
        if r == dst:
            p, o = pairs, offsets
        else:
            c = torch.empty(2, dtype=torch.int64, device=dev)
            dist.recv(c, src, group=group)
            npairs, nimg = int(c[0]), int(c[1])
            p = torch.empty((npairs, 3), dtype=pairs.dtype, device=dev)
            if npairs:
                dist.recv(p, src, group=group)
            o = torch.empty((nimg + 1,), dtype=offsets.dtype, device=dev)
            dist.recv(o, src, group=group)
        parts_p.append(p)
        parts_o.append(o)
    out_o, base = [offsets.new_zeros(1)], 0
    for p, o in zip(parts_p, parts_o):
        out_o.append(o[1:] - o[0] + base)
        base += int(p.shape[0])
    return torch.cat(parts_p), torch.cat(out_o)
