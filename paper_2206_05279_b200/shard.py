"""Multi-GPU sharding of the PILC batch path.

Images / patches are independent containers, so a batch shards by
contiguous index ranges with no data-path exchange: each rank (one process
per GPU) compresses or decompresses its own slice on its own device. The
only communication is the optional gather of the per-rank blob buffers into
one (buffer, offsets) pair on a destination rank -- a host-side
concatenation with rebased offsets, done over the process group's backend
(gloo on CPU tests, NCCL on GPU boxes)."""

from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, end) of rank's share; the first n % world ranks get
    one extra item."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def concat_blobs(parts: list) -> tuple[np.ndarray, np.ndarray]:
    """[(buffer, offsets)] in rank order -> one (buffer, offsets uint64[N+1])."""
    bufs, offs = [], [np.zeros(1, np.uint64)]
    base = 0
    for buf, off in parts:
        off = np.asarray(off, np.uint64)
        bufs.append(np.asarray(buf, np.uint8)[int(off[0]): int(off[-1])])
        offs.append(off[1:] - off[0] + np.uint64(base))
        base += int(off[-1] - off[0])
    return (np.concatenate(bufs) if bufs else np.zeros(0, np.uint8)), np.concatenate(offs)


def gather_blobs(buf: np.ndarray, off: np.ndarray, dst: int = 0, group=None):
    """Gather every rank's (buffer, offsets) to rank `dst` (None elsewhere)."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    got = [None] * world if rank == dst else None
    dist.gather_object((np.asarray(buf, np.uint8), np.asarray(off, np.uint64)), got, dst=dst, group=group)
    return concat_blobs(got) if rank == dst else None


def compress_sharded(images, model=None, config=None, group=None, dst: int = 0):
    """Each rank compresses its contiguous share of `images` (every rank
    passes the whole batch or a view of it); rank `dst` gets the full
    (buffer, offsets) in input order."""
    import torch.distributed as dist

    from .container import CodecConfig, compress_batch

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    s, e = shard_range(len(images), rank, world)
    buf, off = compress_batch(images[s:e], model, config or CodecConfig())
    return gather_blobs(buf, off, dst, group)
