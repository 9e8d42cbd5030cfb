"""Multi-GPU sharding of the PILC batch path.

Images / patches are independent containers, so a batch shards by
contiguous index ranges with no data-path exchange: each rank (one process
per GPU) compresses or decompresses its own slice on its own device. The
only communication is the optional gather of the per-rank results (blob
buffers into one (buffer, offsets) pair with rebased offsets; decoded
images in input order) on a destination rank, over the process group's
backend (gloo on CPU tests, NCCL on GPU boxes) after the data path is done.
One process driving several GPUs uses `devices=[...]` instead (multi.py),
which needs no process group and copies results without pickling."""

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


def compress_sharded(images, model=None, config=None, group=None, dst: int = 0, device=None, codec=None):
    """Each rank compresses its contiguous share of `images` (every rank
    passes the whole batch or a view of it) on its own GPU; rank `dst` gets
    the full (buffer, offsets) in input order, None elsewhere. `codec`
    (images, model, config) -> (buffer, offsets) replaces compress_batch
    (the CPU tests inject the oracle)."""
    import torch.distributed as dist

    from .container import CodecConfig, compress_batch

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    s, e = shard_range(len(images), rank, world)
    cfg = config or CodecConfig()
    if codec is not None:
        buf, off = codec(images[s:e], model, cfg)
    elif e > s:
        buf, off = compress_batch(images[s:e], model, cfg, device=device)
    else:
        buf, off = np.zeros(0, np.uint8), np.zeros(1, np.uint64)
    return gather_blobs(buf, off, dst, group)


def decompress_sharded(buffer, offsets, model=None, group=None, dst: int = 0, device=None, codec=None):
    """Each rank decodes its contiguous share of the blobs (every rank passes
    the whole (buffer, offsets), or at least its share's bytes) on its own
    GPU; rank `dst` gets every image in input order (an (N, H, W, 3) array
    when the shapes agree, else a list), None elsewhere. `codec` (buffer,
    offsets, model) -> images replaces decompress_batch."""
    import torch.distributed as dist

    from .container import check_offsets, decompress_batch

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    offs = check_offsets(offsets)
    s, e = shard_range(offs.size - 1, rank, world)
    sub = np.asarray(buffer, np.uint8)[int(offs[s]): int(offs[e])]
    soff = offs[s: e + 1] - offs[s]
    if e == s:
        imgs = []
    elif codec is not None:
        imgs = codec(sub, soff, model)
    else:
        imgs = decompress_batch(sub, soff, model, device=device)
    got = [None] * world if rank == dst else None
    dist.gather_object(imgs if isinstance(imgs, list) else np.asarray(imgs), got, dst=dst, group=group)
    if rank != dst:
        return None
    parts = [p for p in got if len(p)]
    if parts and all(isinstance(p, np.ndarray) for p in parts) and len({p.shape[1:] for p in parts}) == 1:
        return np.concatenate(parts)
    return [im for p in parts for im in p]
