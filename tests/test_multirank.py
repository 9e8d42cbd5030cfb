"""N>1 host logic on CPU: world_size-2 gloo process group, no GPU.

The data path has no collective (images shard by contiguous ranges); what
crosses ranks is the final gather of per-rank results. These tests drive the
product shard API (shard.compress_sharded / decompress_sharded) over gloo
with the CPU oracle injected as the per-rank codec (there is no GPU here;
tests/test_gpu_codec.py runs the same API on the GPU path) and check the
result is byte-identical to a single-rank batch."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_05279_b200.shard import (concat_blobs, compress_sharded, decompress_sharded, gather_blobs,
                                         shard_range)


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 8192, 4097):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1


def _blobs_for(imgs):
    from oracle import oracle as O

    blobs = [O.compress(im) for im in imgs]
    off = np.zeros(len(blobs) + 1, np.uint64)
    np.cumsum([len(b) for b in blobs], out=off[1:])
    return np.frombuffer(b"".join(blobs), np.uint8), off


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2206_05279_b200.synth import smooth_images

        from oracle import oracle as O

        imgs = smooth_images(9, 8, 8, seed=3)
        s, e = shard_range(len(imgs), rank, world)
        buf, off = _blobs_for(imgs[s:e])
        out = gather_blobs(buf, off, dst=0)
        # the product shard API with the oracle as each rank's codec
        out2 = compress_sharded(imgs, None, None, dst=0, codec=lambda im, m, c: _blobs_for(im))
        full_buf, full_off = _blobs_for(imgs)

        def dec(b, o, m):
            return np.stack([O.decompress(bytes(b[o[i]:o[i + 1]])) for i in range(len(o) - 1)])
        back = decompress_sharded(full_buf, full_off, None, dst=0, codec=dec)
        if rank == 0:
            assert out2[0].tobytes() == out[0].tobytes() and out2[1].tolist() == out[1].tolist()
            assert np.array_equal(back, imgs)
            q.put((out[0].tobytes(), out[1].tolist()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(300)
def test_gloo_world2_gather_matches_single_rank():
    from paper_2206_05279_b200.synth import smooth_images

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    buf, off = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_buf, ref_off = _blobs_for(smooth_images(9, 8, 8, seed=3))
    assert buf == ref_buf.tobytes() and off == ref_off.tolist()


def test_concat_rebases_offsets():
    a = (np.arange(10, dtype=np.uint8), np.array([0, 4, 10], np.uint64))
    b = (np.arange(5, dtype=np.uint8), np.array([0, 5], np.uint64))
    buf, off = concat_blobs([a, b])
    assert off.tolist() == [0, 4, 10, 15] and buf.tolist() == list(range(10)) + list(range(5))
