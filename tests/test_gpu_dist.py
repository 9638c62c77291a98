"""Sharded batches on one GPU: a batch split into 2 and 4 contiguous
shards, each shard's barcodes computed by cr_barcodes_batched, the shards gathered onto rank 0 by
dist.gather_barcodes (world size 2 / 4, gloo over host copies -- the NCCL transport is the same
code on the GPU box) must be byte-identical to the unsharded call's bars and CSR offsets."""
import os
import socket

import numpy as np
import pytest

from workloads import generators as gen

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shard, q):
    import torch
    import torch.distributed as dist
    from paper_2005_12692_b200.dist import gather_barcodes
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pairs, offs = shard
        got = gather_barcodes(torch.from_numpy(pairs), torch.from_numpy(offs))
        q.put((rank, None if got is None else (got[0].numpy(), got[1].numpy())))
    finally:
        dist.destroy_process_group()


def _gather(shards):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = len(shards)
    procs = [ctx.Process(target=_worker, args=(r, world, port, shards[r], q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res[0]


def _batched(cr, imgs, md):
    import torch
    bc, off = cr.barcodes_batched(torch.from_numpy(np.ascontiguousarray(imgs)).cuda(), md)
    return np.ascontiguousarray(bc.pairs.cpu().numpy()), off.cpu().numpy()


@pytest.mark.parametrize("kind", ["c3_like", "c5b_like"])
def test_sharded_batch_equals_unsharded(kind):
    import paper_2005_12692_b200 as cr
    from paper_2005_12692_b200.dist import shard_range
    if kind == "c3_like":
        imgs, md = gen.blobs(2048, 3), 1                       # K7 path (one CTA per image)
    else:
        imgs = np.stack([gen.masked_grf((40, 40, 40), 3.0, 19.0, g)
                         for g in [np.random.default_rng(6)] * 12])  # stacked 3D path
        md = 2
    ref_p, ref_o = _batched(cr, imgs, md)
    for world in (2, 4):
        shards = []
        for r in range(world):
            a, b = shard_range(len(imgs), r, world)
            shards.append(_batched(cr, imgs[a:b], md))
        p, o = _gather(shards)
        assert np.array_equal(o, ref_o), (kind, world)
        assert np.array_equal(p.view(np.uint32), ref_p.view(np.uint32)), (kind, world)
