"""Multi-process (world size 2, gloo, CPU) tests of the batch sharding and the final gather."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_12692_b200.dist import gather_barcodes, shard_range


def test_shard_range_covers_exactly():
    for n in [0, 1, 5, 64, 65536, 65537]:
        for world in [1, 2, 3, 8]:
            got = [shard_range(n, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            for (a, b), (c, d) in zip(got, got[1:]):
                assert b == c and b - a >= d - c >= b - a - 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, nimg=7):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r owns images [start, stop) of a batch of nimg; image i has i % 3 bars (some none)
        start, stop = shard_range(nimg, rank, world)
        rows, offs = [], [0]
        for i in range(start, stop):
            for k in range(i % 3):
                rows.append([k % 2, 100 * i + k, 100 * i + k + 1])
            offs.append(len(rows))
        pairs = torch.tensor(rows, dtype=torch.int32).reshape(-1, 3)
        offsets = torch.tensor(offs, dtype=torch.int64)
        got = gather_barcodes(pairs, offsets)
        q.put((rank, None if got is None else (got[0].tolist(), got[1].tolist())))
    finally:
        dist.destroy_process_group()


def _run(world, nimg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, nimg)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,nimg", [(2, 7), (3, 2)])
def test_gather_to_rank0_gloo(world, nimg):
    """Rank 0 receives every shard's bars and CSR offsets in input order (a rank may own no
    image); the other ranks get None."""
    res = _run(world, nimg)
    exp_rows, exp_offs = [], [0]
    for i in range(nimg):
        for k in range(i % 3):
            exp_rows.append([k % 2, 100 * i + k, 100 * i + k + 1])
        exp_offs.append(len(exp_rows))
    rows, offs = res[0]
    assert rows == exp_rows
    assert offs == exp_offs
    for r in range(1, world):
        assert res[r] is None
