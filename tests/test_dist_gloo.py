"""Multi-process host plumbing on CPU (gloo, world size 2): the row-strip partition, the
ncclUniqueId broadcast, max-over-ranks timing, counter sums and shard gathering that
bench.py uses for N > 1 (the device exchange itself is NCCL inside libaca.so)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_cs_0502039_b200 import dist as adist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims = (16, 8)
        parts = adist.partition(dims, world)
        y0, y1 = parts[rank]
        payload = bytes(range(128)) if rank == 0 else bytes(128)
        uid = adist.broadcast_bytes(payload)
        tmax = adist.reduce_max(1.5 + rank)
        tot = adist.reduce_sum_int(10 + rank)
        full = np.arange(16 * 8, dtype=np.int64).reshape(8, 16)
        local = full[y0:y1].ravel().astype(np.uint64)
        g = adist.gather_shards(local, dims)
        blobs = adist.all_gather_bytes(bytes([rank + 1]) * 192)   # IPC blob exchange (push mode)
        q.put((rank, parts, uid == bytes(range(128)) and blobs == b"\x01" * 192 + b"\x02" * 192, tmax, tot,
               bool(np.array_equal(g, full.astype(np.uint64)))))
    finally:
        dist.destroy_process_group()


def test_partition_rules():
    from paper_cs_0502039_b200 import dist as adist
    assert adist.partition((16384, 16384), 8)[3] == (6144, 8192)
    assert adist.partition((512, 512, 512), 4)[-1] == (384, 512)
    with pytest.raises(ValueError):
        adist.partition((10, 10), 3)


def test_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert [r[0] for r in res] == [0, 1]
    for rank, parts, uid_ok, tmax, tot, gather_ok in res:
        assert parts == [(0, 4), (4, 8)]
        assert uid_ok and tmax == 2.5 and tot == 21 and gather_ok
