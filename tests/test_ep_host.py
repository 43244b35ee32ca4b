"""Host-side expert-parallel logic on CPU: the expert partition and the
handle all-gather over torch.distributed (gloo, world_size 2, 127.0.0.1)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2602_00879_b200 import ep


def test_partition_contiguous_balanced():
    for m in (8, 64, 128, 256):
        for g in (1, 2, 4, 8):
            parts = ep.partition(m, g)
            assert parts[0][0] == 0 and parts[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1
            for e in range(m):
                r = ep.owner_of(e, m, g)
                assert parts[r][0] <= e < parts[r][1]
    with pytest.raises(ValueError):
        ep.partition(4, 9)
    with pytest.raises(ValueError):
        ep.partition(2, 4)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blob = bytes([rank + 1]) * 128
    got = ep.all_gather_handles(blob)
    q.put((rank, got))
    dist.destroy_process_group()


def test_handle_all_gather_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = bytes([1]) * 128 + bytes([2]) * 128
    assert res[0] == want and res[1] == want
