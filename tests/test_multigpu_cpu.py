"""World-size-2 gloo tests of the multi-GPU host logic (no GPU needed).

The data path shards rows with no collective; these tests check the shard
partition, the max-over-ranks timing reduction and the row gather, with the
CPU oracle standing in for each rank's device transform (test-only)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1404_1810_b200.dist import gather_rows, max_over_ranks, shard_rows


def test_shard_rows_partition():
    for total in (0, 1, 7, 65536, 65537):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                s, c = shard_rows(total, world, r)
                seen.extend(range(s, s + c))
            assert seen == list(range(total))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    r = O.restatement()
    rng = np.random.default_rng(3)
    full = rng.standard_normal((total, 2 * n))
    start, cnt = shard_rows(total, world, rank)
    local = np.stack([r.execute(4, O.F_CDFT, n, full[i]) for i in range(start, start + cnt)])
    gathered = gather_rows(torch.tensor(local), total).numpy()
    ms = max_over_ranks(1.0 + rank)
    if rank == 0:
        want = np.stack([r.execute(4, O.F_CDFT, n, full[i]) for i in range(total)])
        q.put((bool(np.array_equal(gathered, want)), ms))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_shard_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 64, 5, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, ms = q.get(timeout=100)
    for p in procs:
        p.join(timeout=60)
    assert ok
    assert ms == 2.0
