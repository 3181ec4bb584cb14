"""Multi-process (world sizes 2 and 4, gloo, CPU) coverage of the M-shard path's host logic: row
blocks, per-rank work on the local block (computed here by the CPU oracle, standing in for the
GPU kernel), max-over-ranks timing and the gather of C — compared with the unsharded oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, n, k, q):
    import sys
    sys.path.insert(0, ROOT)
    from oracle.oracle import EXACT, SAT, Oracle
    from paper_1910_00178_b200 import dist as pdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ora = Oracle()
        a = ora.mat_random_u8(m, k, 0)   # every rank derives the same inputs from the seed
        b = ora.mat_random_i8(n, k, 1)   # B replicated
        r0, r1 = pdist.row_block(m, rank, world)
        ok = True
        for mode in (EXACT, SAT):
            local = ora.gemm(a[r0:r1], b, mode, threads=1) if r1 > r0 else np.zeros((0, n), np.int32)
            full = pdist.gather_rows(torch.from_numpy(local), m, world).numpy()
            ok &= bool((full == ora.gemm(a, b, mode, threads=1)).all())
        t = pdist.reduce_max(1.0 + rank, world)
        s = pdist.reduce_sum(r1 - r0, world)
        q.put((rank, ok, t, s))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m", [(2, 300), (2, 1000), (2, 100), (4, 1000), (4, 300), (4, 100)])
def test_m_shard_gloo(world, m):
    """World sizes 2 and 4 with ragged row blocks (1000 rows over 4 ranks: 256/256/256/232) and
    ranks that own no rows at all (100 rows over 4 ranks)."""
    n, k = 70, 96
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, t, s in res:
        assert ok, f"rank {rank}: gathered C differs from the unsharded oracle"
        assert t == float(world)      # max over ranks
        assert s == float(m)          # rows partition M exactly


def test_row_blocks_partition_and_align():
    from paper_1910_00178_b200 import dist as pdist
    for m in (1, 127, 128, 129, 16384, 16385, 1000):
        for world in (1, 2, 4, 8):
            blocks = [pdist.row_block(m, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0 and a0 <= a1
            assert all(b0 % 128 == 0 for b0, _ in blocks if b0 < m)
