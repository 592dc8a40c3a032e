"""Host-side logic of the multi-GPU (row-partitioned) solve, on CPU.

* partitions (level 0: contiguous, 128-aligned, covering; coarse levels by
  the renumbering's per-rank seed counts -- SURVEY.md §8e) through the
  library's host helpers, across two gloo ranks as dist_setup runs them;
* the agreement on failure that keeps a failing rank from leaving its peers
  in the device barrier;
* the handle exchange the processes run over torch.distributed, with two
  gloo ranks (world_size 2, 127.0.0.1);
* the rank-ordered cross-rank fold of per-rank partial sums that makes every
  rank hold the same bits.
No CUDA kernels run here (the library only needs to load).
"""
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


def test_level0_partition_properties():
    from paper_1302_2547_b200 import distributed as D

    for n in (1, 100, 128, 1000, 65536, 2097152, 2097153):
        for P in (1, 2, 3, 4, 5, 8):
            b = D.partition_rows(n, P)
            assert b[0] == 0 and b[-1] == n
            assert np.all(np.diff(b) >= 0)
            assert np.all(b[1:-1] % 128 == 0) or n < 128 * P
            if n >= 128 * P * 4:
                sizes = np.diff(b)
                assert sizes.max() - sizes.min() <= 256


def test_coarse_bounds_renumbering():
    """The sharded setup's renumbering (csrc/dist_solve.cu coarse_bounds,
    U/aggregation.py:199-203): with the seeds of each rank's rows counted,
    rank q's aggregates are the exclusive-scan block -- equal to numbering
    all seeds globally in ascending order."""
    from paper_1302_2547_b200 import distributed as D

    rng = np.random.default_rng(1)
    n = 5000
    seeds = np.sort(rng.choice(n, size=700, replace=False))
    for P in (1, 2, 3, 8):
        fine = D.partition_rows(n, P)
        counts = [int(np.count_nonzero((seeds >= fine[q]) & (seeds < fine[q + 1]))) for q in range(P)]
        cb = D.coarse_bounds(counts)
        assert cb[0] == 0 and cb[-1] == seeds.shape[0]
        for q in range(P):
            owned = seeds[cb[q]:cb[q + 1]]
            assert np.all((owned >= fine[q]) & (owned < fine[q + 1]))
    with pytest.raises(ValueError):
        D.coarse_bounds([3, -1])


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1302_2547_b200 import distributed as D

    local = bytes([rank]) * D.HANDLE_BYTES
    allh = D.exchange_handles(local)
    # renumbering across ranks exactly as dist_setup does it: per-rank seed
    # counts all-gathered, then the library's exclusive scan
    n = 4000
    seeds = np.sort(np.random.default_rng(7).choice(n, size=600, replace=False))
    fine = D.partition_rows(n, world)
    mine = seeds[(seeds >= fine[rank]) & (seeds < fine[rank + 1])]
    counts = [None] * world
    dist.all_gather_object(counts, int(mine.shape[0]))
    cb = D.coarse_bounds(counts)
    new_ids = cb[rank] + np.arange(mine.shape[0])
    ok_ids = bool(np.array_equal(new_ids, np.searchsorted(seeds, mine)))

    # a failing rank is seen by every rank (so nobody waits on the device)
    class _C:
        virtual = False
        group = None
    agree = D._fail_together(_C(), rank != 1)
    # rank-ordered fold of per-rank partials (what k_xfin does on device)
    rng = np.random.default_rng(rank)
    part = rng.standard_normal(3)
    import torch

    t = torch.tensor(part, dtype=torch.float64)
    parts = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, t)
    tot = np.zeros(3)
    for q in range(world):
        tot = tot + parts[q].numpy()
    out[rank] = (allh, tot.tobytes(), ok_ids, agree)
    dist.destroy_process_group()


def test_two_rank_handle_exchange_renumbering_and_fold():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == bytes([0]) * 64 + bytes([1]) * 64
    assert res[0][1] == res[1][1]  # identical bits on every rank
    assert res[0][2] and res[1][2]  # renumbering = global ascending-seed order
    assert res[0][3] is False and res[1][3] is False
