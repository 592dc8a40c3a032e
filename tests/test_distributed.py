"""Host-side logic of the multi-GPU (row-partitioned) solve, on CPU.

* partitions (level 0: contiguous, 128-aligned, covering; coarse levels by
  seed ownership -- SURVEY.md §8e) through the library's host helpers;
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


def test_coarse_partition_follows_seed_ownership():
    from paper_1302_2547_b200 import distributed as D

    rng = np.random.default_rng(1)
    n = 5000
    seeds = np.sort(rng.choice(n, size=700, replace=False)).astype(np.int32)
    fine = D.partition_rows(n, 4)
    cb = D.partition_coarse(seeds, fine)
    assert cb[0] == 0 and cb[-1] == seeds.shape[0]
    for q in range(4):
        owned = seeds[cb[q]:cb[q + 1]]
        assert np.all((owned >= fine[q]) & (owned < fine[q + 1]))


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1302_2547_b200 import distributed as D

    local = bytes([rank]) * D.HANDLE_BYTES
    allh = D.exchange_handles(local)
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
    out[rank] = (allh, tot.tobytes())
    dist.destroy_process_group()


def test_two_rank_handle_exchange_and_rank_ordered_fold():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == bytes([0]) * 64 + bytes([1]) * 64
    assert res[0][1] == res[1][1]  # identical bits on every rank
