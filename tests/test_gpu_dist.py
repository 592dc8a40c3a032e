"""Multi-process row-partitioned setup and solve (csrc/dist_setup.cu,
dist_solve.cu): two processes share the one GPU of this harness, each
holding only its rows, with CUDA-IPC-mapped peer arenas and the device flag
barrier between phases -- the code path of one process per GPU on an
8xB200 box.  Its hierarchy (per-rank blocks) and residual history must be
bit-identical to the same partition run as virtual ranks in one process,
and the history within 1e-10 of the reference's."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from golden_util import assert_history_close, problem_for

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_block(ip, ix, a, r0, r1):
    import torch

    from paper_1302_2547_b200.device import DeviceCSR, to_device_padded
    e0, e1 = int(ip[r0]), int(ip[r1])
    return DeviceCSR(r1 - r0, ip.shape[0] - 1, to_device_padded((ip[r0:r1 + 1] - e0).astype(np.int32), np.int32),
                     to_device_padded(ix[e0:e1].astype(np.int32), np.int32), to_device_padded(a[e0:e1], np.float64))


def _worker(rank, world, port, case, shard_rows, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1302_2547_b200 as U
    from paper_1302_2547_b200 import distributed as D

    ip, ix, a, g = problem_for(case)
    n = ip.shape[0] - 1
    bounds = D.partition_rows(n, world)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    dh = D.setup_distributed(_local_block(ip, ix, a, r0, r1), n=n, bounds=bounds, group=dist.group.WORLD,
                             shard_rows=shard_rows)
    levels = []
    for l in range(dh.n_levels):
        lv = dh.local_level(l)
        levels.append({k: (v.tobytes() if isinstance(v, np.ndarray) else v) for k, v in lv.items()})
    b = np.ones(r1 - r0)
    x, rep = D.npcg_solve_distributed(dh, U.CycleSpec(), U.Smoother(), b, tol=float(g["tol"]), max_iters=500)
    out[rank] = (np.asarray(rep.residual_history).tobytes(), x.tobytes(), levels, dh.n_levels, dh.n_sharded)
    dh.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("case,shard_rows", [("g2d_dir_64", 200), ("rgg_20000", 1000)])
def test_two_process_setup_and_solve(case, shard_rows):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1302_2547_b200 as U
    from paper_1302_2547_b200 import distributed as D

    ip, ix, a, g = problem_for(case)
    n = ip.shape[0] - 1
    A = U.SparseMatrix(n, n, ip, ix, a)
    world = 2
    dv = D.setup_distributed(A, ranks=world, shard_rows=shard_rows)
    xv, rv = D.npcg_solve_distributed(dv, U.CycleSpec(), U.Smoother(), np.ones(n), tol=float(g["tol"]), max_iters=500)
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, case, shard_rows, out), nprocs=world, join=True)
        res = dict(out)
    bounds = D.partition_rows(n, world)
    hs = [np.frombuffer(res[r][0]) for r in range(world)]
    assert np.array_equal(hs[0], hs[1])
    assert np.array_equal(hs[0], np.asarray(rv.residual_history)), "multi-process history differs from virtual ranks"
    x = np.concatenate([np.frombuffer(res[r][1]) for r in range(world)])
    assert np.array_equal(x, xv)
    assert_history_close(list(hs[0]), g, rtol=1e-10)
    for r in range(world):
        assert res[r][3] == dv.n_levels and res[r][4] == dv.n_sharded
        for l, lv in enumerate(res[r][2]):
            ref = dv.local_level(l, r if l < dv.n_sharded else 0)
            for k, v in ref.items():
                got = lv[k]
                if isinstance(v, np.ndarray):
                    assert got == v.tobytes(), f"rank {r} level {l} {k}"
                else:
                    assert got == v, f"rank {r} level {l} {k}"
