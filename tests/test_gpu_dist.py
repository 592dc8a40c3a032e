"""Multi-process row-partitioned solve (csrc/shard.cu, uaamg_dist_*): two
processes share the one GPU of this harness, each with its own hierarchy,
CUDA-IPC-mapped peer arenas and the device flag barrier between phases.
The residual history must match the single-process solve within round-off
(only the dot folds differ) and the reference's within 1e-10."""
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


def _worker(rank, world, port, case, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1302_2547_b200 as U
    from paper_1302_2547_b200.distributed import npcg_solve_distributed

    ip, ix, a, g = problem_for(case)
    h = U.setup(U.SparseMatrix(ip.shape[0] - 1, ip.shape[0] - 1, ip, ix, a))
    b = np.ones(ip.shape[0] - 1)
    x, rep = npcg_solve_distributed(h, U.CycleSpec(), U.Smoother(), b, tol=float(g["tol"]), max_iters=500,
                                    shard_rows=200)
    out[rank] = (np.asarray(rep.residual_history).tobytes(), x.tobytes())
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["g2d_dir_64"])
def test_two_process_solve(case):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1302_2547_b200 as U

    ip, ix, a, g = problem_for(case)
    h = U.setup(U.SparseMatrix(ip.shape[0] - 1, ip.shape[0] - 1, ip, ix, a))
    x1, r1 = U.npcg_solve(h, U.CycleSpec(), U.Smoother(), np.ones(ip.shape[0] - 1), tol=float(g["tol"]),
                          max_iters=500)
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, case, out), nprocs=world, join=True)
        res = dict(out)
    hs = [np.frombuffer(res[r][0]) for r in range(world)]
    xs = [np.frombuffer(res[r][1]) for r in range(world)]
    assert np.array_equal(hs[0], hs[1]) and np.array_equal(xs[0], xs[1])
    assert_history_close(list(hs[0]), g, rtol=1e-10)
    h1 = np.asarray(r1.residual_history)
    assert hs[0].shape == h1.shape
    assert np.all(np.abs(hs[0] - h1) <= 1e-12 * np.abs(h1) + 1e-15)
    np.testing.assert_allclose(xs[0], x1, rtol=1e-9, atol=1e-12 * np.abs(x1).max())
