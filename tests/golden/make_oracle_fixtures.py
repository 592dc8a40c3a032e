"""Pin the full-size configs C3, C4 and C5 with the CPU oracle.

The reference itself cannot run these sizes in reasonable time (SURVEY.md
section 8d: hours and >100 GB), so their fixtures come from the oracle port
(oracle/uaamg_oracle.c), which is itself pinned bit-exact to the reference
on every hierarchy fixture of tests/golden/make_golden.py and, at the same
family and a smaller size, on C2 (3D 7-pt 128^3) and the solvable C3 graph at
2^18 vertices (rgg_lcc_262144).  Run it on the GPU box host (196 GB, 16
cores; the development container has 62 GB) inside a gpurun lease:

    python tests/golden/make_oracle_fixtures.py --only c4,c5,c3,c3lit --out gpurun_out/fixtures

then copy the .npz files into tests/golden/.  Per config it stores, like
make_golden.py: per-level n, nnz and SHA-256 of (indptr, indices, data) as
int64/int64/float64 and of vertex_to_agg / coarse_vertex_of_agg, n_levels,
complexities, the input digest (int64 layout and the device int32 layout),
the iteration count and the full residual history of
npcg_solve(b = ones, tol = 1e-8, K-cycle, l1), plus the oracle's thread
count and timings.  For the literal C3 graph (SURVEY.md 8d without the
largest-component restriction) it stores the SetupError message instead.
TEST INFRASTRUCTURE ONLY.
"""

import argparse
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(HERE))

from golden_util import sha  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1302_2547_b200 import problems as P  # noqa: E402

CONFIGS = {
    "c4": ("oracle_c4_grid3d27_256", lambda: P.grid3d(256, 27)),
    "c5": ("oracle_c5_grid3d7_512", lambda: P.grid3d(512, 7)),
    "c3": ("oracle_c3_rgg_lcc_8m", lambda: P.random_geometric(1 << 23, 12.0, 0, largest_component=True)),
    "c3lit": ("oracle_c3_rgg_literal_8m", lambda: P.random_geometric(1 << 23, 12.0, 0)),
}


def input_digests(A):
    h32 = hashlib.sha256()
    for arr in (A.indptr, A.indices):
        for k in range(0, arr.shape[0], 1 << 26):  # int32 copies chunk by chunk
            h32.update(memoryview(arr[k:k + (1 << 26)].astype(np.int32)).cast("B"))
    h32.update(memoryview(A.data).cast("B"))
    return {"input_sha": np.array(sha(A.indptr, A.indices, A.data)), "input_sha32": np.array(h32.hexdigest())}


def run(key, out_dir, tol=1e-8):
    name, build = CONFIGS[key]
    t = time.perf_counter()
    A = build()
    print(f"{name}: n={A.n_rows} nnz={A.nnz} built in {time.perf_counter() - t:.1f}s", flush=True)
    out = input_digests(A)
    ip, ix, a = A.indptr, A.indices, A.data
    del A  # the oracle keeps its own copy of level 0
    out["n"] = np.array(ip.shape[0] - 1)
    out["nnz"] = np.array(ix.shape[0])
    out["threads"] = np.array(O.get_num_threads())
    t = time.perf_counter()
    try:
        h = O.setup(ip, ix, a, copy=False)
    except O.OracleError as e:
        out["setup_error"] = np.array(str(e))
        out["setup_seconds"] = np.array(time.perf_counter() - t)
        print(f"    SetupError: {e}", flush=True)
        np.savez_compressed(os.path.join(out_dir, name + ".npz"), **out)
        return
    out["setup_seconds"] = np.array(time.perf_counter() - t)
    print(f"    setup {float(out['setup_seconds']):.1f}s levels={[L.n for L in h.levels]}", flush=True)
    out["n_levels"] = np.array(h.n_levels)
    out["singular"] = np.array(int(h.singular))
    n0 = h.levels[0].n
    nnz0 = max(h.levels[0].nnz, 1)
    out["grid_complexity"] = np.array(sum(L.n for L in h.levels) / n0)
    out["operator_complexity"] = np.array(sum(L.nnz for L in h.levels) / nnz0)
    for l, L in enumerate(h.levels):
        out[f"L{l}_n"] = np.array(L.n)
        out[f"L{l}_nnz"] = np.array(L.nnz)
        out[f"L{l}_csr_sha"] = np.array(sha(L.indptr, L.indices, L.data))
        if L.vertex_to_agg is not None:
            out[f"L{l}_v2a_sha"] = np.array(sha(L.vertex_to_agg))
            out[f"L{l}_seeds_sha"] = np.array(sha(L.coarse_vertex_of_agg))
    del ip, ix, a
    b = np.ones(n0)
    t = time.perf_counter()
    x, rep = O.npcg_solve(h, b, tol=tol, max_iters=500)
    out["solve_seconds"] = np.array(time.perf_counter() - t)
    out["b"] = np.zeros(0)
    out["b_sha"] = np.array(sha(b))
    out["history"] = np.array(rep.residual_history)
    out["iterations"] = np.array(rep.iterations)
    out["converged"] = np.array(int(rep.converged))
    out["x"] = np.zeros(0)
    out["x_sha"] = np.array(sha(x))
    out["tol"] = np.array(tol)
    out["cfg"] = np.array("({}, {})")
    print(f"    solve {float(out['solve_seconds']):.1f}s: {rep.iterations} it, final {rep.residual_history[-1]:.3e}",
          flush=True)
    np.savez_compressed(os.path.join(out_dir, name + ".npz"), **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c4,c5,c3,c3lit")
    ap.add_argument("--out", default=HERE)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    O.set_num_threads(args.threads)
    for key in args.only.split(","):
        run(key, args.out)


if __name__ == "__main__":
    main()
