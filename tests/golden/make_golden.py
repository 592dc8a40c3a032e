"""Generate golden fixtures by running the REFERENCE package itself.

Run in the development container (the reference is not on the GPU box):

    python tests/golden/make_golden.py [--skip-c2]

The reference package is copied to a temporary directory (numba's cache=True
writes next to the sources, and /root/reference is read-only) and imported
from there with the default numba backend.  Outputs are small .npz files in
tests/golden/; large arrays are stored as sha256 digests.  The fixtures pin
(a) the CPU oracle (tests/test_oracle_golden.py) and (b) the B200 path
(tests/test_gpu_parity.py), and the problem builders (tests/test_problems.py).
"""

import argparse
import hashlib
import os
import shutil
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src/uaamg"


def load_reference():
    tmp = tempfile.mkdtemp(prefix="uaamg_ref_")
    shutil.copytree(REF_SRC, os.path.join(tmp, "uaamg"))
    os.environ["NUMBA_CACHE_DIR"] = os.path.join(tmp, "numba_cache")
    sys.path.insert(0, tmp)
    import uaamg  # noqa: E402
    from uaamg import kernels  # noqa: E402
    assert kernels.backend_name == "numba", kernels.backend_name
    return uaamg, kernels


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"  wrote {name}.npz ({os.path.getsize(path) / 1024:.1f} KiB)")


def grid3d_problem(U, n, stencil, bc):
    """3D lattice as a reference GraphProblem (the reference ships no 3D
    generator): +x/+y/+z (7-pt) or all forward (27-pt) neighbours, weight 1,
    Dirichlet boundary weight = number of missing neighbours."""
    edges, boundary = [], []
    for x in range(n):
        for y in range(n):
            for z in range(n):
                v = (x * n + y) * n + z
                miss = 0
                for dx in (-1, 0, 1):
                    for dy in (-1, 0, 1):
                        for dz in (-1, 0, 1):
                            if (dx, dy, dz) == (0, 0, 0):
                                continue
                            if stencil == 7 and abs(dx) + abs(dy) + abs(dz) > 1:
                                continue
                            X, Y, Z = x + dx, y + dy, z + dz
                            if not (0 <= X < n and 0 <= Y < n and 0 <= Z < n):
                                miss += 1
                                continue
                            w = (X * n + Y) * n + Z
                            if w > v:
                                edges.append((v, w, 1.0))
                if bc == "dirichlet" and miss:
                    boundary.append((v, float(miss)))
    return U.GraphProblem(n ** 3, edges, boundary)


def hier_arrays(h, full=True):
    out = {"n_levels": np.int64(h.n_levels), "singular": np.int64(h.singular),
           "grid_complexity": np.float64(h.grid_complexity),
           "operator_complexity": np.float64(h.operator_complexity)}
    for l, lev in enumerate(h.levels):
        A = lev.matrix
        out[f"L{l}_n"] = np.int64(A.n_rows)
        out[f"L{l}_nnz"] = np.int64(A.nnz)
        out[f"L{l}_csr_sha"] = np.array(sha(A.indptr, A.indices, A.data))
        if full and (l > 0 or A.nnz <= 400000):
            out[f"L{l}_indptr"] = A.indptr.astype(np.int32)
            out[f"L{l}_indices"] = A.indices.astype(np.int32)
            out[f"L{l}_data"] = A.data
        if lev.aggregation is not None:
            ag = lev.aggregation
            out[f"L{l}_v2a_sha"] = np.array(sha(ag.vertex_to_agg))
            out[f"L{l}_seeds_sha"] = np.array(sha(ag.coarse_vertex_of_agg))
            if full:
                out[f"L{l}_v2a"] = ag.vertex_to_agg.astype(np.int32)
                out[f"L{l}_seeds"] = ag.coarse_vertex_of_agg.astype(np.int32)
    return out


def solve_arrays(U, h, b, prefix="", x0=None, **kw):
    spec = U.CycleSpec(**{k: v for k, v in kw.items() if k in ("kind", "inner_krylov_steps", "pre_sweeps", "post_sweeps")})
    sm = U.Smoother(**{k: v for k, v in kw.items() if k in ("omega",)}, kind=kw.get("smoother", "l1"))
    tol = kw.get("tol", 1e-8)
    max_iters = kw.get("max_iters", 500)
    t = time.perf_counter()
    x, rep = U.npcg_solve(h, spec, sm, b, tol=tol, max_iters=max_iters, x0=x0)
    dt = time.perf_counter() - t
    print(f"    solve{prefix}: {rep.iterations} it, final {rep.residual_history[-1]:.3e}, {dt:.2f}s")
    return {prefix + "history": np.array(rep.residual_history), prefix + "iterations": np.int64(rep.iterations),
            prefix + "converged": np.int64(rep.converged), prefix + "x": x if x.shape[0] <= 70000 else np.zeros(0),
            prefix + "x_sha": np.array(sha(x)), prefix + "tol": np.float64(tol)}


def make_problems(U):
    """Small reference-assembled problems for builder parity."""
    print("problems")
    out = {}
    cases = {
        "g2d_dir_7": U.generate_structured_grid(7, "dirichlet"),
        "g2d_dir_7_aniso": U.generate_structured_grid(7, "dirichlet", (1.0, 10.0)),
        "g2d_dir_6_float": U.generate_structured_grid(6, "dirichlet", (0.3, 1.7)),
        "g2d_neu_6": U.generate_structured_grid(6, "neumann"),
        "g3d7_dir_4": grid3d_problem(U, 4, 7, "dirichlet"),
        "g3d7_neu_4": grid3d_problem(U, 4, 7, "neumann"),
        "g3d27_dir_4": grid3d_problem(U, 4, 27, "dirichlet"),
    }
    for name, prob in cases.items():
        A = U.assemble_laplacian(prob)
        out[name + "_indptr"] = A.indptr
        out[name + "_indices"] = A.indices
        out[name + "_data"] = A.data
    # random geometric graph: our builder's edge set re-assembled by the reference
    sys.path.insert(0, REPO)
    from paper_1302_2547_b200.problems import random_geometric
    Am, (ei, ej), bnd = random_geometric(600, 12.0, 3, return_edges=True)
    prob = U.GraphProblem(600, [(int(a), int(b), 1.0) for a, b in zip(ei, ej)], [(int(v), 1.0) for v in bnd])
    A = U.assemble_laplacian(prob)
    out["rgg_600_indptr"], out["rgg_600_indices"], out["rgg_600_data"] = A.indptr, A.indices, A.data
    save("problems", **out)


def random_weighted_problem(U, n, seed):
    """Random geometric graph with non-integer weights (exercises order-exact
    floating-point sums in Galerkin/restrict/spmv)."""
    rng = np.random.default_rng(seed)
    P = rng.random((n, 2))
    r = np.sqrt(7.0 / (np.pi * n))
    from scipy.spatial import cKDTree
    pairs = cKDTree(P).query_pairs(r, output_type="ndarray")
    w = rng.uniform(0.25, 2.0, size=pairs.shape[0])
    deg = np.bincount(pairs.ravel(), minlength=n)
    bmask = (deg == 0) | (rng.random(n) < 0.05)
    # every connected component needs a boundary vertex, else a coarse level
    # gets a zero row (the l1 smoother then raises NumericalError)
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    g = coo_matrix((np.ones(pairs.shape[0]), (pairs[:, 0], pairs[:, 1])), shape=(n, n))
    ncomp, lab = connected_components(g, directed=False)
    for c in range(ncomp):
        members = np.flatnonzero(lab == c)
        if not bmask[members].any():
            bmask[members[0]] = True
    bw = rng.uniform(0.1, 1.0, size=n)
    bnd = [(int(v), float(bw[v])) for v in np.flatnonzero(bmask)]
    edges = [(int(a), int(b), float(x)) for (a, b), x in zip(pairs, w)]
    return U.assemble_laplacian(U.GraphProblem(n, edges, bnd))


def make_kernels(U, K):
    print("kernels")
    A = random_weighted_problem(U, 400, 11)
    n = A.n_rows
    rng = np.random.default_rng(5)
    out = {"indptr": A.indptr, "indices": A.indices, "data": A.data}
    x = rng.standard_normal(n)
    b = rng.standard_normal(n)
    out["x"], out["b"] = x, b
    out["spmv"] = K.spmv(A.indptr, A.indices, A.data, x)
    out["diag_of"] = K.diag_of(A.indptr, A.indices, A.data)
    out["l1_diag"] = K.l1_diag(A.indptr, A.indices, A.data)
    out["degrees"] = K.degrees(A.indptr, A.indices)
    idx = rng.integers(0, 1 << 40, size=257).astype(np.int64)
    out["hash_idx"] = idx
    out["hash_u01"] = K.hash_u01(np.uint64(0xDEADBEEF12345678), 5, idx)
    out["scores_p0"] = K.quasi_random_scores(A.indptr, A.indices, np.uint64(0), 0)
    out["scores_s7_p3"] = K.quasi_random_scores(A.indptr, A.indices, np.uint64(7), 3)
    p2, x2 = K.squared_pattern(n, A.indptr, A.indices)
    out["a2_indptr"], out["a2_indices"] = p2, x2
    processed = rng.random(n) < 0.3
    out["processed"] = processed
    s = out["scores_s7_p3"]
    ctr = K.select_centers(p2, x2, s, processed)
    out["select"] = ctr
    owner = K.claim_owners(p2, x2, s, processed, ctr)
    out["claim"] = owner
    # admit on the real buckets of this pass (U/aggregation.py:152-169)
    centers = np.flatnonzero(ctr)
    claimed = np.flatnonzero(owner >= 0)
    claimed = claimed[~ctr[claimed]]
    crank = np.empty(n, dtype=np.int64)
    crank[centers] = np.arange(centers.shape[0])
    rank = crank[owner[claimed]]
    bptr = np.zeros(centers.shape[0] + 1, dtype=np.int64)
    bptr[1:] = np.cumsum(np.bincount(rank, minlength=centers.shape[0]))
    bjs = claimed[np.argsort(rank, kind="stable")]
    out["centers"], out["bucket_ptr"], out["bucket_js"] = centers, bptr, bjs
    for cap in (3, 1 << 62):
        pr = processed.copy()
        v2a = np.full(n, -1, dtype=np.int64)
        K.admit_members(A.indptr, A.indices, A.data, centers.astype(np.int64), bptr, bjs, cap, pr, v2a, 17)
        tag = "cap3" if cap == 3 else "uncapped"
        out[f"admit_{tag}_processed"] = pr
        out[f"admit_{tag}_v2a"] = v2a
    agg = U.aggregate(A, U.AggregationConfig(seed=3))
    out["agg_v2a"], out["agg_seeds"] = agg.vertex_to_agg, agg.coarse_vertex_of_agg
    gp, gi, gv = K.galerkin_coo(A.indptr, A.indices, A.data, agg.vertex_to_agg, agg.n_coarse)
    out["gal_indptr"], out["gal_indices"], out["gal_data"] = gp, gi, gv
    mp, mm = agg.members_csr()
    out["restrict"] = K.restrict(mp, mm, x)
    ec = rng.standard_normal(agg.n_coarse)
    out["e_coarse"] = ec
    out["prolongate"] = K.prolongate_add(agg.vertex_to_agg, ec, x)
    inv_m = 1.0 / out["l1_diag"]
    out["smooth3"] = K.smooth_sweeps(A.indptr, A.indices, A.data, inv_m, x, b, 3)
    # per-pass center record for a whole aggregation (capped) on this graph
    aggc = U.aggregate(A, U.AggregationConfig(seed=9, size_cap=4))
    out["aggcap4_v2a"], out["aggcap4_seeds"] = aggc.vertex_to_agg, aggc.coarse_vertex_of_agg
    save("kernels", **out)


def make_hierarchy(U, name, A, cfg_kw=None, setup_kw=None, solves=(), full=True, b=None):
    cfg_kw = cfg_kw or {}
    setup_kw = setup_kw or {}
    if not isinstance(A, U.SparseMatrix):  # our builder's host CSR -> reference type
        A = U.SparseMatrix(A.n_rows, A.n_cols, A.indptr, A.indices, A.data)
    print(f"{name}: n={A.n_rows} nnz={A.nnz}")
    t = time.perf_counter()
    h = U.setup(A, U.AggregationConfig(**cfg_kw), **setup_kw)
    print(f"    setup {time.perf_counter() - t:.2f}s levels={[l.matrix.n_rows for l in h.levels]}")
    out = hier_arrays(h, full=full)
    out["input_sha"] = np.array(sha(A.indptr, A.indices, A.data))
    if full and A.nnz <= 400000:
        pass  # level 0 arrays already stored
    if b is None:
        b = np.ones(A.n_rows)
    out["b"] = b if b.shape[0] <= 70000 else np.zeros(0)
    out["b_sha"] = np.array(sha(b))
    for tag, kw in solves:
        x0 = kw.pop("x0", None)
        out.update(solve_arrays(U, h, b, prefix=tag, x0=x0, **kw))
        if x0 is not None:
            out[tag + "x0"] = x0
    out["cfg"] = np.array(repr((cfg_kw, setup_kw)))
    save(name, **out)
    return h


def make_reshape(U, P):
    """Subgraph reshaping (reference reshaping.py:215-248): aggregations
    before / after 1 and 2 sweeps, and a setup(reshape_sweeps=1) hierarchy
    with its solve history."""
    print("reshape")
    out = {}
    cases = {
        "g2d16_t5": (P.grid2d(16), U.AggregationConfig(size_cap=5)),       # DisconnectedPair in the reference
        "g2d16_t4": (P.grid2d(16), U.AggregationConfig(size_cap=4)),
        "g2d12": (P.grid2d(12), U.AggregationConfig()),
        "g3d6_t6": (P.grid3d(6, 7), U.AggregationConfig(size_cap=6, seed=1)),
        "g3d6_27_t6": (P.grid3d(6, 27), U.AggregationConfig(size_cap=6)),
        "wgraph_t6": (random_weighted_problem(U, 3000, 4), U.AggregationConfig(size_cap=6, seed=2)),
    }
    for tag, (A, cfg) in cases.items():
        if not isinstance(A, U.SparseMatrix):
            A = U.SparseMatrix(A.n_rows, A.n_cols, A.indptr, A.indices, A.data)
        agg = U.aggregate(A, cfg)
        out[tag + "_indptr"], out[tag + "_indices"], out[tag + "_data"] = A.indptr, A.indices, A.data
        out[tag + "_v2a"], out[tag + "_seeds"] = agg.vertex_to_agg, agg.coarse_vertex_of_agg
        for key, kw in (("rs1", dict(sweeps=1)), ("rs2", dict(sweeps=2)),
                        ("rsj", dict(sweeps=1, smoother=U.Smoother("jacobi"))), ("rs1c8", dict(sweeps=1, pair_cap=8))):
            try:
                r = U.reshape_sweep(A, agg, **kw)
                out[f"{tag}_{key}_v2a"], out[f"{tag}_{key}_seeds"] = r.vertex_to_agg, r.coarse_vertex_of_agg
                res = "ok"
            except ValueError as e:  # DisconnectedPair (the reference raises it from reshape_sweep)
                out[f"{tag}_{key}_error"] = np.array(f"{type(e).__name__}: {e}")
                res = f"{type(e).__name__}"
            print(f"  {tag} {key}: n={A.n_rows} nc={agg.n_coarse} {res}")
    save("reshape", **out)
    make_hierarchy(U, "g2d_dir_20_t4_rs1", P.grid2d(20), cfg_kw={"size_cap": 4, "seed": 1},
                   setup_kw={"reshape_sweeps": 1, "n0": 50}, solves=[("", {})])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c2", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    U, K = load_reference()
    sys.path.insert(0, REPO)
    from paper_1302_2547_b200 import problems as P
    only = set(args.only.split(",")) if args.only else None

    def want(k):
        return only is None or k in only

    if want("problems"):
        make_problems(U)
    if want("kernels"):
        make_kernels(U, K)
    if want("c1"):
        make_hierarchy(U, "c1_grid2d_256", P.grid2d(256), solves=[("", {})])
    if want("g2d64"):
        rng = np.random.default_rng(1)
        make_hierarchy(U, "g2d_dir_64", P.grid2d(64), solves=[
            ("", {}),
            ("vcycle_", {"kind": "vcycle"}),
            ("jacobi_", {"smoother": "jacobi"}),
            ("jacobi_w05_", {"smoother": "jacobi", "omega": 0.5}),
            ("sweeps2_", {"pre_sweeps": 2, "post_sweeps": 2}),
            ("inner0_", {"inner_krylov_steps": 0}),
            ("inner3_", {"inner_krylov_steps": 3}),
            ("x0_", {"x0": rng.standard_normal(64 * 64)}),
            ("tol6_", {"tol": 1e-6}),
            ("maxit5_", {"max_iters": 5}),
        ])
    if want("t5"):
        make_hierarchy(U, "g2d_dir_64_t5", P.grid2d(64), cfg_kw={"size_cap": 5}, solves=[("", {})])
    if want("neu"):
        rng = np.random.default_rng(2)
        b = rng.standard_normal(32 * 32)
        b -= b.mean()
        make_hierarchy(U, "g2d_neu_32", P.grid2d(32, "neumann"), solves=[("", {}), ("vcycle_", {"kind": "vcycle"})], b=b)
    if want("pp2"):
        make_hierarchy(U, "g2d_dir_64_pp2", P.grid2d(64), cfg_kw={"passes_per_level": 2}, solves=[("", {})])
    if want("aniso"):
        make_hierarchy(U, "g2d_aniso_48", P.grid2d(48, "dirichlet", (1.0, 10.0)), cfg_kw={"seed": 5}, solves=[("", {})])
    if want("g3d7"):
        make_hierarchy(U, "g3d7_16", P.grid3d(16, 7), solves=[("", {})])
    if want("g3d27"):
        make_hierarchy(U, "g3d27_10", P.grid3d(10, 27), solves=[("", {})])
    if want("wgraph"):
        A = random_weighted_problem(U, 3000, 4)
        make_hierarchy(U, "wgraph_3000", A, solves=[("", {})])
        make_hierarchy(U, "wgraph_3000_cap6", A, cfg_kw={"size_cap": 6, "seed": 2}, solves=[("", {})])
    if want("rgg"):
        make_hierarchy(U, "rgg_20000", P.random_geometric(20000, 12.0, 0), solves=[("", {})])
    if want("rgg_lcc"):
        # the solvable C3 (largest connected component of the SURVEY 8d RGG)
        # at 2^18 vertices; the 2^23 size is pinned by the oracle
        # (tests/golden/make_oracle_fixtures.py)
        make_hierarchy(U, "rgg_lcc_262144", P.random_geometric(1 << 18, 12.0, 0, largest_component=True),
                       solves=[("", {})], full=False)
    if want("reshape"):
        make_reshape(U, P)
    if want("small"):
        make_hierarchy(U, "g2d_dir_12_n0", P.grid2d(12), setup_kw={"n0": 200}, solves=[("", {})])
        make_hierarchy(U, "g2d_dir_16_ml2", P.grid2d(16), setup_kw={"max_levels": 2}, solves=[("", {})])
    if want("c2") and not args.skip_c2:
        make_hierarchy(U, "c2_grid3d7_128", P.grid3d(128, 7), solves=[("", {})], full=False)


if __name__ == "__main__":
    main()
