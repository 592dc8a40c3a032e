"""Helpers for loading the golden fixtures made by tests/golden/make_golden.py
(outputs of the reference package itself)."""

import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

HIERARCHY_CASES = [
    "c1_grid2d_256", "g2d_dir_64", "g2d_dir_64_t5", "g2d_neu_32", "g2d_dir_64_pp2",
    "g2d_aniso_48", "g3d7_16", "g3d27_10", "wgraph_3000", "wgraph_3000_cap6", "rgg_20000",
    "g2d_dir_12_n0", "g2d_dir_16_ml2", "rgg_lcc_262144",
]

# setup kwargs per case (mirrors make_golden.py)
CASE_CFG = {
    "g2d_dir_64_t5": dict(size_cap=5),
    "g2d_dir_64_pp2": dict(passes_per_level=2),
    "g2d_aniso_48": dict(seed=5),
    "wgraph_3000_cap6": dict(size_cap=6, seed=2),
    "g2d_dir_12_n0": dict(n0=200),
    "g2d_dir_16_ml2": dict(max_levels=2),
}

# solve variants stored in g2d_dir_64.npz: prefix -> npcg kwargs
SOLVE_VARIANTS = {
    "": {},
    "vcycle_": {"kind": "vcycle"},
    "jacobi_": {"smoother": "jacobi"},
    "jacobi_w05_": {"smoother": "jacobi", "omega": 0.5},
    "sweeps2_": {"pre_sweeps": 2, "post_sweeps": 2},
    "inner0_": {"inner_krylov_steps": 0},
    "inner3_": {"inner_krylov_steps": 3},
    "x0_": {},
    "tol6_": {"tol": 1e-6},
    "maxit5_": {"max_iters": 5},
}


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(memoryview(np.ascontiguousarray(a)).cast("B"))
    return h.hexdigest()


def problem_for(name):
    """Rebuild the level-0 matrix of a golden case (host CSR arrays)."""
    from paper_1302_2547_b200 import problems as P
    g = load(name)
    if "L0_indptr" in g:
        ip = g["L0_indptr"].astype(np.int64)
        ix = g["L0_indices"].astype(np.int64)
        a = g["L0_data"]
    else:
        builders = {"c2_grid3d7_128": lambda: P.grid3d(128, 7),
                    "rgg_lcc_262144": lambda: P.random_geometric(1 << 18, 12.0, 0, largest_component=True)}
        A = builders[name]()
        ip, ix, a = A.indptr, A.indices, A.data
    assert sha(ip, ix, a) == str(g["input_sha"]), "input matrix differs from the fixture's"
    return ip, ix, a, g


def assert_hierarchy_equal(g, levels):
    """levels: list of dicts with n, indptr, indices, data, v2a, seeds (numpy,
    any int dtype).  Bit-exact comparison against the fixture."""
    assert len(levels) == int(g["n_levels"]), (len(levels), int(g["n_levels"]))
    for l, L in enumerate(levels):
        assert L["n"] == int(g[f"L{l}_n"]), f"level {l} size"
        ip = np.asarray(L["indptr"], dtype=np.int64)
        ix = np.asarray(L["indices"], dtype=np.int64)
        a = np.asarray(L["data"], dtype=np.float64)
        assert ix.shape[0] == int(g[f"L{l}_nnz"]), f"level {l} nnz"
        assert sha(ip, ix, a) == str(g[f"L{l}_csr_sha"]), f"level {l} matrix differs"
        if f"L{l}_v2a_sha" in g:
            assert L["v2a"] is not None, f"level {l} lacks an aggregation"
            v2a = np.asarray(L["v2a"], dtype=np.int64)
            seeds = np.asarray(L["seeds"], dtype=np.int64)
            assert sha(v2a) == str(g[f"L{l}_v2a_sha"]), f"level {l} vertex_to_agg differs"
            assert sha(seeds) == str(g[f"L{l}_seeds_sha"]), f"level {l} seeds differ"


def assert_history_close(hist, g, prefix="", rtol=1e-10, it_slack=1, atol=1e-13):
    ref = g[prefix + "history"]
    it_ref = int(g[prefix + "iterations"])
    it = len(hist) - 1
    assert abs(it - it_ref) <= it_slack, f"iterations {it} vs reference {it_ref}"
    m = min(len(hist), len(ref))
    h = np.asarray(hist[:m])
    r = ref[:m]
    # relative agreement of the residual history (north star: 1e-10 relative);
    # entries at round-off level (< atol, in units of ||b||) only need to agree
    # to atol -- e.g. a direct coarsest solve leaves ~1e-15 noise.
    err = np.abs(h - r) / np.maximum(np.abs(r), 1e-300)
    err = np.where(np.abs(h - r) <= atol, 0.0, err)
    assert np.all(err <= rtol), f"history mismatch max rel err {err.max():.3e} at {int(err.argmax())}"
