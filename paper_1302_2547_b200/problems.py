"""Vectorised builders for the benchmark problems.

Each builder returns host CSR arrays (int64 indptr/indices, float64 data)
that are bit-identical to the reference's
``assemble_laplacian(GraphProblem(...))`` (reference graph.py:63-82) for the
same graph -- verified at small sizes by tests/test_problems.py against
fixtures made by tests/golden/make_golden.py.  The reference builds a Python
edge list, which is infeasible beyond ~10^6 edges; these builders write the
canonical CSR directly.

Vertex numbering: 2D ``v = r*n + c`` (reference graph.py:97-105); 3D
``i = (x*n + y)*n + z``; random geometric graphs are numbered by
(cell id, point id) for locality.
"""

import numpy as np

from .sparse import SparseMatrix


def _csr_from_offsets(shape_valid, offsets, weights, diag):
    """Assemble a stencil CSR: ``offsets`` sorted ascending (linear index
    offsets, 0 = diagonal), ``shape_valid[k]`` the per-row validity mask of
    offset k, ``weights[k]`` the (positive) edge weight (ignored at 0),
    ``diag`` the per-row diagonal value."""
    n = diag.shape[0]
    cnt = np.zeros(n, dtype=np.int64)
    for m in shape_valid:
        cnt += m
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=indptr[1:])
    nnz = int(indptr[-1])
    indices = np.empty(nnz, dtype=np.int64)
    data = np.empty(nnz, dtype=np.float64)
    pos = indptr[:-1].copy()
    rows = np.arange(n, dtype=np.int64)
    for off, m, w in zip(offsets, shape_valid, weights):
        r = rows[m]
        p = pos[m]
        indices[p] = r + off
        data[p] = diag[m] if off == 0 else -w[m] if isinstance(w, np.ndarray) else -w
        pos[m] += 1
    return indptr, indices, data


def grid2d(n, bc="dirichlet", anisotropy=(1.0, 1.0)):
    """Reference generate_structured_grid + assemble_laplacian
    (graph.py:85-123, 63-82).  Diagonal = edge weights accumulated in the
    reference's edge-list order (up, left, right, down), then + boundary."""
    if n < 2:
        raise ValueError(f"grid size must be >= 2, got {n}")
    if bc not in ("dirichlet", "neumann"):
        raise ValueError(f"unknown boundary condition {bc!r}")
    wh, wv = float(anisotropy[0]), float(anisotropy[1])
    N = n * n
    v = np.arange(N, dtype=np.int64)
    r, c = v // n, v % n
    up, left, right, down = r > 0, c > 0, c + 1 < n, r + 1 < n
    diag = np.zeros(N)
    # edge (v-n,v) is listed when the generator visits v-n, (v-1,v) at v-1,
    # then (v,v+1) and (v,v+n) at v: that is the accumulation order.
    diag = np.where(up, diag + wv, diag)
    diag = np.where(left, diag + wh, diag)
    diag = np.where(right, diag + wh, diag)
    diag = np.where(down, diag + wv, diag)
    if bc == "dirichlet":
        miss = np.zeros(N)
        miss = np.where(r == 0, miss + wv, miss)
        miss = np.where(r == n - 1, miss + wv, miss)
        miss = np.where(c == 0, miss + wh, miss)
        miss = np.where(c == n - 1, miss + wh, miss)
        diag = np.where(miss > 0, miss + diag, diag)
    offs = [-n, -1, 0, 1, n]
    valid = [up, left, np.ones(N, dtype=bool), right, down]
    wts = [wv, wh, 0.0, wh, wv]
    ip, ix, a = _csr_from_offsets(valid, offs, wts, diag)
    return SparseMatrix(N, N, ip, ix, a, _validate=False)


def grid3d(n, stencil=7, bc="dirichlet", dims=None):
    """3D lattice Laplacian, unit weights; 7-point (face neighbours) or
    27-point (all 26 neighbours).  Dirichlet by elimination: every vertex
    gets boundary weight = number of missing stencil neighbours, so the
    diagonal is 6 / 26 everywhere.  ``dims``
    (nx, ny, nz) builds a box instead of the n^3 cube (vertex
    (x*ny + y)*nz + z)."""
    if stencil not in (7, 27):
        raise ValueError("stencil must be 7 or 27")
    nx, ny, nz = dims if dims is not None else (n, n, n)
    if min(nx, ny, nz) < 2:
        raise ValueError("grid size must be >= 2")
    N = nx * ny * nz
    v = np.arange(N, dtype=np.int64)
    x, y, z = v // (ny * nz), (v // nz) % ny, v % nz
    del v
    offs, valid = [], []
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                if stencil == 7 and abs(dx) + abs(dy) + abs(dz) > 1:
                    continue
                m = np.ones(N, dtype=bool)
                for d, c, nd in ((dx, x, nx), (dy, y, ny), (dz, z, nz)):
                    if d < 0:
                        m &= c > 0
                    elif d > 0:
                        m &= c < nd - 1
                offs.append(dx * ny * nz + dy * nz + dz)
                valid.append(m)
    deg = np.zeros(N)
    for o, m in zip(offs, valid):
        if o != 0:
            deg += m
    if bc == "dirichlet":
        diag = np.full(N, float(stencil - 1))
    else:
        diag = deg
    ip, ix, a = _csr_from_offsets(valid, offs, [1.0] * len(offs), diag)
    return SparseMatrix(N, N, ip, ix, a, _validate=False)


def grid3d_device(n, stencil=7, bc="dirichlet", dims=None):
    """``grid3d`` built directly on the device (csrc: gen_grid3d) as a
    DeviceCSR -- same bits as the host builder, no host assembly (the host
    path needs tens of GB and minutes at the 256^3 / 512^3 configs)."""
    import ctypes

    import torch

    from . import _lib
    from .device import DeviceCSR, device_empty, ptr, stream

    if stencil not in (7, 27):
        raise ValueError("stencil must be 7 or 27")
    if bc not in ("dirichlet", "neumann"):
        raise ValueError(f"unknown boundary condition {bc!r}")
    nx, ny, nz = dims if dims is not None else (n, n, n)
    N = nx * ny * nz
    rp = device_empty(N + 1, np.int32)
    nnz = ctypes.c_int64()
    L = _lib.load()
    neu = int(bc == "neumann")
    _lib.check(L.uaamg_gen_grid3d(nx, ny, nz, stencil, neu, ptr(rp), None, None, ctypes.byref(nnz), stream()))
    ci = device_empty(nnz.value, np.int32)
    av = device_empty(nnz.value, np.float64)
    _lib.check(L.uaamg_gen_grid3d(nx, ny, nz, stencil, neu, ptr(rp), ptr(ci), ptr(av), None, stream()))
    return DeviceCSR(N, N, rp, ci, av)


def random_geometric(N, degree=12.0, seed=0, return_edges=False, largest_component=False):
    """Random geometric graph in the unit cube.

    Points ``default_rng(seed).random((N,3))``; radius r with expected degree
    ``degree``; unit-weight edges for ``|p_i - p_j| <= r``; boundary weight 1
    for vertices within r of a cube face and for isolated vertices (so the
    l1 smoother diagonal is positive).  Vertices are renumbered by
    (cell id, point id) with cells of side >= r.

    ``largest_component``: keep only the largest connected component (its
    vertices keep their relative order and are renumbered 0..m-1; boundary
    weights as above).  The literal C3 graph at 2^23 vertices has ~190
    isolated vertices, which no aggregation pass can merge, so the
    reference's setup stagnates before n <= n0 (SetupError); the largest
    component is the solvable C3."""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    P = rng.random((N, 3))
    r = (3.0 * degree / (4.0 * np.pi * N)) ** (1.0 / 3.0)
    m = max(1, int(np.floor(1.0 / r)))
    cell = np.minimum((P * m).astype(np.int64), m - 1)
    cid = (cell[:, 0] * m + cell[:, 1]) * m + cell[:, 2]
    order = np.lexsort((np.arange(N), cid))
    P = P[order]
    pairs = cKDTree(P).query_pairs(r, output_type="ndarray").astype(np.int64)
    i, j = np.minimum(pairs[:, 0], pairs[:, 1]), np.maximum(pairs[:, 0], pairs[:, 1])
    del pairs
    if largest_component:
        from scipy.sparse import coo_matrix
        from scipy.sparse.csgraph import connected_components
        g = coo_matrix((np.ones(i.shape[0], dtype=np.int8), (i, j)), shape=(N, N)).tocsr()
        _, lab = connected_components(g, directed=False)
        del g
        keep = lab == np.argmax(np.bincount(lab))
        new = np.cumsum(keep) - 1
        e = keep[i]  # both ends share a component
        i, j = new[i[e]], new[j[e]]
        P = P[keep]
        N = int(keep.sum())
    deg = np.bincount(i, minlength=N) + np.bincount(j, minlength=N)
    near_face = np.any((P < r) | (P > 1.0 - r), axis=1)
    bnd = near_face | (deg == 0)
    diag = deg.astype(np.float64) + bnd.astype(np.float64)
    rows = np.concatenate([i, j, np.arange(N)])
    cols = np.concatenate([j, i, np.arange(N)])
    vals = np.concatenate([-np.ones(i.shape[0] * 2), diag])
    A = SparseMatrix.from_coo(N, N, rows, cols, vals)
    if return_edges:
        return A, (i, j), np.flatnonzero(bnd)
    return A


def build_config(name):
    """Named benchmark problems (BASELINE.json configs)."""
    if name == "C1":
        return grid2d(256, "dirichlet")
    if name == "C2":
        return grid3d(128, 7)
    if name == "C3":
        return random_geometric(1 << 23, 12.0, 0, largest_component=True)
    if name == "C3-literal":
        return random_geometric(1 << 23, 12.0, 0)
    if name == "C4":
        return grid3d(256, 27)
    if name == "C5":
        return grid3d(512, 7)
    raise ValueError(f"unknown config {name!r}")
