"""Row-partitioned (multi-GPU) setup and solve -- SURVEY.md §8e.

Level 0 is split into P contiguous row blocks (``partition_rows``); each
rank holds and computes only its rows.  ``setup_distributed`` builds the
hierarchy collectively (csrc/dist_setup.cu): aggregation, renumbering,
members and the Galerkin product run per rank and read halo entries straight
from the owning rank's memory; coarse levels inherit the partition (rank q
owns the aggregates seeded in its rows) until they drop below
``shard_rows``, then they are gathered and replicated.  The hierarchy is
bit-identical to :func:`~.hierarchy.setup`'s for any rank count.
``npcg_solve_distributed`` runs the K-cycle NPCG on it
(csrc/dist_solve.cu).

Two ways to run the P ranks:

* one process per GPU (``rank`` = this process's rank; torch.distributed,
  any backend, carries the one-time exchange of the 64-byte CUDA IPC handles
  of the ranks' arenas -- after that, peers read each other's arenas
  directly, over NVLink on an 8xB200 box);
* ``virtual=True``: all P ranks in this process on one device, launched
  rank by rank (the partition-invariance harness used by the tests).
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .aggregation import AggregationConfig
from .device import DeviceCSR, device_empty, ptr, stream, to_device, to_host, view
from .solvers import NumericalError, SolveReport, _params
from .sparse import SparseMatrix

HANDLE_BYTES = 64
SHARD_ROWS = 1 << 20  # levels with fewer rows are gathered and replicated


def partition_rows(n, ranks):
    """Level-0 row ranges (``ranks + 1`` bounds): equal 128-aligned blocks."""
    out = np.zeros(ranks + 1, dtype=np.int32)
    _lib.check(_lib.load().uaamg_partition_rows(int(n), int(ranks), out.ctypes.data_as(ctypes.c_void_p)))
    return out


def coarse_bounds(seed_counts):
    """Coarse-level row ranges from the per-rank seed counts (the sharded
    setup's renumbering, U/aggregation.py:199-203)."""
    c = np.ascontiguousarray(seed_counts, dtype=np.int64)
    out = np.zeros(c.shape[0] + 1, dtype=np.int32)
    _lib.check(_lib.load().uaamg_coarse_bounds(c.ctypes.data_as(ctypes.c_void_p), int(c.shape[0]),
                                               out.ctypes.data_as(ctypes.c_void_p)))
    return out


def arena_bytes_for(n_local, nnz_local):
    """Arena size of one rank: the level CSRs (all sharded levels), the setup
    state of one level and the solve vectors, with headroom."""
    return int(2.2 * (12 * nnz_local + 4 * n_local) + 260 * n_local + (64 << 20))


def exchange_handles(local, group=None):
    """All-gather each rank's ``HANDLE_BYTES`` handle; returns them concatenated in rank order."""
    import torch.distributed as dist

    if len(local) != HANDLE_BYTES:
        raise ValueError("IPC handles are 64 bytes")
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(local), group=group)
    return b"".join(out)


class Communicator:
    """The ranks of one distributed hierarchy and their peer-readable arenas
    (uaamg_comm_*).  ``rank=None``: virtual ranks in this process."""

    def __init__(self, ranks, rank=None, arena_bytes=1 << 30, group=None):
        self.ranks = int(ranks)
        self.rank = rank
        self.group = group
        L = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(L.uaamg_comm_create(self.ranks, -1 if rank is None else int(rank), int(arena_bytes),
                                       ctypes.byref(h)))
        self._h = h
        if rank is not None:
            ok = False
            try:
                hb = (ctypes.c_ubyte * HANDLE_BYTES)()
                _lib.check(L.uaamg_comm_handle(h, hb))
                allh = exchange_handles(bytes(hb), group)
                buf = ctypes.create_string_buffer(allh, len(allh))
                _lib.check(L.uaamg_comm_connect(h, buf))
                ok = True
            finally:
                if not ok:
                    L.uaamg_comm_free(h)
                    self._h = None

    @property
    def virtual(self):
        return self.rank is None

    @property
    def local_ranks(self):
        return list(range(self.ranks)) if self.virtual else [self.rank]

    def barrier(self):
        if self._h and not self.virtual:
            _lib.check(_lib.load().uaamg_comm_barrier(self._h))

    def quiesce(self):
        """Collective: every rank's device work is done and every rank has
        passed a barrier, so no peer still reads this rank's arena.  The host
        collective goes first, so a rank that failed earlier is not waited
        for on the device."""
        if self._h and not self.virtual:
            import torch.distributed as dist
            flag = [None] * dist.get_world_size(self.group)
            dist.all_gather_object(flag, True, group=self.group)
            torch.cuda.synchronize()
            self.barrier()

    def close(self, collective=True):
        """Release this process's handle; the arenas are freed once the
        hierarchies built on them are gone too.  Multi-process teardown must
        be collective (quiesce first) unless a peer already failed."""
        if not self._h:
            return
        if collective:
            self.quiesce()
        _lib.load().uaamg_comm_free(self._h)
        self._h = None


def _fail_together(comm, ok):
    """Multi-process: all ranks learn whether any rank failed (host collective
    over the torch.distributed group), so a failing rank does not leave its
    peers spinning in the device barrier."""
    if comm.virtual:
        return ok
    import torch.distributed as dist
    flags = [None] * dist.get_world_size(comm.group)
    dist.all_gather_object(flags, bool(ok), group=comm.group)
    return all(flags)


class DistributedHierarchy:
    """A row-partitioned hierarchy (uaamg_dhier).  ``n_levels``,
    ``n_sharded`` (levels 0..n_sharded-1 are row-partitioned), ``singular``,
    complexities and ``setup_seconds`` like :class:`~.hierarchy.Hierarchy`;
    level data through :meth:`local_level` (this process's ranks) and, for
    virtual ranks, the assembled global :meth:`level_matrix` /
    :meth:`level_aggregation`."""

    def __init__(self, comm, handle, owns_comm=True):
        self.comm = comm
        self._h = handle
        self._owns_comm = owns_comm
        info = _lib.DHierInfo()
        _lib.check(_lib.load().uaamg_dhier_get_info(handle, ctypes.byref(info)))
        self.n_levels = int(info.n_levels)
        self.n_sharded = int(info.n_sharded)
        self.singular = bool(info.singular)
        self.grid_complexity = float(info.grid_complexity)
        self.operator_complexity = float(info.operator_complexity)
        self.setup_seconds = float(info.setup_seconds)
        v = self._view(0, self.comm.local_ranks[0])
        self.n = int(v.n)
        self.row_bounds = None

    def _view(self, level, rank):
        v = _lib.DLevelView()
        _lib.check(_lib.load().uaamg_dhier_level(self._h, int(level), int(rank), ctypes.byref(v)))
        return v

    def level_size(self, level):
        v = self._view(level, self.comm.local_ranks[0])
        return int(v.n), int(v.nnz)

    def local_level(self, level, rank=None):
        """Host arrays of level ``level`` as held by ``rank``: row range,
        local CSR (int64 row offsets, global columns), v2a and seeds."""
        rank = self.comm.local_ranks[0] if rank is None else rank
        v = self._view(level, rank)
        n_loc = v.row_end - v.row_begin

        def dl(p, m, dt):
            if m == 0 or not p:
                return np.zeros(0, dtype=dt)
            return to_host(view(p, m, dt, self)).copy()

        rp = dl(v.row_ptr, n_loc + 1, np.int32).astype(np.int64)
        return {
            "n": int(v.n), "nnz": int(v.nnz), "sharded": bool(v.sharded), "row_begin": int(v.row_begin),
            "row_end": int(v.row_end), "indptr": rp, "indices": dl(v.col, int(v.local_nnz), np.int32).astype(np.int64),
            "data": dl(v.val, int(v.local_nnz), np.float64), "n_coarse": int(v.n_coarse),
            "vertex_to_agg": dl(v.vertex_to_agg, n_loc, np.int32).astype(np.int64) if v.n_coarse else None,
            "seeds": dl(v.seeds, int(v.n_seeds), np.int32).astype(np.int64) if v.n_coarse else None,
        }

    def _assemble(self, level):
        if not self.comm.virtual and level < self.n_sharded:
            raise ValueError("global level arrays need every rank (virtual ranks)")
        ranks = self.comm.local_ranks if level < self.n_sharded else self.comm.local_ranks[:1]
        parts = [self.local_level(level, r) for r in ranks]
        return parts

    def level_matrix(self, level):
        """Level ``level`` as one host SparseMatrix (rows of every rank)."""
        parts = self._assemble(level)
        n = parts[0]["n"]
        ips, off = [], 0
        for k, p in enumerate(parts):
            ip = p["indptr"] + off
            ips.append(ip[:-1] if k < len(parts) - 1 else ip)
            off = int(ip[-1])
        return SparseMatrix(n, n, np.concatenate(ips), np.concatenate([p["indices"] for p in parts]),
                            np.concatenate([p["data"] for p in parts]), _validate=False)

    def level_aggregation(self, level):
        """(vertex_to_agg, coarse_vertex_of_agg) of level ``level`` (None on the coarsest)."""
        parts = self._assemble(level)
        if parts[0]["n_coarse"] == 0:
            return None
        return (np.concatenate([p["vertex_to_agg"] for p in parts]), np.concatenate([p["seeds"] for p in parts]))

    def close(self, collective=True):
        """Free the hierarchy (collective for one process per GPU: every rank
        must call it), and its communicator if setup_distributed made it; a
        caller-owned communicator can then carry the next hierarchy."""
        if self._h:
            if collective:
                self.comm.quiesce()
            _lib.load().uaamg_dhier_free(self._h)
            self._h = None
        if self._owns_comm:
            self.comm.close(collective=False)

    def __del__(self):
        try:
            self.close(collective=False)
        except Exception:
            pass


def _setup_params(config, n0, max_levels, singular):
    return _lib.SetupParams(size_cap=0 if config.size_cap is None else int(config.size_cap), seed=int(config.seed),
                            max_passes=int(config.max_passes), passes_per_level=int(config.passes_per_level),
                            n0=int(n0), max_levels=int(max_levels),
                            singular=-1 if singular is None else int(bool(singular)), borrow=0)


def setup_distributed(a, ranks=None, bounds=None, n=None, comm=None, config=AggregationConfig(), n0=100,
                      max_levels=20, singular=None, shard_rows=SHARD_ROWS, arena_bytes=None, group=None):
    """Collective row-partitioned setup (U/hierarchy.py:120-153).

    Virtual ranks (``ranks`` given, or a virtual ``comm``): ``a`` is the
    whole matrix (SparseMatrix or DeviceCSR), split into blocks of
    ``partition_rows``.  One process per GPU: ``a`` is this rank's block
    (a DeviceCSR of its rows with GLOBAL column indices), ``n`` the global
    size, ``bounds`` the P+1 row bounds and ``comm`` a connected
    :class:`Communicator` (or pass ``group`` and let this create one).  A
    caller-owned ``comm`` carries one hierarchy at a time and is reused
    (no arena allocation or handle exchange per setup)."""
    L = _lib.load()
    owns = comm is None
    if (comm is None and group is None) or (comm is not None and comm.virtual):
        # virtual ranks over a whole matrix
        d = a if isinstance(a, DeviceCSR) else a.device()
        n = d.n_rows
        P = int(ranks) if comm is None else comm.ranks
        bounds = partition_rows(n, P)
        rp_h = to_host(d.row_ptr).astype(np.int64)
        blocks = []
        for q in range(P):
            r0, r1 = int(bounds[q]), int(bounds[q + 1])
            e0, e1 = int(rp_h[r0]), int(rp_h[r1])
            rp = (d.row_ptr[r0:r1 + 1] - e0).to(torch.int32).contiguous()
            blocks.append((rp, d.col[e0:e1].contiguous(), d.val[e0:e1].contiguous(), e1 - e0))
        if comm is None:
            if arena_bytes is None:
                arena_bytes = max(arena_bytes_for(int(np.diff(bounds).max()), max(b[3] for b in blocks)), 1 << 26)
            comm = Communicator(P, None, arena_bytes)
    else:
        if comm is None:
            import torch.distributed as dist
            P = dist.get_world_size(group)
            r = dist.get_rank(group)
            if arena_bytes is None:
                arena_bytes = arena_bytes_for(a.n_rows, a.nnz)
                # same arena size on every rank (the largest block's)
                sizes = [None] * P
                dist.all_gather_object(sizes, int(arena_bytes), group=group)
                arena_bytes = max(sizes)
            comm = Communicator(P, r, arena_bytes, group)
        P = comm.ranks
        if n is None or bounds is None:
            raise ValueError("multi-process setup needs the global size n and the row bounds")
        bounds = np.ascontiguousarray(bounds, dtype=np.int32)
        blocks = [(to_device(a.row_ptr, np.int32), to_device(a.col, np.int32), to_device(a.val, np.float64), a.nnz)]
    m = len(blocks)
    VP = ctypes.c_void_p * m
    rps = VP(*[ptr(b[0]) for b in blocks])
    cis = VP(*[ptr(b[1]) for b in blocks])
    avs = VP(*[ptr(b[2]) for b in blocks])
    nnz = (ctypes.c_int64 * m)(*[int(b[3]) for b in blocks])
    Pp = _setup_params(config, n0, max_levels, singular)
    h = ctypes.c_void_p()
    ok = False
    try:
        rc = L.uaamg_dsetup(comm._h, int(n), bounds.ctypes.data_as(ctypes.c_void_p), rps, cis, avs, nnz,
                            ctypes.byref(Pp), int(shard_rows), ctypes.byref(h), stream())
        ok = rc == _lib.UAAMG_OK
        err = None if ok else (rc, _lib.last_error())
    finally:
        if not comm.virtual and not _fail_together(comm, ok):
            if ok:
                _lib.load().uaamg_dhier_free(h)
            if owns:
                comm.close(collective=False)
            if ok:
                raise RuntimeError("sharded setup failed on another rank")
    if not ok:
        if owns:
            comm.close(collective=False)
        _lib.check_code(*err)
    dh = DistributedHierarchy(comm, h, owns_comm=owns)
    dh.row_bounds = bounds
    return dh


def npcg_solve_distributed(dh, cycle_spec, smoother, b, tol=1e-6, max_iters=200, x0=None, use_graphs=True):
    """Collective NPCG solve (U/solvers.py:190-255) on a DistributedHierarchy.

    Virtual ranks: ``b`` / ``x0`` / the returned x are whole vectors.  One
    process per GPU: they are this rank's rows."""
    comm = dh.comm
    host = not isinstance(b, torch.Tensor)
    bd = to_device(b, np.float64)
    bounds = dh.row_bounds
    ranks = comm.local_ranks
    if comm.virtual:
        if bd.shape != (dh.n,):
            raise ValueError("right-hand side size mismatch")
        pieces = [(int(bounds[q]), int(bounds[q + 1])) for q in ranks]
    else:
        r = comm.rank
        pieces = [(0, int(bounds[r + 1] - bounds[r]))]
        if bd.shape != (pieces[0][1],):
            raise ValueError("right-hand side size mismatch (this rank's rows)")
    x0d = to_device(x0, np.float64) if x0 is not None else None
    x = torch.empty_like(bd)
    bs = [bd[a:e].contiguous() for a, e in pieces]
    xs = [torch.empty(e - a, dtype=torch.float64, device=bd.device) for a, e in pieces]
    x0s = [x0d[a:e].contiguous() for a, e in pieces] if x0d is not None else None
    m = len(pieces)
    VP = ctypes.c_void_p * m
    hist = np.zeros(int(max_iters) + 1)
    P = _params(cycle_spec, smoother, tol, max_iters, use_graphs)
    res = _lib.SolveResult()
    rc = _lib.load().uaamg_dsolve(dh._h, ctypes.byref(P), VP(*[ptr(t) for t in bs]),
                                  VP(*[ptr(t) for t in x0s]) if x0s is not None else None,
                                  VP(*[ptr(t) for t in xs]), hist.ctypes.data_as(ctypes.c_void_p),
                                  ctypes.byref(res), stream())
    report = SolveReport(int(res.iterations), hist[: int(res.iterations) + 1].tolist(), bool(res.converged),
                         {"solve_seconds": float(res.solve_seconds), "setup_seconds": dh.setup_seconds,
                          "ranks": comm.ranks})
    if rc == _lib.UAAMG_ENUMERICAL:
        raise NumericalError(_lib.last_error(), report=report)
    _lib.check(rc)
    for (a, e), t in zip(pieces, xs):
        x[a:e] = t
    return (to_host(x) if host else x), report


def grid3d_rows(n, stencil, row_begin, row_end, dims=None):
    """This rank's rows [row_begin, row_end) of the 3D lattice Laplacian of
    problems.grid3d, generated on the device (local row offsets, global
    columns) -- level 0 of the multi-GPU C4/C5 configs without any rank
    holding the whole matrix."""
    nx, ny, nz = dims if dims is not None else (n, n, n)
    L = _lib.load()
    m = row_end - row_begin
    rp = device_empty(m + 1, np.int32)
    nnz = ctypes.c_int64()
    _lib.check(L.uaamg_gen_grid3d_rows(nx, ny, nz, stencil, 0, int(row_begin), int(row_end), ptr(rp), None, None,
                                       ctypes.byref(nnz), stream()))
    ci = device_empty(nnz.value, np.int32)
    av = device_empty(nnz.value, np.float64)
    _lib.check(L.uaamg_gen_grid3d_rows(nx, ny, nz, stencil, 0, int(row_begin), int(row_end), ptr(rp), ptr(ci),
                                       ptr(av), None, stream()))
    return DeviceCSR(m, nx * ny * nz, rp, ci, av)
