"""Aggregation types and the device aggregation driver.

Mirrors the reference module /root/reference/pkg/src/uaamg/aggregation.py:
``AggregationConfig`` (:25-40), ``Aggregation`` (:43-102), ``aggregate``
(:172-203), ``compose`` (:206-216), ``quasi_random_scores`` (:130-133),
``select_coarse_vertices`` (:136-141).  The multi-pass PAA runs on the GPU
(``uaamg_aggregate``): quasi-random scores, distance-3 selection as two
max-hops over A (A^2 is never formed), conflict-free claim, admission, and
renumbering by ascending seed.  Results are bit-identical to the reference.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import ptr, stream, to_device, to_host

_UNLIMITED = 2 ** 62


class AggregationError(ValueError):
    pass


@dataclass(frozen=True)
class AggregationConfig:
    size_cap: int | None = None   # max vertices per aggregate, None = unlimited
    seed: int = 0
    max_passes: int = 20
    passes_per_level: int = 1     # 2 composes two aggregations per level

    def __post_init__(self):
        if self.size_cap is not None and self.size_cap < 1:
            raise AggregationError("size_cap must be >= 1 or None")
        if not 0 <= self.seed < 2 ** 64:
            raise AggregationError("seed must fit in an unsigned 64-bit integer")
        if self.max_passes < 1:
            raise AggregationError("max_passes must be >= 1")
        if self.passes_per_level not in (1, 2):
            raise AggregationError("passes_per_level must be 1 or 2")


class Aggregation:
    """Partition of one level's vertices into aggregates (host view, int64).

    ``vertex_to_agg`` maps vertices to aggregates numbered so that
    ``coarse_vertex_of_agg`` (the seeds) is strictly increasing.  Arrays may
    be backed by device memory and are copied to host on first access.
    """

    __slots__ = ("n_fine", "n_coarse", "_v2a", "_seeds", "_dev_v2a", "_dev_seeds", "_members_ptr", "_members")

    def __init__(self, n_fine, vertex_to_agg=None, coarse_vertex_of_agg=None, *, device_arrays=None):
        self.n_fine = int(n_fine)
        self._members_ptr = None
        self._members = None
        self._dev_v2a = self._dev_seeds = None
        if device_arrays is not None:
            self._dev_v2a, self._dev_seeds = device_arrays
            self._v2a = self._seeds = None
            self.n_coarse = int(self._dev_seeds.shape[0])
            return
        self._v2a = np.ascontiguousarray(vertex_to_agg, dtype=np.int64)
        self._seeds = np.ascontiguousarray(coarse_vertex_of_agg, dtype=np.int64)
        self.n_coarse = int(self._seeds.shape[0])
        if self._v2a.shape[0] != self.n_fine:
            raise AggregationError("vertex_to_agg has wrong length")
        if self.n_fine and (self._v2a.min() < 0 or self._v2a.max() >= self.n_coarse):
            raise AggregationError("aggregate index out of range")

    @property
    def vertex_to_agg(self):
        if self._v2a is None:
            self._v2a = to_host(self._dev_v2a).astype(np.int64)
        return self._v2a

    @property
    def coarse_vertex_of_agg(self):
        if self._seeds is None:
            self._seeds = to_host(self._dev_seeds).astype(np.int64)
        return self._seeds

    def device_vertex_to_agg(self):
        if self._dev_v2a is None:
            self._dev_v2a = to_device(self._v2a, np.int32)
        return self._dev_v2a

    @property
    def agg_sizes(self):
        return np.diff(self.members_csr()[0])

    def members_csr(self):
        """(ptr, members): members of aggregate a are members[ptr[a]:ptr[a+1]], ascending."""
        if self._members_ptr is None:
            v = self.vertex_to_agg
            order = np.argsort(v, kind="stable")
            p = np.zeros(self.n_coarse + 1, dtype=np.int64)
            p[1:] = np.cumsum(np.bincount(v, minlength=self.n_coarse))
            self._members_ptr, self._members = p, order.astype(np.int64)
        return self._members_ptr, self._members

    @property
    def coarsening_ratio(self):
        return self.n_fine / self.n_coarse

    def validate(self, a=None, size_cap=None):
        """Partition invariants (reference aggregation.py:83-99)."""
        sizes = self.agg_sizes
        if np.any(sizes == 0):
            raise AggregationError("empty aggregate")
        if np.any(np.diff(self.coarse_vertex_of_agg) <= 0):
            raise AggregationError("coarse vertices not strictly increasing")
        if not np.array_equal(self.vertex_to_agg[self.coarse_vertex_of_agg], np.arange(self.n_coarse)):
            raise AggregationError("coarse vertex not a member of its aggregate")
        if size_cap is not None and sizes.max(initial=0) > size_cap:
            raise AggregationError(f"aggregate larger than cap {size_cap}")
        if a is not None:
            ptr_, mem = self.members_csr()
            for g in range(self.n_coarse):
                if not _connected(a, mem[ptr_[g]:ptr_[g + 1]]):
                    raise AggregationError(f"aggregate {g} is not connected")

    def __repr__(self):
        return f"Aggregation({self.n_fine} -> {self.n_coarse}, ratio={self.coarsening_ratio:.2f})"


def _connected(a, group):
    if group.shape[0] <= 1:
        return True
    pos = {int(v): k for k, v in enumerate(group)}
    seen = np.zeros(group.shape[0], dtype=bool)
    seen[0] = True
    todo = [0]
    while todo:
        v = group[todo.pop()]
        for q in range(a.indptr[v], a.indptr[v + 1]):
            k = pos.get(int(a.indices[q]))
            if k is not None and not seen[k]:
                seen[k] = True
                todo.append(k)
    return bool(seen.all())


def singleton_aggregation(n):
    idx = np.arange(n, dtype=np.int64)
    return Aggregation(n, idx, idx)


def _device_csr(a):
    from .device import DeviceCSR
    if isinstance(a, DeviceCSR):
        return a
    return a.device()


def quasi_random_scores(a, seed, pass_idx=0):
    """degree + ((i mod 12) + hash(seed, pass, i)) / 12 on the GPU."""
    from . import kernel_table
    return kernel_table.quasi_random_scores(a.indptr, a.indices, np.uint64(seed), int(pass_idx))


def select_coarse_vertices(a2_pattern, scores, processed):
    """Unprocessed vertices beating every unprocessed vertex of their A^2 row."""
    from . import kernel_table
    mask = kernel_table.select_centers(a2_pattern.indptr, a2_pattern.indices, scores, processed)
    return np.flatnonzero(mask)


def aggregate(a, config=AggregationConfig()):
    """Multi-pass parallel aggregation on the GPU (reference aggregation.py:172-203)."""
    d = _device_csr(a)
    n = d.n_rows
    if n == 0:
        raise AggregationError("cannot aggregate an empty matrix")
    v2a = torch.empty(n, dtype=torch.int32, device=d.val.device)
    seeds = torch.empty(n, dtype=torch.int32, device=d.val.device)
    nc = np.zeros(1, dtype=np.int32)
    L = _lib.load()
    cap = 0 if config.size_cap is None else int(config.size_cap)
    _lib.check(L.uaamg_aggregate(n, ptr(d.row_ptr), ptr(d.col), ptr(d.val), int(config.seed), int(config.max_passes),
                                 cap, ptr(v2a), ptr(seeds), nc.ctypes.data, stream()))
    # passes_per_level is a setup() knob (reference hierarchy.py:135-138), not
    # read here -- same as the reference aggregate()
    return Aggregation(n, device_arrays=(v2a, seeds[: int(nc[0])]))


def compose(first, second):
    """Compose two successive aggregations (reference aggregation.py:206-216)."""
    if second.n_fine != first.n_coarse:
        raise AggregationError("aggregations do not chain")
    v2a = second.vertex_to_agg[first.vertex_to_agg]
    seeds = first.coarse_vertex_of_agg[second.coarse_vertex_of_agg]
    return Aggregation(first.n_fine, v2a, seeds)
