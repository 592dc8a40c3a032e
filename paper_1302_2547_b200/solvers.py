"""Solve phase on the GPU.

Mirrors /root/reference/pkg/src/uaamg/solvers.py: ``NumericalError``
(:16-21), ``Smoother`` (:24-36), ``CycleSpec`` (:39-50), ``SolveReport``
(:53-66), ``smoother_inverse_diag`` (:69-81), ``smooth`` (:84-91),
``prolongate_add`` (:94-100), ``restrict`` (:103-109), ``cycle`` (:128-157),
``npcg_solve`` (:190-255).

``npcg_solve`` runs the flexible PCG with the K-cycle preconditioner entirely
on the device (``uaamg_npcg_solve``): each outer iteration is one CUDA-graph
replay; inner-FCG breaks, breakdown, restarts and convergence are device
flags.  Inputs may be numpy (host) or torch CUDA tensors; outputs match.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import ptr, stream, to_device, to_host


class NumericalError(RuntimeError):
    """Breakdown or incompatible data during the solve phase."""

    def __init__(self, message, report=None):
        super().__init__(message)
        self.report = report


@dataclass(frozen=True)
class Smoother:
    kind: str = "l1"   # "l1" (parameter free) or "jacobi" (damped)
    omega: float = 2.0 / 3.0
    sweeps: int = 1

    def __post_init__(self):
        if self.kind not in ("l1", "jacobi"):
            raise ValueError(f"unknown smoother kind {self.kind!r}")
        if not 0 < self.omega <= 1:
            raise ValueError("damping must satisfy 0 < omega <= 1")
        if self.sweeps < 1:
            raise ValueError("sweeps must be >= 1")


@dataclass(frozen=True)
class CycleSpec:
    kind: str = "kcycle"   # "kcycle" or "vcycle"
    inner_krylov_steps: int = 2
    pre_sweeps: int = 1
    post_sweeps: int = 1

    def __post_init__(self):
        if self.kind not in ("kcycle", "vcycle"):
            raise ValueError(f"unknown cycle kind {self.kind!r}")
        if self.inner_krylov_steps < 0:
            raise ValueError("inner_krylov_steps must be >= 0")


@dataclass
class SolveReport:
    iterations: int
    residual_history: list
    converged: bool
    timings: dict = field(default_factory=dict)

    def to_dict(self):
        return {"iterations": self.iterations, "converged": self.converged,
                "residual_history": [float(r) for r in self.residual_history], "timings": dict(self.timings)}


def _params(spec, smoother, tol=1e-6, max_iters=200, use_graphs=True):
    return _lib.SolveParams(kcycle=int(spec.kind == "kcycle"), inner_krylov_steps=int(spec.inner_krylov_steps),
                            pre_sweeps=int(spec.pre_sweeps), post_sweeps=int(spec.post_sweeps),
                            smoother_l1=int(smoother.kind == "l1"), omega=float(smoother.omega), tol=float(tol),
                            max_iters=int(max_iters), use_graphs=int(use_graphs), profile_level0=0)


def smoother_inverse_diag(a, smoother):
    """omega/a_ii (damped Jacobi) or 1/(a_ii + sum_j!=i |a_ij|) (l1), on the GPU."""
    from . import kernel_table
    if smoother.kind == "jacobi":
        m = kernel_table.diag_of(a.indptr, a.indices, a.data)
        scale = smoother.omega
    else:
        m = kernel_table.l1_diag(a.indptr, a.indices, a.data)
        scale = 1.0
    if np.any(m <= 0):
        raise NumericalError(f"non-positive smoother diagonal at row {int(np.flatnonzero(m <= 0)[0])}")
    return scale / m


def smooth(a, smoother, x, b, sweeps=None):
    """Pointwise relaxation sweeps x += M^{-1}(b - A x) (bit-identical rows)."""
    from . import kernel_table
    if sweeps is None:
        sweeps = smoother.sweeps
    inv_m = smoother_inverse_diag(a, smoother)
    return kernel_table.smooth_sweeps(a.indptr, a.indices, a.data, inv_m, np.asarray(x, dtype=np.float64),
                                      np.asarray(b, dtype=np.float64), int(sweeps))


def prolongate_add(agg, e_coarse, x):
    """x_i + e_coarse[aggregate(i)] on the GPU."""
    from . import kernel_table
    e_coarse = np.asarray(e_coarse, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    if e_coarse.shape != (agg.n_coarse,) or x.shape != (agg.n_fine,):
        raise ValueError("prolongation size mismatch")
    return kernel_table.prolongate_add(agg.vertex_to_agg, e_coarse, x)


def restrict(agg, r_fine):
    """Sum of fine entries per aggregate, ascending member order, on the GPU."""
    from . import kernel_table
    r_fine = np.asarray(r_fine, dtype=np.float64)
    if r_fine.shape != (agg.n_fine,):
        raise ValueError("restriction size mismatch")
    p, m = agg.members_csr()
    return kernel_table.restrict(p, m, r_fine)


def _vec_in(v, n, what):
    host = not isinstance(v, torch.Tensor)
    d = to_device(v, np.float64)
    if d.shape != (n,):
        raise ValueError(f"{what} size mismatch")
    return d, host


def cycle(h, spec, smoother, level, b):
    """One multigrid cycle on A_level x = b from a zero guess (device)."""
    lev = h.levels[level]
    n = lev.n
    bd, host = _vec_in(b, n, "cycle right-hand side")
    x = torch.empty(n, dtype=torch.float64, device=bd.device)
    P = _params(spec, smoother)
    _lib.check(_lib.load().uaamg_cycle(h._handle, ctypes.byref(P), h._offset + level, ptr(bd), ptr(x), stream()))
    return to_host(x) if host else x


def npcg_solve(h, cycle_spec, smoother, b, tol=1e-6, max_iters=200, x0=None, use_graphs=True):
    """Flexible PCG with one K-/V-cycle per application, on the device."""
    if tol <= 0:
        raise ValueError("tol must be positive")
    if h._offset != 0:
        raise ValueError("npcg_solve needs the full hierarchy")
    n = h.levels[0].n
    bd, host = _vec_in(b, n, "right-hand side")
    x0d = to_device(x0, np.float64) if x0 is not None else None
    x = torch.empty(n, dtype=torch.float64, device=bd.device)
    hist = np.zeros(int(max_iters) + 1)
    P = _params(cycle_spec, smoother, tol, max_iters, use_graphs)
    res = _lib.SolveResult()
    rc = _lib.load().uaamg_npcg_solve(h._handle, ctypes.byref(P), ptr(bd), ptr(x0d), ptr(x),
                                      hist.ctypes.data_as(ctypes.c_void_p), ctypes.byref(res), stream())
    report = SolveReport(int(res.iterations), hist[: int(res.iterations) + 1].tolist(), bool(res.converged),
                         {"solve_seconds": float(res.solve_seconds), "setup_seconds": h.setup_seconds})
    if rc == _lib.UAAMG_ENUMERICAL:
        raise NumericalError(_lib.last_error(), report=report)
    _lib.check(rc)
    return (to_host(x) if host else x), report
