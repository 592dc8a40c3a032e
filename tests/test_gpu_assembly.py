"""On-device assembly (csrc/assemble.cu) against the reference's own
from_coo / assemble_laplacian outputs (tests/golden/assembly.npz, made by
tests/golden/make_assembly_golden.py): bit-exact CSR."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "assembly.npz"))


@pytest.fixture(scope="module")
def U():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1302_2547_b200 as U

    return U


def _eq(d, ip, ix, a):
    h = d.to_host()
    assert np.array_equal(h.indptr, ip) and np.array_equal(h.indices, ix)
    # bit-exact, including the sign of zero
    assert np.array_equal(h.data.view(np.int64), np.asarray(a).view(np.int64))


def test_from_coo_matches_reference(U):
    from paper_1302_2547_b200.device import DeviceCSR

    nr, nc = (int(v) for v in G["coo_shape"])
    d = DeviceCSR.from_coo(nr, nc, G["coo_rows"], G["coo_cols"], G["coo_vals"])
    _eq(d, G["coo_indptr"], G["coo_indices"], G["coo_data"])


def test_from_coo_rejects_out_of_range(U):
    from paper_1302_2547_b200.device import DeviceCSR
    from paper_1302_2547_b200.sparse import SparseFormatError

    with pytest.raises(SparseFormatError):
        DeviceCSR.from_coo(3, 3, np.array([0, 3]), np.array([0, 1]), np.array([1.0, 2.0]))


def test_assemble_laplacian_matches_reference(U):
    from paper_1302_2547_b200.graph import assemble_laplacian_device

    d = assemble_laplacian_device(int(G["lap_n"]), (G["lap_ei"], G["lap_ej"], G["lap_w"]),
                                  (G["lap_bj"], G["lap_bw"]))
    _eq(d, G["lap_indptr"], G["lap_indices"], G["lap_data"])


def test_assemble_laplacian_validation(U):
    from paper_1302_2547_b200.graph import GraphError, assemble_laplacian_device

    with pytest.raises(GraphError):
        assemble_laplacian_device(4, [(0, 0, 1.0)])
    with pytest.raises(GraphError):
        assemble_laplacian_device(4, [(0, 1, 1.0), (1, 0, 2.0)])
    with pytest.raises(GraphError):
        assemble_laplacian_device(4, [(0, 1, -1.0)])
    with pytest.raises(GraphError):
        assemble_laplacian_device(4, [(0, 1, 1.0)], [(2, 1.0), (2, 3.0)])


def test_grid2d_through_device_assembly_solves_like_host(U):
    """A 2D grid assembled on the device gives the same hierarchy and history
    as the host builder (the reference's generator + assembly)."""
    from paper_1302_2547_b200 import problems
    from paper_1302_2547_b200.graph import assemble_laplacian_device

    n = 40
    A = problems.grid2d(n)
    v = np.arange(n * n)
    r, c = v // n, v % n
    right = v[c + 1 < n]
    down = v[r + 1 < n]
    # the reference generator's edge order: per vertex, right then down
    ei = np.concatenate([right, down])
    ej = np.concatenate([right + 1, down + n])
    order = np.lexsort((np.r_[np.zeros(right.size), np.ones(down.size)], ei))
    ei, ej = ei[order], ej[order]
    miss = (r == 0).astype(float) + (r == n - 1) + (c == 0) + (c == n - 1)
    bj = v[miss > 0]
    d = assemble_laplacian_device(n * n, (ei, ej, np.ones(ei.size)), (bj, miss[miss > 0]))
    _eq(d, A.indptr, A.indices, A.data)


@pytest.mark.parametrize("n,bc,aniso", [(31, "dirichlet", (1.0, 1.0)), (24, "dirichlet", (0.3, 1.7)),
                                        (20, "neumann", (1.0, 0.1))])
def test_reference_api_grid_problem(U, n, bc, aniso):
    """generate_structured_grid + assemble_laplacian (device assembly) ==
    the host builder (itself pinned to the reference's assembly)."""
    from paper_1302_2547_b200 import problems

    P = U.generate_structured_grid(n, bc, aniso)
    A = U.assemble_laplacian(P)
    B = problems.grid2d(n, bc, aniso)
    assert np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices)
    assert np.array_equal(A.data, B.data)
    assert P.singular == (bc == "neumann")
