"""Problem builders vs the reference's own assembly (GraphProblem +
assemble_laplacian), fixtures from tests/golden/make_golden.py."""

import numpy as np
import pytest

from golden_util import load
from paper_1302_2547_b200 import problems as P


@pytest.fixture(scope="module")
def g():
    return load("problems")


CASES = {
    "g2d_dir_7": lambda: P.grid2d(7, "dirichlet"),
    "g2d_dir_7_aniso": lambda: P.grid2d(7, "dirichlet", (1.0, 10.0)),
    "g2d_dir_6_float": lambda: P.grid2d(6, "dirichlet", (0.3, 1.7)),
    "g2d_neu_6": lambda: P.grid2d(6, "neumann"),
    "g3d7_dir_4": lambda: P.grid3d(4, 7, "dirichlet"),
    "g3d7_neu_4": lambda: P.grid3d(4, 7, "neumann"),
    "g3d27_dir_4": lambda: P.grid3d(4, 27, "dirichlet"),
    "rgg_600": lambda: P.random_geometric(600, 12.0, 3),
}


@pytest.mark.parametrize("name", list(CASES))
def test_builder_bitexact(g, name):
    A = CASES[name]()
    assert np.array_equal(A.indptr, g[name + "_indptr"])
    assert np.array_equal(A.indices, g[name + "_indices"])
    assert np.array_equal(A.data, g[name + "_data"]), "values differ"


def test_grid3d_sizes():
    A = P.grid3d(8, 7)
    assert A.n_rows == 512 and A.nnz == 512 * 7 - 6 * 64
    A27 = P.grid3d(6, 27)
    assert A27.nnz == (3 * 6 - 2) ** 3
