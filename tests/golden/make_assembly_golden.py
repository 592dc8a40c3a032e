"""Golden fixtures for the on-device assembly (csrc/assemble.cu), made by
running the REFERENCE's own SparseMatrix.from_coo and assemble_laplacian
(U/sparse.py:56-74, U/graph.py:20-82) in this container:

    python tests/golden/make_assembly_golden.py

Writes tests/golden/assembly.npz: (1) random triplets with heavy duplication
(segments up to 700 entries, so np.add.reduceat's pairwise summation is
exercised), exact cancellations and -0.0 values, and the reference CSR;
(2) a random float-weighted graph with boundary weights and its reference
Laplacian."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import load_reference, save  # noqa: E402


def main():
    U, _ = load_reference()
    from uaamg.graph import GraphProblem, assemble_laplacian
    from uaamg.sparse import SparseMatrix

    rng = np.random.default_rng(2024)
    out = {}
    # (1) triplets
    nr, nc = 300, 250
    m = 40000
    rows = rng.integers(0, nr, m)
    cols = rng.integers(0, nc, m)
    # a few very long duplicate segments
    hot = rng.integers(0, m, 2500)
    rows[hot[:1200]] = 7
    cols[hot[:1200]] = 11
    rows[hot[1200:1900]] = 123
    cols[hot[1200:1900]] = 45
    vals = rng.standard_normal(m) * 10.0 ** rng.uniform(-6, 6, m)
    # exact cancellation pairs and signed zeros
    vals[:200:2] = 3.25
    rows[1:200:2], cols[1:200:2] = rows[:200:2], cols[:200:2]
    vals[1:200:2] = -3.25
    vals[200:210] = -0.0
    A = SparseMatrix.from_coo(nr, nc, rows, cols, vals)
    out.update(coo_rows=rows, coo_cols=cols, coo_vals=vals, coo_shape=np.array([nr, nc]),
               coo_indptr=A.indptr, coo_indices=A.indices, coo_data=A.data)
    # (2) Laplacian of a random weighted graph with boundary weights
    n = 2000
    ei = rng.integers(0, n, 12000)
    ej = rng.integers(0, n, 12000)
    keep = ei != ej
    ei, ej = ei[keep], ej[keep]
    lo, hi = np.minimum(ei, ej), np.maximum(ei, ej)
    _, first = np.unique(lo * n + hi, return_index=True)
    first = np.sort(first)
    ei, ej = ei[first], ej[first]  # unique edges, original orientation kept
    w = rng.uniform(0.1, 3.0, ei.shape[0]) * 10.0 ** rng.uniform(-3, 3, ei.shape[0])
    bj = np.sort(rng.choice(n, 150, replace=False))
    bw = rng.uniform(0.5, 2.0, 150)
    P = GraphProblem(n, [(int(a), int(b), float(c)) for a, b, c in zip(ei, ej, w)],
                     [(int(a), float(b)) for a, b in zip(bj, bw)])
    L = assemble_laplacian(P)
    out.update(lap_n=np.array(n), lap_ei=ei, lap_ej=ej, lap_w=w, lap_bj=bj, lap_bw=bw, lap_indptr=L.indptr,
               lap_indices=L.indices, lap_data=L.data)
    save("assembly", **out)


if __name__ == "__main__":
    main()
