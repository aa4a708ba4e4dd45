"""The persistent drivers (persist.cu) over the shapes that change their work
split, bit-identical to the canonical oracle (oracle/krylov.py + CanonOps):

* fused v2 (k <= 32, unpermuted rows): one CTA per SM owning canonical blocks
  me and me + G -- a single partial block (n < 1024), ragged last blocks,
  CTAs owning one and two blocks, E = 2 (n > 303104) up to the largest
  persistent size (606208), k = 0, k in the last column group, k = 32;
* v1 (k = 33 and sigma-permuted rows) on the same matrices;
* SELL-32 and CSR storage.
Matrices are random non-symmetric, diagonally dominant, with ragged rows
(1..9 entries) so the SpMV's predicated batches see every tail length.
"""

import numpy as np
import pytest

from conftest import gpu, random_space_arrays

pytestmark = gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_1406_2831_b200 as P
    return P


def ragged_matrix(n, seed):
    """Random sparse A = D + N: rows with 0..8 off-diagonals at random
    columns, |D| ~ 3, sorted columns (canonical CSR)."""
    from paper_1406_2831_b200.workloads import CSR
    r = np.random.default_rng(seed)
    cnt = r.integers(0, 9, size=n)
    rows = np.repeat(np.arange(n), cnt)
    cols = r.integers(0, n, size=rows.size)
    vals = r.uniform(-1.0, 1.0, size=rows.size)
    rows = np.concatenate([rows, np.arange(n)])
    cols = np.concatenate([cols, np.arange(n)])
    vals = np.concatenate([vals, 2.5 + r.uniform(0.0, 1.0, size=n)])
    import scipy.sparse as sp
    S = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    S.sum_duplicates()
    S.sort_indices()
    return CSR(n, S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data.copy())


def _space(P, S):
    return P.RecycleSpace(U=S.U, Ut=S.Ut, C=S.C, Ct=S.Ct, Dc=S.Dc, Chat=S.Chat,
                          Ccheck=S.Ccheck)


CASES = [
    # n, k, fmt (2 = SELL-32, 1 = CSR)
    (1000, 0, 2),
    (1000, 5, 2),
    (16389, 10, 2),
    (16389, 10, 1),
    (200_000, 20, 2),
    (200_000, 32, 2),
    (200_000, 33, 2),      # k > 32: v1 kernel
    (400_000, 8, 2),       # E = 2
    (606_208, 3, 1),       # largest E = 2 size, CSR
]

# above PERSISTENT_MAX_N the persistent driver refuses; the graph driver runs
GRAPH_CASES = [
    (700_001, 6, 2),       # E = 4
    (1_300_000, 0, 2),     # E = 8, k = 0
    (1_300_000, 9, 1),     # E = 8, CSR
]


@pytest.mark.parametrize("n,k,fmt", CASES)
def test_persistent_bitwise_vs_oracle(pkg, canon, n, k, fmt):
    from oracle import krylov as O
    from paper_1406_2831_b200 import solvers as S
    from paper_1406_2831_b200.device import DeviceMatrix, to_device
    A = ragged_matrix(n, seed=n + k)
    b = np.random.default_rng(n).standard_normal(n)
    Sp = random_space_arrays(A, k, seed=11, ops=canon) if k else None
    M = DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values, fmt=fmt)
    assert M.format == {1: "csr", 2: "sell32"}[fmt]
    for tol, max_itn in ((1e-14, 7), (1e-9, 400)):
        cfg = pkg.SolverConfig(tol=tol, max_itn=max_itn, seed=5)
        xo, ho = O.rbicgstab(A, b, recycle=Sp, config=O.Config(tol=tol, max_itn=max_itn, seed=5),
                             ops=canon)
        xg, hg = S.solve_device(M, to_device(b), None, _space(pkg, Sp) if k else None, cfg,
                                use_graph=2)
        # the driver that actually ran: single cluster for tiny systems,
        # the fused kernel up to k = 32, the nine-barrier kernel above
        # (a 16-CTA cluster needs a GPC with 16 free SMs; without one the
        # fused kernel runs instead)
        want = {"cluster", "fused"} if (A.n <= 16384 and k <= 10) else \
            ({"fused"} if k <= 32 else {"persistent"})
        assert S.LAST_SOLVE["driver"] in want, (S.LAST_SOLVE["driver"], want)
        assert hg.status == ho.status
        assert hg.resid == ho.resid
        assert hg.matvecs == ho.matvecs
        assert np.array_equal(xg.cpu().numpy(), xo)


def test_persistent_sigma_rows_use_v1(pkg, canon):
    """sigma-permuted SELL rows run the v1 persistent kernel: still bitwise."""
    from oracle import krylov as O
    from paper_1406_2831_b200 import solvers as S
    from paper_1406_2831_b200.device import DeviceMatrix, to_device
    A = ragged_matrix(70_000, seed=3)
    b = np.random.default_rng(1).standard_normal(A.n)
    Sp = random_space_arrays(A, 6, seed=2, ops=canon)
    M = DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values, fmt=3)
    assert M.format == "sell32-sigma"
    cfg = pkg.SolverConfig(tol=1e-9, max_itn=60, seed=2)
    xo, ho = O.rbicgstab(A, b, recycle=Sp, config=O.Config(tol=1e-9, max_itn=60, seed=2),
                         ops=canon)
    xg, hg = S.solve_device(M, to_device(b), None, _space(pkg, Sp), cfg, use_graph=2)
    assert S.LAST_SOLVE["driver"] == "persistent"
    assert (hg.status, hg.resid, hg.matvecs) == (ho.status, ho.resid, ho.matvecs)
    assert np.array_equal(xg.cpu().numpy(), xo)


@pytest.mark.parametrize("n,k,fmt", GRAPH_CASES)
def test_large_n_graph_bitwise_and_persistent_refused(pkg, canon, n, k, fmt):
    from oracle import krylov as O
    from paper_1406_2831_b200 import _lib, solvers as S
    from paper_1406_2831_b200.device import DeviceMatrix, to_device
    A = ragged_matrix(n, seed=n + k)
    b = np.random.default_rng(n).standard_normal(n)
    Sp = random_space_arrays(A, k, seed=11, ops=canon) if k else None
    M = DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values, fmt=fmt)
    cfg = pkg.SolverConfig(tol=1e-9, max_itn=400, seed=5)
    xo, ho = O.rbicgstab(A, b, recycle=Sp, config=O.Config(tol=1e-9, max_itn=400, seed=5),
                         ops=canon)
    xg, hg = S.solve_device(M, to_device(b), None, _space(pkg, Sp) if k else None, cfg)
    assert S.LAST_SOLVE["driver"] == "graph"
    assert (hg.status, hg.resid, hg.matvecs) == (ho.status, ho.resid, ho.matvecs)
    assert np.array_equal(xg.cpu().numpy(), xo)
    with pytest.raises(_lib.KrbError):
        S.solve_device(M, to_device(b), None, None, cfg, use_graph=2)


def test_graph_recaptured_for_a_new_matrix_of_the_same_shape(pkg, canon):
    """The graph driver bakes the SpMV's matrix into its kernel parameters:
    a solve on a NEW matrix of the same shape (its arrays partly at freed
    addresses of the previous one) must re-capture, not reuse a graph that
    reads freed memory (bench.py's C5 step caught this)."""
    import gc
    from oracle import krylov as O
    from paper_1406_2831_b200 import solvers as S
    from paper_1406_2831_b200.device import DeviceMatrix, to_device
    n = 700_001
    b = np.random.default_rng(0).standard_normal(n)
    cfg = pkg.SolverConfig(tol=1e-10, max_itn=25, seed=1)
    for seed in (1, 2, 3):
        A = ragged_matrix(n, seed=seed)
        M = DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
        xg, hg = S.solve_device(M, to_device(b), None, None, cfg)
        assert S.LAST_SOLVE["driver"] == "graph"
        xo, ho = O.rbicgstab(A, b, config=O.Config(tol=1e-10, max_itn=25, seed=1), ops=canon)
        assert (hg.status, hg.resid, hg.matvecs) == (ho.status, ho.resid, ho.matvecs), seed
        assert np.array_equal(xg.cpu().numpy(), xo)
        del M, xg
        gc.collect()
