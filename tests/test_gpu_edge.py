"""Edge cases on every device driver (host loop, CUDA graph, fused persistent
kernel, multi-rhs batch), bit-identical to the canonical oracle: tiny and
ragged sizes (n = 1 .. 33, one partial canonical block, one partial SELL
slice), zero right-hand side, exact initial guess, max_itn = 0 and 1, k = 0
and k = 1."""

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


def _tiny(n, seed):
    from test_gpu_persistent import ragged_matrix
    return ragged_matrix(n, seed)


def _space(P, S):
    return P.RecycleSpace(U=S.U, Ut=S.Ut, C=S.C, Ct=S.Ct, Dc=S.Dc, Chat=S.Chat,
                          Ccheck=S.Ccheck)


CASES = [  # n, k, rhs kind, x_init kind, max_itn
    (1, 0, "rand", None, 50),
    (2, 1, "rand", None, 50),
    (31, 0, "zero", None, 50),
    (33, 1, "rand", "exact", 50),
    (33, 1, "rand", None, 0),
    (257, 2, "rand", None, 1),
    (1029, 3, "rand", "rand", 60),
]


@pytest.mark.parametrize("n,k,rhs,x0,max_itn", CASES)
def test_edge_cases_all_drivers(pkg, canon, n, k, rhs, x0, max_itn):
    import time
    from oracle import krylov as O
    from paper_1406_2831_b200 import solvers as S
    A = _tiny(n, seed=n)
    r = np.random.default_rng(n + k)
    b = np.zeros(n) if rhs == "zero" else r.standard_normal(n)
    if x0 == "exact":
        import scipy.sparse.linalg as spla
        xi = spla.spsolve(A.to_scipy().tocsc(), b)
        b = A.to_scipy() @ xi       # consistent pair, r0 rounds to ~0
    else:
        xi = r.standard_normal(n) if x0 == "rand" else None
    Sp = random_space_arrays(A, k, seed=2, ops=canon) if k else None
    cfg = pkg.SolverConfig(tol=1e-10, max_itn=max_itn, seed=3)
    xo, ho = O.rbicgstab(A, b, x_init=xi, recycle=Sp,
                         config=O.Config(tol=1e-10, max_itn=max_itn, seed=3), ops=canon)
    space = _space(pkg, Sp) if k else None
    Asp = pkg.SparseMatrix.from_csr(A)
    for mode in (0, 1, 2):
        xg, hg = S._device_solve(Asp, b, xi, space, cfg, "rbicgstab", time.perf_counter(),
                                 use_graph=mode)
        assert (hg.status, hg.resid, hg.matvecs) == (ho.status, ho.resid, ho.matvecs), mode
        assert np.array_equal(xg, xo), mode
    out = pkg.rbicgstab_solve_batch(Asp, [b, b], x_inits=[xi, xi], recycle=space,
                                    configs=[cfg, cfg])
    for xg, hg in out:
        assert (hg.status, hg.resid, hg.matvecs) == (ho.status, ho.resid, ho.matvecs)
        assert np.array_equal(xg, xo)
    if rhs == "zero":
        assert ho.status == "converged" and ho.iterations == 0
    if max_itn == 0:
        assert ho.status == "max_itn"
