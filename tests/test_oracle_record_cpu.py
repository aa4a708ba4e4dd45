"""CPU: the oracle's record_iterates restatement (oracle/krylov.py
rbicgstab(record=True)) equals krecycle's own recording (solvers.py:284-286,
321-323, 344-347) bit for bit, run live against the unmodified reference
installed in baseline/_ref (one BLAS thread)."""

import os
import sys

import numpy as np
import pytest
from threadpoolctl import threadpool_limits

from conftest import REPO

REF = os.path.join(REPO, "baseline", "_ref")


@pytest.fixture(scope="module")
def K():
    if not os.path.isdir(os.path.join(REF, "krecycle")):
        pytest.skip("krecycle not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import krecycle
    return krecycle


@pytest.mark.parametrize("k,tol", [(0, 1e-9), (5, 1e-9), (5, 0.5)])
def test_record_iterates_refops_equals_reference(K, k, tol):
    from oracle import krylov as O
    from oracle.ops import RefOps
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence("c1", small=True)
    A, b = seq.matrix(1), seq.rhs(1, 0)
    KA = K.SparseMatrix(A.n, A.n, A.row_ptr, A.col_idx, A.values)
    r = np.random.default_rng(9)
    with threadpool_limits(1):
        S = K.biorthonormalize(r.standard_normal((A.n, k)), r.standard_normal((A.n, k)),
                               KA) if k else None
        xk, hk = K.rbicgstab_solve(KA, b, recycle=S, config=K.SolverConfig(
            tol=tol, max_itn=300, seed=3, record_iterates=True))
        xo, ho = O.rbicgstab(A, b, recycle=S, ops=RefOps(), record=True,
                             config=O.Config(tol=tol, max_itn=300, seed=3))
    assert hk.resid == ho.resid
    assert len(hk.iterates) == len(ho.iterates)
    for a, c in zip(hk.iterates, ho.iterates):
        assert np.array_equal(a, c)
    for a, c in zip(hk.residual_vectors, ho.residual_vectors):
        assert np.array_equal(a, c)
    assert len(hk.omega_steps) == len(ho.omega_steps)
    for (s1, t1, o1), (s2, t2, o2) in zip(hk.omega_steps, ho.omega_steps):
        assert np.array_equal(s1, s2) and np.array_equal(t1, t2) and o1 == o2
    assert np.array_equal(xk, xo)
