"""CPU: the host ILUTP factorization (libkrb krb_ilutp_factor, csrc/ilutp.cu)
equals krecycle.ilutp_factor (ilutp.py:131-281) bit for bit -- L, U and the
column permutation -- run live against the unmodified reference installed
in baseline/_ref: BASELINE stencils (no pivoting needed), random sparse
matrices with weak diagonals (column swaps), a fill limit, the exact
(drop_tol = 0) factorization, and the FactorizationError cases."""

import os
import sys

import numpy as np
import pytest

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


def _weak_diag(n, seed, per_row=5, diag_scale=0.05):
    r = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        js = r.choice(n, size=per_row, replace=False)
        for j in js:
            if j != i:
                rows.append(i)
                cols.append(int(j))
                vals.append(r.standard_normal())
        rows.append(i)
        cols.append(i)
        vals.append(diag_scale * r.standard_normal())
    return np.array(rows), np.array(cols), np.array(vals)


def _pair(K, P, rows=None, cols=None, vals=None, csr=None, n=None):
    if csr is not None:
        KA = K.SparseMatrix(csr.n, csr.n, csr.row_ptr, csr.col_idx, csr.values)
    else:
        KA = K.SparseMatrix.from_triplets(n, n, rows, cols, vals)
    PA = P.SparseMatrix(KA.nrows, KA.ncols, KA.row_ptr, KA.col_idx, KA.values)
    return KA, PA


def _same(Fk, Fp):
    for f in ("L", "U"):
        a, b = getattr(Fk, f), getattr(Fp, f)
        assert np.array_equal(a.row_ptr, b.row_ptr), f
        assert np.array_equal(a.col_idx, b.col_idx), f
        assert np.array_equal(np.asarray(a.values), np.asarray(b.values)), f
    assert np.array_equal(Fk.perm, Fp.perm)


CASES = [("c1", True), ("c2", True), ("c5", True), ("c1", False)]


@pytest.mark.parametrize("name,small", CASES)
def test_factor_bitwise_stencils(K, name, small):
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200.ilutp import ilutp_factor
    from paper_1406_2831_b200.workloads import make_sequence
    KA, PA = _pair(K, P, csr=make_sequence(name, small=small).matrix(1))
    Fk = K.ilutp_factor(KA, drop_tol=1e-4, pivot_tol=0.1)
    Fp = ilutp_factor(PA, drop_tol=1e-4, pivot_tol=0.1)
    _same(Fk, Fp)


@pytest.mark.parametrize("seed,drop,piv,fill", [(1, 1e-4, 0.1, None), (2, 1e-3, 1.0, None),
                                                (3, 1e-2, 0.5, 4), (6, 1e-3, 0.5, 8),
                                                (4, 0.0, 0.1, None), (5, 1e-4, 0.0, 3)])
def test_factor_bitwise_pivoting(K, seed, drop, piv, fill):
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200.ilutp import ilutp_factor
    n = 300
    rows, cols, vals = _weak_diag(n, seed)
    KA, PA = _pair(K, P, rows, cols, vals, n=n)
    try:
        Fk = K.ilutp_factor(KA, drop_tol=drop, pivot_tol=piv, fill_limit=fill)
    except K.FactorizationError as e:      # the same failure, same message
        from paper_1406_2831_b200.ilutp import FactorizationError
        with pytest.raises(FactorizationError, match=str(e)):
            ilutp_factor(PA, drop_tol=drop, pivot_tol=piv, fill_limit=fill)
        return
    Fp = ilutp_factor(PA, drop_tol=drop, pivot_tol=piv, fill_limit=fill)
    if piv > 0:
        assert np.any(Fk.perm != np.arange(n)), "case should pivot"
    _same(Fk, Fp)


def test_factorization_errors(K):
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200.ilutp import FactorizationError, ilutp_factor
    # an empty row
    A = P.SparseMatrix.from_triplets(3, 3, [0, 2], [0, 2], [1.0, 1.0])
    with pytest.raises(FactorizationError, match="row 1 is empty"):
        ilutp_factor(A)
    KA = K.SparseMatrix.from_triplets(3, 3, [0, 2], [0, 2], [1.0, 1.0])
    with pytest.raises(K.FactorizationError, match="row 1 is empty"):
        K.ilutp_factor(KA)
    with pytest.raises(ValueError):
        ilutp_factor(P.SparseMatrix.from_triplets(2, 3, [0, 1], [0, 1], [1.0, 1.0]))


def test_oracle_split_operator_refops_equals_reference(K):
    """The oracle's split-ILUTP operand with RefOps (SuperLU solves, as
    ilutp.py) reproduces krecycle's preconditioned solves bit for bit: a
    BiCGSTAB and an RBiCG generation solve on the preconditioned operator
    (driver.py:98-103 form: CountingOperator(SplitPreconditionedOperator),
    b -> apply_left(b))."""
    from threadpoolctl import threadpool_limits
    from oracle import krylov as O
    from oracle.ops import RefOps
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence("c1", small=True)
    A, b = seq.matrix(1), seq.rhs(1, 0)
    KA = K.SparseMatrix(A.n, A.n, A.row_ptr, A.col_idx, A.values)
    F = K.ilutp_factor(KA)
    op = K.SplitPreconditionedOperator(KA, F)
    bh = K.apply_left(F, b)
    with threadpool_limits(1):
        _, hk = K.bicgstab_solve(K.CountingOperator(op), bh, config=K.SolverConfig(seed=2))
        _, ho = O.bicgstab(op, bh, config=O.Config(seed=2), ops=RefOps())
        assert hk.resid == ho.resid and hk.final_true_resid == ho.final_true_resid
        _, _, gk, ck = K.rbicg_solve(K.CountingOperator(op), bh, b_dual=np.ones(A.n),
                                     config=K.SolverConfig(seed=0, s=10))
        _, _, go, co = O.rbicg(op, bh, b_dual=np.ones(A.n), ops=RefOps(),
                               config=O.Config(seed=0, s=10))
    assert gk.resid == go.resid and gk.resid_dual == go.resid_dual
    assert len(ck) == len(co) and np.array_equal(ck[0].V, co[0].V)
