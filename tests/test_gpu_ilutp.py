"""ILUTP split preconditioning on the device (reference ilutp.py):

* the four triangular solves (L^{-1}, L^{-H}, U^{-1}, U^{-H}; level-scheduled
  kernels, csrc/precond.cu) and the operator L^{-1} A P U^{-1} with its
  adjoint equal the canonical oracle (oracle/canon.c canon_trsv) bit for bit,
  with x in shared memory (n <= 25600) and in global memory, with and
  without column pivoting -- and the reference's SuperLU application to
  rounding;
* the solvers on the preconditioned operator (BiCGSTAB, recycled BiCGSTAB,
  the RBiCG generation solve with its harvest) equal the oracle bit for bit,
  and the ``precond=`` form equals the operator form;
* the whole preconditioned sequence (the reference driver's own default
  path, driver.py:98-168) against krecycle's driver.run_sequence, run by
  tests/golden/make_golden_full.py at 1/2/4/8 BLAS threads.
"""

import os

import numpy as np
import pytest

from conftest import REPO, random_space_arrays

pytestmark = pytest.mark.gpu

FULL = os.path.join(REPO, "tests", "golden", "reference_full.npz")


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1406_2831_b200 as P
    return P


def _weak(n, seed):
    r = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        for j in r.choice(n, size=5, replace=False):
            if j != i:
                rows.append(i)
                cols.append(int(j))
                vals.append(r.standard_normal())
        rows.append(i)
        cols.append(i)
        vals.append(0.05 * r.standard_normal() + 3.0 * (i % 7 == 0))
    return np.array(rows), np.array(cols), np.array(vals)


def _matrix(kind, P):
    from paper_1406_2831_b200.workloads import c1_sequence, make_sequence
    if kind == "c1s":
        A = make_sequence("c1", small=True).matrix(1)
    elif kind == "c1":
        A = make_sequence("c1").matrix(1)
    elif kind == "c1big":          # n = 28900 > 25600: x in global memory
        A = c1_sequence(m=170, num=2).matrix(1)
    else:                          # weak diagonal: the factorization pivots
        rows, cols, vals = _weak(700, 3)
        S = P.SparseMatrix.from_triplets(700, 700, rows, cols, vals)
        return S
    return P.SparseMatrix.from_csr(A)


KINDS = ["c1s", "c1", "c1big", "pivot"]


@pytest.mark.parametrize("kind", KINDS)
def test_triangular_solves_and_operator_bitwise(P, canon, kind):
    from oracle.ops import CsrOperand, SplitOperand
    A = _matrix(kind, P)
    F = P.ilutp_factor(A, pivot_tol=0.5 if kind == "pivot" else 0.1)
    if kind == "pivot":
        assert np.any(F.perm != np.arange(A.nrows))
    so = SplitOperand(CsrOperand.of(A), F)
    x = np.random.default_rng(1).standard_normal(A.nrows)
    for which, key in (("lower", "L"), ("lower_h", "Lt"), ("upper", "U"), ("upper_h", "Ut")):
        got = F.device().host_apply(which, x)
        assert np.array_equal(got, canon.trsv(so, key, x)), which
    # the reference's own application (SuperLU) agrees to rounding
    luL, luU = so.superlu()
    assert np.allclose(P.apply_left(F, x), luL.solve(x), rtol=1e-10, atol=1e-12)
    assert np.allclose(P.apply_right_h(F, x), luU.solve(x[F.perm], trans="H"),
                       rtol=1e-10, atol=1e-12)
    op = P.SplitPreconditionedOperator(A, F)
    assert np.array_equal(op.matvec(x), canon.matvec(so, x))
    assert np.array_equal(op.rmatvec(x), canon.rmatvec(so, x))


@pytest.mark.parametrize("kind", ["c1s", "c1big"])
def test_preconditioned_solvers_bitwise(P, canon, kind):
    from oracle import krylov as O
    from oracle.ops import CsrOperand, SplitOperand
    A = _matrix(kind, P)
    F = P.ilutp_factor(A)
    so = SplitOperand(CsrOperand.of(A), F)
    b = np.random.default_rng(2).standard_normal(A.nrows)
    bh = P.apply_left(F, b)
    assert np.array_equal(bh, canon.trsv(so, "L", b))
    op = P.CountingOperator(P.SplitPreconditionedOperator(A, F))
    cfg = P.SolverConfig(tol=1e-10, max_itn=200, seed=3)
    ocfg = O.Config(tol=1e-10, max_itn=200, seed=3)
    x, h = P.bicgstab_solve(op, bh, config=cfg)
    xo, ho = O.bicgstab(so, bh, config=ocfg, ops=canon)
    assert (h.status, h.resid, h.matvecs) == (ho.status, ho.resid, ho.matvecs)
    assert h.final_true_resid == ho.final_true_resid
    assert np.array_equal(x, xo)
    assert op.n_matvec == h.total_matvecs
    # recycled, with a space built on the preconditioned operator
    S = random_space_arrays(so, 4, seed=5, ops=canon)
    Sg = P.RecycleSpace(U=S.U, Ut=S.Ut, C=S.C, Ct=S.Ct, Dc=S.Dc, Chat=S.Chat, Ccheck=S.Ccheck)
    x2, h2 = P.rbicgstab_solve(op, bh, recycle=Sg, config=cfg)
    xo2, ho2 = O.rbicgstab(so, bh, recycle=S, config=ocfg, ops=canon)
    assert (h2.status, h2.resid, h2.matvecs) == (ho2.status, ho2.resid, ho2.matvecs)
    assert np.array_equal(x2, xo2)
    # precond= form: bh = L^{-1} b, x = P U^{-1} y, true residual on (A, b)
    x3, h3 = P.bicgstab_solve(A, b, precond=F, config=cfg)
    assert h3.resid == h.resid
    assert np.array_equal(x3, P.apply_right(F, x))
    r = b - A.to_scipy() @ x3
    assert abs(h3.final_true_resid - np.linalg.norm(r) / np.linalg.norm(b)) <= \
        1e-6 * max(h3.final_true_resid, 1e-300)


def test_preconditioned_generation_bitwise(P, canon):
    """RBiCG on the preconditioned operator (and its adjoint) with the
    per-cycle harvest: histories, cycles, the harvested space."""
    from oracle import krylov as O
    from oracle.ops import CsrOperand, SplitOperand
    A = _matrix("c1", P)
    F = P.ilutp_factor(A)
    so = SplitOperand(CsrOperand.of(A), F)
    b = P.apply_left(F, np.random.default_rng(4).standard_normal(A.nrows))
    op = P.SplitPreconditionedOperator(A, F)
    state, ostate = {"S": None}, {"S": None}

    def harvest(c):
        state["S"] = P.update_recycle_space(op, [c], state["S"], 6)

    def oharvest(c):
        ostate["S"] = O.update_recycle_space(so, [c], ostate["S"], 6, ops=canon)

    cfg = P.SolverConfig(tol=1e-10, max_itn=200, s=3, seed=0)
    x, xt, h, cyc = P.rbicg_solve(op, b, b_dual=np.ones(A.nrows), config=cfg,
                                  cycle_callback=harvest)
    xo, xto, ho, cyco = O.rbicg(so, b, b_dual=np.ones(A.nrows), ops=canon,
                                config=O.Config(tol=1e-10, max_itn=200, s=3, seed=0),
                                cycle_callback=oharvest)
    assert (h.status, h.resid, h.resid_dual, h.matvecs) == \
        (ho.status, ho.resid, ho.resid_dual, ho.matvecs)
    assert np.array_equal(x, xo) and np.array_equal(xt, xto)
    assert len(cyc) == len(cyco) >= 1
    for c1, c2 in zip(cyc, cyco):
        assert np.array_equal(c1.V, c2.V) and np.array_equal(c1.Vt, c2.Vt)
    assert (state["S"] is None) == (ostate["S"] is None)
    if state["S"] is not None and state["S"].k:
        assert state["S"].k == ostate["S"].k
        assert np.array_equal(state["S"].C, ostate["S"].C)


@pytest.mark.parametrize("tag,name,small", [("c1s", "c1", True), ("c1", "c1", False)])
def test_preconditioned_sequence_vs_reference_driver(P, tag, name, small):
    """run_sequence(policy='verbatim', precond='ilutp') -- the reference
    driver's default path -- against krecycle's driver.run_sequence: per
    sequence matvecs within the reference's thread-count envelope +- 2 %,
    every solve converged."""
    from paper_1406_2831_b200.sequence import run_sequence
    from paper_1406_2831_b200.workloads import make_sequence
    if not os.path.exists(FULL):
        pytest.skip("no fixture")
    G = np.load(FULL, allow_pickle=False)
    ts = [t for t in (1, 2, 4, 8, 16) if f"ilutp/{tag}/t{t}/iters" in G]
    if not ts:
        pytest.skip("ilutp fixture missing")
    res = run_sequence(make_sequence(name, small=small), policy="verbatim", baseline=True,
                       api=P, precond="ilutp")
    mv = np.array([G[f"ilutp/{tag}/t{t}/matvecs"] for t in ts])
    bmv = np.array([G[f"ilutp/{tag}/t{t}/base_matvecs"] for t in ts])
    gm = np.array([h.total_matvecs for h in res.recycling.histories])
    gb = np.array([h.total_matvecs for h in res.baseline.histories])
    print(f"\nilutp {tag}: gpu rec matvecs {gm.tolist()} dims {res.space_dims} base "
          f"{gb.tolist()}; reference rec {mv.min(0).tolist()}..{mv.max(0).tolist()} "
          f"base {bmv.min(0).tolist()}..{bmv.max(0).tolist()}")
    assert all(h.status == "converged" for h in res.recycling.histories)
    assert all(h.status == "converged" for h in res.baseline.histories)
    assert mv.sum(1).min() * 0.98 - 2 <= gm.sum() <= mv.sum(1).max() * 1.02 + 2
    assert bmv.sum(1).min() * 0.98 - 2 <= gb.sum() <= bmv.sum(1).max() * 1.02 + 2
