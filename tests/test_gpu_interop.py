"""Drop-in interop with the reference's own objects: krecycle
(installed unmodified into baseline/_ref, the reference arm's install) hands
its SparseMatrix, RecycleSpace, CountingOperator and CapturedCycle objects to
this package's solvers, and this package's objects go back into krecycle's
functions.  Each crossing must work and give the same answer as the
same-package path."""

import os
import sys

import numpy as np
import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu

REF = os.path.join(REPO, "baseline", "_ref")


@pytest.fixture(scope="module")
def K():
    if not os.path.isdir(os.path.join(REF, "krecycle")):
        pytest.skip("krecycle not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import krecycle
    return krecycle


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1406_2831_b200 as P
    return P


@pytest.fixture(scope="module")
def system():
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence("c2", small=True)
    return seq.matrix(1), seq.rhs(1, 0), seq.matrix(2)


def _kmat(K, A):
    return K.SparseMatrix(A.n, A.n, A.row_ptr, A.col_idx, A.values)


def test_reference_objects_into_device_solvers(K, P, system):
    A, b, _ = system
    from paper_1406_2831_b200.workloads import sine_basis
    KA = _kmat(K, A)
    U = sine_basis((16, 16, 16), 8)
    KS = K.biorthonormalize(U, U, KA)                  # numpy RecycleSpace (reference)
    cfg = P.SolverConfig(tol=1e-9, max_itn=400, seed=1)
    # reference SparseMatrix + reference RecycleSpace + reference CountingOperator
    op = K.CountingOperator(KA)
    x1, h1 = P.rbicgstab_solve(op, b, recycle=KS, config=cfg)
    # the same through this package's own objects
    M = P.SparseMatrix.from_csr(A)
    S2 = P.RecycleSpace(U=KS.U, Ut=KS.Ut, C=KS.C, Ct=KS.Ct, Dc=KS.Dc, Chat=KS.Chat,
                        Ccheck=KS.Ccheck)
    op2 = P.CountingOperator(M)
    x2, h2 = P.rbicgstab_solve(op2, b, recycle=S2, config=cfg)
    assert h1.resid == h2.resid and h1.status == h2.status
    assert np.array_equal(x1, x2)
    # the reference's meter sees every product (operators.py:82-88)
    assert op.n_matvec == op2.n_matvec == h1.total_matvecs
    # the reference's refresh + our solver, and krecycle's result is close
    xk, hk = K.rbicgstab_solve(KA, b, recycle=KS, config=K.SolverConfig(
        tol=1e-9, max_itn=400, seed=1))
    # (iteration counts are compared against the reference's own envelope in
    # test_gpu_parity_full.py; here: both converge to the same solution)
    assert hk.status == h1.status == "converged"
    assert np.linalg.norm(x1 - xk) <= 1e-6 * np.linalg.norm(xk)


def test_reference_captured_cycle_into_device_update(K, P, system):
    """A CapturedCycle built the reference's way (numpy V / Vt n x ncols)
    through update_recycle_space on the device equals the device-built
    cycle's update bit for bit."""
    A, b, _ = system
    M = P.SparseMatrix.from_csr(A)
    cyc_dev = []
    P.rbicg_solve(M, b, b_dual=np.ones(A.n), config=P.SolverConfig(
        tol=1e-9, max_itn=300, s=10, seed=0), cycle_callback=cyc_dev.append)
    assert cyc_dev
    c = cyc_dev[0]
    kc = K.CapturedCycle(V=c.V, Vt=c.Vt, tri=c.tri, first_index=c.first_index)
    pc = P.CapturedCycle(V=c.V, Vt=c.Vt, tri=c.tri, first_index=c.first_index)
    assert pc.ncols == kc.ncols and pc.last_index == kc.last_index
    S_dev = P.update_recycle_space(M, [c], None, 6)
    S_ref_obj = P.update_recycle_space(M, [kc], None, 6)
    S_host = P.update_recycle_space(M, [pc], None, 6)
    for S in (S_ref_obj, S_host):
        assert S.k == S_dev.k
        for f in ("U", "Ut", "C", "Ct", "Chat", "Ccheck"):
            assert np.array_equal(getattr(S, f), getattr(S_dev, f))


def test_device_objects_into_reference_functions(K, P, system):
    """This package's RecycleSpace (device-resident, lazy host views) and
    CapturedCycle (device blocks) are accepted by krecycle's own CPU code."""
    A, b, A2 = system
    KA = _kmat(K, A)
    M = P.SparseMatrix.from_csr(A)
    r = np.random.default_rng(5)
    S = P.biorthonormalize(r.standard_normal((A.n, 6)), r.standard_normal((A.n, 6)), M)
    xk, hk = K.rbicgstab_solve(KA, b, recycle=S, config=K.SolverConfig(tol=1e-9, seed=1))
    assert hk.status == "converged"
    assert hk.final_true_resid <= 1.1e-9
    cycles = []
    P.rbicg_solve(M, b, b_dual=np.ones(A.n), config=P.SolverConfig(
        tol=1e-9, max_itn=300, s=10, seed=0), cycle_callback=cycles.append)
    Sk = K.update_recycle_space(KA, cycles[:1], None, 6)
    Sd = P.update_recycle_space(M, cycles[:1], None, 6)
    assert Sk.k == Sd.k
    # same space up to rounding (different summation orders)
    assert np.linalg.norm(Sk.C - Sd.C) <= 1e-6 * np.linalg.norm(Sk.C)
    # krecycle's refresh of a device space onto the next operator
    Sr = K.refresh_images(S, _kmat(K, A2))
    assert Sr.k == S.k
    # the package's SparseMatrix as krecycle's operator (duck-typed protocol)
    xs, hs = K.bicgstab_solve(M, b, config=K.SolverConfig(tol=1e-9, seed=2))
    assert hs.status == "converged"
