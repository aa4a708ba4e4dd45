"""Multi-right-hand-side path (batch.cu): a batch of
solves with one matrix and one recycle space is bit-identical, right-hand
side by right-hand side, to the separate single solves (which are pinned to
the oracle elsewhere) -- solutions, residual histories, matvec counts and
statuses -- including rhs that stop at different iterations (converged,
max_itn), x_init starts, k = 0 and chunks of more than four."""

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


def _space(P, S):
    return P.RecycleSpace(U=S.U, Ut=S.Ut, C=S.C, Ct=S.Ct, Dc=S.Dc, Chat=S.Chat,
                          Ccheck=S.Ccheck)


def _same(single, batched):
    (x1, h1), (x2, h2) = single, batched
    assert h1.status == h2.status
    assert h1.resid == h2.resid
    assert h1.matvecs == h2.matvecs
    assert h1.final_true_resid == h2.final_true_resid
    assert np.array_equal(np.asarray(x1), np.asarray(x2))


def _matrix(kind):
    if kind == "ragged":
        from test_gpu_persistent import ragged_matrix
        return ragged_matrix(50_003, seed=7)
    from paper_1406_2831_b200.workloads import make_sequence
    return make_sequence("c3", small=True).matrix(3)


@pytest.mark.parametrize("kind,k,nrhs", [("ragged", 6, 4), ("c3", 10, 3), ("ragged", 0, 2),
                                         ("c3", 0, 5), ("ragged", 33, 1)])
def test_batch_bitwise_vs_single(pkg, canon, kind, k, nrhs):
    A = _matrix(kind)
    Sp = pkg.SparseMatrix.from_csr(A)
    space = _space(pkg, random_space_arrays(A, k, seed=3, ops=canon)) if k else None
    r = np.random.default_rng(nrhs + k)
    bs = [r.standard_normal(A.n) for _ in range(nrhs)]
    # different stopping points: tight tol / short max_itn on some rhs
    cfgs = [pkg.SolverConfig(tol=(1e-10, 1e-6, 1e-12, 1e-8, 1e-9)[j % 5],
                             max_itn=(400, 400, 9, 400, 30)[j % 5], seed=11 + j)
            for j in range(nrhs)]
    x0s = [None] * nrhs
    if nrhs > 1:
        x0s[1] = r.standard_normal(A.n) * 1e-3
    if k:
        batched = pkg.rbicgstab_solve_batch(Sp, bs, x_inits=x0s, recycle=space, configs=cfgs)
    else:
        batched = pkg.bicgstab_solve_batch(Sp, bs, x_inits=x0s, configs=cfgs)
    assert len(batched) == nrhs
    for j in range(nrhs):
        if k:
            single = pkg.rbicgstab_solve(Sp, bs[j], x_init=x0s[j], recycle=space, config=cfgs[j])
        else:
            single = pkg.bicgstab_solve(Sp, bs[j], x_init=x0s[j], config=cfgs[j])
        _same(single, batched[j])
    statuses = {h.status for _, h in batched}
    if nrhs >= 3:
        assert "max_itn" in statuses and "converged" in statuses


def test_batch_counts_matvecs(pkg):
    """a CountingOperator is metered exactly as by the separate solves"""
    A = _matrix("ragged")
    Sp = pkg.SparseMatrix.from_csr(A)
    r = np.random.default_rng(0)
    bs = [r.standard_normal(A.n) for _ in range(3)]
    cfgs = [pkg.SolverConfig(tol=1e-8, seed=j) for j in range(3)]
    op1, op2 = pkg.CountingOperator(Sp), pkg.CountingOperator(Sp)
    pkg.bicgstab_solve_batch(op1, bs, configs=cfgs)
    for j in range(3):
        pkg.bicgstab_solve(op2, bs[j], config=cfgs[j])
    assert op1.n_matvec == op2.n_matvec > 0


@pytest.mark.parametrize("policy", ["verbatim", "first"])
def test_sequence_batched_schedule_identical(pkg, policy):
    """run_sequence(batch=True) == the one-by-one schedule on C3 (4 rhs per
    matrix): every recycling and baseline history, statuses and meters."""
    from paper_1406_2831_b200.sequence import run_sequence
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence("c3", small=True)
    r1 = run_sequence(seq, policy=policy, systems=8, batch=True)
    r2 = run_sequence(seq, policy=policy, systems=8, batch=False)
    for a, b in ((r1.recycling, r2.recycling), (r1.baseline, r2.baseline)):
        assert [h.resid for h in a.histories] == [h.resid for h in b.histories]
        assert [h.matvecs for h in a.histories] == [h.matvecs for h in b.histories]
        assert [h.status for h in a.histories] == [h.status for h in b.histories]
        assert a.total_matvecs == b.total_matvecs
    assert r1.space_dims == r2.space_dims
