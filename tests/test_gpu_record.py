"""record_iterates on the device (reference solvers.py:40-56; recording at
:168-172, :209-218, :281-286, :340-346): per-iteration iterates
(x - U xc for the recycled solver), residual vectors and (s, t, omega)
steps, bit for bit against the canonical oracle, with a half-step exit and
with full iterations, with and without a recycle space."""

import numpy as np
import pytest

from conftest import random_space_arrays

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1406_2831_b200 as P
    return P


FIELDS = ("U", "Ut", "C", "Ct", "Dc", "Chat", "Ccheck")


@pytest.mark.parametrize("k,tol", [(0, 1e-9), (6, 1e-9), (6, 1e-3), (0, 0.9)])
def test_record_iterates_bitwise_vs_oracle(P, canon, k, tol):
    from oracle import krylov as O
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence("c2", small=True)
    A, b = seq.matrix(1), seq.rhs(1, 0)
    S = random_space_arrays(A, k, seed=4, ops=canon) if k else None
    Sg = P.RecycleSpace(**{f: getattr(S, f) for f in FIELDS}) if k else None
    cfg = P.SolverConfig(tol=tol, max_itn=200, seed=2, record_iterates=True)
    x, h = P.rbicgstab_solve(P.SparseMatrix.from_csr(A), b, recycle=Sg, config=cfg)
    xo, ho = O.rbicgstab(A, b, recycle=S, ops=canon, record=True,
                         config=O.Config(tol=tol, max_itn=200, seed=2))
    assert h.resid == ho.resid and h.status == ho.status
    assert len(h.iterates) == len(ho.iterates) == len(h.resid)
    assert len(h.residual_vectors) == len(h.resid)
    assert len(h.omega_steps) == len(ho.omega_steps)
    for a, c in zip(h.iterates, ho.iterates):
        assert np.array_equal(a, c)
    for a, c in zip(h.residual_vectors, ho.residual_vectors):
        assert np.array_equal(a, c)
    for (s1, t1, o1), (s2, t2, o2) in zip(h.omega_steps, ho.omega_steps):
        assert np.array_equal(s1, s2) and np.array_equal(t1, t2) and o1 == o2
    assert np.array_equal(h.iterates[-1], x)
    assert np.array_equal(x, xo)


def test_record_off_leaves_fields_none(P):
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence("c1", small=True)
    _, h = P.bicgstab_solve(P.SparseMatrix.from_csr(seq.matrix(0)), seq.rhs(0, 0))
    assert h.iterates is None and h.residual_vectors is None and h.omega_steps is None
