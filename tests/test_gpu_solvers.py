"""Solver-level parity on the B200.

* vs the canonical CPU oracle (oracle/krylov.py with CanonOps): residual
  histories, matvec counts, statuses and solutions bit-identical;
* vs the reference (golden fixtures produced by krecycle itself, and the
  RefOps restatement): relative residual histories within the reference's own
  noise floor over the first 50 iterations (north-star bar 1e-8 where the
  reference itself is reproducible to that level), final true residual <= tol,
  matvec counts within +-2%.
"""

import numpy as np
import pytest

from conftest import golden_csr, gpu, random_space_arrays

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


def _rel_hist_diff(a, b, m=51):
    a = np.asarray(a)[:m]
    b = np.asarray(b)[:m]
    L = min(len(a), len(b))
    return float(np.max(np.abs(a[:L] - b[:L]) / np.abs(b[:L]))) if L else 0.0


@pytest.mark.parametrize("cfg", ["c1", "c2", "c4", "c5"])
def test_bicgstab_bitwise_vs_canon_oracle(pkg, canon, cfg):
    from oracle import krylov as O
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence(cfg, small=True)
    for j in range(seq.num_matrices):
        A, b = seq.matrix(j), seq.rhs(j, 0)
        x_o, h_o = O.bicgstab(A, b, config=O.Config(tol=seq.tol, max_itn=400, seed=j),
                              ops=canon)
        x_g, h_g = pkg.bicgstab_solve(pkg.SparseMatrix.from_csr(A), b,
                                      config=pkg.SolverConfig(tol=seq.tol, max_itn=400,
                                                              seed=j))
        assert h_g.status == h_o.status
        assert h_g.resid == h_o.resid
        assert h_g.matvecs == h_o.matvecs
        assert np.array_equal(x_g, x_o)
        assert h_g.final_true_resid == h_o.final_true_resid


@pytest.mark.parametrize("cfg,k", [("c1", 10), ("c2", 20), ("c4", 30), ("c5", 30)])
def test_rbicgstab_bitwise_vs_canon_oracle(pkg, canon, cfg, k):
    from oracle import krylov as O
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence(cfg, small=True)
    A0, A1 = seq.matrix(0), seq.matrix(1)
    S = random_space_arrays(A1, k, seed=5, ops=canon)
    b = seq.rhs(1, 0)
    cfgo = O.Config(tol=seq.tol, max_itn=400, seed=2)
    x_o, h_o = O.rbicgstab(A1, b, recycle=S, config=cfgo, ops=canon)
    x_g, h_g = pkg.rbicgstab_solve(pkg.SparseMatrix.from_csr(A1), b,
                                   recycle=_space(pkg, S),
                                   config=pkg.SolverConfig(tol=seq.tol, max_itn=400,
                                                           seed=2))
    assert h_g.status == h_o.status
    assert h_g.resid == h_o.resid
    assert h_g.matvecs == h_o.matvecs
    assert np.array_equal(x_g, x_o)


def test_bicgstab_vs_reference_golden(pkg, golden):
    for j in range(3):
        p = f"bicgstab/c1s{j}/"
        A = golden_csr(golden, p)
        b = golden[p + "b"]
        x, h = pkg.bicgstab_solve(pkg.SparseMatrix.from_csr(A), b,
                                  config=pkg.SolverConfig(tol=1e-8, max_itn=500,
                                                          seed=int(golden[p + "seed"])))
        ref = golden[p + "resid"]
        noise = max(_rel_hist_diff(golden[p + "resid_8thr"], ref),
                    _rel_hist_diff(golden[p + "resid_exactdot"], ref),
                    float(np.max(golden[p + "resid_variant_reldiff"])))
        assert _rel_hist_diff(h.resid, ref) <= max(1e-8, 10 * noise)
        assert h.status == str(golden[p + "status"])
        assert abs(h.total_matvecs - golden[p + "matvecs"][-1]) <= max(2, 0.02 * golden[p + "matvecs"][-1])
        assert h.final_true_resid <= 1e-8 * 1.1


def test_rbicgstab_vs_reference_golden(pkg, golden):
    p = "rbicgstab/rand300/"
    A = golden_csr(golden, p)
    b = golden[p + "b"]
    S = pkg.RecycleSpace(**{f: golden[p + "space/" + f] for f in
                            ("U", "Ut", "C", "Ct", "Dc", "Chat", "Ccheck")})
    x, h = pkg.rbicgstab_solve(pkg.SparseMatrix.from_csr(A), b, recycle=S,
                               config=pkg.SolverConfig(tol=1e-10, max_itn=300, seed=3))
    ref = golden[p + "resid"]
    floor = max(_rel_hist_diff(golden[p + "resid_8thr"], ref),
                _rel_hist_diff(golden[p + "resid_exactdot"], ref),
                float(np.max(golden[p + "resid_variant_reldiff"])))
    assert _rel_hist_diff(h.resid, ref) <= max(1e-8, 10 * floor)
    assert h.status == "converged"
    assert h.total_matvecs == golden[p + "matvecs"][-1]
    assert np.allclose(x, golden[p + "x"], rtol=1e-8, atol=1e-12)
    # x_init path: one counted product
    x2, h2 = pkg.rbicgstab_solve(pkg.SparseMatrix.from_csr(A), b,
                                 x_init=golden[p + "xinit"], recycle=S,
                                 config=pkg.SolverConfig(tol=1e-10, max_itn=300, seed=3))
    assert h2.matvecs[0] == 1
    ref2 = golden[p + "xinit_resid"]
    floor2 = _rel_hist_diff(golden[p + "xinit_resid_exactdot"], ref2)
    assert _rel_hist_diff(h2.resid, ref2) <= max(1e-8, 10 * floor2)
    assert h2.final_true_resid <= 1.1e-10


def test_counting_operator_and_errors(pkg):
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence("c1", small=True)
    A = pkg.SparseMatrix.from_csr(seq.matrix(0))
    op = pkg.CountingOperator(A)
    x, h = pkg.bicgstab_solve(op, seq.rhs(0, 0))
    assert op.n_matvec == h.total_matvecs and op.n_rmatvec == 0
    with pytest.raises(ValueError):
        pkg.bicgstab_solve(A, np.ones(A.nrows + 1))
    with pytest.raises(AttributeError):   # not an IlutpFactors (the reference
        pkg.bicgstab_solve(A, seq.rhs(0, 0), precond=object())   # fails alike)
    # max_itn = 0 -> immediate max_itn, one history entry
    x, h = pkg.bicgstab_solve(A, seq.rhs(0, 0), config=pkg.SolverConfig(max_itn=0))
    assert h.status == "max_itn" and h.iterations == 0
    # zero rhs -> converged at entry
    x, h = pkg.bicgstab_solve(A, np.zeros(A.nrows))
    assert h.status == "converged" and h.iterations == 0 and np.all(x == 0)


def test_graph_and_host_loop_agree(pkg):
    from paper_1406_2831_b200 import solvers as S
    from paper_1406_2831_b200.workloads import make_sequence
    import time
    seq = make_sequence("c2", small=True)
    A = pkg.SparseMatrix.from_csr(seq.matrix(0))
    b = seq.rhs(0, 0)
    cfg = pkg.SolverConfig(tol=1e-8, max_itn=300)
    x1, h1 = S._device_solve(A, b, None, None, cfg, "bicgstab", time.perf_counter(), use_graph=1)
    x2, h2 = S._device_solve(A, b, None, None, cfg, "bicgstab", time.perf_counter(), use_graph=0)
    assert h1.resid == h2.resid and np.array_equal(x1, x2)
    # second graph launch (cached graph) reproduces the first
    x3, h3 = S._device_solve(A, b, None, None, cfg, "bicgstab", time.perf_counter(), use_graph=1)
    assert h3.resid == h1.resid and np.array_equal(x3, x1)
    # persistent cooperative kernel (default driver)
    x4, h4 = S._device_solve(A, b, None, None, cfg, "bicgstab", time.perf_counter(), use_graph=2)
    assert h4.resid == h1.resid and np.array_equal(x4, x1)


@pytest.mark.parametrize("cfg,k", [("c1", 10), ("c2", 20), ("c4", 30), ("c5", 30)])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_drivers_bitwise_with_space(pkg, canon, cfg, k, mode):
    """Host loop, CUDA graph and persistent kernel: identical to the oracle,
    including half-step exits and breakdown paths exercised by max_itn."""
    import time
    from oracle import krylov as O
    from paper_1406_2831_b200 import solvers as S
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence(cfg, small=True)
    A = seq.matrix(2)
    Sp = random_space_arrays(A, k, seed=9, ops=canon)
    b = seq.rhs(2, 0)
    for max_itn in (7, 400):
        cfgp = pkg.SolverConfig(tol=seq.tol, max_itn=max_itn, seed=4)
        xo, ho = O.rbicgstab(A, b, recycle=Sp, config=O.Config(tol=seq.tol, max_itn=max_itn,
                                                               seed=4), ops=canon)
        xg, hg = S._device_solve(pkg.SparseMatrix.from_csr(A), b, None, _space(pkg, Sp), cfgp,
                                 "rbicgstab", time.perf_counter(), use_graph=mode)
        assert hg.status == ho.status and hg.resid == ho.resid
        assert hg.matvecs == ho.matvecs and np.array_equal(xg, xo)


@pytest.mark.parametrize("cfg,k", [("c2", 20), ("c5", 30)])
def test_value_coding_variants_same_bits(pkg, canon, cfg, k):
    """The value-coded SpMV kernels (diagonal form, row templates) and the
    plain offset-coded one inside the graph drivers: RBiCGSTAB and the RBiCG
    generation solve give the same bits under every setting, equal to the
    oracle's."""
    import time
    from oracle import krylov as O
    from paper_1406_2831_b200 import _lib, device as D, solvers as S
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence(cfg, small=True)
    A = seq.matrix(1)
    Sp = random_space_arrays(A, k, seed=4, ops=canon)
    b = seq.rhs(1, 0)
    conf = dict(tol=seq.tol, max_itn=120, seed=2)
    x_o, h_o = O.rbicgstab(A, b, recycle=Sp, config=O.Config(**conf), ops=canon)
    xb_o, xbt_o, hb_o, cyc_o = O.rbicg(A, b, b[::-1].copy(), config=O.Config(s=6, **conf),
                                       ops=canon)
    for vc in (1, 2, 0):
        with _lib.tuning(value_coding=vc):
            M = pkg.SparseMatrix.from_csr(A)
            dm = D.device_matrix(M)
            assert dm.format == ("sell32-dict-vc" if vc else "sell32-dict")
            if vc:
                assert dm.stream_stats["diagonal_form"] == (vc == 1)
            x, h = S._device_solve(M, b, None, _space(pkg, Sp), pkg.SolverConfig(**conf),
                                   "rbicgstab", time.perf_counter(), use_graph=1)
            assert h.resid == h_o.resid and h.status == h_o.status
            assert np.array_equal(x, x_o)
            with _lib.tuning(graph_mode=1):
                xb, xbt, hb, cyc = pkg.rbicg_solve(M, b, b[::-1].copy(),
                                                   config=pkg.SolverConfig(s=6, **conf))
            assert hb.resid == hb_o.resid and np.array_equal(xb, xb_o)
            assert np.array_equal(xbt, xbt_o) and len(cyc) == len(cyc_o)


def test_graph_cache_not_reused_for_other_constants(pkg, canon):
    """The value-coded diagonal table travels BY VALUE in the captured
    graph's kernel parameters: a later matrix with the same pattern and sizes
    but other constants -- possibly at the very addresses of the freed arrays
    of the first -- must get its own graph (each solve equals the oracle)."""
    import gc
    import time
    from oracle import krylov as O
    from paper_1406_2831_b200 import device as D, solvers as S
    from paper_1406_2831_b200.workloads import CSR, make_sequence
    seq = make_sequence("c5", small=True)
    A1 = seq.matrix(1)
    b = seq.rhs(1, 0)
    conf = dict(tol=seq.tol, max_itn=60, seed=3)
    mats = [A1, CSR(A1.n, A1.row_ptr, A1.col_idx, A1.values * 1.5),
            CSR(A1.n, A1.row_ptr, A1.col_idx, A1.values * 0.75), A1]
    for A in mats:
        x_o, h_o = O.bicgstab(A, b, config=O.Config(**conf), ops=canon)
        M = pkg.SparseMatrix.from_csr(A)
        assert D.device_matrix(M).stream_stats.get("diagonal_form")
        x, h = S._device_solve(M, b, None, None, pkg.SolverConfig(**conf), "bicgstab",
                               time.perf_counter(), use_graph=1)
        assert h.resid == h_o.resid and np.array_equal(x, x_o)
        del M
        D.MATRICES.clear()
        gc.collect()
