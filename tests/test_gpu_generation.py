"""Recycle-space generation on the B200:
rbicg_solve with device Lanczos capture, update_recycle_space,
biorthonormalize / refresh_images, and the sequence policy — bit-identical to
the canonical CPU oracle, and within the reference's noise floor of the
reference's own outputs (golden fixtures)."""

import types

import numpy as np
import pytest

from conftest import golden_csr, gpu, random_space_arrays

pytestmark = gpu

FIELDS = ("U", "Ut", "C", "Ct", "Dc", "Chat", "Ccheck")


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_1406_2831_b200 as P
    return P


def oracle_api(ops):
    """The oracle restatement behind the product's API names (checker)."""
    import paper_1406_2831_b200 as P
    from oracle import krylov as O
    from oracle.ops import CsrOperand
    return types.SimpleNamespace(
        SparseMatrix=types.SimpleNamespace(from_csr=CsrOperand.of),
        CountingOperator=P.CountingOperator,
        SolverConfig=P.SolverConfig,
        rbicg_solve=lambda A, b, **kw: O.rbicg(A, b, ops=ops, **kw),
        rbicgstab_solve=lambda A, b, **kw: O.rbicgstab(A, b, ops=ops, **kw),
        bicgstab_solve=lambda A, b, **kw: O.bicgstab(A, b, ops=ops, **kw),
        update_recycle_space=lambda A, c, p, k, **kw: O.update_recycle_space(
            A, c, p, k, ops=ops, **kw),
        refresh_images=lambda S, A, **kw: O.refresh_images(S, A, ops=ops, **kw),
    )


def _same_space(S_gpu, S_or):
    assert S_gpu.k == S_or.k
    for f in FIELDS:
        a, b = np.asarray(getattr(S_gpu, f)), np.asarray(getattr(S_or, f))
        assert a.shape == b.shape, f
        assert np.array_equal(a, b), f


def validate_space(space, A, tol=1e-10):
    """Every defining identity of a recycle space (reference
    tests/conftest.py:49-78), evaluated with scipy on the host copy."""
    if space.k == 0:
        return
    S = A.to_scipy()
    U, Ut, C, Ct, Dc = space.U, space.Ut, space.C, space.Ct, space.Dc
    k = space.k
    assert np.linalg.norm(S @ U - C) <= tol * max(np.linalg.norm(C), 1.0)
    assert np.linalg.norm(S.T @ Ut - Ct) <= tol * max(np.linalg.norm(Ct), 1.0)
    G = Ct.T @ C
    off = G - np.diag(np.diag(G))
    assert np.linalg.norm(off) <= tol * np.linalg.norm(G)
    assert np.all(np.diag(G) > 0)
    assert np.allclose(np.diag(G), Dc, rtol=tol, atol=tol)
    assert np.allclose(space.Chat, Ct / Dc, rtol=tol, atol=tol)
    assert np.allclose(space.Ccheck, C / Dc, rtol=tol, atol=tol)
    assert np.linalg.norm(space.Chat.T @ C - np.eye(k)) <= tol * k
    assert np.linalg.norm(space.Ccheck.T @ Ct - np.eye(k)) <= tol * k


@pytest.mark.parametrize("cfg,k", [("c1", 10), ("c2", 20), ("c5", 30)])
def test_biorthonormalize_and_refresh_bitwise(P, canon, cfg, k):
    from oracle import krylov as O
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence(cfg, small=True)
    A0, A1 = seq.matrix(0), seq.matrix(1)
    r = np.random.default_rng(k)
    U, Ut = r.standard_normal((A0.n, k)), r.standard_normal((A0.n, k))
    Ag = P.SparseMatrix.from_csr(A0)
    S_g = P.biorthonormalize(U, Ut, Ag)
    S_o = O.biorthonormalize(U, Ut, A0, ops=canon)
    _same_space(S_g, S_o)
    validate_space(S_g, A0)
    R_g = P.refresh_images(S_g, P.SparseMatrix.from_csr(A1))
    R_o = O.refresh_images(S_o, A1, ops=canon)
    _same_space(R_g, R_o)
    validate_space(R_g, A1)


@pytest.mark.parametrize("cfg,k", [("c1", 10), ("c2", 20)])
def test_rbicg_harvest_bitwise_vs_canon_oracle(P, canon, cfg, k):
    from oracle import krylov as O
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence(cfg, small=True)
    A = seq.matrix(0)
    b = seq.rhs(0, 0)
    dims_g, dims_o = [], []
    st_g, st_o = {"s": None}, {"s": None}
    Ag = P.CountingOperator(P.SparseMatrix.from_csr(A))

    def hg(c):
        st_g["s"] = P.update_recycle_space(Ag, [c], st_g["s"], k, res_tol=4.0)
        dims_g.append(st_g["s"].k)

    from oracle.ops import CsrOperand
    Ao = P.CountingOperator(CsrOperand.of(A))

    def ho(c):
        st_o["s"] = O.update_recycle_space(Ao, [c], st_o["s"], k, res_tol=4.0, ops=canon)
        dims_o.append(st_o["s"].k)

    cfg_ = P.SolverConfig(tol=seq.tol, max_itn=600, k=k, s=25, seed=0)
    xg, xtg, hg_, cyc_g = P.rbicg_solve(Ag, b, b_dual=np.ones(A.n), config=cfg_,
                                        cycle_callback=hg)
    xo, xto, ho_, cyc_o = O.rbicg(Ao, b, b_dual=np.ones(A.n), config=cfg_,
                                  cycle_callback=ho, ops=canon)
    assert hg_.status == ho_.status
    assert hg_.resid == ho_.resid
    assert hg_.resid_dual == ho_.resid_dual
    assert hg_.matvecs == ho_.matvecs
    assert np.array_equal(xg, xo) and np.array_equal(xtg, xto)
    assert len(cyc_g) == len(cyc_o)
    for cg, co in zip(cyc_g, cyc_o):
        assert cg.first_index == co.first_index
        assert np.array_equal(cg.V, co.V) and np.array_equal(cg.Vt, co.Vt)
        tri = cg.tri   # lazily built on first access (solvers.py:524-540)
        assert isinstance(tri, np.ndarray) and tri.shape == (3, cg.ncols)
        assert cg.tri is tri and np.isfinite(tri[1, :-1]).all()
    assert dims_g == dims_o
    assert (Ag.n_matvec, Ag.n_rmatvec) == (Ao.n_matvec, Ao.n_rmatvec)
    if st_g["s"] is not None and st_g["s"].k:
        _same_space(st_g["s"], st_o["s"])
        validate_space(st_g["s"], A)


def test_rbicg_with_space_and_default_dual(P, canon):
    """rbicg deflated by an existing space, b_dual drawn on the device from
    the seeded stream (solvers.py:485-486), x_init / x_init_dual paths."""
    from oracle import krylov as O
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence("c2", small=True)
    A = seq.matrix(1)
    S = random_space_arrays(A, 6, seed=3, ops=canon)
    b = seq.rhs(1, 0)
    Sg = P.RecycleSpace(**{f: getattr(S, f) for f in FIELDS})
    cfg = P.SolverConfig(tol=1e-8, max_itn=400, s=10, seed=7)
    r = np.random.default_rng(0)
    x0, xt0 = r.standard_normal(A.n), r.standard_normal(A.n)
    for kw in ({}, {"x_init": x0, "x_init_dual": xt0}):
        xg, xtg, hg, cg = P.rbicg_solve(P.SparseMatrix.from_csr(A), b, recycle=Sg,
                                        config=cfg, **kw)
        xo, xto, ho, co = O.rbicg(A, b, recycle=S, config=cfg, ops=canon, **kw)
        assert hg.status == ho.status
        assert hg.resid == ho.resid and hg.resid_dual == ho.resid_dual
        assert hg.matvecs == ho.matvecs
        assert np.array_equal(xg, xo) and np.array_equal(xtg, xto)
        assert len(cg) == len(co)
        for a, b_ in zip(cg, co):
            assert a.first_index == b_.first_index
            assert np.array_equal(a.V, b_.V) and np.array_equal(a.Vt, b_.Vt)


@pytest.mark.parametrize("tag", ["c1s", "c2s"])
def test_generation_vs_reference_golden(P, golden, tag):
    """The reference's own rbicg + harvest run (golden): histories within the
    noise floor, same cycle count, harvested dimensions and final status."""
    p = f"gen/{tag}/"
    A0 = golden_csr(golden, p + "A0/")
    k = int(golden[p + "k"])
    dims = []
    st = {"s": None}
    op = P.CountingOperator(P.SparseMatrix.from_csr(A0))

    def harvest(c):
        st["s"] = P.update_recycle_space(op, [c], st["s"], k, res_tol=4.0)
        dims.append(st["s"].k)

    _, _, h, cycles = P.rbicg_solve(op, golden[p + "b0"], b_dual=np.ones(A0.n),
                                    config=P.SolverConfig(tol=1e-8, max_itn=600, k=k,
                                                          s=25, seed=0),
                                    cycle_callback=harvest)
    ref = golden[p + "rbicg_resid"]
    L = min(len(ref), len(h.resid), 51)
    rel = np.max(np.abs(np.asarray(h.resid[:L]) - ref[:L]) / ref[:L])
    floor = float(np.max(golden[p + "rbicg_variant_reldiff"]))
    assert rel <= max(1e-8, 2 * floor), (rel, floor)
    statuses = {str(golden[p + "rbicg_status"])} | set(map(str, golden[p + "rbicg_variant_status"]))
    assert h.status in statuses, (h.status, statuses)
    its = np.append(golden[p + "rbicg_variant_iters"], len(ref) - 1)
    slack = max(2, 0.02 * its.max(), 0.5 * (its.max() - its.min()))
    assert its.min() - slack <= h.iterations <= its.max() + slack


@pytest.mark.parametrize("cfg,policy", [("c1", "first"), ("c3", "verbatim")])
def test_sequence_policy_matches_oracle(P, canon, cfg, policy):
    """The whole sequence policy on the device equals the same policy driven
    over the canonical oracle: every history, space dimension, aux count."""
    from paper_1406_2831_b200.sequence import run_sequence
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence(cfg, small=True)
    r_g = run_sequence(seq, policy=policy, systems=4)
    r_o = run_sequence(make_sequence(cfg, small=True), policy=policy, systems=4,
                       api=oracle_api(canon))
    assert r_g.space_dims == r_o.space_dims
    for hg, ho in zip(r_g.recycling.histories, r_o.recycling.histories):
        assert hg.status == ho.status
        assert hg.resid == ho.resid
        assert hg.matvecs == ho.matvecs
    assert r_g.recycling.aux_matvecs == r_o.recycling.aux_matvecs
    assert r_g.baseline.total_matvecs == r_o.baseline.total_matvecs
    assert abs(r_g.savings - r_o.savings) < 1e-12


@pytest.mark.parametrize("cfg,k", [("c1", 6), ("c2", 6), ("c2", 0), ("c4", 0)])
def test_rbicg_drivers_bitwise(P, canon, cfg, k, monkeypatch):
    """persistent kernel (per cycle; k = 0 takes the fused P+M+Q phase),
    CUDA graph and host loop give the same bits: histories, cycles (ring
    columns) and solutions."""
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence(cfg, small=True)
    A = seq.matrix(1)
    Sg = None
    if k:
        S = random_space_arrays(A, k, seed=3, ops=canon)
        Sg = P.RecycleSpace(**{f: getattr(S, f) for f in FIELDS})
    b = seq.rhs(1, 0)
    cfg_ = P.SolverConfig(tol=1e-9, max_itn=300, s=10, seed=5)
    out = {}
    from paper_1406_2831_b200 import _lib
    for mode in ("2", "1", "0"):
        with _lib.tuning(graph_mode=int(mode)):
            out[mode] = P.rbicg_solve(P.SparseMatrix.from_csr(A), b, b_dual=np.ones(A.n),
                                      recycle=Sg, config=cfg_)
    ref = out["2"]
    assert len(ref[3]) >= 2
    for mode in ("1", "0"):
        x, xt, h, cyc = out[mode]
        assert h.resid == ref[2].resid and h.resid_dual == ref[2].resid_dual
        assert h.matvecs == ref[2].matvecs and h.status == ref[2].status
        assert np.array_equal(x, ref[0]) and np.array_equal(xt, ref[1])
        assert len(cyc) == len(ref[3])
        for c1, c2 in zip(cyc, ref[3]):
            assert c1.first_index == c2.first_index
            assert np.array_equal(c1.V, c2.V) and np.array_equal(c1.Vt, c2.Vt)


@pytest.mark.parametrize("near", [0, 1, 3, 40])
def test_near_null_eligibility_subset_bitwise(P, canon, near):
    """The device eigen-residual filter computes only the near-null columns;
    the decision must equal the oracle's full computation (recycling.py:348-358)
    whether none, some or all of the Ritz values are near-null, with complex
    pairs and a non-finite value among them."""
    import torch
    from oracle import krylov as O
    from paper_1406_2831_b200 import update as UP
    rs = np.random.default_rng(7 + near)
    n, m = 5000, 47
    W = rs.standard_normal((n, m))
    AW = rs.standard_normal((n, m))
    VR = rs.standard_normal((m, m)) + 1j * rs.standard_normal((m, m))
    theta = (rs.uniform(1.0, 2.0, m) + 1j * rs.uniform(-1.0, 1.0, m)).astype(np.complex128)
    theta[rs.permutation(m)[:near]] *= 1e-5          # near-null
    theta[0] = np.inf
    Wd = torch.as_tensor(np.ascontiguousarray(W.T), device="cuda")
    AWd = torch.as_tensor(np.ascontiguousarray(AW.T), device="cuda")
    for res_tol in (0.0, 4.0, 1e9):
        got = UP.near_null_eligibility(theta, VR, Wd, AWd, res_tol)
        want = O.near_null_eligibility(theta, VR, W, AW, res_tol, canon)
        assert np.array_equal(got, want), (near, res_tol)


def test_sequence_with_pinned_inputs_prefetches_and_matches(P):
    """Page-locked host matrices are uploaded one system ahead on a side copy
    stream (device.prefetch_matrix); the results equal the pageable run's."""
    from paper_1406_2831_b200 import device as D
    from paper_1406_2831_b200.sequence import run_sequence
    from paper_1406_2831_b200.workloads import CSR, SequenceSpec, make_sequence
    seq = make_sequence("c2", small=True)
    nm = seq.num_matrices
    mats = {i: seq.matrix(i) for i in range(nm)}
    pm = {i: CSR(A.n, D.pinned_copy(A.row_ptr), D.pinned_copy(A.col_idx),
                 D.pinned_copy(A.values)) for i, A in mats.items()}
    pseq = SequenceSpec(seq.name, seq.n, seq.k, seq.tol, nm, seq.rhs_per_matrix,
                        lambda i: pm[i], seq.rhs, s=seq.s, max_itn=seq.max_itn,
                        meta=seq.meta)
    issued = []
    orig = D.PREFETCH.issue
    D.PREFETCH.issue = lambda A: issued.append(orig(A)) or issued[-1]
    try:
        r_p = run_sequence(pseq, baseline=False)
    finally:
        D.PREFETCH.issue = orig
    assert issued and all(issued), issued
    assert not D.PREFETCH.items
    r_g = run_sequence(seq, baseline=False)
    assert len(r_p.recycling.histories) == len(r_g.recycling.histories) == nm
    for hp, hg in zip(r_p.recycling.histories, r_g.recycling.histories):
        assert hp.status == hg.status and hp.resid == hg.resid and hp.matvecs == hg.matvecs


def test_rbicg_deferred_cycle_launch_paths(P, canon):
    """The next harvest cycle is launched when the callback starts host work
    (device.flush_pending), right after a callback that never flushes, or
    immediately without a callback: the solve is the same in every case; a
    callback that raises drops the deferred launch and the next solve runs."""
    from paper_1406_2831_b200 import device as D
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence("c2", small=True)
    A, b = seq.matrix(0), seq.rhs(0, 0)
    cfg = P.SolverConfig(tol=seq.tol, max_itn=600, k=8, s=25, seed=0)
    ones = np.ones(A.n)

    def run(cb):
        return P.rbicg_solve(P.SparseMatrix.from_csr(A), b, b_dual=ones, config=cfg,
                             cycle_callback=cb)

    seen = []
    ref = run(None)
    flushed = run(lambda c: (D.flush_pending(), seen.append(c.first_index)))
    plain = run(lambda c: seen.append(-c.first_index))
    for out in (flushed, plain):
        assert out[2].resid == ref[2].resid and out[2].matvecs == ref[2].matvecs
        assert np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1])
        assert [c.first_index for c in out[3]] == [c.first_index for c in ref[3]]
        for c1, c2 in zip(out[3], ref[3]):
            assert np.array_equal(c1.V, c2.V)
    assert len(ref[3]) > 1 and len(seen) == 2 * len(ref[3])

    class Boom(Exception):
        pass

    def bad(c):
        raise Boom()

    with pytest.raises(Boom):
        run(bad)
    assert not D._PENDING
    again = run(None)
    assert again[2].resid == ref[2].resid


def test_pageable_int64_prefetch_background_matches(P):
    """Plain pageable numpy inputs with int64 column indices (the reference
    SparseMatrix's dtype): prefetch_matrix stages them on a background
    thread (int64 -> int32 inside the staging copy); the solve equals the
    one that uploads on first use, bit for bit."""
    import numpy as np
    from paper_1406_2831_b200 import device as D
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence("c2", small=True)
    A = seq.matrix(1)
    b = seq.rhs(1, 0)
    ci64 = A.col_idx.astype(np.int64)
    # the cast staging itself, across several pipeline chunks
    big = np.random.default_rng(0).integers(0, 2**31 - 1, size=3_000_001, dtype=np.int64)
    got = D.to_device(big, np.int32).cpu().numpy()
    assert got.dtype == np.int32 and np.array_equal(got, big.astype(np.int32))
    cfg = P.SolverConfig(tol=1e-10, max_itn=500, seed=3)
    M1 = P.SparseMatrix(A.n, A.n, A.row_ptr, ci64, A.values)
    x1, h1 = P.bicgstab_solve(M1, b, config=cfg)
    M2 = P.SparseMatrix(A.n, A.n, A.row_ptr.copy(), ci64.copy(), A.values.copy())
    assert D.prefetch_matrix(M2)
    x2, h2 = P.bicgstab_solve(M2, b, config=cfg)
    assert not D.PREFETCH.items
    assert h1.resid == h2.resid and np.array_equal(x1, x2)
