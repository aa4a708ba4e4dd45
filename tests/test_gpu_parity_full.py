"""GPU vs the REFERENCE at full BASELINE sizes (C1: all 6 systems; C2:
systems 0, 5, 9), against tests/golden/reference_full.npz, which
tests/golden/make_golden_full.py wrote by running krecycle itself at every
OpenBLAS thread count in (1, 2, 4, 8, 16).

The reference is not reproducible below its own rounding noise: each thread
count is a valid run of it and they differ (e.g. C1
system 0 BiCGSTAB: 207..230 iterations).  The bar, per system, with NO
multiplier on the reference's own spread:

* residual history, first 50 iterations:  max_i |h_gpu - h_ref1| / h_ref1
  <= max(1e-8, S) where S = the largest such difference between any two of
  the reference's own runs -- its thread counts plus two runs with its dots
  in other valid summation orders (exactly rounded; pairwise), i.e. what
  another BLAS would give (the north-star 1e-8 wherever the reference is
  reproducible to that level, else its own spread);
* matvecs within [min_ref - 2 %, max_ref + 2 %] of the reference runs;
* the same final status class, and final true residual <= tol when
  converged.

The measured deviation is printed for every case (pytest -s shows it).
The bitwise equality GPU == CanonOps oracle at these sizes is asserted too.
"""

import hashlib
import os

import numpy as np
import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu

FULL = os.path.join(REPO, "tests", "golden", "reference_full.npz")


@pytest.fixture(scope="module")
def G():
    if not os.path.exists(FULL):
        pytest.skip("reference_full.npz not generated")
    return np.load(FULL, allow_pickle=False)


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1406_2831_b200 as P
    return P


def csr_hash(csr):
    h = hashlib.sha256()
    for a in (csr.row_ptr, csr.col_idx, csr.values):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def threads(G):
    return [int(t) for t in G["meta/threads"]] if "meta/threads" in G else [1, 2, 4, 8, 16]


def run_tags(G, prefix):
    """Every stored valid run of the reference for a case: its BLAS thread
    counts, the alternative dot orders (make_golden_full.py VARIANTS) and the
    seeded random block splits (random_block_variants: the thread-count
    family generalised to any split of the vectors)."""
    tags = [f"t{t}" for t in threads(G)]
    if "meta/variants" in G:
        tags += [str(v) for v in G["meta/variants"]]
    parts = prefix.split("/")
    if len(parts) >= 3 and f"meta/rblock/{parts[1]}/{parts[2]}" in G:
        tags += [str(v) for v in G[f"meta/rblock/{parts[1]}/{parts[2]}"]]
    return [tg for tg in tags if f"{prefix}/{tg}/resid51" in G]


def reldiff(a, b, m=51):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    L = min(len(a), len(b), m)
    return float(np.max(np.abs(a[:L] - b[:L]) / b[:L])) if L else 0.0


def spread(runs, m=51):
    ts = list(runs)
    S = 0.0
    for i, a in enumerate(ts):
        for b in ts[i + 1:]:
            S = max(S, reldiff(runs[a], runs[b], m), reldiff(runs[b], runs[a], m))
    return S


# Beyond this relative spread the reference's own valid runs are
# decorrelated: a history comparison there measures chaos, not parity.
CHAOS = 1e-2


def envelope(G, prefix):
    """The reference's own spread over its valid runs (thread counts,
    alternative dot orders, random block splits): the largest pairwise
    history difference over the first 50 iterations; the window m* <= 51
    over which the runs stay correlated (spread < CHAOS) and the spread
    there."""
    runs = {tg: G[f"{prefix}/{tg}/resid51"] for tg in run_tags(G, prefix)}
    S = spread(runs)
    m = 51
    while m > 1 and spread(runs, m) >= CHAOS:
        m -= 1
    mv = [int(G[f"{prefix}/{t}/matvecs"]) for t in runs]
    st = {str(G[f"{prefix}/{t}/status"]) for t in runs}
    return runs, S, mv, st, m, spread(runs, m)


def check(h, G, prefix, tol, label):
    runs, S, mv, st, m, Sm = envelope(G, prefix)
    dev = reldiff(h.resid, runs["t1"])
    lo, hi = min(mv) * 0.98, max(mv) * 1.02
    print(f"\n{label}: gpu {h.iterations} its / {h.total_matvecs} mv ({h.status}); "
          f"reference mv {min(mv)}..{max(mv)} over {len(runs)} valid runs; history dev vs "
          f"ref@1 {dev:.2e}, reference spread {S:.2e}")
    if S < CHAOS:
        bar = max(1e-8, S)
        assert dev <= bar, (label, dev, bar)
    else:
        # the reference's runs decorrelate inside the first 50 iterations:
        # the history is compared over the window where they still agree
        devm = reldiff(h.resid, runs["t1"], m)
        bar = max(1e-8, Sm)
        print(f"   chaotic: reference runs agree to {Sm:.2e} over the first {m} entries; "
              f"gpu dev there {devm:.2e}")
        assert devm <= bar, (label, m, devm, bar)
    assert lo <= h.total_matvecs <= hi, (label, h.total_matvecs, mv)
    conv = "converged" in st
    assert (h.status == "converged") == conv or h.status in st, (label, h.status, st)
    if h.status == "converged":
        assert h.final_true_resid <= 1.1 * tol, (label, h.final_true_resid)


CASES = [("c1", j) for j in range(6)] + [("c2", j) for j in (0, 5, 9)]


@pytest.mark.parametrize("name,j", CASES)
def test_full_size_solvers_vs_reference(P, G, canon, name, j):
    from oracle import krylov as O
    from paper_1406_2831_b200.workloads import make_sequence, sine_basis
    if f"mat/{name}/{j}/sha" not in G:
        pytest.skip("case not in the fixture")
    seq = make_sequence(name)
    A = seq.matrix(j)
    b = seq.rhs(j, 0)
    assert csr_hash(A) == str(G[f"mat/{name}/{j}/sha"]), "generator drifted from the golden"
    M = P.SparseMatrix.from_csr(A)
    cfg = P.SolverConfig(tol=seq.tol, max_itn=seq.max_itn, seed=j)
    _, hb = P.bicgstab_solve(M, b, config=cfg)
    check(hb, G, f"bicgstab/{name}/{j}", seq.tol, f"bicgstab {name}/{j}")
    U = sine_basis(tuple(seq.meta["grid"]), seq.k)
    Ut = U
    S = P.biorthonormalize(U, Ut, M)
    assert S.k == int(G[f"rbicgstab/{name}/{j}/t1/k"])
    x, hr = P.rbicgstab_solve(M, b, recycle=S, config=cfg)
    check(hr, G, f"rbicgstab/{name}/{j}", seq.tol, f"rbicgstab {name}/{j} k={S.k}")
    # and the GPU is the canonical oracle bit for bit at this size
    So = O.biorthonormalize(U, Ut, A, ops=canon)
    xo, ho = O.rbicgstab(A, b, recycle=So, ops=canon,
                         config=O.Config(tol=seq.tol, max_itn=seq.max_itn, seed=j))
    assert (hr.status, hr.resid, hr.matvecs) == (ho.status, ho.resid, ho.matvecs)
    assert np.array_equal(x, xo)


def _seq_tags(G, prefix):
    tags = [f"t{t}" for t in threads(G)]
    if "meta/variants" in G:
        tags += [str(v) for v in G["meta/variants"]]
    return [tg for tg in tags if f"{prefix}/{tg}/iters" in G]


def _seq_check(G, prefix, res, label):
    ts = _seq_tags(G, prefix)
    if not ts:
        pytest.skip(f"{prefix} not in the fixture")
    mv = np.array([G[f"{prefix}/{t}/matvecs"] for t in ts])          # (runs, systems)
    dims = [list(G[f"{prefix}/{t}/space_dims"]) for t in ts]
    gm = np.array([h.total_matvecs for h in res.recycling.histories])
    S0 = max(reldiff(G[f"{prefix}/{a}/resid51_0"], G[f"{prefix}/{b}/resid51_0"])
             for a in ts for b in ts if a != b) if len(ts) > 1 else 0.0
    dev0 = reldiff(res.recycling.histories[0].resid, G[f"{prefix}/t1/resid51_0"])
    print(f"\n{label}: gpu matvecs {gm.tolist()} dims {res.space_dims}; reference "
          f"matvecs min {mv.min(0).tolist()} max {mv.max(0).tolist()} dims {dims}; "
          f"system-0 history dev {dev0:.2e} (reference spread {S0:.2e})")
    assert dev0 <= max(1e-8, S0)
    lo, hi = mv.min(0) * 0.98, mv.max(0) * 1.02
    total_lo, total_hi = mv.sum(1).min() * 0.98, mv.sum(1).max() * 1.02
    assert total_lo <= gm.sum() <= total_hi, (gm.sum(), mv.sum(1))
    return gm, lo, hi


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_full_size_policy_vs_reference(P, G, name):
    """The sequence policy ('first': RBiCG + harvest on system 0, refresh +
    guarded RBiCGSTAB after) on the device vs the same policy over the
    reference's own functions: per-sequence matvecs within the reference's
    thread-count envelope +-2 %."""
    from paper_1406_2831_b200.sequence import run_sequence
    from paper_1406_2831_b200.workloads import make_sequence
    res = run_sequence(make_sequence(name), policy="first", baseline=False, api=P)
    _seq_check(G, f"policy/{name}first", res, f"policy {name}")


def test_verbatim_policy_vs_reference_driver(P, G):
    """Our 'verbatim' schedule vs krecycle's own driver.run_sequence (ILUTP
    replaced by the identity) on full C1: RBiCG + harvest at every matrix
    change, and the baseline track."""
    from paper_1406_2831_b200.sequence import run_sequence
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence("c1")
    res = run_sequence(seq, policy="verbatim", baseline=True, api=P)
    _seq_check(G, "driver/c1", res, "driver c1")
    ts = [t for t in _seq_tags(G, "driver/c1") if f"driver/c1/{t}/base_iters" in G]
    bi = np.array([G[f"driver/c1/{t}/base_iters"] for t in ts])
    gb = np.array([h.iterations for h in res.baseline.histories])
    assert bi.sum(1).min() * 0.98 <= gb.sum() <= bi.sum(1).max() * 1.02, (gb, bi)
