"""Generate golden fixtures by running the REFERENCE itself (krecycle from
/root/reference/pkg/src) on seeded inputs.  Runs in the build container only
(the reference does not exist on the GPU box); the .npz outputs are committed.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

All reference runs use OPENBLAS_NUM_THREADS=1 (threadpoolctl) so they are
bit-reproducible; the 8-thread rerun of each solver case is stored beside it
as the reference's own noise floor.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from threadpoolctl import threadpool_limits  # noqa: E402

import krecycle as K  # noqa: E402
from paper_1406_2831_b200 import workloads as W  # noqa: E402

warnings.simplefilter("ignore")


def ref_matrix(csr):
    return K.SparseMatrix(csr.n, csr.n, csr.row_ptr, csr.col_idx, csr.values)


def csr_arrays(prefix, csr, out):
    out[prefix + "row_ptr"] = csr.row_ptr
    out[prefix + "col_idx"] = csr.col_idx
    out[prefix + "values"] = csr.values


def hist_arrays(prefix, h, out):
    out[prefix + "resid"] = np.asarray(h.resid)
    out[prefix + "matvecs"] = np.asarray(h.matvecs)
    out[prefix + "status"] = np.array(h.status)
    out[prefix + "final_true_resid"] = np.array(h.final_true_resid)
    out[prefix + "rhs_norm"] = np.array(h.rhs_norm)
    if h.resid_dual:
        out[prefix + "resid_dual"] = np.asarray(h.resid_dual)


def space_arrays(prefix, s, out):
    for f in ("U", "Ut", "C", "Ct", "Dc", "Chat", "Ccheck"):
        out[prefix + f] = np.asarray(getattr(s, f))


def random_sparse(rng, n, per_row=4, dominance=2.0):
    """tests/conftest.py:30-46 pattern (sparse random, dominant diagonal)."""
    rows, cols, vals = [], [], []
    for i in range(n):
        js = rng.choice(n, size=min(per_row, n), replace=False)
        for j in js:
            if j == i:
                continue
            rows.append(i)
            cols.append(int(j))
            vals.append(rng.standard_normal())
        rows.append(i)
        cols.append(i)
        vals.append(dominance * per_row * (1.0 + rng.uniform()))
    A = K.SparseMatrix.from_triplets(n, n, np.array(rows), np.array(cols),
                                     np.array(vals))
    return W.CSR(n, A.row_ptr.astype(np.int64), A.col_idx.astype(np.int32),
                 np.asarray(A.values)), rng.standard_normal(n)


def case_spmv(out):
    rng = np.random.default_rng(11)
    mats = {
        "dense40": None,
        "rand200": random_sparse(np.random.default_rng(5), 200)[0],
        "c1s": W.make_sequence("c1", small=True).matrix(0),
        "c4s": W.c4_sequence(n=1500, num=1).matrix(0),
    }
    D = rng.standard_normal((40, 40))
    D[np.abs(D) < 0.3] = 0.0
    rr, cc = np.nonzero(D)
    A = K.SparseMatrix.from_triplets(40, 40, rr, cc, D[rr, cc])
    mats["dense40"] = W.CSR(40, A.row_ptr.astype(np.int64),
                            A.col_idx.astype(np.int32), np.asarray(A.values))
    for name, csr in mats.items():
        RA = ref_matrix(csr)
        x = rng.standard_normal(csr.n) * np.exp(rng.uniform(-8, 8, csr.n))
        csr_arrays(f"spmv/{name}/", csr, out)
        out[f"spmv/{name}/x"] = x
        out[f"spmv/{name}/Ax"] = RA.matvec(x)
        out[f"spmv/{name}/AHx"] = RA.rmatvec(x)


def exact_dot(a, b):
    """Exactly rounded dot: Dekker-split exact products summed by math.fsum."""
    import math
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    f = 134217729.0

    def split(x):
        c = f * x
        hi = c - (c - x)
        return hi, x - hi

    p = a * b
    ah, al = split(a)
    bh, bl = split(b)
    e = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    return np.float64(math.fsum(np.concatenate([p, e])))


def _exact_numpy():
    """numpy namespace whose vdot / linalg.norm are exactly rounded: running
    the reference's solvers with it measures how far a *different but valid*
    summation order moves the histories (the reference's noise floor)."""
    import types
    ns = types.SimpleNamespace(**{k: getattr(np, k) for k in dir(np)
                                  if not k.startswith("__")})
    ns.vdot = exact_dot
    ns.linalg = types.SimpleNamespace(norm=lambda x: np.sqrt(exact_dot(x, x)))
    return ns


def _numpy_with_dot(dotf):
    import types
    ns = types.SimpleNamespace(**{k: getattr(np, k) for k in dir(np)
                                  if not k.startswith("__")})
    ns.vdot = dotf
    ns.linalg = types.SimpleNamespace(norm=lambda x: np.sqrt(dotf(x, x)))
    return ns


_DOT_VARIANTS = (
    exact_dot,                                              # exactly rounded
    lambda a, b: np.float64(np.sum(np.asarray(a) * np.asarray(b))),   # pairwise
    lambda a, b: np.float64(np.dot(np.asarray(a)[::-1], np.asarray(b)[::-1])),
    lambda a, b: np.float64(sum(np.dot(np.asarray(a)[i:i + 97], np.asarray(b)[i:i + 97])
                                for i in range(0, len(a), 97))),   # blocked
)


def _solver_pair(fn):
    """Run at 1 thread (golden), at 8 threads, and with exactly rounded dots
    (the latter two bound the reference's own noise floor)."""
    import krecycle.solvers as KS
    with threadpool_limits(1):
        g = fn()
    with threadpool_limits(8):
        f = fn()
    KS.np = _exact_numpy()
    try:
        with threadpool_limits(1):
            e = fn()
    finally:
        KS.np = np
    return g, f, e


def case_bicgstab(out):
    seq = W.make_sequence("c1", small=True)
    for j in range(seq.num_matrices):
        csr, b = seq.matrix(j), seq.rhs(j, 0)
        RA = ref_matrix(csr)
        cfg = K.SolverConfig(tol=1e-8, max_itn=500, seed=j)
        (x, h), (_, hf), (_, he) = _solver_pair(
            lambda: K.bicgstab_solve(RA, b, config=cfg))
        p = f"bicgstab/c1s{j}/"
        csr_arrays(p, csr, out)
        out[p + "b"] = b
        out[p + "seed"] = np.array(j)
        out[p + "x"] = x
        hist_arrays(p, h, out)
        out[p + "resid_8thr"] = np.asarray(hf.resid)
        out[p + "resid_exactdot"] = np.asarray(he.resid)
        out[p + "resid_variant_reldiff"] = np.asarray(
            _variant_reldiffs(lambda: K.bicgstab_solve(RA, b, config=cfg), h.resid))


def _variant_reldiffs(fn, ref_resid, m=51):
    """Max relative history difference (first m entries) of the reference
    rerun with each alternative dot order of _DOT_VARIANTS."""
    import krecycle.solvers as KS
    out = []
    for dotf in _DOT_VARIANTS:
        KS.np = _numpy_with_dot(dotf)
        try:
            with threadpool_limits(1):
                _, hx = fn()
        finally:
            KS.np = np
        L = min(len(hx.resid), len(ref_resid), m)
        a, r = np.asarray(hx.resid[:L]), np.asarray(ref_resid[:L])
        out.append(float(np.max(np.abs(a - r) / r)))
    return out


def case_rbicgstab(out):
    rng = np.random.default_rng(1234)
    csr, b = random_sparse(rng, 300)
    RA = ref_matrix(csr)
    U = rng.standard_normal((300, 5))
    Ut = rng.standard_normal((300, 5))
    with threadpool_limits(1):
        space = K.biorthonormalize(U, Ut, RA)
    p = "rbicgstab/rand300/"
    csr_arrays(p, csr, out)
    out[p + "b"] = b
    out[p + "U_raw"] = U
    out[p + "Ut_raw"] = Ut
    space_arrays(p + "space/", space, out)
    cfg = K.SolverConfig(tol=1e-10, max_itn=300, seed=3)
    (x, h), (_, hf), (_, he) = _solver_pair(
        lambda: K.rbicgstab_solve(RA, b, recycle=space, config=cfg))
    out[p + "x"] = x
    hist_arrays(p, h, out)
    out[p + "resid_8thr"] = np.asarray(hf.resid)
    out[p + "resid_exactdot"] = np.asarray(he.resid)
    out[p + "resid_variant_reldiff"] = np.asarray(_variant_reldiffs(
        lambda: K.rbicgstab_solve(RA, b, recycle=space, config=cfg), h.resid))
    # x_init path (one counted product)
    x0 = rng.standard_normal(300)
    (x2, h2), _, (_, h2e) = _solver_pair(
        lambda: K.rbicgstab_solve(RA, b, x_init=x0, recycle=space, config=cfg))
    out[p + "xinit"] = x0
    out[p + "xinit_x"] = x2
    hist_arrays(p + "xinit_", h2, out)
    out[p + "xinit_resid_exactdot"] = np.asarray(h2e.resid)


def case_generation(out):
    """rbicg + per-cycle update_recycle_space (driver.py:116-126 harvest),
    refresh_images onto the next matrix, then rbicgstab with the space."""
    for tag, seq, k in (("c1s", W.make_sequence("c1", small=True), 10),
                        ("c2s", W.make_sequence("c2", small=True), 20)):
        A0, A1 = seq.matrix(0), seq.matrix(1)
        RA0, RA1 = ref_matrix(A0), ref_matrix(A1)
        b0, b1 = seq.rhs(0, 0), seq.rhs(1, 0)
        p = f"gen/{tag}/"
        csr_arrays(p + "A0/", A0, out)
        csr_arrays(p + "A1/", A1, out)
        out[p + "b0"] = b0
        out[p + "b1"] = b1
        out[p + "k"] = np.array(k)
        with threadpool_limits(1):
            state = {"space": None, "dims": []}

            def harvest(cyc, _st=state):
                _st["space"] = K.update_recycle_space(RA0, [cyc], _st["space"],
                                                      k, res_tol=4.0)
                _st["dims"].append(_st["space"].k)

            cfg = K.SolverConfig(tol=seq.tol, max_itn=600, k=k, s=25, seed=0)
            _, _, hr, cycles = K.rbicg_solve(RA0, b0, b_dual=np.ones(seq.n),
                                             config=cfg, cycle_callback=harvest)
            hist_arrays(p + "rbicg_", hr, out)
            # the same harvest run with the solvers' dots in other valid
            # orders: the reference's own noise envelope for rbicg
            import krecycle.solvers as KS
            var_diff, var_it, var_st = [], [], []
            for dotf in _DOT_VARIANTS:
                KS.np = _numpy_with_dot(dotf)
                try:
                    sv = {"s": None}

                    def hv(cyc, _sv=sv):
                        _sv["s"] = K.update_recycle_space(RA0, [cyc], _sv["s"], k,
                                                          res_tol=4.0)

                    _, _, hx, _ = K.rbicg_solve(RA0, b0, b_dual=np.ones(seq.n),
                                                config=K.SolverConfig(
                                                    tol=seq.tol, max_itn=600, k=k,
                                                    s=25, seed=0),
                                                cycle_callback=hv)
                finally:
                    KS.np = np
                L = min(len(hx.resid), len(hr.resid), 51)
                var_diff.append(float(np.max(np.abs(np.asarray(hx.resid[:L]) -
                                                    np.asarray(hr.resid[:L])) /
                                             np.asarray(hr.resid[:L]))))
                var_it.append(hx.iterations)
                var_st.append(hx.status)
            out[p + "rbicg_variant_reldiff"] = np.asarray(var_diff)
            out[p + "rbicg_variant_status"] = np.asarray(var_st)
            out[p + "rbicg_variant_iters"] = np.asarray(var_it)
            out[p + "harvest_dims"] = np.asarray(state["dims"])
            out[p + "ncycles"] = np.array(len(cycles))
            if cycles:
                out[p + "cycle0_V"] = cycles[0].V
                out[p + "cycle0_Vt"] = cycles[0].Vt
            # one update from scratch with res_tol = 0 keeps a non-trivial k
            sp0 = K.update_recycle_space(RA0, cycles[:2], None, k)
            space_arrays(p + "upd0/", sp0, out)
            ref = K.refresh_images(sp0, RA1)
            space_arrays(p + "refresh/", ref, out)
            scfg = K.SolverConfig(tol=seq.tol, max_itn=600, seed=1)
            x, h = K.rbicgstab_solve(RA1, b1, recycle=ref, config=scfg)
            out[p + "rbicgstab_x"] = x
            hist_arrays(p + "rbicgstab_", h, out)
            xb, hb = K.bicgstab_solve(RA1, b1, config=scfg)
            hist_arrays(p + "bicgstab_", hb, out)


def case_policy(out):
    """The sequence policy (paper_1406_2831_b200/sequence.py)
    driven over the reference's own functions."""
    import types
    from paper_1406_2831_b200.sequence import run_sequence
    api = types.SimpleNamespace(
        SparseMatrix=types.SimpleNamespace(from_csr=ref_matrix),
        CountingOperator=K.CountingOperator, SolverConfig=K.SolverConfig,
        rbicg_solve=K.rbicg_solve, rbicgstab_solve=K.rbicgstab_solve,
        bicgstab_solve=K.bicgstab_solve,
        update_recycle_space=K.update_recycle_space,
        refresh_images=K.refresh_images)
    for tag, name, policy in (("c1s", "c1", "first"), ("c3s", "c3", "verbatim")):
        with threadpool_limits(1):
            res = run_sequence(W.make_sequence(name, small=True), policy=policy,
                               systems=4, api=api)
        p = f"policy/{tag}/"
        out[p + "space_dims"] = np.asarray(res.space_dims)
        out[p + "rec_aux"] = np.array(res.recycling.aux_matvecs)
        out[p + "base_total"] = np.array(res.baseline.total_matvecs)
        out[p + "rec_total"] = np.array(res.recycling.total_matvecs)
        for j, h in enumerate(res.recycling.histories):
            hist_arrays(p + f"rec{j}_", h, out)
        for j, h in enumerate(res.baseline.histories):
            hist_arrays(p + f"base{j}_", h, out)
        out[p + "rec_mv"] = np.asarray(res.recycling.per_system_matvecs)
        # the same policy with the solvers' dots evaluated in other valid
        # orders: the envelope of the reference's own per-system counts
        import krecycle.solvers as KS
        env = []
        for dotf in _DOT_VARIANTS:
            KS.np = _numpy_with_dot(dotf)
            try:
                with threadpool_limits(1):
                    rx = run_sequence(W.make_sequence(name, small=True),
                                      policy=policy, systems=4, api=api)
            finally:
                KS.np = np
            env.append(rx.recycling.per_system_matvecs)
        out[p + "rec_mv_variants"] = np.asarray(env)


def main():
    out = {}
    case_spmv(out)
    case_bicgstab(out)
    case_rbicgstab(out)
    case_generation(out)
    case_policy(out)
    out["meta/numpy"] = np.array(np.__version__)
    import scipy
    out["meta/scipy"] = np.array(scipy.__version__)
    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
