"""Full-size parity fixtures: the REFERENCE itself (krecycle from
/root/reference/pkg/src) run on the BASELINE configs C1 and C2 at their full
sizes, at every OpenBLAS thread count in THREADS -- each one a valid
configuration of the reference, whose results differ in the last bits of
every BLAS reduction.  Runs in the build container only;
the small summary arrays go to tests/golden/reference_full.npz (committed).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_full.py [group ...]

Cases (every solver case stores, per thread count: the first 51 relative
residuals, iterations, matvecs, status, final true residual):

* bicgstab/c1/j, rbicgstab/c1/j   -- all 6 C1 systems; rbicgstab with the k =
  10 space biorthonormalize(U, U, A_j), U = the k lowest grid sine modes;
  besides the thread counts, two more valid runs of the reference with its
  dots in other summation orders (vexact: exactly rounded; vpair: numpy's
  pairwise sum) -- what another BLAS would give;
* bicgstab/c2/j, rbicgstab/c2/j   -- C2 systems 0, 5, 9, k = 20;
* policy/c1first, policy/c2first  -- the sequence policy (sequence.py,
  policy "first") over the reference's own functions: RBiCG + harvest on
  system 0, refresh + guarded RBiCGSTAB after (the round-1 C2 bench step);
* driver/c1, driver/c2s           -- the reference's OWN driver.run_sequence
  with the ILUTP split preconditioner replaced by the identity (verbatim
  policy: RBiCG + harvest at every matrix change);
* ilutp/c1s, ilutp/c1             -- the reference's driver.run_sequence as
  shipped: ILUTP split preconditioning, verbatim policy (C1-small, full C1).

The matrices are identified by a sha256 of their CSR arrays, so the GPU
tests (which regenerate them with paper_1406_2831_b200.workloads on the
box) first prove they solve the same systems.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time
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
THREADS = (1, 2, 3, 4, 6, 8, 16)
OUT = os.path.join(HERE, "reference_full.npz")
SPACE_SEED = 777


def csr_hash(csr) -> str:
    h = hashlib.sha256()
    for a in (csr.row_ptr, csr.col_idx, csr.values):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def vec_hash(v) -> str:
    return hashlib.sha256(np.ascontiguousarray(v, dtype=np.float64).tobytes()).hexdigest()


def ref_matrix(csr):
    return K.SparseMatrix(csr.n, csr.n, csr.row_ptr, csr.col_idx, csr.values)


def put_hist(out, p, h):
    out[p + "resid51"] = np.asarray(h.resid[:51])
    out[p + "iters"] = np.array(h.iterations)
    out[p + "matvecs"] = np.array(h.total_matvecs)
    out[p + "status"] = np.array(h.status)
    out[p + "final_true_resid"] = np.array(h.final_true_resid)


def space_basis(seq):
    """The recycle basis of the rbicgstab cases: the k lowest sine modes of
    the grid (workloads.sine_basis), U = Ut -- well conditioned, so the
    reference's own runs agree where the iteration itself is stable."""
    grid = seq.meta["grid"]
    return W.sine_basis(tuple(grid), seq.k)


def _numpy_with_dot(dotf):
    import types
    ns = types.SimpleNamespace(**{k: getattr(np, k) for k in dir(np)
                                  if not k.startswith("__")})
    ns.vdot = dotf
    ns.linalg = types.SimpleNamespace(norm=lambda x: np.sqrt(dotf(x, x)))
    return ns


def _exact_dot(a, b):
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


# the reference's solvers with other valid summation orders for their dots
# (what another BLAS would do): exactly rounded, and numpy's pairwise sum
VARIANTS = {"vexact": _exact_dot,
            "vpair": lambda a, b: np.float64(np.sum(np.asarray(a) * np.asarray(b))),
            "vrev": lambda a, b: np.float64(np.dot(np.asarray(a)[::-1], np.asarray(b)[::-1])),
            "vblk": lambda a, b: np.float64(sum(np.dot(np.asarray(a)[i:i + 97],
                                                       np.asarray(b)[i:i + 97])
                                                for i in range(0, len(a), 97)))}


def _blocked_dot(B):
    """Partial sums over consecutive blocks of B elements, added in order:
    the order a BLAS splitting the vector over n / B threads (or cache
    blocks) gives -- the thread-count family generalised to any split."""
    def dot(a, b):
        a = np.asarray(a, dtype=np.float64).ravel()
        b = np.asarray(b, dtype=np.float64).ravel()
        m = len(a) // B
        head = np.einsum("ij,ij->i", a[:m * B].reshape(m, B), b[:m * B].reshape(m, B))
        tail = np.dot(a[m * B:], b[m * B:])
        return np.float64((np.cumsum(head)[-1] if m else 0.0) + tail)
    return dot


def random_block_variants(n, count=16, seed=2024):
    """count block sizes log-uniform in [64, n / 2] (seeded)."""
    r = np.random.default_rng(seed)
    Bs = np.unique(np.exp(r.uniform(np.log(64), np.log(n / 2), count)).astype(int))
    return {f"vb{int(B)}": _blocked_dot(int(B)) for B in Bs}


def solver_cases(out, name, systems, only_random=False):
    seq = W.make_sequence(name)
    for j in systems:
        A = seq.matrix(j)
        b = seq.rhs(j, 0)
        RA = ref_matrix(A)
        U = space_basis(seq)
        out[f"mat/{name}/{j}/sha"] = np.array(csr_hash(A))
        out[f"mat/{name}/{j}/b_sha"] = np.array(vec_hash(b))
        cfg = K.SolverConfig(tol=seq.tol, max_itn=seq.max_itn, seed=j)
        import krecycle.solvers as KS
        runs = [(f"t{th}", th, None) for th in THREADS] + \
               [(v, 1, f) for v, f in VARIANTS.items()]
        rb = random_block_variants(A.n)
        out[f"meta/rblock/{name}/{j}"] = np.asarray(list(rb))
        runs = ([] if only_random else runs) + [(v, 1, f) for v, f in rb.items()]
        for tag, th, dotf in runs:
            t0 = time.time()
            if dotf is not None:
                KS.np = _numpy_with_dot(dotf)
            try:
                with threadpool_limits(th):
                    _, h = K.bicgstab_solve(RA, b, config=cfg)
                    put_hist(out, f"bicgstab/{name}/{j}/{tag}/", h)
                    S = K.biorthonormalize(U, U, RA)
                    out[f"rbicgstab/{name}/{j}/{tag}/k"] = np.array(S.k)
                    _, hr = K.rbicgstab_solve(RA, b, recycle=S, config=cfg)
                    put_hist(out, f"rbicgstab/{name}/{j}/{tag}/", hr)
            finally:
                KS.np = np
            print(f"{name} {j} {tag}: bicgstab {h.iterations} {h.status}, rbicgstab "
                  f"{hr.iterations} {hr.status} ({time.time() - t0:.1f}s)", flush=True)


def ref_api():
    import types
    return types.SimpleNamespace(
        SparseMatrix=types.SimpleNamespace(from_csr=ref_matrix),
        CountingOperator=K.CountingOperator, SolverConfig=K.SolverConfig,
        rbicg_solve=K.rbicg_solve, rbicgstab_solve=K.rbicgstab_solve,
        bicgstab_solve=K.bicgstab_solve, update_recycle_space=K.update_recycle_space,
        refresh_images=K.refresh_images)


def put_seq(out, p, rec, space_dims):
    out[p + "space_dims"] = np.asarray(space_dims)
    out[p + "iters"] = np.asarray([h.iterations for h in rec.histories])
    out[p + "matvecs"] = np.asarray([h.total_matvecs for h in rec.histories])
    out[p + "status"] = np.asarray([h.status for h in rec.histories])
    out[p + "aux"] = np.array(rec.aux_matvecs)
    out[p + "resid51_0"] = np.asarray(rec.histories[0].resid[:51])
    out[p + "resid51_1"] = np.asarray(rec.histories[1].resid[:51])


def policy_cases(out, name):
    from paper_1406_2831_b200.sequence import run_sequence
    seq = W.make_sequence(name)
    for j in range(seq.num_matrices):
        out[f"mat/{name}/{j}/sha"] = np.array(csr_hash(seq.matrix(j)))
    import krecycle.solvers as KS
    runs = [(f"t{th}", th, None) for th in THREADS] + \
           [(v, 1, f) for v, f in VARIANTS.items()]
    for tag, th, dotf in runs:
        t0 = time.time()
        if dotf is not None:
            KS.np = _numpy_with_dot(dotf)
        try:
            with threadpool_limits(th):
                res = run_sequence(W.make_sequence(name), policy="first", baseline=False,
                                   api=ref_api())
        finally:
            KS.np = np
        put_seq(out, f"policy/{name}first/{tag}/", res.recycling, res.space_dims)
        print(f"policy {name} {tag}: {[h.iterations for h in res.recycling.histories]} "
              f"dims {res.space_dims} ({time.time() - t0:.1f}s)", flush=True)


class _SeqAdapter:
    """A workloads sequence seen through krecycle's ParametricSequence
    interface (matrix(i) -> SparseMatrix, rhs[i][kappa])."""

    def __init__(self, seq):
        self.seq = seq
        self.num_matrices = seq.num_matrices
        self.rhs_per_matrix = seq.rhs_per_matrix
        self.rhs = [[seq.rhs(i, kap) for kap in range(seq.rhs_per_matrix)]
                    for i in range(seq.num_matrices)]

    def matrix(self, i):
        return ref_matrix(self.seq.matrix(i))


def driver_cases(out, tag, seq, threads=THREADS):
    """The reference's driver.run_sequence itself, preconditioner = identity
    (ilutp_factor / SplitPreconditionedOperator / apply_left patched in the
    driver module only; everything else is the reference's own code)."""
    import krecycle.driver as KD
    saved = (KD.ilutp_factor, KD.SplitPreconditionedOperator, KD.apply_left)
    KD.ilutp_factor = lambda A, **kw: None
    KD.SplitPreconditionedOperator = lambda A, f: A
    KD.apply_left = lambda f, b: np.asarray(b)
    import krecycle.solvers as KS
    runs = [(f"t{th}", th, None) for th in threads] + \
           [(v, 1, f) for v, f in VARIANTS.items()]
    try:
        for rt, th, dotf in runs:
            t0 = time.time()
            if dotf is not None:
                KS.np = _numpy_with_dot(dotf)
            try:
                with threadpool_limits(th):
                    res = KD.run_sequence(_SeqAdapter(seq), tol=seq.tol,
                                          max_itn=seq.max_itn, k=seq.k, s=seq.s, seed=0)
            finally:
                KS.np = np
            put_seq(out, f"driver/{tag}/{rt}/", res.recycling, res.space_dims)
            out[f"driver/{tag}/{rt}/base_iters"] = np.asarray(
                [h.iterations for h in res.baseline.histories])
            out[f"driver/{tag}/{rt}/base_aux"] = np.array(res.baseline.aux_matvecs)
            print(f"driver {tag} {rt}: {[h.iterations for h in res.recycling.histories]} "
                  f"dims {res.space_dims} ({time.time() - t0:.1f}s)", flush=True)
    finally:
        KD.ilutp_factor, KD.SplitPreconditionedOperator, KD.apply_left = saved


def ilutp_driver_cases(out, tag, seq, threads=(1, 2, 4, 8)):
    """The reference's OWN driver.run_sequence, unmodified: ILUTP split
    preconditioning (drop_tol 1e-4, pivot_tol 0.1), verbatim policy."""
    import krecycle.driver as KD
    for th in threads:
        t0 = time.time()
        with threadpool_limits(th):
            res = KD.run_sequence(_SeqAdapter(seq), tol=seq.tol, max_itn=seq.max_itn,
                                  k=seq.k, s=seq.s, seed=0)
        put_seq(out, f"ilutp/{tag}/t{th}/", res.recycling, res.space_dims)
        out[f"ilutp/{tag}/t{th}/base_iters"] = np.asarray(
            [h.iterations for h in res.baseline.histories])
        out[f"ilutp/{tag}/t{th}/base_matvecs"] = np.asarray(
            [h.total_matvecs for h in res.baseline.histories])
        out[f"ilutp/{tag}/t{th}/base_resid51_0"] = np.asarray(
            res.baseline.histories[0].resid[:51])
        print(f"ilutp {tag} t{th}: {[h.iterations for h in res.recycling.histories]} "
              f"base {[h.iterations for h in res.baseline.histories]} dims {res.space_dims} "
              f"({time.time() - t0:.1f}s)", flush=True)


GROUPS = {
    "c1": lambda out: solver_cases(out, "c1", range(6)),
    "c2": lambda out: solver_cases(out, "c2", (0, 5, 9)),
    "c1rb": lambda out: solver_cases(out, "c1", range(6), only_random=True),
    "c2rb": lambda out: solver_cases(out, "c2", (0, 5, 9), only_random=True),
    "policy": lambda out: (policy_cases(out, "c1"), policy_cases(out, "c2")),
    "driver": lambda out: (driver_cases(out, "c1", W.make_sequence("c1")),
                           driver_cases(out, "c2s", W.make_sequence("c2", small=True))),
    "ilutp": lambda out: (ilutp_driver_cases(out, "c1s", W.make_sequence("c1", small=True)),
                          ilutp_driver_cases(out, "c1", W.make_sequence("c1"))),
}


def main():
    groups = sys.argv[1:] or list(GROUPS)
    out = dict(np.load(OUT)) if os.path.exists(OUT) else {}
    for g in groups:
        GROUPS[g](out)
        np.savez_compressed(OUT, **out)     # incremental: a long run keeps its parts
    import scipy
    out["meta/numpy"] = np.array(np.__version__)
    out["meta/scipy"] = np.array(scipy.__version__)
    out["meta/threads"] = np.asarray(THREADS)
    out["meta/variants"] = np.asarray(list(VARIANTS))
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
