"""Seeded synthetic sequences for the five BASELINE configurations (C1-C5).

The reference ships no generator for any BASELINE config,
so these are written here, vectorised, and feed the *same* CSR arrays to the
CPU oracle and to the GPU path.  Conventions:

* PDE operators use physical 1/h^2 scaling; convection is second-order central
  (the coefficient template is the reference's ``example1_operator``,
  /root/reference/pkg/src/krecycle/problems.py:50-57, rescaled by 1/h^2).
* "(s E - K)" is realised with K = -L_h, i.e. the system matrix is s*E + L_h
  with L_h the convection-diffusion operator (positive-real spectrum).
* C3: 20 matrices (5 shifts x 4 p-values) x 4 right-hand sides = 80 solves.
* Every CSR is canonical (rows sorted by column, no duplicates), row_ptr int64,
  col_idx int32, values float64.

The public benchmark model of the paper (PMOR membrane, n=60,020) is not
available; C3 stands in for it.  All inputs are synthetic.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np


@dataclass
class CSR:
    """Plain host CSR triple (canonical)."""

    n: int
    row_ptr: np.ndarray   # int64 (n+1)
    col_idx: np.ndarray   # int32 (nnz)
    values: np.ndarray    # float64 (nnz)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values, self.col_idx, self.row_ptr),
                             shape=(self.n, self.n))


# ---------------------------------------------------------------------------
# structured-grid stencils
# ---------------------------------------------------------------------------

def _stencil_csr(dims, offsets, coeffs, diag, chunk_rows=1 << 22) -> CSR:
    """CSR of a constant-coefficient stencil with a per-row diagonal.

    ``dims`` = (mx, my, mz) with x fastest; ``offsets`` = list of (dx,dy,dz)
    (must include (0,0,0) whose coefficient is replaced by ``diag``).
    Columns come out sorted because offsets are visited in increasing linear
    offset order and every valid neighbour has a distinct linear offset.
    """
    mx, my, mz = dims
    n = mx * my * mz
    lin = [dx + mx * (dy + my * dz) for dx, dy, dz in offsets]
    order = np.argsort(lin, kind="stable")
    offsets = [offsets[i] for i in order]
    coeffs = [coeffs[i] for i in order]
    lin = [lin[i] for i in order]
    noff = len(offsets)

    counts = np.zeros(n, dtype=np.int64)
    cols_parts, vals_parts = [], []
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        rows = np.arange(r0, r1, dtype=np.int64)
        x = rows % mx
        y = (rows // mx) % my
        z = rows // (mx * my)
        valid = np.empty((r1 - r0, noff), dtype=bool)
        cols = np.empty((r1 - r0, noff), dtype=np.int32)
        vals = np.empty((r1 - r0, noff), dtype=np.float64)
        for t, (dx, dy, dz) in enumerate(offsets):
            v = np.ones(r1 - r0, dtype=bool)
            if dx:
                v &= (x + dx >= 0) & (x + dx < mx)
            if dy:
                v &= (y + dy >= 0) & (y + dy < my)
            if dz:
                v &= (z + dz >= 0) & (z + dz < mz)
            valid[:, t] = v
            cols[:, t] = (rows + lin[t]).astype(np.int32, copy=False) if n < 2**31 else 0
            if (dx, dy, dz) == (0, 0, 0):
                vals[:, t] = diag[r0:r1]
            else:
                vals[:, t] = coeffs[t]
        counts[r0:r1] = valid.sum(axis=1)
        cols_parts.append(cols[valid])
        vals_parts.append(vals[valid])
        del valid, cols, vals
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    col_idx = np.concatenate(cols_parts) if len(cols_parts) > 1 else cols_parts[0]
    values = np.concatenate(vals_parts) if len(vals_parts) > 1 else vals_parts[0]
    return CSR(n=n, row_ptr=row_ptr, col_idx=np.ascontiguousarray(col_idx),
               values=np.ascontiguousarray(values))


def _cd_offsets_7(h, w):
    """-Lap + w.grad, 1/h^2 scaling, central convection (7-point)."""
    wx, wy, wz = w
    d = 1.0 / (h * h)
    offs = [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0),
            (0, 0, -1), (0, 0, 1)]
    co = [6.0 * d,
          -d - wx / (2 * h), -d + wx / (2 * h),
          -d - wy / (2 * h), -d + wy / (2 * h),
          -d - wz / (2 * h), -d + wz / (2 * h)]
    return offs, co


def _cd_offsets_27(h, w):
    """27-point diffusion (26 u_c - sum of the 26 neighbours)/(9 h^2), which is
    consistent with -Lap, plus central convection on the six faces."""
    wx, wy, wz = w
    d = 1.0 / (9.0 * h * h)
    offs, co = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                offs.append((dx, dy, dz))
                if (dx, dy, dz) == (0, 0, 0):
                    co.append(26.0 * d)
                    continue
                c = -d
                if dy == 0 and dz == 0:
                    c += dx * wx / (2 * h)
                elif dx == 0 and dz == 0:
                    c += dy * wy / (2 * h)
                elif dx == 0 and dy == 0:
                    c += dz * wz / (2 * h)
                co.append(c)
    return offs, co


# ---------------------------------------------------------------------------
# sequence container
# ---------------------------------------------------------------------------

@dataclass
class SequenceSpec:
    """A sequence of systems A_i x = b_{i,kappa} (solved strictly in order)."""

    name: str
    n: int
    k: int
    tol: float
    num_matrices: int
    rhs_per_matrix: int
    matrix_fn: Callable[[int], CSR]
    rhs_fn: Callable[[int, int], np.ndarray]
    s: int = 25
    max_itn: int = 1000
    meta: dict = field(default_factory=dict)
    _cache: dict = field(default_factory=dict, repr=False)

    def matrix(self, i: int) -> CSR:
        if i not in self._cache:
            if len(self._cache) >= 2:
                self._cache.pop(next(iter(self._cache)))
            self._cache[i] = self.matrix_fn(i)
        return self._cache[i]

    def rhs(self, i: int, kappa: int = 0) -> np.ndarray:
        return self.rhs_fn(i, kappa)

    @property
    def num_systems(self) -> int:
        return self.num_matrices * self.rhs_per_matrix


def _normal(seed, n):
    return np.random.default_rng(seed).standard_normal(n)


def c1_sequence(m: int = 128, num: int = 6) -> SequenceSpec:
    """C1: 2D 5-point -Lap u + 20 u_x + 10 u_y on an m x m interior grid;
    A_j = A0 + 0.1 j I; b_j ~ N(0,1) from seed j, unit norm; k=10, tol 1e-8."""
    h = 1.0 / (m + 1)
    d = 1.0 / (h * h)
    offs = [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0)]
    co = [4 * d, -d - 20 / (2 * h), -d + 20 / (2 * h), -d - 10 / (2 * h),
          -d + 10 / (2 * h)]
    n = m * m
    base = np.full(n, 4 * d)

    def mat(j):
        return _stencil_csr((m, m, 1), offs, co, base + 0.1 * j)

    def rhs(j, kappa):
        b = _normal(j, n)
        return b / np.linalg.norm(b)

    return SequenceSpec("c1", n, 10, 1e-8, num, 1, mat, rhs,
                        meta={"grid": (m, m), "stencil": 5})


def c2_sequence(m: int = 64, num: int = 10) -> SequenceSpec:
    """C2: 3D 7-point m^3, convection (30,20,10); (s_j E + L_h) with E = diag
    U[1,2] (seed 0), s_j = logspace(-2, 0, num); b fixed (seed 0) for the first
    5 systems then N(0,1) from seed j; k=20, tol 1e-8."""
    h = 1.0 / (m + 1)
    offs, co = _cd_offsets_7(h, (30.0, 20.0, 10.0))
    n = m ** 3
    E = np.random.default_rng(0).uniform(1.0, 2.0, n)
    shifts = np.logspace(-2, 0, num)

    def mat(j):
        return _stencil_csr((m, m, m), offs, co, shifts[j] * E + co[0])

    def rhs(j, kappa):
        return _normal(0 if j < 5 else j, n)

    return SequenceSpec("c2", n, 20, 1e-8, num, 1, mat, rhs,
                        meta={"grid": (m, m, m), "stencil": 7,
                              "shifts": shifts.tolist()})


def c3_sequence(m: int = 128, n_s: int = 5, n_p: int = 4, nrhs: int = 4,
                k1_per_row: int = 4) -> SequenceSpec:
    """C3: (s E + L_h - p K1) B e_i on m^3 (7-point, convection (30,20,10)),
    K1 random with 4 off-diagonal entries per row (uniform columns, N(0,0.05)),
    s in logspace(-2,0,5) x p in linspace(0,0.5,4) -> 20 matrices x 4 rhs."""
    import scipy.sparse as sp
    h = 1.0 / (m + 1)
    offs, co = _cd_offsets_7(h, (30.0, 20.0, 10.0))
    n = m ** 3
    E = np.random.default_rng(0).uniform(1.0, 2.0, n)
    rng = np.random.default_rng(1)
    rows = np.repeat(np.arange(n, dtype=np.int64), k1_per_row)
    cols = rng.integers(0, n - 1, size=n * k1_per_row)
    cols = cols + (cols >= rows)               # never the diagonal
    vals = rng.normal(0.0, 0.05, size=n * k1_per_row)
    K1 = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    K1.sum_duplicates()
    K1.sort_indices()
    L = _stencil_csr((m, m, m), offs, co, np.full(n, co[0])).to_scipy()
    svals = np.logspace(-2, 0, n_s)
    pvals = np.linspace(0.0, 0.5, n_p)
    grid = [(s, p) for s in svals for p in pvals]
    B = np.random.default_rng(2).standard_normal((nrhs, n))

    def mat(j):
        s, p = grid[j]
        A = (sp.diags(s * E) + L - p * K1).tocsr()
        A.sum_duplicates()
        A.sort_indices()
        return CSR(n, A.indptr.astype(np.int64), A.indices.astype(np.int32),
                   A.data.astype(np.float64))

    def rhs(j, kappa):
        return B[kappa].copy()

    return SequenceSpec("c3", n, 20, 1e-10, len(grid), nrhs, mat, rhs,
                        meta={"grid": (m, m, m), "stencil": "7+K1",
                              "pairs": grid})


def _power_law_lengths(rng, n, lo=3, hi=200, mean=27.0):
    """Truncated discrete power law P(L) ~ L^-a on [lo, hi], a fitted so the
    mean row length is ``mean``."""
    L = np.arange(lo, hi + 1, dtype=np.float64)

    def mean_of(a):
        w = L ** (-a)
        return float((w * L).sum() / w.sum())

    a_lo, a_hi = 0.0, 4.0
    for _ in range(80):
        a = 0.5 * (a_lo + a_hi)
        if mean_of(a) > mean:
            a_lo = a
        else:
            a_hi = a
    w = L ** (-a)
    return rng.choice(L.astype(np.int64), size=n, p=w / w.sum()), a


def c4_sequence(n: int = 4_000_000, num: int = 8) -> SequenceSpec:
    """C4: unstructured power-law rows (3..200 nnz, mean ~27, diagonal
    included), uniform random off-diagonal columns, N(0,1) values; diagonal
    1.2 x the row's absolute off-diagonal sum; the largest off-diagonal of 5%
    of rows flips sign; A_j = A + 0.05 j I; N(0,1) rhs from seed j; k=30."""
    import scipy.sparse as sp
    rng = np.random.default_rng(4)
    lens, _ = _power_law_lengths(rng, n)
    noff = lens - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), noff)
    cols = rng.integers(0, n - 1, size=rows.shape[0])
    cols = cols + (cols >= rows)
    vals = rng.standard_normal(rows.shape[0])
    O = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    O.sum_duplicates()
    O.sort_indices()
    del rows, cols, vals
    absv = np.abs(O.data)
    rowsum = np.add.reduceat(absv, O.indptr[:-1]) if O.nnz else np.zeros(n)
    rowsum[np.diff(O.indptr) == 0] = 0.0
    flip = np.flatnonzero(rng.uniform(size=n) < 0.05)
    flip = flip[np.diff(O.indptr)[flip] > 0]
    if flip.size:
        # position of the largest |a_ij| within each flipped row
        starts = O.indptr[flip]
        ends = O.indptr[flip + 1]
        pos = np.empty(flip.size, dtype=np.int64)
        for t in range(flip.size):   # ~5% of rows; short rows
            seg = absv[starts[t]:ends[t]]
            pos[t] = starts[t] + int(np.argmax(seg))
        O.data[pos] = -O.data[pos]
    base = (O + sp.diags(1.2 * rowsum)).tocsr()
    base.sum_duplicates()
    base.sort_indices()
    diag_pos = _diag_positions(base.indptr, base.indices, n)
    bvals = base.data.copy()
    rp = base.indptr.astype(np.int64)
    ci = base.indices.astype(np.int32)
    del O, base

    def mat(j):
        v = bvals.copy()
        v[diag_pos] = v[diag_pos] + 0.05 * j
        return CSR(n, rp, ci, v)

    def rhs(j, kappa):
        return _normal(j, n)

    # max_itn 3000: system 0 (sigma = 0) needs 1909 BiCGSTAB iterations at
    # n = 4 M (319 / 582 / 779 at n = 20 k / 200 k / 1 M; the reference
    # algorithm on the CPU: 370 / 659 at 20 k / 200 k), so the default 1000
    # would stop it at max_itn (tools/c4_convergence.py)
    return SequenceSpec("c4", n, 30, 1e-8, num, 1, mat, rhs, max_itn=3000,
                        meta={"rows": n, "pattern": "power-law 3..200"})


def _diag_positions(indptr, indices, n, chunk=1 << 22):
    """Index into the CSR value array of each row's diagonal entry."""
    out = []
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        lo, hi = int(indptr[r0]), int(indptr[r1])
        rows = np.repeat(np.arange(r0, r1, dtype=np.int64), np.diff(indptr[r0:r1 + 1]))
        out.append(lo + np.flatnonzero(indices[lo:hi] == rows))
    hit = np.concatenate(out) if out else np.zeros(0, dtype=np.int64)
    if hit.shape[0] != n:
        raise ValueError("every row needs a stored diagonal")
    return hit


def c5_sequence(m: int = 256, num: int = 8) -> SequenceSpec:
    """C5: 27-point m^3, convection (50,25,10), (s_j E + L_h) with E U[1,2]
    (seed 0), s_j = logspace(-3,-1,num); N(0,1) rhs from seed j; k=30 and
    s=28, so the recycle update's candidate basis holds m = k + s + 2 = 60
    stored vectors (BASELINE configs[4]).

    The matrices differ only on the diagonal: the stencil CSR is built once
    and every matrix shares its row_ptr / col_idx arrays (a fresh value array
    per matrix with the shifted diagonal), so eight 449 M-nnz systems hold
    one index structure in host memory."""
    h = 1.0 / (m + 1)
    offs, co = _cd_offsets_27(h, (50.0, 25.0, 10.0))
    n = m ** 3
    E = np.random.default_rng(0).uniform(1.0, 2.0, n)
    shifts = np.logspace(-3, -1, num)
    dcoef = co[offs.index((0, 0, 0))]
    base = {}

    def mat(j):
        if not base:
            B = _stencil_csr((m, m, m), offs, co, np.zeros(n))
            base["csr"] = B
            base["diag"] = _diag_positions(B.row_ptr, B.col_idx, n)
        B, dpos = base["csr"], base["diag"]
        v = B.values.copy()
        v[dpos] = shifts[j] * E + dcoef
        return CSR(n, B.row_ptr, B.col_idx, v)

    def rhs(j, kappa):
        return _normal(j, n)

    return SequenceSpec("c5", n, 30, 1e-8, num, 1, mat, rhs, s=28,
                        meta={"grid": (m, m, m), "stencil": 27, "m_basis": 60,
                              "s": 28, "shifts": shifts.tolist()})


CONFIGS = {
    "c1": c1_sequence,
    "c2": c2_sequence,
    "c3": c3_sequence,
    "c4": c4_sequence,
    "c5": c5_sequence,
}

# Reduced-size variants with the same structure, for parity tests whose CPU
# oracle has to finish in seconds.
SMALL = {
    "c1": lambda: c1_sequence(m=32, num=3),
    "c2": lambda: c2_sequence(m=16, num=3),
    "c3": lambda: c3_sequence(m=16, n_s=2, n_p=2, nrhs=2),
    "c4": lambda: c4_sequence(n=20_000, num=3),
    "c5": lambda: c5_sequence(m=16, num=3),
}


def make_sequence(name: str, small: bool = False) -> SequenceSpec:
    table = SMALL if small else CONFIGS
    if name not in table:
        raise ValueError(f"unknown config {name!r}; choose from {sorted(table)}")
    return table[name]()


def sine_basis(grid, k: int) -> np.ndarray:
    """n x k basis of the k lowest discrete sine modes of a structured grid
    (x fastest): sin(pi p x) sin(pi q y) [sin(pi r z)] ordered by p^2 + q^2
    (+ r^2), ties by (p, q, r).  These approximate the small-eigenvalue
    modes of the Laplacian part of the C1-C5 operators, so a recycle space
    built from them is well conditioned (unlike a random basis pair, whose
    biorthonormalization amplifies rounding by ~1e2-1e3 and makes the
    reference's own runs disagree at different BLAS thread counts)."""
    dims = list(grid)
    axes = [(np.arange(m) + 1.0) / (m + 1.0) for m in dims]
    R = int(np.ceil(k ** (1.0 / len(dims)))) + 2
    import itertools
    modes = sorted(itertools.product(range(1, R + 1), repeat=len(dims)),
                   key=lambda t: (sum(v * v for v in t), t))[:k]
    cols = []
    for mode in modes:
        f = np.sin(np.pi * mode[0] * axes[0])
        for d in range(1, len(dims)):
            f = np.multiply.outer(np.sin(np.pi * mode[d] * axes[d]), f)
        cols.append(f.ravel())
    return np.stack(cols, axis=1)


def bytes_per_iteration(n: int, nnz: int, k: int) -> int:
    """Algorithmic HBM bytes of one RBiCGSTAB iteration:
    24 nnz + 32 n k + 216 n for k > 0, 24 nnz + 184 n for k = 0
    (fp64 values, int32 column indices)."""
    if k > 0:
        return 24 * nnz + 32 * n * k + 216 * n
    return 24 * nnz + 184 * n


def spmv_bytes(n: int, nnz: int) -> int:
    """Algorithmic bytes of one SpMV: 12 nnz + 4 (n+1) + 16 n."""
    return 12 * nnz + 4 * (n + 1) + 16 * n
