"""The k = 0 fused kernel with the operator on chip (csrc/persist0.cu),
bit-identical to the canonical oracle and to the other k = 0 drivers:

* stencil operators whose rows and halo fit in shared memory (every CTA on
  chip), forced off chip (tuning p0_onchip=0: the same kernel gathering from
  global memory), and the previous fused kernel (tuning persist0=0);
* scattered random columns (halo over budget: CTAs fall back per CTA) and a
  mix of banded and scattered rows (some CTAs on chip, some not);
* one CTA per block (nb <= #SMs), two blocks per CTA, a partial last block,
  a single block (cluster driver disabled), SELL-32 and CSR storage,
  breakdown-free early exits at the half step (tight tol / max_itn).
"""

import numpy as np
import pytest

from conftest import gpu

pytestmark = gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_1406_2831_b200 as P
    return P


def stencil7(m, shift=0.05, seed=0):
    """3-D 7-point convection-diffusion-like operator on an m^3 grid."""
    import scipy.sparse as sp
    from paper_1406_2831_b200.workloads import CSR
    r = np.random.default_rng(seed)
    n = m ** 3
    I = sp.identity(m, format="csr")
    T = sp.diags([-1.0 - 0.1, 2.0, -1.0 + 0.1], [-1, 0, 1], shape=(m, m), format="csr")
    A = (sp.kron(sp.kron(T, I), I) + sp.kron(sp.kron(I, T), I) + sp.kron(sp.kron(I, I), T)).tocsr()
    A = A + sp.diags(shift + 0.01 * r.uniform(size=n))
    A = A.tocsr()
    A.sum_duplicates()
    A.sort_indices()
    return CSR(n, A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.copy())


def banded_mixed(n, seed):
    """rows below n/2: 1..9 entries within +-3000 of the diagonal (small
    halo); rows above: random columns over the whole range (huge halo)."""
    import scipy.sparse as sp
    from paper_1406_2831_b200.workloads import CSR
    r = np.random.default_rng(seed)
    cnt = r.integers(0, 9, size=n)
    rows = np.repeat(np.arange(n), cnt)
    near = np.clip(rows + r.integers(-3000, 3001, size=rows.size), 0, n - 1)
    far = r.integers(0, n, size=rows.size)
    cols = np.where(rows < n // 2, near, far)
    vals = r.uniform(-1.0, 1.0, size=rows.size)
    rows = np.concatenate([rows, np.arange(n)])
    cols = np.concatenate([cols, np.arange(n)])
    vals = np.concatenate([vals, 2.5 + r.uniform(0.0, 1.0, size=n)])
    S = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    S.sum_duplicates()
    S.sort_indices()
    return CSR(n, S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data.copy())


def _matrix(kind, n):
    if kind == "stencil":
        return stencil7(int(round(n ** (1 / 3))))
    if kind == "mixed":
        return banded_mixed(n, seed=n)
    from test_gpu_persistent import ragged_matrix
    return ragged_matrix(n, seed=n)


CASES = [
    # kind, n (stencil: m^3), fmt
    ("stencil", 64 ** 3, 2),     # the C2 grid: two blocks per CTA, on chip
    ("stencil", 40 ** 3, 1),     # CSR, 63 blocks: one per CTA
    ("stencil", 27 ** 3, 2),     # partial last block
    ("mixed", 250_000, 2),       # some CTAs on chip, some not
    ("random", 200_000, 2),      # every CTA off chip
    ("random", 30_000, 1),
]


@pytest.mark.parametrize("kind,n,fmt", CASES)
def test_persist0_bitwise(pkg, canon, monkeypatch, kind, n, fmt):
    from oracle import krylov as O
    from paper_1406_2831_b200 import _lib, solvers as S
    from paper_1406_2831_b200.device import DeviceMatrix, to_device
    A = _matrix(kind, n)
    b = np.random.default_rng(A.n).standard_normal(A.n)
    M = DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values, fmt=fmt)
    for tol, max_itn in ((1e-14, 9), (1e-9, 600)):
        cfg = pkg.SolverConfig(tol=tol, max_itn=max_itn, seed=5)
        xo, ho = O.rbicgstab(A, b, config=O.Config(tol=tol, max_itn=max_itn, seed=5), ops=canon)
        for env in ({}, {"p0_onchip": 0}, {"p0_grid_half": 1}, {"persist0": 0}):
            with _lib.tuning(**env):
                xg, hg = S.solve_device(M, to_device(b), None, None, cfg, use_graph=2)
            assert S.LAST_SOLVE["driver"] == "fused", env
            assert hg.status == ho.status, env
            assert hg.resid == ho.resid, env
            assert hg.matvecs == ho.matvecs, env
            assert np.array_equal(xg.cpu().numpy(), xo), env


def test_persist0_single_block(pkg, canon, monkeypatch):
    """n < 1024 with the cluster driver disabled: one CTA, one partial block."""
    from oracle import krylov as O
    from paper_1406_2831_b200 import solvers as S
    from paper_1406_2831_b200.device import DeviceMatrix, to_device
    from test_gpu_persistent import ragged_matrix
    from paper_1406_2831_b200 import _lib
    A = ragged_matrix(777, seed=1)
    b = np.random.default_rng(2).standard_normal(A.n)
    M = DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values, fmt=2)
    cfg = pkg.SolverConfig(tol=1e-12, max_itn=300, seed=1)
    xo, ho = O.rbicgstab(A, b, config=O.Config(tol=1e-12, max_itn=300, seed=1), ops=canon)
    with _lib.tuning(cluster=0):
        xg, hg = S.solve_device(M, to_device(b), None, None, cfg, use_graph=2)
    assert S.LAST_SOLVE["driver"] == "fused"
    assert (hg.status, hg.resid, hg.matvecs) == (ho.status, ho.resid, ho.matvecs)
    assert np.array_equal(xg.cpu().numpy(), xo)
