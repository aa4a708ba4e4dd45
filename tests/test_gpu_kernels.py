"""Kernel-level parity on the B200: every libkrb primitive against the CPU
oracle (oracle/canon.c) — bit-exact — and against the reference's numpy/scipy
results (golden fixtures) where the reference's order is reproducible."""

import numpy as np
import pytest

from conftest import golden_csr, gpu

pytestmark = gpu


@pytest.fixture(scope="module")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_1406_2831_b200 import device
    device.require_cuda()
    return device


def _tensor(a):
    from paper_1406_2831_b200.device import to_device
    return to_device(a)


def _cols(X):
    """numpy n x k -> device (k, n)."""
    return _tensor(np.ascontiguousarray(np.asarray(X).T))


@pytest.mark.parametrize("name", ["dense40", "rand200", "c1s", "c4s"])
def test_spmv_bitwise_vs_reference_golden(dev, golden, name):
    p = f"spmv/{name}/"
    csr = golden_csr(golden, p)
    M = dev.DeviceMatrix(csr.n, csr.row_ptr, csr.col_idx, csr.values)
    x = golden[p + "x"]
    y = M.spmv(_tensor(x)).cpu().numpy()
    yt = M.spmv(_tensor(x), transpose=True).cpu().numpy()
    assert np.array_equal(y, golden[p + "Ax"])      # scipy csr_matvec, bitwise
    assert np.array_equal(yt, golden[p + "AHx"])    # scipy rmatvec, bitwise


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
@pytest.mark.parametrize("fmt", [0, 1, 2, 3, 4])
def test_spmv_formats_bitwise(dev, canon, cfg, fmt):
    from oracle.ops import CsrOperand
    from paper_1406_2831_b200.workloads import make_sequence
    A = make_sequence(cfg, small=True).matrix(1)
    M = dev.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values, fmt=fmt)
    x = np.random.default_rng(3).standard_normal(A.n)
    op = CsrOperand.of(A)
    assert np.array_equal(M.spmv(_tensor(x)).cpu().numpy(), canon.matvec(op, x))
    assert np.array_equal(M.spmv(_tensor(x), transpose=True).cpu().numpy(),
                          canon.rmatvec(op, x))
    assert np.array_equal(M.spmv(_tensor(x)).cpu().numpy(), op._csr @ x)


@pytest.mark.parametrize("cfg,expect", [("c1", "sell32-dict-vc"), ("c2", "sell32-dict-vc"),
                                        ("c5", "sell32-dict-vc"), ("c3", "sell32"),
                                        ("c4", "sell32-sigma")])
def test_offset_coded_format_choice(dev, cfg, expect):
    """Stencil matrices (<= 255 distinct diagonals) get the offset-coded
    SELL-32 stream automatically, their transposes too -- with value tables
    for their constant diagonals (constant-coefficient stencils: all of K's
    diagonals but the main one of s E - K); C3's random K1 columns and C4's
    power-law rows do not qualify."""
    from paper_1406_2831_b200.workloads import make_sequence
    A = make_sequence(cfg, small=True).matrix(1)
    M = dev.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
    assert M.format == expect
    x = np.random.default_rng(5).standard_normal(A.n)
    S = A.to_scipy()
    assert np.array_equal(M.spmv(_tensor(x)).cpu().numpy(), S @ x)
    assert np.array_equal(M.spmv(_tensor(x), transpose=True).cpu().numpy(), S.T.tocsr() @ x)
    X = np.random.default_rng(6).standard_normal((A.n, 11))
    Y = M.spmm(_cols(X)).cpu().numpy().T
    for c in range(11):
        assert np.array_equal(Y[:, c], S @ X[:, c])


@pytest.mark.parametrize("n", [31, 32, 33, 95, 1000, 4099])
def test_offset_coded_ragged_slices(dev, n):
    """Mixed slices: banded rows with random gaps (non-uniform slices next to
    uniform ones), empty rows, a partial last slice, 255 distinct offsets
    (the limit) and one more (falls back to plain SELL-32)."""
    import scipy.sparse as sp
    r = np.random.default_rng(n)
    offs = np.arange(-127, 128)            # 255 distinct diagonals
    rows, cols = [], []
    for i in range(n):
        if i % 97 == 5:
            continue                        # empty row
        sel = offs if (i // 32) % 3 == 0 else offs[r.random(offs.size) < 0.3]
        c = i + sel
        c = c[(c >= 0) & (c < n)]
        rows.extend([i] * c.size)
        cols.extend(c.tolist())
    vals = r.standard_normal(len(rows)) * np.exp(r.uniform(-6, 6, len(rows)))
    S = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    S.sort_indices()
    x = r.standard_normal(n)
    M = dev.DeviceMatrix(n, S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data)
    if n > 127:
        assert M.format == "sell32-dict"     # random values: no constant diagonal
    assert np.array_equal(M.spmv(_tensor(x)).cpu().numpy(), S @ x)
    assert np.array_equal(M.spmv(_tensor(x), transpose=True).cpu().numpy(), S.T.tocsr() @ x)
    # 256 distinct offsets: no dictionary
    if n > 200:
        S2 = S.tolil()
        S2[n - 1, n - 1 - 200] = 1.0
        S2 = S2.tocsr()
        S2.sort_indices()
        M2 = dev.DeviceMatrix(n, S2.indptr.astype(np.int64), S2.indices.astype(np.int32), S2.data)
        assert M2.format in ("sell32", "sell32-sigma", "csr")
        assert np.array_equal(M2.spmv(_tensor(x)).cpu().numpy(), S2 @ x)


def _banded(n, offs, r, const_offs, gaps=5):
    """Banded matrix on the diagonals `offs`: the diagonals in const_offs
    carry ONE value each (bit-identical), the others random values; rows of
    every third slice group lose entries (one of `gaps` random subsets per
    row: non-uniform slices, several row templates per warp)."""
    import scipy.sparse as sp
    cval = {int(o): float(r.standard_normal() * np.exp(r.uniform(-5, 5))) for o in const_offs}
    subsets = [offs[r.random(offs.size) < 0.6] for _ in range(int(gaps))]
    rows, cols, vals = [], [], []
    for i in range(n):
        if i % 211 == 7:
            continue                        # empty row
        sel = offs if (not gaps or (i // 32) % 3) else subsets[r.integers(len(subsets))]
        for o in sel:
            c = i + int(o)
            if 0 <= c < n:
                rows.append(i)
                cols.append(c)
                vals.append(cval[int(o)] if int(o) in cval else float(r.standard_normal()))
    S = sp.csr_matrix((np.array(vals), (rows, cols)), shape=(n, n))
    S.sort_indices()
    return S


@pytest.mark.parametrize("n", [64, 1000, 4099, 40000])
@pytest.mark.parametrize("nvar", [0, 1, 3])
def test_value_coded_bitwise(dev, n, nvar):
    """Value-coded format: constant diagonals served from the value tables,
    varying ones from the stream; uniform and ragged slices, empty rows, a
    partial last slice.  Products, transposed products and multi-column
    products are bit-identical to scipy and to the same matrix with the value
    tables switched off."""
    from paper_1406_2831_b200 import _lib
    r = np.random.default_rng(1000 * n + nvar)
    offs = np.array([-40, -33, -32, -31, -1, 0, 1, 2, 31, 32, 33, 50, 51])
    var = set(r.choice(offs, size=nvar, replace=False).tolist())
    S = _banded(n, offs, r, [o for o in offs if int(o) not in var])
    x = r.standard_normal(n)
    X = r.standard_normal((n, 9))
    args = (n, S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data)
    M = dev.DeviceMatrix(*args, fmt=4)
    assert M.format == "sell32-dict-vc", M.format
    assert M.stream_stats["const_diagonals"] == offs.size - nvar
    coo = S.tocoo()
    assert M.stream_stats["const_entries"] == int(np.isin(coo.col - coo.row,
                                                          [o for o in offs if int(o) not in var]).sum())
    assert 1 <= M.stream_stats["templates"] <= 1024
    y, yt = M.spmv(_tensor(x)).cpu().numpy(), M.spmv(_tensor(x), transpose=True).cpu().numpy()
    Y = M.spmm(_cols(X)).cpu().numpy().T
    Yt = M.spmm(_cols(X), transpose=True).cpu().numpy().T
    St = S.T.tocsr()
    assert np.array_equal(y, S @ x) and np.array_equal(yt, St @ x)
    for c in range(9):
        assert np.array_equal(Y[:, c], S @ X[:, c])
        assert np.array_equal(Yt[:, c], St @ X[:, c])
    assert M.stream_stats["diagonal_form"] == (n >= 1000)   # 13 diagonals, mostly full
    with _lib.tuning(value_coding=2):           # the row-template kernel
        assert np.array_equal(M.spmv(_tensor(x)).cpu().numpy(), y)
        assert np.array_equal(M.spmv(_tensor(x), transpose=True).cpu().numpy(), yt)
    with _lib.tuning(value_coding=0):
        M0 = dev.DeviceMatrix(*args, fmt=4)
        assert M0.format == "sell32-dict"
        assert np.array_equal(M0.spmv(_tensor(x)).cpu().numpy(), y)
        assert np.array_equal(M0.spmv(_tensor(x), transpose=True).cpu().numpy(), yt)


def test_value_coded_sparse_diagonals_use_row_templates(dev):
    """Few entries per row spread over many diagonals (less than half of the
    n x ndict positions filled), and a matrix with more than 32 diagonals:
    value-coded through the row templates, not the diagonal form."""
    import scipy.sparse as sp
    r = np.random.default_rng(4)
    n = 6000
    for offs, per_row in ((np.arange(-30, 31, 2), 6), (np.arange(-25, 26), 40)):
        cval = {int(o): float(r.standard_normal()) for o in offs}
        kinds = [np.sort(r.choice(offs, size=per_row, replace=False)) for _ in range(6)]
        rows, cols, vals = [], [], []
        for i in range(n):
            for o in kinds[(i // 64) % 6]:
                if 0 <= i + int(o) < n:
                    rows.append(i); cols.append(i + int(o)); vals.append(cval[int(o)])
        S = sp.csr_matrix((np.array(vals), (rows, cols)), shape=(n, n))
        S.sort_indices()
        M = dev.DeviceMatrix(n, S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data, fmt=4)
        assert M.format == "sell32-dict-vc" and not M.stream_stats["diagonal_form"]
        x = r.standard_normal(n)
        assert np.array_equal(M.spmv(_tensor(x)).cpu().numpy(), S @ x)
        assert np.array_equal(M.spmv(_tensor(x), transpose=True).cpu().numpy(), S.T.tocsr() @ x)


def test_value_coded_special_values_and_shared_pattern(dev):
    """-0.0 / +0.0 and NaN payloads on a diagonal are different bit patterns
    (such a diagonal is not constant); a later matrix on the SAME pattern with
    random values is not value-coded while the first one stays so."""
    r = np.random.default_rng(77)
    n = 3000
    offs = np.array([-32, -1, 0, 1, 32])
    S = _banded(n, offs, r, offs, gaps=0)
    d = S.data.copy()
    main = np.flatnonzero(S.indices == np.repeat(np.arange(n), np.diff(S.indptr)))
    up = np.flatnonzero(S.indices == np.repeat(np.arange(n), np.diff(S.indptr)) + 1)
    d[main] = 0.0
    d[main[::7]] = -0.0                      # same value, other bits
    d[up[5]] = np.nan
    args = (n, S.indptr.astype(np.int64), S.indices.astype(np.int32))
    M = dev.DeviceMatrix(*args, d)
    assert M.format == "sell32-dict-vc"
    assert M.stream_stats["const_diagonals"] == 3
    import scipy.sparse as sp
    S1 = sp.csr_matrix((d, S.indices, S.indptr), shape=(n, n))
    x = r.standard_normal(n)
    y = M.spmv(_tensor(x)).cpu().numpy()
    assert np.array_equal(y, S1 @ x, equal_nan=True)
    assert np.array_equal(np.signbit(y), np.signbit(S1 @ x))
    d2 = r.standard_normal(S.nnz)
    M2 = dev.DeviceMatrix(*args, d2)
    assert M2.pattern_info()[0] == M.pattern_info()[0]
    assert M2.format == "sell32-dict" and M.format == "sell32-dict-vc"
    S2 = sp.csr_matrix((d2, S.indices, S.indptr), shape=(n, n))
    assert np.array_equal(M2.spmv(_tensor(x)).cpu().numpy(), S2 @ x)
    assert np.array_equal(M2.spmv(_tensor(x), transpose=True).cpu().numpy(), S2.T.tocsr() @ x)
    assert np.array_equal(M.spmv(_tensor(x)).cpu().numpy(), y, equal_nan=True)
    assert np.array_equal(M.spmv(_tensor(x), transpose=True).cpu().numpy(),
                          S1.T.tocsr() @ x, equal_nan=True)


def test_value_coded_falls_back_on_too_many_templates(dev):
    """More than 1024 distinct row sequences: no templates, the matrix stays
    plainly offset-coded (constant diagonals or not) and correct."""
    r = np.random.default_rng(9)
    n = 20000
    offs = np.arange(-8, 9)
    S = _banded(n, offs, r, offs, gaps=4000)
    M = dev.DeviceMatrix(n, S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data)
    assert M.format == "sell32-dict"
    x = r.standard_normal(n)
    assert np.array_equal(M.spmv(_tensor(x)).cpu().numpy(), S @ x)
    assert np.array_equal(M.spmv(_tensor(x), transpose=True).cpu().numpy(), S.T.tocsr() @ x)


def test_sell_sigma_chosen_for_power_law(dev):
    from paper_1406_2831_b200.workloads import c4_sequence
    A = c4_sequence(n=50_000, num=1).matrix(0)
    M = dev.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
    assert M.format == "sell32-sigma"
    x = np.random.default_rng(1).standard_normal(A.n)
    assert np.array_equal(M.spmv(_tensor(x)).cpu().numpy(), A.to_scipy() @ x)


def test_spmv_empty_rows_and_tiny(dev):
    import scipy.sparse as sp
    from paper_1406_2831_b200.workloads import CSR
    D = np.zeros((37, 37))
    D[3, 5] = 2.0
    D[36, 0] = -1.5
    D[10, 10] = 4.0
    S = sp.csr_matrix(D)
    A = CSR(37, S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data)
    M = dev.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
    x = np.arange(37, dtype=np.float64) - 7.0
    assert np.array_equal(M.spmv(_tensor(x)).cpu().numpy(), S @ x)
    assert np.array_equal(M.spmv(_tensor(x), transpose=True).cpu().numpy(),
                          S.T.tocsr() @ x)


@pytest.mark.parametrize("n", [1, 255, 256, 257, 4096, 100_003, 700_001, 5_000_000])
def test_dot_bitwise(dev, canon, n):
    from paper_1406_2831_b200.recycling import dot
    r = np.random.default_rng(n)
    x = r.standard_normal(n)
    y = r.standard_normal(n) * np.exp(r.uniform(-5, 5, n))
    got = float(dot(_tensor(x), _tensor(y)).cpu().numpy()[0])
    assert got == float(canon.dot(x, y))
    assert abs(got - float(np.dot(x, y))) <= 1e-12 * np.abs(x * y).sum()


@pytest.mark.parametrize("n,k", [(1000, 1), (4096, 10), (300_001, 20), (2_000_000, 30)])
def test_projection_primitives_bitwise(dev, canon, n, k):
    from paper_1406_2831_b200 import recycling as R
    r = np.random.default_rng(k)
    M = r.standard_normal((n, k))
    v = r.standard_normal(n)
    y = r.standard_normal(k)
    Md = _cols(M)
    assert np.array_equal(R.tdot(Md, _tensor(v)).cpu().numpy(), canon.tdot(M, v))
    base = r.standard_normal(n)
    got = R.gemv(Md, _tensor(y), base=_tensor(base), sign=-1).cpu().numpy()
    assert np.array_equal(got, base - canon.gemv(M, y))
    got = R.gemv(Md, _tensor(y), base=_tensor(base), sign=+1).cpu().numpy()
    assert np.array_equal(got, base + canon.gemv(M, y))
    assert np.array_equal(R.colnorms(Md).cpu().numpy(), canon.colnorms(M))


@pytest.mark.parametrize("n,na,nc", [(500, 3, 4), (70_000, 20, 20), (1_000_000, 47, 47),
                                     (262_144, 40, 40), (5_000, 130, 30), (3_001, 1, 64)])
def test_gram_gemm_bitwise(dev, canon, n, na, nc):
    from paper_1406_2831_b200 import recycling as R
    r = np.random.default_rng(na)
    X = r.standard_normal((n, na))
    Y = r.standard_normal((n, nc))
    G = R.gram(_cols(X), _cols(Y)).cpu().numpy()
    assert np.array_equal(G, canon.gram(X, Y))
    Z = r.standard_normal((na, 7))
    out = R.gemm(_cols(X), Z).cpu().numpy().T
    assert np.array_equal(out, canon.gemm(X, Z))


@pytest.mark.parametrize("seed", [0, 1, 7, 104729, 2**40 + 3])
@pytest.mark.parametrize("n", [1, 1000, 1_234_567])
def test_pcg64_matches_numpy(dev, seed, n):
    import ctypes
    import torch
    from paper_1406_2831_b200 import _lib
    from paper_1406_2831_b200.solvers import pcg64_words
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.call("krb_uniform_pcg64", n, *pcg64_words(seed), -1.0, 1.0,
              ctypes.c_void_p(out.data_ptr()), dev.stream_ptr())
    ref = np.random.default_rng(seed).uniform(-1.0, 1.0, size=n)
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("mode", ["0", "8", "12", "24", "122", None])
@pytest.mark.parametrize("n,m,nc", [(1_000, 3, 1), (1_001, 47, 9), (129, 20, 20), (262_144, 40, 40), (5_003, 64, 64),
                                    (70_001, 200, 30), (70_002, 47, 47), (262_146, 26, 26),
                                    (4_096, 19, 20), (98, 5, 2)])
def test_gemm_shapes_bitwise(dev, canon, monkeypatch, mode, n, m, nc):
    """row kernel (gemm_mode 0) and the TMA-tiled kernel with 8 / 12 /
    24 columns per thread, 12 columns x 2 rows per thread (122), and the
    default choice (None): full tiles, partial last tiles (odd remainders),
    idle column groups, odd leading dimensions (row-kernel fallback)"""
    from paper_1406_2831_b200 import _lib, recycling as R
    r = np.random.default_rng(m + nc)
    X = r.standard_normal((n, m))
    Z = r.standard_normal((m, nc))
    with _lib.tuning(**({} if mode is None else {"gemm_mode": int(mode)})):
        out = R.gemm(_cols(X), Z).cpu().numpy().T
    assert np.array_equal(out, canon.gemm(X, Z))


@pytest.mark.parametrize("n,k", [(1, 1), (1_000, 3), (262_144, 47), (70_001, 20), (5_000_003, 2)])
def test_colscale_div_bitwise(dev, n, k):
    """X[:, j] / s[j] (recycling.py:307-308, 333-340): numpy's correctly
    rounded division, element for element"""
    from paper_1406_2831_b200 import recycling as R
    r = np.random.default_rng(n + k)
    X = r.standard_normal((n, k))
    sv = r.uniform(0.1, 10.0, size=k)
    Xd = _cols(X)
    R.colscale_div(Xd, _tensor(sv))
    assert np.array_equal(Xd.cpu().numpy().T, X / sv)


@pytest.mark.parametrize("n,parts", [(1, [1]), (1_000, [3, 2]), (262_144, [20, 27]),
                                     (70_001, [0, 5, 7])])
def test_assemble_scaled_bitwise(dev, n, parts):
    """[parts] stacked and divided column-wise (the hstack + scaling of
    recycling.py:326-340 done as scaled copies, krb_colscale_div_to): the
    same bits as numpy's hstack then division; sources untouched."""
    from paper_1406_2831_b200 import recycling as R
    r = np.random.default_rng(n + len(parts))
    blocks = [r.standard_normal((n, k)) for k in parts]
    m = sum(parts)
    sv = r.uniform(0.1, 10.0, size=m)
    devs = [_cols(B) for B in blocks]
    before = [d.clone() for d in devs]
    out = R.assemble_scaled(devs, _tensor(sv))
    assert np.array_equal(out.cpu().numpy().T, np.hstack(blocks) / sv)
    for d, b0 in zip(devs, before):
        assert np.array_equal(d.cpu().numpy(), b0.cpu().numpy())
    C = blocks[-1]
    got = R.colscale_div_to(_cols(C), _tensor(sv[-C.shape[1]:] if C.shape[1] else sv[:0]))
    assert np.array_equal(got.cpu().numpy().T, C / sv[m - C.shape[1]:])


@pytest.mark.parametrize("cfg", ["c2", "c4"])
def test_spmv_adjoint_and_linearity(dev, cfg):
    """The reference's operator properties (tests/test_sparse.py:78-102):
    (A x, y) = (x, A^T y) and A (a x + b y) = a A x + b A y, to rounding."""
    import torch
    from paper_1406_2831_b200 import device as D
    from paper_1406_2831_b200.workloads import make_sequence
    A = make_sequence(cfg, small=True).matrix(0)
    M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
    r = np.random.default_rng(3)
    x, y = r.standard_normal(A.n), r.standard_normal(A.n)
    xd, yd = _tensor(x), _tensor(y)
    Ax = M.spmv(xd).cpu().numpy()
    Aty = M.spmv(yd, transpose=True).cpu().numpy()
    lhs, rhs = Ax @ y, x @ Aty
    assert abs(lhs - rhs) <= 1e-12 * (np.abs(Ax) @ np.abs(y) + 1.0)
    a, b = 0.75, -1.25
    comb = M.spmv(_tensor(a * x + b * y)).cpu().numpy()
    Ay = M.spmv(yd).cpu().numpy()
    assert np.allclose(comb, a * Ax + b * Ay, rtol=1e-12, atol=1e-12 * np.abs(Ax).max())


def _csr_of(S):
    from paper_1406_2831_b200.workloads import CSR
    S = S.tocsr()
    S.sort_indices()
    return CSR(S.shape[0], S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data)


@pytest.mark.parametrize("cfg", ["c2", "c4", "c5"])
def test_shared_pattern_values_and_transpose(dev, cfg):
    """Matrices of a sequence with one sparsity pattern share the structure
    work (SELL layout, offset codes, transpose permutation): every product
    stays bit-identical to scipy, the pattern outlives the matrix that built
    it, and a different pattern of the same size is not shared."""
    import scipy.sparse as sp
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence(cfg, small=True)
    A1, A2 = seq.matrix(0), seq.matrix(1)
    assert np.array_equal(A1.col_idx, A2.col_idx) or cfg == "c4"
    r = np.random.default_rng(9)
    x = r.standard_normal(A1.n)
    M1 = dev.DeviceMatrix(A1.n, A1.row_ptr, A1.col_idx, A1.values)
    y1t = M1.spmv(_tensor(x), transpose=True).cpu().numpy()      # builds the transpose
    assert np.array_equal(y1t, A1.to_scipy().T.tocsr() @ x)
    # same pattern, new values (scaled diagonal shift of the first matrix)
    S2 = A1.to_scipy() + 0.37 * sp.identity(A1.n, format="csr")
    B2 = _csr_of(S2)
    same = np.array_equal(B2.row_ptr, A1.row_ptr) and np.array_equal(B2.col_idx, A1.col_idx)
    M2 = dev.DeviceMatrix(B2.n, B2.row_ptr, B2.col_idx, B2.values)
    p1, p2 = M1.pattern_info(), M2.pattern_info()
    if same:
        assert p1[0] == p2[0] and p2[1] >= 2 and p2[2]
    assert np.array_equal(M2.spmv(_tensor(x)).cpu().numpy(), S2 @ x)
    assert np.array_equal(M2.spmv(_tensor(x), transpose=True).cpu().numpy(), S2.T.tocsr() @ x)
    X = r.standard_normal((A1.n, 9))
    Y = M2.spmm(_cols(X), transpose=True).cpu().numpy().T
    for c in range(9):
        assert np.array_equal(Y[:, c], S2.T.tocsr() @ X[:, c])
    # the builder goes away; the pattern stays with M2
    del M1
    import gc
    gc.collect()
    assert np.array_equal(M2.spmv(_tensor(x)).cpu().numpy(), S2 @ x)
    assert np.array_equal(M2.spmv(_tensor(x), transpose=True).cpu().numpy(), S2.T.tocsr() @ x)
    # a third matrix attaches to the surviving pattern
    S3 = S2 * 1.5
    B3 = _csr_of(S3)
    M3 = dev.DeviceMatrix(B3.n, B3.row_ptr, B3.col_idx, B3.values)
    if same:
        assert M3.pattern_info()[0] == p2[0]
    assert np.array_equal(M3.spmv(_tensor(x), transpose=True).cpu().numpy(), S3.T.tocsr() @ x)
    # same n and nnz, one column moved: its own pattern
    cols = B3.col_idx.copy()
    row = int(np.argmax(np.diff(B3.row_ptr) >= 2))
    b0, e0 = B3.row_ptr[row], B3.row_ptr[row + 1]
    free = sorted(set(range(B3.n)) - set(cols[b0:e0].tolist()))
    cols[e0 - 1] = free[-1] if free[-1] > cols[e0 - 2] else cols[e0 - 1]
    S4 = sp.csr_matrix((B3.values, cols, B3.row_ptr), shape=(B3.n, B3.n))
    S4.sort_indices()
    B4 = _csr_of(S4)
    M4 = dev.DeviceMatrix(B4.n, B4.row_ptr, B4.col_idx, B4.values)
    if not np.array_equal(B4.col_idx, B3.col_idx):
        assert M4.pattern_info()[0] != M3.pattern_info()[0]
    assert np.array_equal(M4.spmv(_tensor(x)).cpu().numpy(), S4 @ x)
    assert np.array_equal(M4.spmv(_tensor(x), transpose=True).cpu().numpy(), S4.T.tocsr() @ x)
