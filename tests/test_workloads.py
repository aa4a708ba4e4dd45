"""CPU: the seeded generators produce the BASELINE shapes, canonical CSR."""

import numpy as np
import pytest

from paper_1406_2831_b200 import workloads as W


def test_c1_c2_exact_sizes():
    a = W.make_sequence("c1").matrix(0)
    assert (a.n, a.nnz) == (16384, 81408)
    b = W.make_sequence("c2").matrix(0)
    assert (b.n, b.nnz) == (262144, 1810432)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_small_variants_canonical(name):
    s = W.make_sequence(name, small=True)
    for j in range(min(2, s.num_matrices)):
        A = s.matrix(j)
        S = A.to_scipy()
        assert S.has_canonical_format
        assert A.col_idx.dtype == np.int32 and A.row_ptr.dtype == np.int64
        d = S.diagonal()
        assert np.all(d != 0)
        assert s.rhs(j, 0).shape == (A.n,)


def test_stencil_nnz_formula():
    # 27-point on m^3: (3m-2)^3 ; 7-point: 7m^3 - 6m^2
    m = 12
    assert W.c5_sequence(m=m, num=1).matrix(0).nnz == (3 * m - 2) ** 3
    assert W.c2_sequence(m=m, num=1).matrix(0).nnz == 7 * m ** 3 - 6 * m ** 2


def test_bytes_formula():
    assert W.bytes_per_iteration(16384, 81408, 10) == 24 * 81408 + 32 * 16384 * 10 + 216 * 16384
