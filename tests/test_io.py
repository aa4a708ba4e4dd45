"""Run-report CSV and KRSP recycle snapshots (paper_1406_2831_b200/io.py)
against files written by the reference's own krecycle.io
(tests/golden/make_io_golden.py): byte-identical output, same parser
errors; the device reload (recycle_load) is a GPU test."""

import os
import struct
import types

import numpy as np
import pytest

from conftest import gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _fixed_histories():
    from paper_1406_2831_b200.solvers import ConvergenceHistory as H
    h1 = H(solver="rbicgstab", resid=[1.0, 0.5, 1.0 / 3.0, 2.5e-9],
           matvecs=[0, 2, 4, 6], seconds=[0.0, 0.00123, 0.0024567, 0.0037],
           status="converged")
    h2 = H(solver="bicgstab", resid=[1.0, 0.125], matvecs=[1, 3],
           seconds=[0.0, 1.5e-7], status="max_itn")
    h3 = H(solver="rbicg")
    return [h1, h2, h3]


def _fixed_space():
    r = np.random.default_rng(2024)
    U, Ut = r.standard_normal((37, 3)), r.standard_normal((37, 3))
    return types.SimpleNamespace(n=37, k=3, U=U, Ut=Ut)


def test_history_write_matches_reference(tmp_path):
    from paper_1406_2831_b200 import io
    from paper_1406_2831_b200.sequence import RunReport
    p = tmp_path / "h.csv"
    io.history_write(p, _fixed_histories())
    assert p.read_bytes() == open(os.path.join(HERE, "history_ref.csv"), "rb").read()
    p2 = tmp_path / "h2.csv"
    io.history_write(p2, RunReport(label="x", histories=_fixed_histories()))
    assert p2.read_bytes() == p.read_bytes()
    p3 = tmp_path / "empty.csv"
    io.history_write(p3, [])
    assert p3.read_text().strip() == "system_index,solver,iteration,resid,matvecs_cum,seconds_cum"


def test_recycle_save_matches_reference(tmp_path):
    from paper_1406_2831_b200 import io
    p = tmp_path / "s.krsp"
    io.recycle_save(p, _fixed_space())
    ref = open(os.path.join(HERE, "space_ref.krsp"), "rb").read()
    assert p.read_bytes() == ref
    n, U, Ut = io._read(p)
    S = _fixed_space()
    assert n == 37 and np.array_equal(U, S.U) and np.array_equal(Ut, S.Ut)
    with pytest.raises(ValueError, match="empty"):
        io.recycle_save(tmp_path / "e.krsp", types.SimpleNamespace(n=5, k=0))


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XXXX" + b[4:], "bad magic"),
    (lambda b: b[:10], "truncated recycle-space header"),
    (lambda b: b[:4] + struct.pack("<I", 2) + b[8:], "unsupported"),
    (lambda b: b[:-8], "truncated recycle-space payload"),
])
def test_recycle_file_errors(tmp_path, mutate, msg):
    from paper_1406_2831_b200 import io
    ref = open(os.path.join(HERE, "space_ref.krsp"), "rb").read()
    p = tmp_path / "bad.krsp"
    p.write_bytes(mutate(ref))
    with pytest.raises(ValueError, match=msg):
        io._read(p)


@gpu
def test_recycle_load_rebuilds_images(tmp_path, canon):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import io
    from paper_1406_2831_b200.workloads import make_sequence
    seq = make_sequence("c1")
    A = seq.matrix(1)
    r = np.random.default_rng(3)
    U, Ut = r.standard_normal((A.n, 6)), r.standard_normal((A.n, 6))
    p = tmp_path / "c1.krsp"
    io.recycle_save(p, types.SimpleNamespace(n=A.n, k=6, U=U, Ut=Ut))
    Sp = P.SparseMatrix.from_csr(A)
    S1 = io.recycle_load(p, Sp)
    S2 = P.biorthonormalize(U, Ut, Sp)
    assert S1.k == S2.k > 0
    for name in ("U", "Ut", "C", "Ct", "Chat", "Ccheck"):
        assert np.array_equal(getattr(S1, name), getattr(S2, name)), name
    with pytest.raises(ValueError, match="does not match"):
        io.recycle_load(p, P.SparseMatrix.from_csr(make_sequence("c1", small=True).matrix(0)))
