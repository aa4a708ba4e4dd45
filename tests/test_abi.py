"""CPU: the C-ABI library loads and exports every symbol include/krb.h
declares; the ctypes table covers them all.  No compute calls (no GPU)."""

import os
import re

from conftest import REPO


def _declared():
    src = open(os.path.join(REPO, "include", "krb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(krb_[a-z0-9_]+)\s*\(", src))


def test_header_symbols_exported():
    from paper_1406_2831_b200 import _lib
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 20
    for name in sorted(names):
        assert hasattr(lib, name), f"{name} declared in krb.h but not exported"
    assert names == set(_lib.SIGNATURES), names ^ set(_lib.SIGNATURES)
    assert lib.krb_abi_version() == 1


def test_library_is_sm100a():
    import subprocess
    so = os.path.join(REPO, "paper_1406_2831_b200", "libkrb.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_errors_without_gpu_are_loud():
    import numpy as np
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import _lib
    A = P.SparseMatrix.from_triplets(2, 2, [0, 1], [0, 1], [1.0, 2.0])
    with pytest.raises(_lib.KrbError):
        P.bicgstab_solve(A, np.ones(2))
