"""Shared test setup.

Markers: ``gpu`` = needs a CUDA device (run on the B200 via gpurun); the rest
run on CPU.  The oracle (oracle/) is imported only here in tests, as the
checker.
"""

import os
import sys

import numpy as np
import pytest

REPO = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN, allow_pickle=False)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def canon():
    from oracle.ops import CanonOps
    return CanonOps()


def golden_csr(g, prefix):
    from paper_1406_2831_b200.workloads import CSR
    rp = g[prefix + "row_ptr"]
    return CSR(len(rp) - 1, rp, g[prefix + "col_idx"], g[prefix + "values"])


def random_space_arrays(A, k, seed=0, ops=None):
    """Random biorthonormalized space built by the oracle (canonical ops)."""
    from oracle import krylov as O
    r = np.random.default_rng(seed)
    n = A.n if hasattr(A, "n") else A.nrows
    U = r.standard_normal((n, k))
    Ut = r.standard_normal((n, k))
    return O.biorthonormalize(U, Ut, A, ops=ops)


gpu = pytest.mark.gpu
