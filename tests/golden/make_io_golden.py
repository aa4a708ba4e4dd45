"""Golden files for the I/O formats, written by the
REFERENCE's own krecycle.io from fixed inputs -- run in the build container
only (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_io_golden.py

* history_ref.csv  -- krecycle.io.history_write of two fixed histories
* space_ref.krsp   -- krecycle.io.recycle_save of a fixed (U, Ut) pair
  (n = 37, k = 3, seeded normal bases; images rebuilt on load)
"""
import os

import numpy as np
from krecycle import io as rio
from krecycle.recycling import RecycleSpace
from krecycle.solvers import ConvergenceHistory

HERE = os.path.dirname(os.path.abspath(__file__))


def fixed_histories(cls):
    h1 = cls(solver="rbicgstab", resid=[1.0, 0.5, 1.0 / 3.0, 2.5e-9],
             matvecs=[0, 2, 4, 6], seconds=[0.0, 0.00123, 0.0024567, 0.0037],
             status="converged")
    h2 = cls(solver="bicgstab", resid=[1.0, 0.125], matvecs=[1, 3],
             seconds=[0.0, 1.5e-7], status="max_itn")
    h3 = cls(solver="rbicg")   # empty history: summary row with nan
    return [h1, h2, h3]


def fixed_space():
    r = np.random.default_rng(2024)
    return r.standard_normal((37, 3)), r.standard_normal((37, 3))


if __name__ == "__main__":
    rio.history_write(os.path.join(HERE, "history_ref.csv"), fixed_histories(ConvergenceHistory))
    U, Ut = fixed_space()
    space = RecycleSpace(U=U, Ut=Ut, C=U, Ct=Ut, Dc=np.ones(3), Chat=Ut, Ccheck=U)
    rio.recycle_save(os.path.join(HERE, "space_ref.krsp"), space)
    print("wrote history_ref.csv, space_ref.krsp")
