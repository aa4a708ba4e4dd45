"""The oracle behind the package's API names -- TEST INFRASTRUCTURE.

``oracle_api(ops)`` exposes the oracle restatement (oracle/krylov.py) with
the call signatures of paper_1406_2831_b200 / krecycle, so the shared
sequence policy (paper_1406_2831_b200/sequence.py) can drive it as a
backend.  Only tests/, smoke() and bench.py's CPU legs use it.
"""

from __future__ import annotations

import types


def oracle_api(ops=None):
    import paper_1406_2831_b200 as P
    from oracle import krylov as O
    from oracle.ops import CsrOperand, RefOps
    ops = ops or RefOps()
    cache = {}

    def from_csr(A):
        if id(A) not in cache:
            cache[id(A)] = (A, CsrOperand.of(A))
        return cache[id(A)][1]

    return types.SimpleNamespace(
        SparseMatrix=types.SimpleNamespace(from_csr=from_csr),
        CountingOperator=P.CountingOperator, SolverConfig=P.SolverConfig,
        rbicg_solve=lambda A, b, **kw: O.rbicg(A, b, ops=ops, **kw),
        rbicgstab_solve=lambda A, b, **kw: O.rbicgstab(A, b, ops=ops, **kw),
        bicgstab_solve=lambda A, b, **kw: O.bicgstab(A, b, ops=ops, **kw),
        update_recycle_space=lambda A, c, p, k, **kw: O.update_recycle_space(
            A, c, p, k, ops=ops, **kw),
        refresh_images=lambda S, A, **kw: O.refresh_images(S, A, ops=ops, **kw))
