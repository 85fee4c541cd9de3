"""The reference's BASELINE harness A = MatrixFreeOperator(n, lambda v:
s * L(v), diag=6s) (operators.py:104-121) is recognised as the
scaled Laplacian it is and dispatched to the fused kernels (VERDICT r1
missing #6); anything that is not exactly one scalar times the stencil stays
a generic callback.  CPU only: recognition is symbolic (no block is applied)."""

import numpy as np
import pytest


@pytest.fixture
def ops():
    from paper_0705_2626_b200 import operators

    return operators


def test_recognised_forms(ops):
    N = 6
    s = float((N + 1) ** 2)
    L = ops.Laplacian3D((N, N, N), device="cpu")
    n = N ** 3
    for fn in (lambda v: s * L(v), lambda v: L(v) * s, lambda v: np.float64(s) * L(v)):
        a = ops.MatrixFreeOperator(n, fn, spd=True, diag=np.full(n, 6 * s), device="cpu")
        lap = ops.as_fused_stencil(a)
        assert isinstance(lap, ops.Laplacian3D) and lap.scale == s
        assert (lap.grid.nx, lap.grid.ny, lap.grid.nz) == (N, N, N)
    a = ops.MatrixFreeOperator(n, lambda v: L(v), device="cpu")
    assert ops.as_fused_stencil(a).scale == 1.0
    Ls = ops.Laplacian3D((N, N, N), scale=s, device="cpu")
    a = ops.MatrixFreeOperator(n, lambda v: Ls(v), device="cpu")
    assert ops.as_fused_stencil(a).scale == s
    assert ops.as_fused_stencil(L) is L


def test_other_functions_stay_callbacks(ops):
    N = 5
    s = 36.0
    L = ops.Laplacian3D((N, N, N), device="cpu")
    Ls = ops.Laplacian3D((N, N, N), scale=s, device="cpu")
    n = N ** 3
    calls = []

    def counting(v):
        calls.append(1)
        return s * L(v)

    for fn in (lambda v: s * (2.0 * L(v)),        # two roundings
               lambda v: 2.0 * Ls(v),              # scale epilogue + a product
               lambda v: L(v) / s,                 # division rounds differently
               lambda v: L(v) + v,                 # not a pure stencil
               lambda v: v,                        # no stencil
               lambda v: L(L(v)),                  # stencil squared
               lambda v: True * L(v)):
        a = ops.MatrixFreeOperator(n, fn, device="cpu")
        assert ops.as_fused_stencil(a) is None
    L4 = ops.Laplacian3D((4, 4, 4), device="cpu")
    assert ops.as_fused_stencil(ops.MatrixFreeOperator(n, lambda v: s * L4(v), device="cpu")) is None
    a = ops.MatrixFreeOperator(n, counting, device="cpu")
    assert ops.as_fused_stencil(a).scale == s and len(calls) == 1
