"""CPU-side checks of the boundary: the C-ABI library loads, exports every
symbol include/b200lobpcg.h declares, and the host-side logic (small dense
algebra, closed form) matches the reference's known answers.  No GPU needed.
"""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "b200lobpcg.h").read_text()
    return sorted(set(re.findall(r"\b(b2l_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_0705_2626_b200 import _lib

    lib = _lib.load()
    syms = header_symbols()
    assert {"b2l_stencil7", "b2l_gram", "b2l_residual", "b2l_update"} <= set(syms)
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} lacks a ctypes signature"
    assert lib.b2l_abi_version() == _lib.ABI_VERSION


def test_library_is_sm100a_only():
    import subprocess

    from paper_0705_2626_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for bad in ("sm_80", "sm_90", "sm_103"):
        assert bad not in out


def test_error_path_reports_message():
    from paper_0705_2626_b200 import _lib

    lib = _lib.load()
    # odd ld is rejected before any CUDA call
    rc = lib.b2l_stencil7(None, None, 4, 4, 4, 3, None, 0, 0, 1.0, None)
    assert rc != 0
    assert b"ld must be even" in lib.b2l_last_error()


def test_cholesky_known_answers():
    from paper_0705_2626_b200.small import NotSPD, cholesky

    # test_multivec.py:110-113 style hand example
    g = np.array([[4.0, 2.0], [2.0, 5.0]])
    np.testing.assert_allclose(cholesky(g), [[2.0, 1.0], [0.0, 2.0]])
    # dependent second column -> pivot 1
    g = np.array([[1.0, 1.0, 0.0], [1.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    with pytest.raises(NotSPD) as e:
        cholesky(g)
    assert e.value.pivot == 1
    # pivot floor
    g = np.array([[1.0, 1.0 - 1e-10], [1.0 - 1e-10, 1.0]])
    cholesky(g)
    with pytest.raises(NotSPD):
        cholesky(g, pivot_floor=1e-8)


def test_gen_sym_eig_matches_oracle():
    from oracle import lobpcg_oracle as orc
    from paper_0705_2626_b200.small import gen_sym_eig

    rng = np.random.Generator(np.random.PCG64(3))
    for k in (3, 7, 12):
        a = rng.standard_normal((k, k))
        a = a + a.T
        b = rng.standard_normal((k, k))
        b = b @ b.T + k * np.eye(k)
        v1, c1 = gen_sym_eig(a, b, 2)
        v2, c2 = orc.pencil_smallest(a, b, 2)
        # dpotrf vs the reference's row-wise Cholesky: rounding-level only
        np.testing.assert_allclose(v1, v2, rtol=1e-13)
        np.testing.assert_allclose(np.abs(c1), np.abs(c2), rtol=1e-10, atol=1e-12)


def test_scaled_cholesky_inverse_orthonormalizes():
    from paper_0705_2626_b200.small import scaled_cholesky

    rng = np.random.Generator(np.random.PCG64(5))
    x = rng.standard_normal((200, 6)) * np.array([1e-3, 1, 10, 1e3, 2, 5])
    reff, minv = scaled_cholesky(x.T @ x)
    q = x @ minv
    np.testing.assert_allclose(q.T @ q, np.eye(6), atol=1e-12)
    np.testing.assert_allclose(q @ reff, x, rtol=1e-12, atol=1e-12)


def test_exact_eigenvalues_match_oracle_closed_form():
    from oracle import lobpcg_oracle as orc
    from paper_0705_2626_b200.problems import exact_eigenvalues

    for dims, m in [((20, 20, 20), 10), ((8, 9, 10), 10), ((464, 464, 464), 8)]:
        np.testing.assert_allclose(exact_eigenvalues(dims, m), orc.closed_form_smallest(*dims, m),
                                   rtol=1e-15)
    s = float(129 ** 2)
    np.testing.assert_allclose(exact_eigenvalues((128,) * 3, 10, scale=s)[0],
                               s * 12 * np.sin(np.pi / 258) ** 2, rtol=1e-14)


def test_iter_state_layout_matches_library():
    import ctypes

    from paper_0705_2626_b200 import _lib

    lib = _lib.load()
    assert lib.b2l_iter_state_size() == ctypes.sizeof(_lib.b2l_iter_state)
