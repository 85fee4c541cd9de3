"""End-to-end parity of the GPU solve() against the reference's own outputs.

Criteria (SURVEY 8c parity protocol, BASELINE.json north_star):
  * eigenvalues within 1e-8 relative of the reference at matched iterations
    and of the closed form on converging runs;
  * iteration counts within +-1 of the reference on well-conditioned
    converging cases;
  * residual norms <= tol (or <= the reference's own final residual);
  * status strings identical.
"""

import numpy as np

import pytest
import torch

from tests.conftest import golden20_band, locks_in_band, trajectory_band_ok

pytestmark = pytest.mark.gpu

REL = 1e-8


@pytest.fixture(scope="module")
def pk():
    assert torch.cuda.is_available()
    import paper_0705_2626_b200 as pk

    return pk


def scaled(pk, N):
    s = float((N + 1) ** 2)
    return pk.Laplacian3D((N, N, N), scale=s), s


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)) / np.abs(np.asarray(b))


def test_golden_trajectory(pk, golden):
    """20^3 unscaled, m=10, Jacobi, tol 1e-6, seed 2 -> Converged @180
    (pkg/demos/convergence_history.csv)."""
    g = golden20_band(golden)
    a = pk.laplacian3d((20, 20, 20))
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=10, tol=1e-6, max_iter=200, seed=2))
    assert rep.status == "Converged"
    # The reference itself moves between 180 and 197 iterations under
    # rounding-level perturbations (golden20_band); hold the GPU run to that
    # band +-1, and each column's lock iteration to the widened lock band.
    its = g["all_iterations"]
    assert its.min() - 1 <= rep.iterations_used <= its.max() + 1, rep.iterations_used
    ok, lo, hi = locks_in_band(rep.lock_iterations, g["all_locks"])
    assert ok, (rep.lock_iterations, lo, hi)
    ritz = np.array([h.ritz for h in rep.history])
    ok, worst = trajectory_band_ok(ritz, g)
    assert ok, worst
    exact = pk.exact_eigenvalues((20, 20, 20), 10)
    assert rel(rep.eigenvalues, exact).max() < 1e-8
    assert rel(rep.eigenvalues, g["eigenvalues"]).max() < 1e-10
    assert np.all(rep.residual_norms <= np.maximum(1e-6, 10 * g["residual_norms"]))


def test_c1_matched_iterations(pk, golden):
    """BASELINE configs[0]: 32^3 scaled, m=4, no T, tol 1e-6, 200 it."""
    g = golden("c1_32cubed_m4_200it.npz")
    a, _ = scaled(pk, 32)
    rep = pk.solve(a, config=pk.SolverConfig(block_size=4, tol=1e-6, max_iter=200, seed=0))
    assert rep.status == str(g["status"]) == "MaxIterReached"
    assert rep.iterations_used == 200
    assert rel(rep.eigenvalues, g["eigenvalues"]).max() <= REL
    ritz = np.array([h.ritz for h in rep.history])
    assert rel(ritz, g["hist_ritz"]).max() <= 1e-6
    assert rel(ritz[-1], g["hist_ritz"][-1]).max() <= REL
    np.testing.assert_allclose(rep.residual_norms, g["residual_norms"], rtol=0.5)


@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_seeds_1_2_matched_iterations(pk, golden, name, seed):
    """Seeds 1 and 2 of the BASELINE shapes (SURVEY 8c harness rules) against
    the real reference at a matched iteration count (make_seeds.py): status,
    iterations, Ritz values at 1e-8 relative, the whole Ritz history at 1e-6,
    residual norms within a factor of two."""
    N, m, jac, diag_b, tol, max_iter = {
        "c1": (32, 4, False, False, 1e-6, 120), "c2": (48, 10, True, False, 1e-8, 60),
        "c3": (40, 16, True, False, 1e-6, 60), "c5": (24, 32, True, True, 1e-6, 40)}[name]
    g = golden("seeds12.npz")
    k = f"{name}_s{seed}_"
    a, _ = scaled(pk, N)
    b = None
    if diag_b:
        b = pk.DiagonalOperator(
            np.random.Generator(np.random.PCG64(1000 + seed)).uniform(1.0, 2.0, N ** 3))
    rep = pk.solve(a, b=b, t=pk.jacobi_preconditioner(a) if jac else None,
                   config=pk.SolverConfig(block_size=m, tol=tol, max_iter=max_iter, seed=seed))
    assert rep.status == str(g[k + "status"]) == "MaxIterReached"
    assert rep.iterations_used == int(g[k + "iterations_used"])
    assert rel(rep.eigenvalues, g[k + "eigenvalues"]).max() <= REL
    ritz = np.array([h.ritz for h in rep.history])
    assert rel(ritz, g[k + "hist_ritz"]).max() <= 1e-6
    assert np.array_equal(rep.converged, g[k + "converged"])
    np.testing.assert_allclose(rep.residual_norms, g[k + "residual_norms"], rtol=1.0)


def test_c1_converging_time_to_tol(pk, golden):
    """C1 with max_iter=1000 converges.  Its triple eigenvalue cluster makes
    the converged iteration count chaotic: the reference itself, with its
    operator scaled by 1..8 ulp, ends anywhere in 359..612 iterations and
    sometimes as BasisFallback (golden c1_1000it_band.npz); with +-1 ulp noise
    in its Ritz-update coefficients, in 338..427 (c1_1000it_band_coef.npz).
    The GPU run is held to the union band (+-10%) and to the closed form."""
    g = golden("c1_32cubed_m4_1000it.npz")
    band = golden("c1_1000it_band.npz")
    band2 = golden("c1_1000it_band_coef.npz")
    a, s = scaled(pk, 32)
    rep = pk.solve(a, config=pk.SolverConfig(block_size=4, tol=1e-6, max_iter=1000, seed=0))
    assert rep.status == "Converged" or rep.status.startswith("BasisFallback")
    its = np.concatenate([[int(g["iterations_used"])], band["iterations"], band2["iterations"]])
    assert 0.9 * its.min() <= rep.iterations_used <= 1.1 * its.max(), rep.iterations_used
    exact = pk.exact_eigenvalues((32, 32, 32), 4, scale=s)
    assert rel(rep.eigenvalues, exact).max() <= REL
    assert rel(rep.eigenvalues, g["eigenvalues"]).max() <= REL
    # the exit-refresh residual of a soft-locked member of the triple cluster
    # is not controlled after its lock (the cluster's Ritz vectors keep
    # rotating): the reference's own band spans 4e-7 .. 4.6e-5 (two orders of
    # magnitude); hold it to two orders above the band's worst run
    rmax = max(float(g["residual_norms"].max()), float(band["residual_max"].max()))
    assert np.all(rep.residual_norms <= np.maximum(1e-6, 100 * rmax))
    locked = [h.residual_norms[j] for h in rep.history for j in h.locked_now]
    assert all(r < 1e-6 for r in locked)   # every lock on a residual below tol


def test_small_laplacian_closed_form(pk, golden):
    g = golden("lap5_m4_jacobi.npz")
    a = pk.laplacian3d((5, 5, 5))
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=4, tol=1e-8, max_iter=300))
    assert rep.all_converged
    assert abs(rep.iterations_used - int(g["iterations_used"])) <= 1
    np.testing.assert_allclose(rep.eigenvalues, pk.exact_eigenvalues((5, 5, 5), 4), rtol=1e-8)
    # test_lobpcg.py:211-225 bounds the final residuals by 1.01 tol; the exit
    # refresh rotates the triple cluster, and the reference's own final
    # residual reaches 1.114e-8 with its operator scaled by 1 +- k ulp,
    # |k| <= 16 (lap5_band.npz): that band bounds ours
    band = golden("lap5_band.npz")
    assert np.all(rep.residual_norms <= 1.01 * max(1e-8, float(band["residual_max"].max())))
    locked = [h.residual_norms[j] for h in rep.history for j in h.locked_now]
    assert all(r < 1e-8 for r in locked)
    x = rep.eigenvectors
    assert np.abs(x.T @ x - np.eye(4)).max() <= 1e-8


def test_lap10(pk, golden):
    g = golden("lap10_m5_jacobi.npz")
    a = pk.laplacian3d((10, 10, 10))
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=5, tol=1e-8, max_iter=300))
    assert rep.status == str(g["status"])
    assert abs(rep.iterations_used - int(g["iterations_used"])) <= 1
    assert rel(rep.eigenvalues, g["eigenvalues"]).max() <= 1e-10


def test_generalized_diag_pencil(pk, golden):
    """Generic A (DiagonalOperator callback) + diagonal B fused as weights
    (test_lobpcg.py:371-382)."""
    g = golden("diag_pencil_n30_m4.npz")
    n = 30
    a = pk.DiagonalOperator(np.arange(1.0, n + 1.0))
    b = pk.DiagonalOperator(g["bdiag"])
    rep = pk.solve(a, b=b, config=pk.SolverConfig(block_size=4, tol=1e-10, max_iter=300))
    assert rep.all_converged
    np.testing.assert_allclose(rep.eigenvalues, g["dense_vals"], rtol=1e-10)
    x = rep.eigenvectors
    assert np.abs(x.T @ (g["bdiag"][:, None] * x) - np.eye(4)).max() <= 1e-8
    assert abs(rep.iterations_used - int(g["iterations_used"])) <= 2


def test_laplacian_diag_b(pk, golden):
    """12^3 scaled Laplacian, B = diag(U[1,2]), Jacobi (C5 code path)."""
    g = golden("lap12_m6_diagB.npz")
    a, _ = scaled(pk, 12)
    rep = pk.solve(a, b=pk.DiagonalOperator(g["bdiag"]), t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=6, tol=1e-6, max_iter=150, seed=0))
    assert rep.status == str(g["status"])
    assert abs(rep.iterations_used - int(g["iterations_used"])) <= 1
    assert rel(rep.eigenvalues, g["eigenvalues"]).max() <= REL
    assert np.all(np.abs(rep.lock_iterations - g["lock_iterations"]) <= 1)


def test_c3_reduced(pk, golden):
    """48^3, m=16, Jacobi, tol 1e-6, 300 it: partial soft locking (k < m)."""
    g = golden("c3r_48cubed_m16_300it.npz")
    a, _ = scaled(pk, 48)
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=16, tol=1e-6, max_iter=300, seed=0))
    assert rep.status == str(g["status"])
    assert rep.iterations_used == int(g["iterations_used"])
    assert rel(rep.eigenvalues, g["eigenvalues"]).max() <= REL
    # columns right at the lock threshold: the reference's own 1-2 ulp
    # perturbations lock 9 or 10 of 16 (golden c3r_band.npz)
    band = golden("c3r_band.npz")
    counts = np.concatenate([[int(g["converged"].sum())], band["converged"]])
    assert counts.min() <= int(rep.converged.sum()) <= counts.max()


def test_c5_reduced(pk, golden):
    """32^3, m=64, diagonal B, Jacobi, 200 it (large-block Gram path)."""
    g = golden("c5r_32cubed_m64_diagB_200it.npz")
    N = 32
    bd = np.random.Generator(np.random.PCG64(1000)).uniform(1.0, 2.0, N ** 3)
    a, _ = scaled(pk, N)
    rep = pk.solve(a, b=pk.DiagonalOperator(bd), t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=64, tol=1e-6, max_iter=200, seed=0))
    assert rep.status == str(g["status"])
    assert rel(rep.eigenvalues, g["eigenvalues"]).max() <= REL
    assert abs(int(rep.converged.sum()) - int(g["converged"].sum())) <= 1


def test_single_point_and_exact_guess(pk):
    rep = pk.solve(pk.laplacian3d((1, 1, 1)), config=pk.SolverConfig(block_size=1))
    assert rep.all_converged and rep.iterations_used == 0
    np.testing.assert_allclose(rep.eigenvalues, [6.0], rtol=1e-14)
    a = pk.DiagonalOperator(np.arange(1.0, 11.0))
    rep = pk.solve(a, x0=np.eye(10)[:, :3], config=pk.SolverConfig(block_size=3, tol=1e-8))
    assert rep.iterations_used == 0 and rep.all_converged
    np.testing.assert_allclose(rep.eigenvalues, [1.0, 2.0, 3.0], atol=1e-12)


def test_input_validation(pk):
    a = pk.laplacian3d((4, 4, 4))
    with pytest.raises(ValueError):
        pk.solve(a, x0=np.ones((64, 2)), config=pk.SolverConfig(block_size=3))
    x0 = np.random.default_rng(0).standard_normal((64, 2))
    x0[3, 1] = np.nan
    with pytest.raises(ValueError):
        pk.solve(a, x0=x0, config=pk.SolverConfig(block_size=2))
    with pytest.raises(ValueError):
        pk.solve(a, config=pk.SolverConfig(block_size=65))
    with pytest.raises(ValueError):
        pk.SolverConfig(tol=0.0).validate()
    with pytest.raises(ValueError, match="shape"):
        pk.solve(a, t=lambda w: w[:, :1], config=pk.SolverConfig(block_size=3, max_iter=5))
    with pytest.raises(ValueError, match="non-finite"):
        pk.solve(a, t=lambda w: w * float("nan"), config=pk.SolverConfig(block_size=3, max_iter=5))
    with pytest.raises(ValueError, match="degenerate"):
        pk.solve(a, x0=np.ones((64, 2)), config=pk.SolverConfig(block_size=2))


def test_generic_preconditioner_callback(pk):
    """A user lambda preconditioner (CUDA tensor in, CUDA tensor out) gives
    the same run as the built-in Jacobi it imitates."""
    a = pk.laplacian3d((8, 8, 8))
    cfg = pk.SolverConfig(block_size=4, tol=1e-8, max_iter=200)
    r1 = pk.solve(a, t=pk.jacobi_preconditioner(a), config=cfg)
    r2 = pk.solve(a, t=lambda w: (1.0 / 6.0) * w, config=cfg)
    # the fused and the callback paths round differently (different Gram
    # kernels), so the runs agree to rounding, not bit for bit
    assert abs(r1.iterations_used - r2.iterations_used) <= 2
    np.testing.assert_allclose(r1.eigenvalues, r2.eigenvalues, rtol=1e-10)


def test_bitwise_reproducible(pk):
    a, _ = scaled(pk, 24)
    cfg = pk.SolverConfig(block_size=6, tol=1e-8, max_iter=60, seed=3)
    t = pk.jacobi_preconditioner(a)
    r1 = pk.solve(a, t=t, config=cfg)
    r2 = pk.solve(a, t=t, config=cfg)
    assert np.array_equal(r1.eigenvalues, r2.eigenvalues)
    assert np.array_equal(r1.eigenvectors, r2.eigenvectors)


def test_relative_tol_and_history_flags(pk):
    a = pk.laplacian3d((6, 6, 6))
    rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=3, tol=1e-8, max_iter=300,
                                          relative_tol=True, lock_history=False,
                                          check_invariants=True))
    assert rep.all_converged
    assert all(h.ritz is None for h in rep.history)
    np.testing.assert_allclose(rep.eigenvalues, pk.exact_eigenvalues((6, 6, 6), 3), rtol=1e-8)


def test_interleaved_runs_match_solo_runs(pk):
    """Two LOBPCGRun objects stepped alternately (they share the library's
    side stream, workspaces and caches) give the same histories as when each
    runs alone."""
    from paper_0705_2626_b200 import lobpcg as lb

    def make(N, m, seed):
        a, _ = scaled(pk, N)
        cfg = pk.SolverConfig(block_size=m, tol=1e-8, max_iter=30, seed=seed)
        return lambda: lb.LOBPCGRun(a, t=pk.jacobi_preconditioner(a), config=cfg)

    mk1, mk2 = make(24, 10, 1), make(20, 8, 2)
    solo = []
    for mk in (mk1, mk2):
        r = mk()
        while r.step():
            pass
        solo.append(np.array([h.ritz for h in r.history]))
    r1, r2 = mk1(), mk2()
    more1 = more2 = True
    while more1 or more2:
        if more1:
            more1 = r1.step()
        if more2:
            more2 = r2.step()
    for r, ref in zip((r1, r2), solo):
        got = np.array([h.ritz for h in r.history])
        assert got.shape == ref.shape and np.array_equal(got, ref)


def test_timer_entered_mid_run_matches_solo(pk):
    """A step that leaves the native loop (a timer entered mid-run sends it
    down the Python path) must read the reductions the native step's passes
    wrote into the mapped host buffers, not stale device copies."""
    N, m = 48, 10
    a = pk.Laplacian3D((N, N, N), scale=float((N + 1) ** 2))
    t = pk.jacobi_preconditioner(a)
    cfg = pk.SolverConfig(block_size=m, tol=1e-8, max_iter=30, seed=0)
    solo = pk.solve(a, t=t, config=cfg)
    run = pk.LOBPCGRun(a, t=t, config=cfg)
    for _ in range(6):
        assert run.step()
    assert run._native is not None

    def timer(name, fn):
        return fn()

    with pk.device_options(timer=timer):
        for _ in range(4):
            run.step()
    while run.step():
        pass
    rep = run.report()
    assert rep.status == solo.status and rep.iterations_used == solo.iterations_used
    a_ = np.array([h.ritz for h in rep.history])
    b_ = np.array([h.ritz for h in solo.history])
    np.testing.assert_allclose(a_, b_, rtol=1e-12)


_REPAIR_CASE = """
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_0705_2626_b200 as pk
N, m = 64, 10
a = pk.Laplacian3D((N, N, N), scale=float((N + 1) ** 2))
run = pk.LOBPCGRun(a, t=pk.jacobi_preconditioner(a),
                   config=pk.SolverConfig(block_size=m, tol=1e-8, max_iter=150, seed=0))
while run.step():
    pass
rep = run.report()
print(json.dumps(dict(repairs=run.drift_repairs, status=rep.status, it=rep.iterations_used,
                      ritz=[list(map(float, h.ritz)) for h in rep.history],
                      eig=list(map(float, rep.eigenvalues)))))
"""


def test_native_drift_repair_matches_python_repair():
    """The drift repair inside the native loop (one X^T A X Gram, the folded
    rotation, one no-update F1 pass) against the Python repair path
    (B2L_NATIVE_REPAIR=0: rotations + Grams + residual as separate kernels)
    on the same problem: same repair count, status and iterations, Ritz
    trajectory equal to rounding."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parents[1])
    out = {}
    for mode in ("1", "0"):
        env = dict(os.environ, B2L_NATIVE_REPAIR=mode)
        r = subprocess.run([sys.executable, "-c", _REPAIR_CASE.format(root=root)], env=env,
                           capture_output=True, text=True, timeout=600, cwd=root)
        assert r.returncode == 0, r.stderr[-2000:]
        out[mode] = json.loads(r.stdout.strip().splitlines()[-1])
    nat, py = out["1"], out["0"]
    # the two repairs round differently (one folded rotation vs two applied
    # ones), and later drift tests against 1e-11 are decided on drift that
    # accumulated from rounding: the repair count may move by one or two
    assert nat["repairs"] >= 1 and py["repairs"] >= 1
    assert abs(nat["repairs"] - py["repairs"]) <= 2
    assert nat["status"] == py["status"] and nat["it"] == py["it"]
    np.testing.assert_allclose(np.array(nat["ritz"]), np.array(py["ritz"]), rtol=1e-7)
    np.testing.assert_allclose(nat["eig"], py["eig"], rtol=1e-9)


@pytest.mark.parametrize("diag_b,rel_tol,m", [(False, False, 10), (True, True, 6), (False, True, 16)])
def test_native_repair_under_forced_drift(pk, monkeypatch, diag_b, rel_tol, m):
    """The native drift repair in the configurations the steady state runs
    (identity / diagonal B, absolute / relative tol, m = 6 / 10 / 16, with
    columns locking on the way): with the drift limit lowered to 1e-15 the
    repair fires every few iterations; the native loop (the repair inside
    b2l_fast_iteration) and the Python repair path must land on the same
    eigenpairs."""
    from paper_0705_2626_b200 import lobpcg as lb

    N = 24
    s = float((N + 1) ** 2)
    a = pk.Laplacian3D((N, N, N), scale=s)
    b = None
    if diag_b:
        b = pk.DiagonalOperator(np.random.Generator(np.random.PCG64(4)).uniform(1.0, 2.0, N ** 3))
    cfg = pk.SolverConfig(block_size=m, tol=1e-7 if rel_tol else 1e-6, max_iter=60, seed=1,
                          relative_tol=rel_tol)
    monkeypatch.setattr(lb, "DRIFT_LIMIT", 1e-15)
    out = []
    for fused in (True, False):
        with pk.device_options(fused=fused):
            run = pk.LOBPCGRun(a, b=b, t=pk.jacobi_preconditioner(a), config=cfg)
            assert (run._native is not None) == fused
            while run.step():
                pass
            out.append((run.report(), run.drift_repairs))
    (nat, nrep), (py, prep) = out
    assert nrep >= 5 and prep >= 5, (nrep, prep)
    assert nat.status == py.status
    assert abs(nat.iterations_used - py.iterations_used) <= 1
    np.testing.assert_allclose(nat.eigenvalues, py.eigenvalues, rtol=1e-9)
    assert np.any(~nat.history[-1].active) or nat.iterations_used == 60


@pytest.mark.parametrize("name,N,m,tol", [("n20", 20, 10, 1e-6), ("n16", 16, 8, 1e-8)])
def test_seed_sweep_against_reference(pk, golden, name, N, m, tol):
    """Seeds 0..15 run to convergence, against the REAL reference on the same
    seeds (seed_sweep.npz, make_seed_sweep.py): the reference converges on
    every seed (one BasisFallback on 20^3) in 188..379 / 174..241 iterations.
    The B200 path must not fail or stall where the reference converges: every
    seed reaches the tolerance and the closed form, no run is much longer than
    the reference's longest, and the median sits on the reference's.  (This
    pins the Rayleigh-Ritz step's congruence and cluster gap -- with the
    explicit-inverse congruence one 16^3 run stalls at max_iter, with the
    cluster gap at the tolerance one 20^3 run stalls for 200 iterations -- and
    the F1 pair kernel's narrow-stage scratch layout, whose bug turned every
    dropped-P fallback of these runs into Failed(BasisDegeneracy).)"""
    g = golden("seed_sweep.npz")
    ref_its = g[name + "_iterations"]
    s = float((N + 1) ** 2)
    a = pk.Laplacian3D((N, N, N), scale=s)
    exact = pk.exact_eigenvalues((N, N, N), m, scale=s)
    its = []
    for seed in range(16):
        rep = pk.solve(a, t=pk.jacobi_preconditioner(a),
                       config=pk.SolverConfig(block_size=m, tol=tol, max_iter=1500, seed=seed))
        assert rep.status == "Converged" or rep.status.startswith("BasisFallback"), \
            (seed, rep.status)
        assert rep.all_converged, (seed, rep.status)
        assert rel(rep.eigenvalues, exact).max() <= REL, seed
        its.append(rep.iterations_used)
    assert max(its) <= 1.25 * ref_its.max(), (max(its), int(ref_its.max()))
    assert min(its) >= 0.9 * ref_its.min(), (min(its), int(ref_its.min()))
    assert abs(np.median(its) - np.median(ref_its)) <= 0.05 * np.median(ref_its), \
        (np.median(its), np.median(ref_its))


def test_stalled_run_is_refreshed(pk):
    """24^3, m = 9 (the block cuts a triple eigenvalue), absolute tol 1e-8 at
    |A| = 7,500, seed 1757: the reference converges at iteration 752 (oracle,
    bit-exact).  On the fused path the carried diag(Lambda) / AX drift above
    the tolerance around iteration 420 and two columns would stall at
    residuals of 1e-7 until max_iter; the stall watch recomputes A X, A P and
    runs the reference's own repair on them, after which the run converges."""
    N, m = 24, 9
    s = float((N + 1) ** 2)
    a = pk.Laplacian3D((N, N, N), scale=s)
    run = pk.LOBPCGRun(a, t=pk.jacobi_preconditioner(a),
                       config=pk.SolverConfig(block_size=m, tol=1e-8, max_iter=3000, seed=1757))
    while run.step():
        pass
    rep = run.report()
    assert rep.all_converged, rep.status
    assert rep.iterations_used <= 1.25 * 752, rep.iterations_used
    assert run.ax_refreshes <= 3
    assert rel(rep.eigenvalues, pk.exact_eigenvalues((N, N, N), m, scale=s)).max() <= REL
    # a healthy run never triggers the watch
    run2 = pk.LOBPCGRun(a, t=pk.jacobi_preconditioner(a),
                        config=pk.SolverConfig(block_size=m, tol=1e-8, max_iter=3000, seed=1759))
    while run2.step():
        pass
    assert run2.ax_refreshes == 0 and run2.report().all_converged


def test_c1_outcome_distribution_matches_reference(pk, golden):
    """A single converging C1 run lands anywhere in the reference's chaotic
    band, which cannot catch a change of behaviour.  Here the GPU runs the
    SAME 32 perturbed problems as the reference's own distribution
    (c1_band32.npz: operator scale (N+1)^2 (1 + k 2^-52), k = +-1..16; the
    kernel's scale epilogue rounds the same single product s * L(v)), and
    the outcome distributions must agree: how many runs converge (the rest
    end in BasisFallback), how many lock their second column by iteration
    215, and the median iteration count.  (A plain tridiagonal QR in the
    Rayleigh-Ritz step, B2L_RR_ALIGN=0, fails this: 10 of 32 converge against
    the reference's 27 -- DESIGN.md; the default aligned QR gives 32 / 22, the
    dsyevr sequence 24 / 15-19.)"""
    band = golden("c1_band32.npz")
    N = 32
    base = float((N + 1) ** 2)
    its, conv, early = [], 0, 0
    for k in band["ulps"]:
        a = pk.Laplacian3D((N, N, N), scale=base * (1.0 + int(k) * 2.0 ** -52))
        rep = pk.solve(a, config=pk.SolverConfig(block_size=4, tol=1e-6, max_iter=1000, seed=0))
        assert rep.status == "Converged" or rep.status.startswith("BasisFallback"), rep.status
        its.append(rep.iterations_used)
        conv += rep.status == "Converged"
        early += sorted(rep.lock_iterations)[1] <= 215
    ref_conv = int(sum(str(x) == "Converged" for x in band["status"]))
    ref_early = int(sum(sorted(l)[1] <= 215 for l in band["lock_iterations"]))
    n = len(its)
    # two independent binomials over 32 runs at p ~ 0.8 / 0.7: the sd of their
    # difference is ~3.2 / ~3.7 runs; hold both to 3 sd (the plain QR's 10 vs
    # 27 converged is 5 sd away)
    assert abs(conv - ref_conv) <= 10, (conv, ref_conv, n)
    assert abs(early - ref_early) <= 11, (early, ref_early, n)
    assert abs(np.median(its) - np.median(band["iterations"])) <= 0.1 * np.median(band["iterations"])


def test_c1_outcome_distribution_128_runs(pk, golden):
    """The same comparison over 128 perturbed C1@1000 problems (k = +-1..64;
    c1_band128.npz from the REAL reference: 117 of 128 end Converged, 107 lock
    their second column by iteration 215, median 408 iterations, quartiles
    404 / 411).  Every run must reach the tolerance on all four pairs; the
    GPU's median iteration count must sit on the reference's, and the share
    of runs that never need a basis fallback and of early second locks must
    stay in the reference's class (measured: 128 / 83 with the default
    aligned-QR Rayleigh-Ritz step, 97 / 68 with the dsyevr sequence, 93 / 61
    with the MRRR stages, 39 / 17 with a plain tridiagonal QR).  What the
    alignment is and why it matters: DESIGN.md."""
    band = golden("c1_band128.npz")
    N = 32
    base = float((N + 1) ** 2)
    its, conv, early = [], 0, 0
    for k in band["ulps"]:
        s = base * (1.0 + int(k) * 2.0 ** -52)
        a = pk.Laplacian3D((N, N, N), scale=s)
        rep = pk.solve(a, config=pk.SolverConfig(block_size=4, tol=1e-6, max_iter=1000, seed=0))
        assert rep.status == "Converged" or rep.status.startswith("BasisFallback"), rep.status
        assert bool(np.all(rep.converged)), (int(k), rep.status)
        exact = pk.exact_eigenvalues((N, N, N), 4, scale=s)
        np.testing.assert_allclose(rep.eigenvalues, exact, rtol=1e-8)
        its.append(rep.iterations_used)
        conv += rep.status == "Converged"
        early += sorted(rep.lock_iterations)[1] <= 215
    ref_its = np.asarray(band["iterations"])
    assert abs(np.median(its) - np.median(ref_its)) <= 0.03 * np.median(ref_its), np.median(its)
    assert conv >= 97, (conv, "reference 117 of 128; dsyevr sequence 97; plain QR 39")
    assert early >= 68, (early, "reference 107 of 128; dsyevr sequence 68; plain QR 17")
