"""blockeig-bench on the B200 path, following the
reference's tests/test_cli.py: flags and exit codes, the JSON record, the
history CSV and the LOBX eigenvector container (CPU), and in-process runs on
the GPU (JSON/CSV/LOBX outputs, constraints flow, sweeps)."""

import json

import numpy as np
import pytest
import torch

from paper_0705_2626_b200.cli import (
    EXIT_ERROR,
    EXIT_OK,
    EXIT_PARTIAL,
    build_parser,
    load_eigenvectors,
    main,
    save_eigenvectors,
)

gpu = pytest.mark.gpu


def run_json(tmp_path, extra, name="out.json"):
    path = tmp_path / name
    code = main(extra + ["-json", str(path), "-verb", "0"])
    return code, (json.loads(path.read_text()) if path.exists() else None)


# ------------------------------------------------------------ CPU: parsing


def test_parser_defaults():
    a = build_parser().parse_args([])
    assert (a.n, a.m, a.seed, a.tol, a.itr) == ([10, 10, 10], 5, 0, 1e-6, 200)
    assert (a.pcgitr, a.precond, a.verb, a.full_out) == (0, "jacobi", 1, 0)
    assert (a.scaled, a.device, a.ngpu) == (0, None, 1)


def test_parser_vrand_and_n_eigs_are_synonyms():
    assert build_parser().parse_args(["-vrand", "7"]).m == 7
    assert build_parser().parse_args(["-n_eigs", "7"]).m == 7


def test_unknown_flag_and_invalid_values():
    assert main(["-bogus", "3"]) == EXIT_ERROR
    for bad in (["-n", "0", "1", "1"], ["-tol", "0"], ["-tol", "-1e-6"], ["-itr", "0"],
                ["-vrand", "0"], ["-pcgitr", "-1"], ["-precond", "ilu"], ["-verb", "-1"],
                ["-ngpu", "0"]):
        assert main(bad) == EXIT_ERROR, bad


def test_sweep_value_validation():
    args = ["-n", "3", "3", "3", "-verb", "0", "-sweep", "inner_iter"]
    assert main(args + ["-sweep_values", ""]) == EXIT_ERROR
    assert main(args + ["-sweep_values", "1,x"]) == EXIT_ERROR
    assert main(args + ["-sweep_values", "-2"]) == EXIT_ERROR
    bs = ["-n", "3", "3", "3", "-verb", "0", "-sweep", "block_size"]
    assert main(bs + ["-sweep_values", "0,2"]) == EXIT_ERROR


# ---------------------------------------------------------- CPU: LOBX files


def test_eigenvector_file_round_trip(tmp_path):
    x = np.random.Generator(np.random.PCG64(5)).standard_normal((40, 3))
    path = tmp_path / "vecs.bin"
    save_eigenvectors(path, x)
    np.testing.assert_array_equal(load_eigenvectors(path), x)
    # byte layout: <4sIQQ header, then column-major little-endian f64
    raw = path.read_bytes()
    assert raw[:4] == b"LOBX" and int.from_bytes(raw[4:8], "little") == 1
    assert int.from_bytes(raw[8:16], "little") == 40 and int.from_bytes(raw[16:24], "little") == 3
    np.testing.assert_array_equal(np.frombuffer(raw[24:], "<f8"), x.ravel(order="F"))


def test_eigenvector_file_error_cases(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"\x00" * 4)
    with pytest.raises(ValueError, match="truncated"):
        load_eigenvectors(bad)
    good = tmp_path / "good.bin"
    save_eigenvectors(good, np.ones((4, 2)))
    raw = bytearray(good.read_bytes())
    (tmp_path / "magic.bin").write_bytes(b"XXXX" + bytes(raw[4:]))
    with pytest.raises(ValueError, match="magic"):
        load_eigenvectors(tmp_path / "magic.bin")
    ver = bytearray(raw)
    ver[4] = 99
    (tmp_path / "version.bin").write_bytes(bytes(ver))
    with pytest.raises(ValueError, match="version"):
        load_eigenvectors(tmp_path / "version.bin")
    (tmp_path / "short.bin").write_bytes(bytes(raw[:-8]))
    with pytest.raises(ValueError):
        load_eigenvectors(tmp_path / "short.bin")
    with pytest.raises(ValueError):
        save_eigenvectors(tmp_path / "x.bin", np.ones(3))


def test_reference_lobx_interoperates(tmp_path, golden):
    """A file in the reference's exact layout loads, and ours is byte-equal
    to what the reference writer produces for the same block
    (cli.py:63-75: header then tobytes(order='F'))."""
    import struct

    x = np.arange(12.0).reshape(4, 3) / 7.0
    ref = struct.pack("<4sIQQ", b"LOBX", 1, 4, 3) + x.astype("<f8").tobytes(order="F")
    save_eigenvectors(tmp_path / "ours.bin", x)
    assert (tmp_path / "ours.bin").read_bytes() == ref


# ------------------------------------------------------------ GPU: runs


@pytest.fixture
def needs_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")


@gpu
def test_block_larger_than_grid_rejected(needs_gpu):
    assert main(["-n", "2", "2", "2", "-vrand", "9", "-verb", "0"]) == EXIT_ERROR


@gpu
def test_single_point_grid_run(needs_gpu, tmp_path):
    code, rec = run_json(tmp_path, ["-n", "1", "1", "1", "-vrand", "1"])
    assert code == EXIT_OK and rec["iterations"] == 0
    np.testing.assert_allclose(rec["eigenvalues"], [6.0], rtol=1e-12)
    assert rec["status"] == "Converged" and rec["rel_errors"][0] < 1e-12


@gpu
def test_json_record_schema(needs_gpu, tmp_path):
    code, rec = run_json(tmp_path, ["-n", "4", "4", "4", "-vrand", "3", "-tol", "1e-8"])
    assert code == EXIT_OK
    assert set(rec) == {"config", "eigenvalues", "analytic", "rel_errors", "iterations",
                        "history", "setup_sec", "solve_sec", "status"}
    assert rec["config"]["n"] == [4, 4, 4] and rec["config"]["m"] == 3
    assert rec["config"]["preconditioner"] == "jacobi"
    assert len(rec["eigenvalues"]) == len(rec["analytic"]) == 3
    assert rec["history"] == []
    assert all(e < 1e-8 for e in rec["rel_errors"])
    assert json.loads(json.dumps(rec)) == rec


@gpu
def test_runs_are_bit_reproducible(needs_gpu, tmp_path):
    argv = ["-n", "5", "5", "5", "-vrand", "4", "-seed", "3", "-tol", "1e-8"]
    c1, r1 = run_json(tmp_path, argv, "a.json")
    c2, r2 = run_json(tmp_path, argv, "b.json")
    assert c1 == c2 == EXIT_OK
    assert (r1["eigenvalues"], r1["iterations"], r1["status"]) == \
        (r2["eigenvalues"], r2["iterations"], r2["status"])


@gpu
def test_verbosity(needs_gpu, capsys):
    assert main(["-n", "3", "3", "3", "-vrand", "2", "-verb", "0"]) == EXIT_OK
    assert capsys.readouterr().out == ""
    assert main(["-n", "3", "3", "3", "-vrand", "2"]) == EXIT_OK
    out = capsys.readouterr().out
    assert "eigenvalue" in out and "analytic" in out


@gpu
def test_partial_convergence_exit_code(needs_gpu, tmp_path):
    code, rec = run_json(tmp_path, ["-n", "8", "8", "8", "-vrand", "3", "-tol", "1e-12",
                                    "-itr", "2"])
    assert code == EXIT_PARTIAL and rec["status"] == "MaxIterReached"


@gpu
def test_inner_pcg_reduces_outer_iterations(needs_gpu, tmp_path):
    base = ["-n", "10", "10", "10", "-vrand", "5", "-tol", "1e-6"]
    c0, r0 = run_json(tmp_path, base + ["-pcgitr", "0"], "p0.json")
    c10, r10 = run_json(tmp_path, base + ["-pcgitr", "10"], "p10.json")
    assert c0 == c10 == EXIT_OK
    assert r10["iterations"] < r0["iterations"]
    assert r10["config"]["preconditioner"] == "pcg:10"


@gpu
def test_history_outputs(needs_gpu, tmp_path):
    code, rec = run_json(tmp_path, ["-n", "3", "3", "3", "-vrand", "2", "-full_out", "1",
                                    "-csv", str(tmp_path / "h.csv")])
    assert code == EXIT_OK
    rows = rec["history"]
    assert len(rows) == 2 * (rec["iterations"] + 1)
    assert set(rows[0]) == {"iter", "j", "ritz", "resid", "active"}
    assert rows[0]["iter"] == 0 and rows[-1]["iter"] == rec["iterations"]
    lines = (tmp_path / "h.csv").read_text().splitlines()
    assert lines[0] == "iter,j,ritz,resid,active"
    assert len(lines) == 1 + 2 * (rec["iterations"] + 1)
    first = lines[1].split(",")
    assert first[0] == "0" and first[1] == "0" and first[4] in ("0", "1")
    float(first[2]), float(first[3])


@gpu
def test_out_evecs_and_constraints_flow(needs_gpu, tmp_path):
    grid = ["-n", "5", "5", "5"]
    ev = tmp_path / "first5.bin"
    c1, r1 = run_json(tmp_path, grid + ["-vrand", "5", "-tol", "1e-8", "-out_evecs", str(ev)],
                      "s1.json")
    assert c1 == EXIT_OK
    x = load_eigenvectors(ev)
    assert x.shape == (125, 5) and np.abs(x.T @ x - np.eye(5)).max() <= 1e-8
    c2, r2 = run_json(tmp_path, grid + ["-vrand", "5", "-tol", "1e-8", "-constraints", str(ev)],
                      "s2.json")
    assert c2 == EXIT_OK
    assert all(e < 1e-8 for e in r2["rel_errors"])
    assert min(r2["eigenvalues"]) > max(r1["eigenvalues"]) - 1e-10
    wrong = tmp_path / "wrong.bin"
    save_eigenvectors(wrong, np.ones((8, 1)))
    assert main(["-n", "3", "3", "3", "-vrand", "2", "-verb", "0", "-constraints",
                 str(wrong)]) == EXIT_ERROR
    assert main(["-n", "3", "3", "3", "-verb", "0", "-constraints",
                 str(tmp_path / "absent.bin")]) == EXIT_ERROR


@gpu
def test_sweeps(needs_gpu, tmp_path):
    csv_path, json_path = tmp_path / "sweep.csv", tmp_path / "sweep.json"
    code = main(["-n", "10", "10", "10", "-vrand", "1", "-verb", "0", "-sweep", "inner_iter",
                 "-sweep_values", "0,2,10", "-csv", str(csv_path), "-json", str(json_path)])
    assert code == EXIT_OK
    lines = csv_path.read_text().splitlines()
    assert lines[0] == "pcgitr,iterations,solve_sec" and len(lines) == 4
    assert [int(ln.split(",")[0]) for ln in lines[1:]] == [0, 2, 10]
    iters = [int(ln.split(",")[1]) for ln in lines[1:]]
    assert iters[-1] < iters[0]
    rec = json.loads(json_path.read_text())
    assert rec["sweep"] == "inner_iter" and [r["pcgitr"] for r in rec["rows"]] == [0, 2, 10]
    bs = tmp_path / "bs.csv"
    assert main(["-n", "4", "4", "4", "-verb", "0", "-sweep", "block_size", "-sweep_values",
                 "1,2", "-csv", str(bs)]) == EXIT_OK
    lines = bs.read_text().splitlines()
    assert lines[0] == "block_size,iterations,solve_sec" and len(lines) == 3


@gpu
def test_scaled_flag_matches_harness(needs_gpu, tmp_path):
    """-scaled 1: operator s*L with s = (N+1)^2, the analytic column scaled
    with it (the BASELINE harness)."""
    from paper_0705_2626_b200 import exact_eigenvalues

    code, rec = run_json(tmp_path, ["-n", "12", "12", "12", "-vrand", "4", "-tol", "1e-8",
                                    "-scaled", "1", "-itr", "300"])
    assert code == EXIT_OK
    assert all(e < 1e-8 for e in rec["rel_errors"])
    np.testing.assert_allclose(rec["analytic"], exact_eigenvalues((12, 12, 12), 4, scale=169.0),
                               rtol=1e-14)
