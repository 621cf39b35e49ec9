"""File formats and the command line (paper_1003_2022_b200.pgmio / cli),
pinned to golden files written by the reference's own pgmio / cli
(tests/golden/make_golden_io.py; reference tests: pkg/tests/test_io_cli.py).
Format and exit-code tests run on CPU; the filtering subcommands need the
GPU."""

import struct

import numpy as np
import pytest

from conftest import golden
from paper_1003_2022_b200 import cli, pgmio


@pytest.fixture(scope="module")
def g():
    return golden("io_cli.npz")


def test_pgm_bytes_match_reference(tmp_path, g):
    p8, p16 = tmp_path / "a.pgm", tmp_path / "b.pgm"
    pgmio.write_pgm(p8, g["img8"], 255)
    pgmio.write_pgm(p16, g["img16"], 65535)
    assert p8.read_bytes() == g["pgm8"].tobytes()
    assert p16.read_bytes() == g["pgm16"].tobytes()
    for path, img, mv in ((p8, g["img8"], 255), (p16, g["img16"], 65535)):
        back, maxval = pgmio.read_pgm(path)
        assert maxval == mv and back.dtype == img.dtype and np.array_equal(back, img)


def test_raw_plane_bytes_match_reference(tmp_path, g):
    p = tmp_path / "c.f64"
    pgmio.write_raw_plane(p, g["plane"])
    assert p.read_bytes() == g["raw"].tobytes()
    assert np.array_equal(pgmio.read_raw_plane(p), g["plane"])
    raw = p.read_bytes()
    assert raw[:4] == b"RUF8" and struct.unpack("<II", raw[4:12]) == (5, 3)


def test_quantize_matches_reference(g):
    q = pgmio.quantize(g["q_in"], 255)
    assert q.dtype == np.uint8 and np.array_equal(q, g["q8"])
    q16 = pgmio.quantize(np.array([70000.0, 12.3, 0.5, 1.5]), 65535)
    assert q16.dtype == np.uint16 and np.array_equal(q16, g["q16"])


def test_pgm_header_comments_and_errors(tmp_path):
    p = tmp_path / "c.pgm"
    p.write_bytes(b"P5\n# a comment\n3 # width\n2\n255\n" + bytes(range(6)))
    data, maxval = pgmio.read_pgm(p)
    assert maxval == 255 and data.tolist() == [[0, 1, 2], [3, 4, 5]]
    for body in (b"P2\n3 2\n255\n" + bytes(6), b"P5\n3 2\n255\n" + bytes(5), b"P5\n3 2\n",
                 b"P5\n3 2\n70000\n" + bytes(6), b"P5\n0 2\n255\n", b"P5\n2 1\n9\n" + bytes([3, 10])):
        p.write_bytes(body)
        with pytest.raises(ValueError):
            pgmio.read_pgm(p)
    with pytest.raises(ValueError):
        pgmio.write_pgm(tmp_path / "x.pgm", np.zeros((3, 3)), 255)  # float samples
    with pytest.raises(ValueError):
        pgmio.write_pgm(tmp_path / "x.pgm", np.full((2, 2), 300, np.int32), 255)
    bad = tmp_path / "bad.f64"
    bad.write_bytes(b"RUF8" + struct.pack("<II", 4, 4) + bytes(10))
    with pytest.raises(ValueError):
        pgmio.read_raw_plane(bad)


def test_atomic_write_leaves_no_partial_file(tmp_path):
    target = tmp_path / "keep.pgm"
    target.write_bytes(b"old")

    with pytest.raises(TypeError):
        pgmio.atomic_write_bytes(target, object())  # write fails mid-way
    assert target.read_bytes() == b"old"
    assert [p.name for p in tmp_path.iterdir()] == ["keep.pgm"]


def test_cli_exit_codes_match_reference(tmp_path, g):
    src = tmp_path / "in.pgm"
    src.write_bytes(g["cli_in"].tobytes())
    dst = str(tmp_path / "o.pgm")
    assert cli.main(["filter", "--in", str(tmp_path / "nope.pgm"), "--out", dst, "--size", "2"]) \
        == int(g["rc_missing"]) == 4
    assert cli.main(["filter", "--in", str(src), "--size", "-2", "--out", dst]) == int(g["rc_badsize"]) == 5
    assert cli.main(["filter", "--in", str(src), "--out", dst, "--size", "2", "--elongation", "50",
                     "--orientation", str(np.pi / 8)]) == int(g["rc_infeasible"]) == 3
    with pytest.raises(SystemExit) as e:
        cli.main(["filter", "--in", str(src)])  # argparse usage error
    assert e.value.code == 2


@pytest.mark.gpu
def test_cli_filter_and_adapt_match_reference_cli(cuda, tmp_path, g):
    src = tmp_path / "in.pgm"
    src.write_bytes(g["cli_in"].tobytes())
    runs = {
        "filter": ["filter", "--in", str(src), "--size", "3", "--elongation", "2", "--orientation", "0.4"],
        "filter2": ["filter", "--in", str(src), "--size", "6", "--elongation", "3", "--orientation", "2.0",
                    "--iterations", "2"],
        "adapt": ["adapt", "--in", str(src), "--noise-sigma", "10"],
    }
    for k, argv in runs.items():
        dst = tmp_path / (k + ".f64")
        assert cli.main(argv + ["--out", str(dst)]) == 0
        got, ref = pgmio.read_raw_plane(dst), g["cli_" + k]
        # the reference's own fast path is accurate to ~1e-12 at this size;
        # adapt's elongation map is ill-conditioned: 2e-8
        tol = 2e-8 if k == "adapt" else 1e-9
        assert np.abs(got - ref).max() <= tol * np.abs(ref).max(), k
    dst = tmp_path / "filter.pgm"
    assert cli.main(runs["filter"] + ["--out", str(dst)]) == 0
    assert dst.read_bytes() == g["cli_filter_pgm"].tobytes()


@pytest.mark.gpu
def test_cli_filter_three_directions_and_bench(cuda, tmp_path, g, capsys):
    import oracle
    from paper_1003_2022_b200 import scales3_from_params
    src = tmp_path / "in.pgm"
    src.write_bytes(g["cli_in"].tobytes())
    dst = tmp_path / "o3.f64"
    assert cli.main(["filter", "--in", str(src), "--out", str(dst), "--size", "5", "--elongation", "2",
                     "--orientation", "0.3", "--directions", "3"]) == 0
    img, _ = pgmio.read_pgm(src)
    ref = oracle.dense3(img.astype(float), scales3_from_params(5.0, 2.0, 0.3))
    assert np.abs(pgmio.read_raw_plane(dst) - ref).max() < 1e-9 * np.abs(ref).max()
    assert cli.main(["bench", "--n", "256", "--scales", "1,16,256", "--runs", "2"]) == 0
    out = capsys.readouterr().out
    assert "size_s\tmean_s" in out and "max/min mean ratio" in out


# --- lookup-table files (solver.save_lut / load_lut, cli lut-build / lut-inspect)


def test_lut_file_round_trip_matches_reference_bytes(tmp_path):
    from paper_1003_2022_b200 import solver
    g = golden("lut_file.npz")
    p = tmp_path / "ref.lut"
    p.write_bytes(g["lut_bytes"].tobytes())
    lut = solver.load_lut(p)
    assert np.array_equal(lut.rho_grid, g["rho_grid"]) and np.array_equal(lut.phi_grid, g["phi_grid"])
    assert np.array_equal(lut.entries, g["entries"])
    q = tmp_path / "ours.lut"
    solver.save_lut(lut, q)
    assert q.read_bytes() == p.read_bytes()
    # lut-build here: the same table to the host solver's accuracy
    r = tmp_path / "built.lut"
    assert cli.main(["lut-build", "--out", str(r), "--rho-points", "8", "--phi-points", "6",
                     "--rho-max", "4.5"]) == 0
    built = solver.load_lut(r)
    assert np.array_equal(built.rho_grid, g["rho_grid"])
    assert np.abs(built.entries - g["entries"]).max() < 1e-13


def test_lut_file_errors(tmp_path):
    from paper_1003_2022_b200 import solver
    g = golden("lut_file.npz")
    good = g["lut_bytes"].tobytes()
    cases = [b"XXXX" + good[4:], good[:4] + (2).to_bytes(4, "little") + good[8:], good[:-8]]
    bad_grid = bytearray(good)
    bad_grid[16:24] = bad_grid[24:32]  # rho_grid[0] == rho_grid[1]
    cases.append(bytes(bad_grid))
    for i, body in enumerate(cases):
        p = tmp_path / f"bad{i}.lut"
        p.write_bytes(body)
        with pytest.raises(ValueError):
            solver.load_lut(p)
    assert cli.main(["lut-inspect", "--in", str(tmp_path / "missing.lut")]) == 4
    assert cli.main(["lut-inspect", "--in", str(tmp_path / "bad0.lut")]) == 5


@pytest.mark.gpu
def test_lut_inspect_and_adapt_with_a_table_file(cuda, tmp_path, g, capsys):
    from paper_1003_2022_b200 import default_lut, solver
    lg = golden("lut_file.npz")
    p = tmp_path / "ref.lut"
    p.write_bytes(lg["lut_bytes"].tobytes())
    assert cli.main(["lut-inspect", "--in", str(p)]) == 0
    ours = capsys.readouterr().out.splitlines()
    ref = str(lg["inspect"]).splitlines()
    assert ours[:3] == ref[:3]  # table size, elongation and orientation ranges
    assert float(ours[3].split(":")[1]) < 1e-12 and float(ref[3].split(":")[1]) < 1e-12
    num = lambda line: np.array([float(v) for v in line.split("[")[1].rstrip("]").split()])  # noqa: E731
    assert np.abs(num(ours[4]) - num(ref[4])).max() < 1e-12
    # adapt with the default table written to a file == adapt with the default table
    t = tmp_path / "default.lut"
    solver.save_lut(default_lut(), t)
    src = tmp_path / "in.pgm"
    src.write_bytes(g["cli_in"].tobytes())
    a, b = tmp_path / "a.f64", tmp_path / "b.f64"
    assert cli.main(["adapt", "--in", str(src), "--out", str(a), "--noise-sigma", "10"]) == 0
    assert cli.main(["adapt", "--in", str(src), "--out", str(b), "--noise-sigma", "10", "--lut", str(t)]) == 0
    from paper_1003_2022_b200 import pgmio
    assert np.array_equal(pgmio.read_raw_plane(a), pgmio.read_raw_plane(b))
