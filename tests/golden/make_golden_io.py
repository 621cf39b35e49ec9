"""Golden fixtures for the command line and its file formats, generated
from the REAL reference (build container only: imports /root/reference).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_io.py

Recorded (pkg/src/rubs/pgmio.py, cli.py):
  * the bytes write_pgm writes for an 8-bit and a 16-bit image, and
    write_raw_plane for a float64 plane;
  * quantize on edge values;
  * `rubs filter` and `rubs adapt` outputs (.f64) for a small noisy stripe
    PGM (the reference test's recipe, test_io_cli.py:108-114), and the
    exit codes of its failure cases;
  * (lut_file.npz) the bytes `rubs lut-build` writes for an 8 x 6 table up
    to elongation 4.5, the table it loads back, and `rubs lut-inspect`'s
    report of it (solver.py:351-395, cli.py:142-176).
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from rubs import cli, pgmio  # noqa: E402
from rubs.oracle import stripe_image  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(7)
    g = {}
    with tempfile.TemporaryDirectory() as d:
        img8 = rng.integers(0, 256, (5, 7)).astype(np.uint8)
        pgmio.write_pgm(os.path.join(d, "a.pgm"), img8, 255)
        g["img8"], g["pgm8"] = img8, np.frombuffer(open(os.path.join(d, "a.pgm"), "rb").read(), np.uint8)
        img16 = rng.integers(0, 65536, (4, 3)).astype(np.uint16)
        pgmio.write_pgm(os.path.join(d, "b.pgm"), img16, 65535)
        g["img16"], g["pgm16"] = img16, np.frombuffer(open(os.path.join(d, "b.pgm"), "rb").read(), np.uint8)
        plane = rng.standard_normal((3, 5))
        pgmio.write_raw_plane(os.path.join(d, "c.f64"), plane)
        g["plane"], g["raw"] = plane, np.frombuffer(open(os.path.join(d, "c.f64"), "rb").read(), np.uint8)
        q = np.array([-0.2, 0.0, 0.5, 1.5, 2.5, 255.9, 300.0, 127.5, 128.5])
        g["q_in"], g["q8"] = q, pgmio.quantize(q, 255)
        g["q16"] = pgmio.quantize(np.array([70000.0, 12.3, 0.5, 1.5]), 65535)
        # CLI: a noisy stripe image as PGM (reference recipe), filtered / adapted
        noisy = stripe_image((40, 48), period=6.0, angle=0.5) * 200.0 + rng.normal(0.0, 10.0, (40, 48))
        src = os.path.join(d, "in.pgm")
        pgmio.write_pgm(src, pgmio.quantize(noisy, 255), 255)
        g["cli_in"] = np.frombuffer(open(src, "rb").read(), np.uint8)
        runs = {
            "filter": ["filter", "--in", src, "--size", "3", "--elongation", "2", "--orientation", "0.4"],
            "filter2": ["filter", "--in", src, "--size", "6", "--elongation", "3", "--orientation", "2.0",
                        "--iterations", "2"],
            "adapt": ["adapt", "--in", src, "--noise-sigma", "10"],
        }
        for k, argv in runs.items():
            dst = os.path.join(d, k + ".f64")
            assert cli.main(argv + ["--out", dst]) == 0
            g["cli_" + k] = pgmio.read_raw_plane(dst)
        dst = os.path.join(d, "filter.pgm")
        assert cli.main(runs["filter"] + ["--out", dst]) == 0
        g["cli_filter_pgm"] = np.frombuffer(open(dst, "rb").read(), np.uint8)
        g["rc_missing"] = cli.main(["filter", "--in", os.path.join(d, "nope.pgm"), "--out", dst,
                                    "--size", "2"])
        g["rc_badsize"] = cli.main(runs["filter"][:-6] + ["--size", "-2", "--out", dst])
        g["rc_infeasible"] = cli.main(["filter", "--in", src, "--out", dst, "--size", "2",
                                       "--elongation", "50", "--orientation", str(np.pi / 8)])
    np.savez_compressed(os.path.join(OUT, "io_cli.npz"), **g)


def lut_file():
    import contextlib
    import io
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.lut")
        assert cli.main(["lut-build", "--out", p, "--rho-points", "8", "--phi-points", "6",
                         "--rho-max", "4.5"]) == 0
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            assert cli.main(["lut-inspect", "--in", p]) == 0
        from rubs import solver
        lut = solver.load_lut(p)
        np.savez_compressed(os.path.join(OUT, "lut_file.npz"),
                            lut_bytes=np.frombuffer(open(p, "rb").read(), np.uint8),
                            rho_grid=lut.rho_grid, phi_grid=lut.phi_grid, entries=lut.entries,
                            inspect=np.array(buf.getvalue()))


if __name__ == "__main__":
    main()
    lut_file()
