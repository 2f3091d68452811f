"""The CLI mirror of kronmul/cli.py: file format and argument errors on CPU;
``mul`` / ``bench`` through the GPU path (-m gpu), with the reference's
CSV schema (the header line byte-identical, 7 fields per row)."""
import os
import subprocess
import sys

import pytest

from paper_0712_4046_b200.cli import (CSV_HEADER, CommandError, main, parse_degree_grid, read_poly_file,
                                      write_poly_file)
from paper_0712_4046_b200.modpoly import ModPoly

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXAMPLE_F = "1000003\n4\n274 610 887 621\n"
EXAMPLE_G = "1000003\n4\n553 298 424 790\n"
EXAMPLE_H = (151522, 418982, 788467, 82836, 43043, 964034, 490590)


@pytest.fixture
def poly_files(tmp_path):
    f, g = tmp_path / "f.txt", tmp_path / "g.txt"
    f.write_text(EXAMPLE_F)
    g.write_text(EXAMPLE_G)
    return f, g


def test_header_matches_reference_schema():
    # kronmul/cli.py:32
    assert CSV_HEADER == "degree,length,modulus_bits,variant,wall_ns_median,limb_products,ratio_vs_ks1"


def test_poly_file_round_trip_and_errors(tmp_path):
    p = ModPoly((0, 1, 2, 3), 97)
    path = tmp_path / "p.txt"
    write_poly_file(str(path), p)
    assert read_poly_file(str(path)) == p
    bad = tmp_path / "bad.txt"
    bad.write_text("97\n3\n1 2\n")
    with pytest.raises(CommandError):
        read_poly_file(str(bad))
    bad.write_text("97\nx\n")
    with pytest.raises(CommandError):
        read_poly_file(str(bad))
    with pytest.raises(CommandError):
        read_poly_file(str(tmp_path / "missing.txt"))


def test_parse_degree_grid():
    assert parse_degree_grid("1:10:+3") == [1, 4, 7, 10]
    pts = parse_degree_grid("100:5000:log")
    assert pts[0] == 100 and pts[-1] == 5000 and 15 <= len(pts) <= 20 and pts == sorted(set(pts))
    for bad in ["5", "10:1:log", "1:10:lin", "0:9:+1", "1:9:+0"]:
        with pytest.raises(CommandError):
            parse_degree_grid(bad)


def test_bench_rejects_bad_arguments(capsys):
    assert main(["bench", "--degrees", "nope"]) == 1
    assert "invalid degree grid" in capsys.readouterr().err
    assert main(["bench", "--degrees", "1:4:+1", "--variants", "auto"]) == 1
    assert main(["bench", "--degrees", "1:4:+1", "--reps", "0"]) == 1


def test_mul_modulus_mismatch(poly_files, tmp_path, capsys):
    f, g = poly_files
    other = tmp_path / "other.txt"
    other.write_text("97\n1\n5\n")
    assert main(["mul", str(f), str(other)]) == 1
    assert "modulus mismatch" in capsys.readouterr().err
    assert main(["mul", "--modulus", "7", str(f), str(g)]) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["ks1", "ks2", "ks3", "ks4", "auto"])
def test_mul_command(poly_files, tmp_path, variant):
    f, g = poly_files
    out = tmp_path / "h.txt"
    assert main(["mul", "--modulus", "1000003", "--variant", variant, str(f), str(g), "-o", str(out)]) == 0
    assert read_poly_file(str(out)).coeffs == EXAMPLE_H


@pytest.mark.gpu
def test_bench_csv_schema(tmp_path):
    out = tmp_path / "bench.csv"
    for batch in ("1", "64"):
        assert main(["bench", "--modulus-bits", "8", "--degrees", "2:6:+4", "--variants", "ks1,ks4",
                     "--reps", "3", "--seed", "5", "--count-ops", "--batch", batch, "-o", str(out)]) == 0
        lines = out.read_text().splitlines()
        comments = [ln for ln in lines if ln.startswith("#")]
        assert any("seed=5" in c and "device=" in c for c in comments)
        body = [ln for ln in lines if not ln.startswith("#")]
        assert body[0] == CSV_HEADER
        rows = [ln.split(",") for ln in body[1:]]
        assert len(rows) == 4
        for degree, length, bits, variant, ns, ops, ratio in rows:
            assert int(length) == int(degree) + 1 and bits == "8" and variant in ("ks1", "ks4")
            assert int(ns) > 0 and int(ops) > 0
            if variant == "ks1":
                assert float(ratio) == 1.0


@pytest.mark.gpu
def test_module_entry_point(poly_files, tmp_path):
    f, g = poly_files
    out = tmp_path / "h.txt"
    r = subprocess.run([sys.executable, "-m", "paper_0712_4046_b200", "mul", str(f), str(g), "-o", str(out)],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert read_poly_file(str(out)).coeffs == EXAMPLE_H
