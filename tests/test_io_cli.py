"""File formats and the batch driver (feastlib io.py / cli.py semantics,
test_io.py / test_cli.py cases); CPU except the end-to-end GPU runs."""

import numpy as np
import pytest

from paper_1203_4031_b200.io import (CooMatrix, ParseError, parse_config, parse_coordinate, write_config,
                                     write_coordinate)

HELLO_IN = """s      ! problem kind
d      ! precision
F      ! storage
-5.0e0 ! Emin
5.0e0  ! Emax
2      ! M0
!!!!FEASTPARAM overrides
1      ! print runtime report
8      ! contour points
12     ! tolerance exponent
20     ! loop budget
0      ! criterion kind
"""
HELLO_A = "2 2 4\n1 1 2.0\n1 2 -1.0\n2 1 -1.0\n2 2 2.0\n"


def test_parse_config_fields_and_overrides():
    cfg = parse_config(HELLO_IN)
    assert (cfg.problem, cfg.precision, cfg.uplo, cfg.emin, cfg.emax, cfg.m0) == ("s", "d", "F", -5.0, 5.0, 2)
    assert [cfg.fpm.slot(k) for k in (1, 2, 3, 4, 6)] == [1, 8, 12, 20, 0]
    again = parse_config(write_config(cfg))
    assert (again.emin, again.emax, again.m0, again.fpm.slot(2)) == (-5.0, 5.0, 2, 8)


def test_parse_config_single_precision_tolerance_slot_and_fortran_exponent():
    cfg = parse_config(HELLO_IN.replace("d      ! precision", "c").replace("-5.0e0", "-5.0d0"))
    assert cfg.is_single and cfg.is_complex and cfg.emin == -5.0
    assert cfg.fpm.slot(7) == 12


@pytest.mark.parametrize("bad,line", [("x      ! problem kind", 1), ("q      ! precision", 2),
                                      ("Q      ! storage", 3), ("abc ! Emin", 4), ("2.5    ! M0", 6)])
def test_parse_config_errors_carry_line(bad, line):
    lines = HELLO_IN.splitlines()
    lines[line - 1] = bad
    with pytest.raises(ParseError) as e:
        parse_config("\n".join(lines))
    assert e.value.line == line


def test_parse_config_too_short_and_too_many_overrides():
    with pytest.raises(ParseError):
        parse_config("s\nd\nF\n")
    with pytest.raises(ParseError) as e:
        parse_config(HELLO_IN + "7 ! extra\n")
    assert e.value.line == 13


def test_coordinate_roundtrip_duplicates_and_assembly():
    text = "3 3 5 ! header\n1 1 1.5\n2 1 -2\n2 1 0.25\n3 3 4\n3 2 1e-1\n"
    coo = parse_coordinate(text)
    assert coo.nnz == 5 and list(coo.rows) == [1, 2, 2, 3, 3]
    back = parse_coordinate(write_coordinate(coo))
    assert np.array_equal(back.values, coo.values)
    full = coo.to_dense("L")
    want = np.array([[1.5, -1.75, 0], [-1.75, 0, 0.1], [0, 0.1, 4]])
    assert np.array_equal(full, want)
    ab, kl = coo.to_band("L")
    assert kl == 1 and ab.shape == (3, 3)
    for i in range(3):
        for j in range(3):
            if abs(i - j) <= kl:
                assert ab[kl + i - j, j] == want[i, j]


def test_coordinate_complex_hermitian_mirror():
    coo = parse_coordinate("2 2 3\n1 1 1 0\n2 1 0.5 2\n2 2 3 0\n", complex_values=True)
    a = coo.to_dense("L")
    assert a[0, 1] == np.conj(a[1, 0]) == 0.5 - 2j


@pytest.mark.parametrize("text,line", [("", None), ("2 3 1\n1 1 1\n", 1), ("2 2 1\n1 zz 1.0\n", 2),
                                       ("2 2 1\n3 1 1.0\n", 2), ("2 2 1\n1 1 1.0\n2 2 1.0\n", 3),
                                       ("2 2 2\n1 1 1.0\n", None), ("2 2 1\n1 1\n", 2)])
def test_coordinate_errors(text, line):
    with pytest.raises(ParseError) as e:
        parse_coordinate(text)
    assert e.value.line == line


def test_triangle_violations_rejected():
    coo = CooMatrix(2, 1, np.array([1]), np.array([2]), np.array([1.0]))
    with pytest.raises(ValueError):
        coo.to_dense("L")
    coo = CooMatrix(2, 1, np.array([2]), np.array([1]), np.array([1.0]))
    with pytest.raises(ValueError):
        coo.to_dense("U")


@pytest.fixture
def hello(tmp_path):
    (tmp_path / "hello.in").write_text(HELLO_IN)
    (tmp_path / "hello.A").write_text(HELLO_A)
    return str(tmp_path / "hello")


def test_cli_missing_files_and_parse_errors_exit_two(tmp_path, capsys):
    from paper_1203_4031_b200.cli import run_driver
    assert run_driver(str(tmp_path / "nothing")) == 2
    assert "nothing.in" in capsys.readouterr().err
    (tmp_path / "only.in").write_text(HELLO_IN)
    assert run_driver(str(tmp_path / "only")) == 2
    assert "only.A" in capsys.readouterr().err
    (tmp_path / "gen.in").write_text(HELLO_IN.replace("s      ! problem kind", "g"))
    (tmp_path / "gen.A").write_text(HELLO_A)
    assert run_driver(str(tmp_path / "gen")) == 2
    assert "gen.B" in capsys.readouterr().err
    (tmp_path / "bad.in").write_text(HELLO_IN)
    (tmp_path / "bad.A").write_text("2 2 1\n1 zz 1.0\n")
    assert run_driver(str(tmp_path / "bad")) == 2
    assert "line 2" in capsys.readouterr().err


def test_cli_unknown_format(hello, capsys):
    from paper_1203_4031_b200.cli import run_driver
    assert run_driver(hello, fmt="coo") == 2
    assert "unknown format" in capsys.readouterr().err


def test_coo_to_csr_matches_dense_assembly():
    coo = parse_coordinate("3 3 5\n1 1 1.0\n2 1 -1.0\n2 1 -0.5\n2 2 2.0\n3 3 4.0\n")
    for uplo in ("F", "L"):
        assert np.array_equal(coo.to_csr(uplo).to_dense(), coo.to_dense(uplo))


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["sparse", "dense", "banded"])
def test_cli_helloworld_gpu(hello, capsys, fmt):
    from paper_1203_4031_b200.cli import run_driver
    assert run_driver(hello, fmt=fmt) == 0
    out = capsys.readouterr().out
    assert "mode found/subspace 2 2" in out
    assert "1 1.000000000000000e+00" in out
    assert "2 3.000000000000000e+00" in out
    assert "==>FEAST has successfully converged" in out


@pytest.mark.gpu
def test_cli_interval_error_exit_one(tmp_path, capsys):
    from paper_1203_4031_b200.cli import run_driver
    (tmp_path / "bad.in").write_text(HELLO_IN.replace("-5.0e0", "7.0e0"))
    (tmp_path / "bad.A").write_text(HELLO_A)
    assert run_driver(str(tmp_path / "bad")) == 1
    assert "Emin>=Emax" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_helloworld_gpu_iterative(hello, capsys):
    from paper_1203_4031_b200.cli import main
    assert main([hello, "--solver", "iterative", "--iter-tol", "1e-12"]) == 0
    out = capsys.readouterr().out
    assert "mode found/subspace 2 2" in out
    assert "1 1.000000000000000e+00" in out
