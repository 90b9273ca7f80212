"""Seeded inputs and text fixtures (paper_2401_04658_b200.matrix vs tila.matrix behaviour).

The cases follow the reference's pkg/tests/test_matrix.py: determinism of
random_matrix, exact fixture round trips, and a FixtureFormatError naming the
offending line for every malformed file.
"""

import numpy as np
import pytest

from oracle import tila_port
from paper_2401_04658_b200 import matrix as M


def test_random_matrix_matches_oracle_seeds():
    for rows, cols, seed in [(1, 1, 0), (7, 3, 5), (64, 64, 123)]:
        for prec in M.PRECISIONS:
            a = M.random_matrix(rows, cols, seed, prec)
            b = tila_port.random_matrix(rows, cols, seed, prec)
            assert a.dtype == b.dtype and np.array_equal(a, b)


def test_random_matrix_properties():
    a = M.random_matrix(50, 40, 3)
    assert a.dtype == np.float64 and np.array_equal(a, M.random_matrix(50, 40, 3))
    assert not np.array_equal(a, M.random_matrix(50, 40, 4))
    assert np.all(np.abs(a) <= 1.0) and np.all(np.isfinite(a))
    assert M.random_matrix(3, 3, 0, "single").dtype == np.float32
    for bad in [(0, 3, 0), (3, 0, 0), (3, 3, -1)]:
        with pytest.raises(ValueError):
            M.random_matrix(*bad)
    with pytest.raises(ValueError):
        M.random_matrix(3, 3, 0, "half")


@pytest.mark.parametrize("prec", M.PRECISIONS)
def test_fixture_round_trip_exact(tmp_path, prec):
    a = M.random_matrix(17, 9, 11, prec) * np.array(1e-30 if prec == "single" else 1e-300)
    a = a.astype(M.dtype_for(prec))
    a[0, 0], a[1, 1] = 0.0, -0.0
    p = tmp_path / "m.txt"
    M.save_fixture(a, p)
    b = M.load_fixture(p)
    assert b.dtype == a.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))
    M.save_fixture(b, tmp_path / "m2.txt")
    assert (tmp_path / "m2.txt").read_text() == p.read_text()


def test_reference_written_fixture_parses(tmp_path):
    p = tmp_path / "r.txt"
    p.write_text("2 3 double\n0.5 -1 2.5\n1e-3 0 -0.25\n")
    assert np.array_equal(M.load_fixture(p), np.array([[0.5, -1, 2.5], [1e-3, 0, -0.25]]))


@pytest.mark.parametrize("text,match", [
    ("", "missing header"),
    ("2 2\n1 2\n3 4\n", "line 1"),
    ("2 x double\n1 2\n3 4\n", "line 1"),
    ("2 2 quad\n1 2\n3 4\n", "line 1: unknown precision"),
    ("0 2 double\n", "line 1: invalid shape"),
    ("2 2 double\n1 2\n3\n", "line 3"),
    ("2 2 double\n1 nan\n3 4\n", "line 2.*non-finite"),
    ("2 2 double\n1 inf\n3 4\n", "line 2.*non-finite"),
    ("2 2 double\n1 abc\n3 4\n", "line 2.*unparseable"),
    ("3 2 double\n1 2\n3 4\n", "line 4"),
    ("1 2 double\n1 2\n3 4\n", "trailing data"),
])
def test_fixture_errors_name_the_line(tmp_path, text, match):
    p = tmp_path / "bad.txt"
    p.write_text(text)
    with pytest.raises(M.FixtureFormatError, match=match):
        M.load_fixture(p)


def test_save_fixture_rejects_bad_arrays(tmp_path):
    with pytest.raises(ValueError):
        M.save_fixture(np.zeros(3), tmp_path / "a.txt")
    with pytest.raises(ValueError):
        M.save_fixture(np.zeros((2, 2), np.float16), tmp_path / "a.txt")


def test_attention_config():
    c = M.AttentionConfig(n=8, d=4, block=16, lam=0.9)
    assert c.dv == 4 and c.precision == "double"
    assert M.AttentionConfig(n=8, d=4, block=2, lam=1.0, dv=7).dv == 7
    for kw in [dict(n=0), dict(d=0), dict(block=0), dict(lam=0.0), dict(lam=1.5),
               dict(precision="half"), dict(dv=0)]:
        args = dict(n=8, d=4, block=4, lam=0.5)
        args.update(kw)
        with pytest.raises(ValueError):
            M.AttentionConfig(**args)


def test_fixture_interop_with_reference(tmp_path):
    """Files written by the reference's tila.matrix parse identically here and back."""
    import os
    import sys
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference sources not present (GPU box)")
    sys.path.insert(0, src)
    try:
        from tila import matrix as ref
    finally:
        sys.path.remove(src)
    for prec in M.PRECISIONS:
        a = M.random_matrix(5, 7, 9, prec)
        ref.save_fixture(a, tmp_path / "ref.txt")
        M.save_fixture(a, tmp_path / "ours.txt")
        assert (tmp_path / "ref.txt").read_text() == (tmp_path / "ours.txt").read_text()
        assert np.array_equal(ref.load_fixture(tmp_path / "ours.txt"), M.load_fixture(tmp_path / "ref.txt"))
