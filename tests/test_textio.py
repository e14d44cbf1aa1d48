"""Matrix text wire format (include/mpsvd/io.hpp,
csrc/textio.cpp) against the reference's proj/src/io.cpp compiled in place.

Mirrors proj/tests/test_io.cpp (the reference side runs in a child process,
oracle/_ref/ref_io): write-then-read is bit-exact for both
precisions with awkward values (signed zeros, 0.1, the smallest normal, 1/3,
random mantissas and exponents, subnormals, infinities), the header records
shape and tag, and a bad tag, a short body, zero dimensions or an unparsable
token are IoError (MPSVD_ERR_IO). Beyond that: our writer's bytes equal the
reference writer's, and each side reads the other's files bit-exactly.
Host-only: no GPU is needed.
"""
from __future__ import annotations

import numpy as np
import pytest

M = pytest.importorskip("paper_2603_11953_b200")

import pyoracle  # noqa: E402

IO_STATUS = 9


def _awkward(dtype, m=9, n=4, seed=5):
    rng = np.random.default_rng(seed)
    fi = np.finfo(dtype)
    mant = rng.uniform(0.5, 1.0, (m, n))
    expo = rng.integers(-60, 60, (m, n))
    a = np.asfortranarray((mant * 2.0 ** expo).astype(dtype))
    a[0, 0] = 0.0
    a[1, 0] = -0.0
    a[2, 0] = dtype(0.1)
    a[3, 0] = fi.tiny
    a[4, 0] = dtype(1.0) / dtype(3.0)
    a[5, 0] = fi.tiny / dtype(8)  # subnormal
    a[6, 0] = -fi.max
    a[7, 0] = np.inf
    a[8, 0] = -np.inf
    return a


def _bits(x):
    return x.view(np.uint32 if x.dtype == np.float32 else np.uint64)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_round_trip_bit_exact(tmp_path, dtype):
    a = _awkward(dtype)
    mat = M.Matrix.from_numpy(a)
    p = tmp_path / "a.txt"
    mat.write_file(p)
    b = M.Matrix.read_file(p)
    assert b.precision == mat.precision and (b.rows, b.cols) == a.shape
    assert np.array_equal(_bits(b.numpy()), _bits(a))
    assert b.bitwise_equal(mat)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_bytes_identical_to_reference_writer(tmp_path, ref, dtype):
    # the reference reads our file and writes it back byte for byte: same
    # value formatting, and it parses every value we wrote exactly
    a = _awkward(dtype, m=13, n=5, seed=9)
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    M.Matrix.from_numpy(a).write_file(ours)
    assert ref.io_roundtrip(ours, theirs) == 0
    assert ours.read_bytes() == theirs.read_bytes()
    assert np.array_equal(_bits(M.Matrix.read_file(theirs).numpy()), _bits(a))


def test_header_records_shape_and_tag(tmp_path):
    p = tmp_path / "h.txt"
    M.Matrix(3, 2, M.Precision.WORKING).write_file(p)
    lines = p.read_text().splitlines()
    assert lines[0] == "3 2 f32"
    assert len(lines) == 1 + 2 and lines[1].split() == ["0", "0", "0"]


@pytest.mark.parametrize("text", [
    "2 2 f99\n1 2 3 4\n",      # unknown tag
    "2 2 f32\n1 2 3\n",        # one value short
    "0 2 f32\n",               # zero dimension
    "2 2 f64\n1 2 bogus 4\n",  # unparsable token
    "2 2 f64\n1 2 3x 4\n",     # trailing garbage in a token
    "",                        # no header
])
def test_parse_errors_are_io_errors_like_the_reference(tmp_path, ref, text):
    p = tmp_path / "bad.txt"
    p.write_text(text)
    with pytest.raises(M.MpsvdError) as e:
        M.Matrix.read_file(p)
    assert e.value.status == IO_STATUS
    assert ref.io_roundtrip(p, tmp_path / "out.txt") == IO_STATUS


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(M.MpsvdError) as e:
        M.Matrix.read_file(tmp_path / "does_not_exist.txt")
    assert e.value.status == IO_STATUS
