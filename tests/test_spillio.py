"""Layer-directory spill I/O through the library (csrc/spillio.cu; SURVEY.md
§8f ranks 2-3). Host-only: runs without a GPU.

* the parallel writer produces the bytes of storage.write_matrix_as_layer,
  itself byte-identical to the reference's writer (tests/test_cpu_boundary);
* the parallel reader returns the rows the reference's loader returns,
  counts every delivery (exactly once, criterion 2), and raises the
  reference's error classes on damaged input (oocgnn/errors.py).
"""

import os
import sys

import numpy as np
import pytest

from helpers import REFERENCE_SRC
from paper_2605_09402_b200 import chunks as C
from paper_2605_09402_b200 import storage as S
from paper_2605_09402_b200.errors import (BadMagicError, ConsistencyError,
                                          CoverageError, TruncatedFileError,
                                          VersionMismatchError)


def _files(root):
    out = {}
    for base, _, names in os.walk(root):
        for n in names:
            p = os.path.join(base, n)
            out[os.path.relpath(p, root)] = open(p, "rb").read()
    return out


@pytest.mark.parametrize("dtype", ["f32", "f16"])
@pytest.mark.parametrize("v,dim,parts", [(1, 3, 1), (1003, 7, 3),
                                         (4096, 64, 8), (10, 2, 16)])
def test_writer_bytes_match_format_writer(tmp_path, dtype, v, dim, parts):
    m = np.random.default_rng(v).uniform(-1, 1, (v, dim)).astype(np.float32)
    S.write_matrix_as_layer(tmp_path / "a", m, partitions=parts, dtype=dtype)
    C.write_layer_output(tmp_path / "b", m, partitions=parts, dtype=dtype,
                         threads=4)
    assert _files(tmp_path / "a") == _files(tmp_path / "b")


@pytest.mark.parametrize("dtype", ["f32", "f16"])
def test_reader_matches_reference_loader(tmp_path, dtype):
    m = np.random.default_rng(3).uniform(-1, 1, (5000, 24)).astype(np.float32)
    S.write_matrix_as_layer(tmp_path / "l", m, partitions=5, dtype=dtype,
                            spill_rows=333)
    meta, rows, nbytes, delivery = C.load_layer_input(tmp_path / "l",
                                                      threads=3)
    np.testing.assert_array_equal(rows, m.astype(S.NP_DTYPES[dtype]))
    assert (delivery == 1).all()
    assert nbytes == 5000 * (24 * (4 if dtype == "f32" else 2) + 8)
    if REFERENCE_SRC.exists():
        sys.path.insert(0, str(REFERENCE_SRC))
        from oocgnn.storage import load_layer_matrix
        np.testing.assert_array_equal(rows.astype(np.float32),
                                      load_layer_matrix(tmp_path / "l"))


def test_reader_reads_generated_feature_spills(tmp_path):
    """generate_synthetic's 4 MiB feature spills (many files, one
    partition) -- the reference dataset layout."""
    S.generate_synthetic("uniform", 20_000, 4, 100, 7, tmp_path / "d")
    _, rows, _, delivery = C.load_layer_input(tmp_path / "d" / "features")
    want = S.load_layer_matrix(tmp_path / "d" / "features")
    np.testing.assert_array_equal(rows, want)
    assert (delivery == 1).all()


def _layer(tmp_path):
    m = np.arange(60, dtype=np.float32).reshape(20, 3)
    S.write_matrix_as_layer(tmp_path / "l", m, partitions=2, spill_rows=4)
    return tmp_path / "l", tmp_path / "l" / "part_0" / "spill_0"


def test_reader_rejects_bad_magic(tmp_path):
    d, f = _layer(tmp_path)
    b = bytearray(f.read_bytes())
    b[:4] = b"XXXX"
    f.write_bytes(bytes(b))
    with pytest.raises(BadMagicError):
        C.load_layer_input(d)


def test_reader_rejects_truncation(tmp_path):
    d, f = _layer(tmp_path)
    f.write_bytes(f.read_bytes()[:5000])
    with pytest.raises(TruncatedFileError):
        C.load_layer_input(d)


def test_reader_rejects_version(tmp_path):
    d, f = _layer(tmp_path)
    b = bytearray(f.read_bytes())
    b[4] = 9
    f.write_bytes(bytes(b))
    with pytest.raises(VersionMismatchError):
        C.load_layer_input(d)


def test_reader_rejects_dtype_mismatch(tmp_path):
    d, _ = _layer(tmp_path)
    meta = (d / "meta.txt").read_text().replace("dtype=f32", "dtype=f16")
    (d / "meta.txt").write_text(meta)
    with pytest.raises(ConsistencyError):
        C.load_layer_input(d)


def test_reader_counts_duplicates_and_gaps(tmp_path):
    d, _ = _layer(tmp_path)
    man = d / "part_0" / "manifest.txt"
    names = man.read_text().split()
    man.write_text("\n".join(names + [names[0]]) + "\n")  # spill read twice
    with pytest.raises(CoverageError):
        C.load_layer_input(d)
    man.write_text("\n".join(names[1:]) + "\n")  # ids 0..3 never arrive
    with pytest.raises(CoverageError):
        C.load_layer_input(d)
