"""Layer directories read straight into HBM (atlas_spill_read_device:
GPUDirect Storage through cuFile, or the pinned-bounce stream when the
cuFile driver is unavailable) must hold exactly the rows the host reader
returns -- itself pinned to the reference's loader (tests/test_spillio.py)
-- with the same delivery counts, byte accounting and error classes."""

import numpy as np
import pytest
import torch

from paper_2605_09402_b200 import _native as N
from paper_2605_09402_b200 import chunks as C
from paper_2605_09402_b200 import storage as S
from paper_2605_09402_b200.errors import (BadMagicError, CoverageError,
                                          TruncatedFileError)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["f32", "f16"])
@pytest.mark.parametrize("v,dim,parts,spill", [(5000, 24, 5, 333),
                                               (1, 3, 1, 0),
                                               (200_000, 100, 8, 4096)])
def test_device_reader_matches_host_reader(tmp_path, dtype, v, dim, parts,
                                           spill):
    m = np.random.default_rng(v).uniform(-1, 1, (v, dim)).astype(np.float32)
    S.write_matrix_as_layer(tmp_path / "l", m, partitions=parts, dtype=dtype,
                            spill_rows=spill or None)
    _, host, hb, hd = C.load_layer_input(tmp_path / "l", threads=4)
    _, dev, db, dd, gds = C.load_layer_device(tmp_path / "l", threads=4)
    assert dev.is_cuda
    np.testing.assert_array_equal(dev.cpu().numpy(), host)
    assert db == hb and (dd == hd).all()
    print("path:", "cuFile" if gds else N.load_library().atlas_gds_status())


def _layer(tmp_path):
    m = np.arange(40, dtype=np.float32).reshape(10, 4)
    S.write_matrix_as_layer(tmp_path / "d", m, partitions=1, spill_rows=4)
    d = tmp_path / "d"
    return d, d / "part_0" / "spill_0"


def test_device_reader_errors(tmp_path):
    d, f = _layer(tmp_path)
    raw = f.read_bytes()
    f.write_bytes(raw[:5000])
    with pytest.raises(TruncatedFileError):
        C.load_layer_device(d)
    b = bytearray(raw)
    b[:4] = b"XXXX"
    f.write_bytes(bytes(b))
    with pytest.raises(BadMagicError):
        C.load_layer_device(d)
    f.write_bytes(raw)
    man = d / "part_0" / "manifest.txt"
    names = man.read_text().split()
    man.write_text("\n".join(names + [names[0]]) + "\n")
    with pytest.raises(CoverageError):
        C.load_layer_device(d)
    torch.cuda.synchronize()
