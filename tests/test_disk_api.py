"""The disk-to-disk drop-in API (row a13: ``run_inference`` / ``run_layer``,
oocgnn/runtime.py:114-264) against the reference's own outputs.

CPU:
* the output spill layout (chunks.write_graduation_layout) is byte-for-byte
  the reference writer's (oocgnn/writer.py:40-115) for the same graduation
  order -- checked against the reference's SpillBufferSet when
  /root/reference is importable;
* a truncated input spill fails with an EngineError and leaves no
  layer_0/ behind (the reference's tests/test_runtime.py:181-195).

GPU (``-m gpu``), on the datasets of every golden case, written here by this
repo's reference-identical generator: ``run_inference`` must reproduce the
reference's layer directories byte for byte (sha256 over every file,
tests/golden/golden.json ``layer_dirs``) and its metrics.csv column for
column -- except ``bytes_read``, which counts what this engine actually read
(each input spill once, whole; the reference re-reads through per-chunk
aligned preads and an LRU of open files). ``bytes_written``
(spill files + cold records) is equal. ``run_layer`` on one layer
reproduces that layer's directory.
"""

import csv
import hashlib
import sys
from pathlib import Path

import numpy as np
import pytest

from helpers import (REFERENCE_SRC, case_weights, golden_manifest)
from paper_2605_09402_b200 import chunks as C
from paper_2605_09402_b200 import storage as S
from paper_2605_09402_b200.errors import EngineError

CSV_BYTES_READ = 8  # column index of bytes_read in CSV_FIELDS


def dir_digest(layer_dir):
    layer_dir = Path(layer_dir)
    h = hashlib.sha256()
    n = total = 0
    for p in sorted(q for q in layer_dir.rglob("*") if q.is_file()):
        data = p.read_bytes()
        h.update(str(p.relative_to(layer_dir)).encode() + b"\0")
        h.update(data)
        n += 1
        total += len(data)
    return {"sha": h.hexdigest(), "files": n, "bytes": total}


@pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference absent")
@pytest.mark.parametrize("v,dim,parts,buf", [(1000, 4, 3, 4096),
                                             (777, 16, 8, 64 << 10),
                                             (50, 3, 1, 1), (5, 2, 8, 100)])
def test_graduation_layout_matches_reference_writer(tmp_path, v, dim, parts,
                                                    buf):
    sys.path.insert(0, str(REFERENCE_SRC))
    from oocgnn.writer import SpillBufferSet
    rng = np.random.default_rng(v)
    rows = rng.uniform(-1, 1, (v, dim)).astype(np.float32)
    order = rng.permutation(v)
    ref = SpillBufferSet(tmp_path / "ref", v, dim, parts, buf, direct=False)
    cuts = np.sort(rng.choice(np.arange(1, v), size=min(6, v - 1),
                              replace=False)) if v > 1 else []
    for batch in np.split(order, cuts):
        ref.scatter(batch, rows[batch])
    ref.flush_all()
    written = C.write_graduation_layout(tmp_path / "ours", rows, order,
                                        parts, buf)
    assert dir_digest(tmp_path / "ours") == dir_digest(tmp_path / "ref")
    assert written == ref.io.spill_bytes_written


def test_truncated_input_fails_and_cleans_output(tmp_path):
    from paper_2605_09402_b200.runtime import PipelineConfig, run_inference
    ds = tmp_path / "broken"
    S.generate_synthetic("uniform", 2000, 6, 8, 3, ds)
    spill = next((ds / "features").glob("part_*/spill_*"))
    with open(spill, "r+b") as f:
        f.truncate(spill.stat().st_size // 2)
    out = tmp_path / "out"
    w = S.random_weights(S.ModelKind.GCN, [8, 4, 2], 5)
    with pytest.raises(EngineError):
        run_inference(ds, w, PipelineConfig(chunk_budget=64 << 10,
                                             partitions=3), out)
    assert not (out / "layer_0").exists()


# --- GPU: every golden case through the disk API ---------------------------

CASES = sorted(k for k in golden_manifest() if not k.startswith("_"))
_DIRS = {}


def _dataset_dir(name, root):
    if name in _DIRS:
        return _DIRS[name]
    d = root / name
    if name == "fig2":
        from helpers import fig2_graph
        feats = np.random.default_rng(3).uniform(-1, 1, (6, 8)).astype(
            np.float32)
        S.write_csr(fig2_graph(), d)
        S.write_matrix_as_layer(d / "features", feats)
    else:
        kind, v, deg, dim, seed, dtype = golden_manifest()["_datasets"][name]
        S.generate_synthetic(kind, v, deg, dim, seed, d, dtype=dtype)
    _DIRS[name] = d
    return d


@pytest.fixture(scope="module")
def data_root(tmp_path_factory):
    return tmp_path_factory.mktemp("disk_api")


def _csv_rows(path):
    with open(path, newline="") as f:
        return [r[:-1] for r in csv.reader(f)]  # minus wall_seconds


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_run_inference_reproduces_reference_directories(case, data_root,
                                                        tmp_path):
    from paper_2605_09402_b200.runtime import PipelineConfig, run_inference
    entry = golden_manifest()[case]
    ds = _dataset_dir(entry["dataset"], data_root)
    out = tmp_path / "out"
    report = run_inference(ds, case_weights(entry),
                           PipelineConfig(**entry["config"],
                                          backend="stable"), out)
    for l, want in enumerate(entry["layer_dirs"]):
        assert dir_digest(out / f"layer_{l}") == want, l
    got = _csv_rows(out / "metrics.csv")
    ref = entry["metrics_csv"]
    assert got[0] == ref[0]
    for g, r in zip(got[1:], ref[1:]):
        assert g[:CSV_BYTES_READ] == r[:CSV_BYTES_READ], (g, r)
        assert g[CSV_BYTES_READ + 1:] == r[CSV_BYTES_READ + 1:], (g, r)
    assert len(report.layers) == len(entry["layers"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["small_sage_tight", "half_gin_slots300",
                                  "uniform_gcn_slots500", "wide_sage"])
def test_run_layer_reproduces_reference_layer(case, data_root, tmp_path):
    from paper_2605_09402_b200.runtime import PipelineConfig, run_layer
    entry = golden_manifest()[case]
    ds = _dataset_dir(entry["dataset"], data_root)
    hdr = S.read_topology_header(ds / S.TOPOLOGY_FILE)
    indeg = S.read_in_degrees(ds / S.INDEGREE_FILE, hdr.num_vertices)
    m = run_layer(ds / S.TOPOLOGY_FILE, indeg, ds / "features",
                  tmp_path / "layer_0", case_weights(entry), 0,
                  PipelineConfig(**entry["config"], backend="stable"))
    assert dir_digest(tmp_path / "layer_0") == entry["layer_dirs"][0]
    ref = entry["metrics_csv"][1]
    assert [str(m.messages), str(m.evictions), str(m.reloads)] == ref[1:4]
    assert str(m.bytes_written) == ref[9]
