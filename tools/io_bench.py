"""Layer-directory I/O and disk-to-disk run_inference on the cfg2 dataset
(diagnostic; results go to profiles/). Prints one JSON line.

* write: a (2.4M x 128) f32 layer output as 8 partition spills with the
  library's parallel writer vs storage.write_matrix_as_layer (numpy);
* read: the 100-d f32 feature set of generate_synthetic (4 MiB spills, the
  reference's dataset layout) with the library's parallel reader (into
  pinned memory) vs a numpy loop over the same files, and straight into
  HBM (atlas_spill_read_device) vs host reader + upload;
* run_inference: dataset directory -> 3 layer directories on disk, both
  transform backends, wall clock (topology + features read, H2D, 3 layers,
  D2H, spill writes).
"""

import json
import shutil
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2605_09402_b200 import chunks as C  # noqa: E402
from paper_2605_09402_b200 import storage as S  # noqa: E402
from paper_2605_09402_b200.runtime import (PipelineConfig,  # noqa: E402
                                           run_inference)


def timed(f):
    t0 = time.perf_counter()
    out = f()
    return out, time.perf_counter() - t0


def numpy_read(layer_dir):
    meta = S.read_layer_meta(layer_dir)
    rows = np.empty((meta.num_vertices, meta.dim), S.NP_DTYPES[meta.dtype])
    for k in range(meta.partitions):
        for name in S.read_manifest(S.part_dir(layer_dir, k)):
            ids, block = S.read_spill_file(S.part_dir(layer_dir, k) / name)
            rows[ids] = block
    return rows


def main():
    root = Path(tempfile.mkdtemp(prefix="iobench_", dir="/tmp"))
    out = {}
    try:
        data, gen_s = timed(lambda: S.generate_synthetic(
            "uniform", 2_400_000, 26, 100, 7, root / "cfg2"))
        out["generate_s"] = gen_s
        feats_dir = root / "cfg2" / "features"
        nbytes = 2_400_000 * 100 * 4
        # read (page cache warm: one untimed pass first)
        C.load_layer_input(feats_dir)
        (_, rows, _, _), t_nat = timed(lambda: C.load_layer_input(feats_dir))
        ref, t_np = timed(lambda: numpy_read(feats_dir))
        assert np.array_equal(rows, ref)
        out["read_features"] = {
            "bytes": nbytes, "files": len(S.read_manifest(
                S.part_dir(feats_dir, 0))),
            "native_gb_s": nbytes / t_nat / 1e9,
            "numpy_gb_s": nbytes / t_np / 1e9}
        # straight into HBM (cuFile or the pinned-bounce stream) vs host
        # reader + one pinned upload
        import torch

        from paper_2605_09402_b200 import _native as N
        C.load_layer_device(feats_dir)
        (_, dev, _, _, gds), t_dev = timed(
            lambda: C.load_layer_device(feats_dir))
        assert np.array_equal(dev.cpu().numpy(), rows)

        def host_then_upload():
            _, r, _, _ = C.load_layer_input(feats_dir)
            t = torch.from_numpy(r).cuda(non_blocking=True)
            torch.cuda.synchronize()
            return t
        _, t_hu = timed(host_then_upload)
        out["read_features_to_hbm"] = {
            "path": "cuFile" if gds else
            N.load_library().atlas_gds_status().decode(),
            "device_reader_gb_s": nbytes / t_dev / 1e9,
            "host_reader_plus_upload_gb_s": nbytes / t_hu / 1e9}
        # write
        m = np.random.default_rng(0).uniform(-1, 1, (2_400_000, 128)).astype(
            np.float32)
        wb = m.nbytes
        _, t_nw = timed(lambda: C.write_layer_output(root / "w1", m, 8))
        _, t_pw = timed(lambda: S.write_matrix_as_layer(root / "w2", m, 8))
        out["write_layer"] = {"bytes": wb, "native_gb_s": wb / t_nw / 1e9,
                              "numpy_gb_s": wb / t_pw / 1e9}
        # disk to disk
        w = S.random_weights(S.ModelKind.GCN, [100, 128, 128, 47], 5)
        runs = {}
        for backend in ("tcgen05", "stable"):
            cfg = PipelineConfig(chunk_budget=8 << 20, hot_slots=2_400_000,
                                 backend=backend)
            run_inference(root / "cfg2", w, cfg, root / f"run_{backend}")
            rep, t = timed(lambda: run_inference(root / "cfg2", w, cfg,
                                                 root / f"run_{backend}"))
            runs[backend] = {"wall_s": t,
                             "edges_per_s_per_layer": 3 * data.num_edges / t,
                             "layer_wall_s": [m.wall_seconds
                                              for m in rep.layers]}
        out["run_inference_disk_to_disk"] = runs
    finally:
        shutil.rmtree(root, ignore_errors=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
