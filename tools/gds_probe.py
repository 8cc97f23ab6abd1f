"""Device spill reader diagnostics: reads one layer dir into HBM through
the bounce path (and through cuFile with ATLAS_GDS=1), printing progress,
so a hang shows where it stops. Usage: gds_probe.py [rows] [dim]"""
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_09402_b200 import _native as N  # noqa: E402
from paper_2605_09402_b200 import chunks as C  # noqa: E402
from paper_2605_09402_b200 import storage as S  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 64
root = Path(tempfile.mkdtemp(prefix="gds_", dir=sys.argv[3] if len(sys.argv) > 3 else "/tmp"))
m = np.random.default_rng(0).uniform(-1, 1, (rows, dim)).astype(np.float32)
S.write_matrix_as_layer(root / "l", m, partitions=4, spill_rows=4096)
print("written", root, flush=True)
print("status:", N.load_library().atlas_gds_status().decode(), flush=True)
t = time.perf_counter()
_, dev, nb, _, gds = C.load_layer_device(root / "l", threads=4)
print("read", "cuFile" if gds else "bounce", f"{time.perf_counter() - t:.3f} s",
      "equal", bool((dev.cpu().numpy() == m).all()), flush=True)
