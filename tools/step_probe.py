"""Host-side timing of back-to-back infer(metrics=False) steps (diagnostic)."""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_09402_b200 import storage as S
from paper_2605_09402_b200.runtime import Engine, PipelineConfig

g, f = S.synthetic_in_memory("uniform", 2_400_000, 26, 100, 7)
w = S.random_weights(S.ModelKind.GCN, [100, 128, 128, 47], 5)
eng = Engine(g, w, PipelineConfig(chunk_budget=8 << 20, hot_slots=2_400_000, backend="tcgen05"))
x = torch.from_numpy(f).cuda()
for _ in range(3):
    eng.infer(x)
torch.cuda.synchronize()
HOST = {}


def _trace(cls, names):
    for n in names:
        f = getattr(cls, n)

        def wrap(*a, _f=f, _n=n, **k):
            t = time.perf_counter()
            try:
                return _f(*a, **k)
            finally:
                HOST.setdefault(_n, []).append(
                    round(1e3 * (time.perf_counter() - t), 2))
        setattr(cls, n, wrap)


from paper_2605_09402_b200 import engine as _E  # noqa: E402
_trace(_E.DeviceLayer, ["reset", "run_resident", "run_fused",
                        "accumulator_ptr"])
_trace(_E, ["transform_device", "transform_typed"])
for trial in range(4):
    HOST.clear()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    hs = []
    evs[0].record()
    for i in range(6):
        t0 = time.perf_counter()
        eng.infer(x, metrics=False)
        hs.append(1e3 * (time.perf_counter() - t0))
        evs[i + 1].record()
    torch.cuda.synchronize()
    print("host ms", [round(h, 2) for h in hs])
    print("dev ms ", [round(evs[i].elapsed_time(evs[i + 1]), 2) for i in range(6)])
    print("  per call host ms:", {k: v for k, v in HOST.items()})
