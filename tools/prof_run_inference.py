import cProfile, pstats, sys, time, tempfile, shutil
from pathlib import Path
sys.path.insert(0, '/root/repo')
from paper_2605_09402_b200 import storage as S
from paper_2605_09402_b200.runtime import PipelineConfig, run_inference
root = Path(tempfile.mkdtemp(dir='/tmp'))
S.generate_synthetic("uniform", 2_400_000, 26, 100, 7, root / "d")
w = S.random_weights(S.ModelKind.GCN, [100, 128, 128, 47], 5)
cfg = PipelineConfig(chunk_budget=8 << 20, hot_slots=2_400_000, backend="tcgen05")
run_inference(root / "d", w, cfg, root / "r")
pr = cProfile.Profile(); pr.enable()
t0=time.perf_counter(); rep = run_inference(root / "d", w, cfg, root / "r"); t=time.perf_counter()-t0
pr.disable()
print("wall", t, [m.wall_seconds for m in rep.layers])
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
shutil.rmtree(root)
