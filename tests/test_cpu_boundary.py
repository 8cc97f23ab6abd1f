"""CPU-only checks of the boundary: formats, chunk plan, library symbols,
and the oracle pinned to the reference's golden vectors."""

import re
from pathlib import Path

import numpy as np
import pytest

from helpers import (REFERENCE_SRC, case_weights, dataset, digest_array,
                     flatten_events, golden_arrays, golden_manifest,
                     oracle_case)
from paper_2605_09402_b200 import _native as N
from paper_2605_09402_b200 import storage as S
from paper_2605_09402_b200.chunks import plan_chunks

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_header_symbol():
    lib = N.load_library()
    header = (ROOT / "include" / "atlas_b200.h").read_text()
    declared = set(re.findall(r"ATLAS_API [a-z0-9_ \*]*?(atlas_[a-z0-9_]+)\(",
                              header))
    assert declared == set(N.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.atlas_abi_version() == 1


def test_no_oracle_import_in_product():
    for p in (ROOT / "paper_2605_09402_b200").rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p


@pytest.mark.parametrize("key", list(golden_manifest()["_plans"]))
def test_plan_chunks_matches_reference(key):
    v, d, t, b = key.split("_")
    plan = plan_chunks(int(v), int(d), t, int(b))
    n, head, tail = golden_manifest()["_plans"][key]
    assert len(plan) == n
    assert [list(x) for x in plan[:3]] == head
    assert [list(x) for x in plan[-1:]] == tail


def test_formats_roundtrip_and_damage(tmp_path):
    g = S.edges_to_csr(np.array([0, 0, 2, 4, 4]), np.array([1, 3, 3, 1, 3]),
                       6)
    S.write_csr(g, tmp_path)
    back = S.read_csr(tmp_path)
    assert np.array_equal(back.offsets, g.offsets)
    assert np.array_equal(back.neighbors, g.neighbors)
    assert np.array_equal(back.in_degrees, [0, 2, 0, 3, 0, 0])
    rng = np.random.default_rng(8)
    for dt in (np.float32, np.float16):
        ids = np.arange(5, 12)
        rows = rng.uniform(-2, 2, (7, 6)).astype(dt)
        S.write_spill_file(tmp_path / f"s_{dt.__name__}", ids, rows)
        bi, br = S.read_spill_file(tmp_path / f"s_{dt.__name__}")
        assert np.array_equal(bi, ids) and br.tobytes() == rows.tobytes()
    w = S.random_weights(S.ModelKind.SAGE, [6, 4, 2], 9, gin_epsilon=0.25)
    S.write_weights(tmp_path / "w.bin", w)
    bw = S.read_weights(tmp_path / "w.bin")
    assert bw.kind == w.kind and bw.gin_epsilon == 0.25
    perm = rng.permutation(40)
    S.write_permutation(tmp_path / "p.bin", perm)
    assert np.array_equal(S.read_permutation(tmp_path / "p.bin"), perm)
    topo = tmp_path / S.TOPOLOGY_FILE
    blob = bytearray(topo.read_bytes())
    blob[:4] = b"NOPE"
    topo.write_bytes(bytes(blob))
    with pytest.raises(S.BadMagicError):
        S.read_csr(tmp_path)
    sp = tmp_path / "s_float32"
    sp.write_bytes(sp.read_bytes()[:-4096])
    with pytest.raises(S.TruncatedFileError):
        S.read_spill_file(sp)


@pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference absent")
def test_files_byte_identical_to_reference(tmp_path):
    import sys
    sys.path.insert(0, str(REFERENCE_SRC))
    import oocgnn.storage as R
    for kind, v, deg, dim, seed, dt in [("uniform", 3000, 6, 8, 3, "f32"),
                                        ("pa", 2000, 5, 16, 12, "f16")]:
        a, b = tmp_path / f"a{kind}", tmp_path / f"b{kind}"
        R.generate_synthetic(kind, v, deg, dim, seed, a, dtype=dt)
        S.generate_synthetic(kind, v, deg, dim, seed, b, dtype=dt)
        for pa in a.rglob("*"):
            if pa.is_file():
                pb = b / pa.relative_to(a)
                assert pa.read_bytes() == pb.read_bytes(), pa


FAST = ["fig2_gcn", "fig2_sage", "fig2_gin", "small_gcn_tight",
        "small_sage_tight", "small_gin_tight", "half_gcn_slots300",
        "half_sage_slots300", "half_gin_slots300", "uniform_gcn_slots500",
        "wide_sage"]


@pytest.mark.parametrize("case", FAST)
def test_oracle_pinned_to_reference_goldens(case):
    entry = golden_manifest()[case]
    for l, (out, m, log) in enumerate(oracle_case(case)):
        g = entry["layers"][l]
        assert digest_array(out) == g["output_sha"]
        assert digest_array(flatten_events(log.victims)) == g["victims_sha"]
        assert digest_array(flatten_events(log.reloads)) == g["reloads_sha"]
        assert digest_array(flatten_events(log.graduated)) == \
            g["graduated_sha"]
        for f in ("messages", "evictions", "reloads", "unique_reloads",
                  "mean_span", "p99_span", "mean_reload_pct", "hot_peak",
                  "hot_slot_count"):
            assert getattr(m, f) == g[f], f


def test_pcg64_restatement_matches_numpy():
    """engine.cu's RandomPolicy draw (PCG64 step, generator-level u32
    buffering, Lemire bounded ints) restated in Python vs numpy."""
    mult = (2549297995355413924 << 64) + 4865540595714422341
    mask64 = (1 << 64) - 1
    for seed in (0, 1, 7):
        st = np.random.default_rng(seed).bit_generator.state
        gen = {"s": st["state"]["state"], "inc": st["state"]["inc"],
               "has": 0, "keep": 0}

        def next32():
            if gen["has"]:
                gen["has"] = 0
                return gen["keep"]
            gen["s"] = (gen["s"] * mult + gen["inc"]) & ((1 << 128) - 1)
            hi, lo = gen["s"] >> 64, gen["s"] & mask64
            x, rot = hi ^ lo, hi >> 58
            out = ((x >> rot) | (x << ((-rot) & 63))) & mask64
            gen["has"], gen["keep"] = 1, out >> 32
            return out & 0xFFFFFFFF

        ref = np.random.default_rng(seed)
        draws = np.random.default_rng(seed + 100).integers(1, 10**6, 3000)
        for n in draws.tolist():
            want = int(ref.integers(n))
            if n == 1:
                got = 0
            else:
                m = next32() * n
                if (m & 0xFFFFFFFF) < n:
                    thr = (0xFFFFFFFF - (n - 1)) % n
                    while (m & 0xFFFFFFFF) < thr:
                        m = next32() * n
                got = m >> 32
            assert got == want


def test_markstein_division(tmp_path):
    """The aggregation kernel's division (aggregate.cu div_rn): RN(m/d) via
    q = RN(m*RN(1/d)), e = fma(-q,d,m), RN(fma(e,r,q)); checked against
    IEEE division on ~1e8 (m, d) pairs (normal or zero quotients)."""
    import subprocess
    src = Path(__file__).resolve().parent / "native" / "markstein_check.c"
    exe = tmp_path / "markstein"
    subprocess.run(["gcc", "-O2", "-mfma", "-o", str(exe), str(src), "-lm"],
                   check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True,
                         text=True).stdout
    assert out.strip().endswith("bad(normal results)=0"), out


GATHER_CASES = [c for c in golden_manifest() if not c.startswith("_")]


@pytest.mark.parametrize("case", GATHER_CASES)
def test_gather_oracle_pinned_to_reference_oracle(case):
    """oracle/gather.py (the f64 oracle behind every tolerance test) equals
    the reference's own ``oracle_inference`` (oocgnn/oracle.py:26-55) as
    make_golden stored it: the last layer rounded to f32, every row for the
    small cases and the first 64 rows otherwise. Same CSR construction,
    same f64 operation order, so the f32 roundings must agree exactly."""
    from oracle import gather as G

    entry = golden_manifest()[case]
    graph, feats = dataset(entry["dataset"])
    w = case_weights(entry)
    outs = G.per_layer(graph.num_vertices, graph.offsets, graph.neighbors,
                       graph.in_degrees, feats, int(w.kind),
                       [(lw.weight, lw.bias) for lw in w.layers],
                       gin_epsilon=w.gin_epsilon)
    want = golden_arrays(case)["oracle64"]
    got = outs[-1].astype(np.float32)[:len(want)]
    np.testing.assert_array_equal(got, want)
    if len(want) == graph.num_vertices:
        assert digest_array(outs[-1].astype(np.float32)) == \
            entry["oracle64_sha"]
    assert float(np.abs(outs[-1]).max().astype(np.float32)) == \
        entry["oracle64_absmax"]


def test_cfg2_scale_golden_is_self_consistent():
    """The benchmark-scale golden (make_golden.py scale, one run of the
    unmodified reference at cfg2): the reference engine's f32 rows sit
    within the reference's own 1e-4 bar of its float64 oracle rows
    (tests/test_acceptance.py:43), and the row sample and metrics are the
    shape the GPU tests expect."""
    import json
    from helpers import GOLDEN
    man = json.loads((GOLDEN / "golden_scale.json").read_text())["cfg2_gcn"]
    arrays = dict(np.load(GOLDEN / "cfg2_gcn.npz"))
    assert man["num_edges"] == 62_399_647 and len(man["layers"]) == 3
    assert len(arrays["rows"]) == 2048
    for l, lay in enumerate(man["layers"]):
        assert lay["messages"] == man["num_edges"]
        d = np.abs(arrays[f"L{l}_out_rows"].astype(np.float64)
                   - arrays[f"L{l}_oracle_rows"])
        assert d.max() <= 1e-4
        assert abs(lay["output_absmax"] - lay["oracle_absmax"]) <= 1e-6
