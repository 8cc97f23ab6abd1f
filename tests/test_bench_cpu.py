"""bench.py's roofline bookkeeping on CPU: the algorithmic-byte formulas
 against hand counts on a tiny graph, and the
per-layer transform roofline object."""

import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402
from helpers import fig2_graph  # noqa: E402
from paper_2605_09402_b200 import gat as G  # noqa: E402
from paper_2605_09402_b200 import storage as S  # noqa: E402


class _AggFirst:
    def transform_first(self, l):
        return False


def test_agg_bytes_gcn_hand_count():
    g = fig2_graph()  # 6 vertices, 5 edges
    w = S.random_weights(S.ModelKind.GCN, [8, 4, 2], 1)
    got = bench.agg_bytes(g, w, (0, 6), [4, 4], _AggFirst())
    e, v = 5, 6
    # layer 0: 8-d f32 source rows per edge, u32 ids, CSC/degree, records
    assert got[0] == e * 8 * 4 + 4 * e + 12 * v + 4 * 8 * v
    assert got[1] == e * 4 * 4 + 4 * e + 12 * v + 4 * 4 * v


def test_agg_bytes_sage_reads_self_rows():
    g = fig2_graph()
    w = S.random_weights(S.ModelKind.SAGE, [8, 4, 2], 1)
    got = bench.agg_bytes(g, w, (0, 6), [2, 4], _AggFirst())
    e, v = 5, 6
    # f16 input, self row read once per destination, 2d-wide records
    assert got[0] == e * 8 * 2 + 4 * e + 12 * v + v * 8 * 2 + 4 * 16 * v


def test_gat_bytes_drop_el_sector_for_line_aligned_rows():
    g = fig2_graph()
    w = G.random_gat_weights([8, 8, 3], 2, seed=1)
    f32 = [G.ZLayout(lw.heads, lw.head_dim, 4) for lw in w.layers]
    f16 = [G.ZLayout(lw.heads, lw.head_dim, 2) for lw in w.layers]
    assert all(lay.line_rows for lay in f32)
    assert not any(lay.line_rows for lay in f16)
    a = bench.gat_agg_bytes(g, w, f32, (0, 6), 4)
    b = bench.gat_agg_bytes(g, w, f16, (0, 6), 4)
    assert [y - x for x, y in zip(a, b)] == [32 * 5] * len(a)
    # line-aligned f32 layouts start rows on 128-byte lines
    assert all(lay.ldz * 4 % 128 == 0 for lay in f32)
    assert all(lay.ncols <= lay.ldz for lay in f32)


def test_transform_roofline_object():
    w = S.random_weights(S.ModelKind.GCN, [8, 4, 2], 1)
    steps = [[SimpleNamespace(transform_ms=0.5), SimpleNamespace(
        transform_ms=0.25)]] * 2
    out = bench.transform_roofline(w, _AggFirst(), steps, [4, 4],
                                   {"hbm_gbs": 1000.0}, nloc=10 ** 7,
                                   nrows=10 ** 7)
    l0, l1 = out["layers"]
    m = 10 ** 7
    assert (l0["rows"], l0["k"], l0["n"]) == (m, 8, 4)
    assert l0["bytes"] == m * 8 * 4 + m * 4 * 4 + 4 * 8 * 4
    assert np.isclose(l0["hbm_gbs"], l0["bytes"] / 0.5e-3 / 1e9, rtol=1e-3)
    assert np.isclose(l0["hbm_frac"], l0["hbm_gbs"] / 1000.0, atol=1e-3)
    # last layer writes f32
    assert l1["bytes"] == m * 4 * 4 + m * 2 * 4 + 2 * 4 * 4
    assert out["bound"] == "hbm"
