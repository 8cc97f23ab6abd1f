"""GAT model definition and its float64 oracle (CPU). The reference has no
GAT, so the oracle is pinned against an independent per-edge
restatement rather than reference golden vectors (parity unpinned)."""

import numpy as np
import pytest

from oracle import gat as OG
from paper_2605_09402_b200 import gat as G
from paper_2605_09402_b200 import storage as S
from paper_2605_09402_b200.errors import ConfigError, VersionMismatchError


def hub_graph(v=300, seed=4):
    """Random graph with zero in-degree vertices, a 100-in-degree hub and
    self loops (the GAT kernel's edge cases)."""
    rng = np.random.default_rng(seed)
    src = rng.integers(0, v, 5 * v)
    dst = rng.integers(20, v, 5 * v)          # 0..19 get no in-edges
    src = np.concatenate([src, np.arange(100), [27, 28]])
    dst = np.concatenate([dst, np.full(100, 25), [27, 28]])
    return S.edges_to_csr(src, dst, v)


@pytest.mark.parametrize("heads,dims", [(1, [8, 4, 3]), (4, [12, 16, 19]),
                                        (3, [5, 9, 2])])
def test_oracle_vectorised_matches_loops(heads, dims):
    g = hub_graph()
    w = G.random_gat_weights(dims, heads, seed=3)
    x = np.random.default_rng(1).uniform(-1, 1, (g.num_vertices, dims[0]))
    h = x
    for i, lw in enumerate(w.layers):
        concat = i < len(w.layers) - 1
        a = OG.gat_layer(g.offsets, g.neighbors, h, lw.weight, lw.attn_l,
                         lw.attn_r, lw.bias, lw.heads, concat)
        b = OG.gat_layer_loops(g.offsets, g.neighbors, h, lw.weight,
                               lw.attn_l, lw.attn_r, lw.bias, lw.heads,
                               concat)
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)
        h = np.maximum(a, 0) if concat else a


def test_zero_in_degree_gives_bias():
    g = hub_graph()
    w = G.random_gat_weights([6, 8, 5], 2, seed=9)
    x = np.random.default_rng(2).uniform(-1, 1, (g.num_vertices, 6))
    out = OG.gat_per_layer(g.offsets, g.neighbors, x, w.oracle_layers())
    lw0, lw1 = w.layers
    np.testing.assert_allclose(out[0][:20], np.maximum(lw0.bias, 0)[None]
                               .repeat(20, 0), atol=0)
    mean_b = lw1.bias.astype(np.float64).reshape(2, 5).mean(0)
    np.testing.assert_allclose(out[1][:20], mean_b[None].repeat(20, 0),
                               atol=1e-15)


def test_weights_roundtrip(tmp_path):
    w = G.random_gat_weights([32, 16, 7], 4, seed=5)
    G.write_gat_weights(tmp_path / "w.awts", w)
    r = G.read_gat_weights(tmp_path / "w.awts")
    assert r.negative_slope == np.float32(w.negative_slope)
    for a, b in zip(w.layers, r.layers):
        for f in ("weight", "attn_l", "attn_r", "bias"):
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
        assert (a.in_dim, a.heads, a.head_dim) == (b.in_dim, b.heads,
                                                   b.head_dim)
    # a v1 (GCN/SAGE/GIN) file is not a GAT file
    S.write_weights(tmp_path / "v1.awts",
                    S.random_weights(S.ModelKind.GCN, [4, 3], 1))
    with pytest.raises(VersionMismatchError):
        G.read_gat_weights(tmp_path / "v1.awts")


def test_hidden_width_must_split_into_heads():
    with pytest.raises(ConfigError):
        G.random_gat_weights([8, 10, 3], 4, seed=0)


@pytest.mark.parametrize("itemsize", [4, 2])
def test_extended_weight_emits_el_er(itemsize):
    """z_ext = h . W_ext^T holds z, then el and er at the layout's
    16-byte-aligned columns."""
    w = G.random_gat_weights([24, 19], 4, seed=2)
    lw = w.layers[0]
    lay = G.ZLayout(lw.heads, lw.head_dim, itemsize)
    assert lay.el_col % lay.epc == 0 and lay.ldz % lay.epc == 0
    assert lay.head_stride % lay.epc == 0 and lay.head_stride >= 19
    assert lay.el_col == 4 * lay.head_stride
    assert lay.ldz >= lay.er_col + lw.heads
    h = np.random.default_rng(0).uniform(-1, 1, (50, 24))
    ext = G.extended_weight(lw, lay).astype(np.float64)
    zx = h @ ext.T
    z = (h @ lw.weight.astype(np.float64).T).reshape(50, 4, 19)
    el = np.einsum("vhf,hf->vh", z, lw.attn_l.astype(np.float64))
    er = np.einsum("vhf,hf->vh", z, lw.attn_r.astype(np.float64))
    zs = zx[:, :lay.el_col].reshape(50, 4, lay.head_stride)
    np.testing.assert_allclose(zs[:, :, :19], z, atol=1e-6)
    np.testing.assert_array_equal(zs[:, :, 19:], 0)
    np.testing.assert_allclose(zx[:, lay.el_col:lay.el_col + 4], el,
                               atol=1e-5)
    np.testing.assert_allclose(zx[:, lay.er_col:lay.er_col + 4], er,
                               atol=1e-5)


def test_gat_subset_oracle_matches_whole_layer():
    """oracle.gat.gat_layer_at (destination subsets, used by the IGB-Medium
    scale check) == gat_layer's rows for those destinations."""
    import numpy as np
    from oracle import gat as OG
    from paper_2605_09402_b200 import storage as S
    from paper_2605_09402_b200.gat import random_gat_weights
    g, _ = S.synthetic_in_memory("uniform", 500, 6, 4, 3)
    w = random_gat_weights([12, 16, 5], 4, seed=2).layers[0]
    h = np.random.default_rng(1).uniform(-1, 1, (500, 12))
    full = OG.gat_layer(g.offsets, g.neighbors, h, w.weight, w.attn_l,
                        w.attn_r, w.bias, w.heads, concat=True)
    dests = np.array([0, 7, 99, 250, 499])
    src = np.repeat(np.arange(500), np.diff(g.offsets))
    dst = np.asarray(g.neighbors, np.int64)
    lists = [src[dst == t] for t in dests]
    offs = np.concatenate([[0], np.cumsum([len(x) for x in lists])])
    srcs = np.concatenate(lists)
    uniq, inv = np.unique(srcs, return_inverse=True)
    got = OG.gat_layer_at(dests, offs, inv, h[uniq], h[dests], w.weight,
                          w.attn_l, w.attn_r, w.bias, w.heads, concat=True)
    np.testing.assert_allclose(got, full[dests], rtol=0, atol=1e-12)
