"""Float64 GAT oracle (TEST INFRASTRUCTURE ONLY) — parity UNPINNED.

The reference has no GAT, so there is nothing of the
reference's to pin this to. It restates the semantics SURVEY.md A.5 fixes
for BASELINE config 3, in the reference oracle's own conventions
(oocgnn/oracle.py:26-55: float64, edges (src -> dst) from the CSR, ReLU
between layers, none after the last):

    z_u      = W h_u                       reshaped (H, F)
    el_u[h]  = a_l[h] . z_u[h]             er_v[h] = a_r[h] . z_v[h]
    e_uv[h]  = LeakyReLU_slope(el_u[h] + er_v[h])          (slope 0.2)
    alpha_uv = softmax over the in-edges of v of e_uv      (per head)
    out_v[h] = sum_u alpha_uv[h] z_u[h] + b[h]
    hidden layers concatenate the heads (H*F), the last averages them (F);
    zero in-degree -> out_v = b (like the max(1, d_in) convention); no
    self-loops are added (consistent with the reference GCN).

Two independent restatements are kept: ``gat_layers`` (vectorised, scipy
segment sums) and ``gat_layer_loops`` (a per-destination Python walk for
small graphs), and the tests check them against each other.
"""

import numpy as np


def leaky(x, slope):
    return np.where(x >= 0, x, slope * x)


def _edges(offsets, neighbors):
    v = len(offsets) - 1
    src = np.repeat(np.arange(v, dtype=np.int64), np.diff(offsets))
    return src, np.asarray(neighbors, dtype=np.int64)


def gat_layer(offsets, neighbors, h, weight, attn_l, attn_r, bias, heads,
              concat, slope=0.2):
    """One layer in float64; returns (V, H*F) if concat else (V, F)."""
    h = np.asarray(h, np.float64)
    v = h.shape[0]
    hf = weight.shape[0]
    f = hf // heads
    z = (h @ np.asarray(weight, np.float64).T).reshape(v, heads, f)
    el = np.einsum("vhf,hf->vh", z, np.asarray(attn_l, np.float64))
    er = np.einsum("vhf,hf->vh", z, np.asarray(attn_r, np.float64))
    src, dst = _edges(offsets, neighbors)
    e = leaky(el[src] + er[dst], slope)                      # (E, H)
    emax = np.full((v, heads), -np.inf)
    np.maximum.at(emax, dst, e)
    p = np.exp(e - emax[dst])
    s = np.zeros((v, heads))
    np.add.at(s, dst, p)
    alpha = p / s[dst]
    out = np.zeros((v, heads, f))
    np.add.at(out, dst, alpha[:, :, None] * z[src])
    out += np.asarray(bias, np.float64).reshape(heads, f)
    return out.reshape(v, hf) if concat else out.mean(axis=1)


def gat_layer_loops(offsets, neighbors, h, weight, attn_l, attn_r, bias,
                    heads, concat, slope=0.2):
    """Same layer, walked destination by destination (small graphs)."""
    h = np.asarray(h, np.float64)
    v = h.shape[0]
    hf = weight.shape[0]
    f = hf // heads
    z = (h @ np.asarray(weight, np.float64).T).reshape(v, heads, f)
    al, ar = np.asarray(attn_l, np.float64), np.asarray(attn_r, np.float64)
    b = np.asarray(bias, np.float64).reshape(heads, f)
    ins = [[] for _ in range(v)]
    for u in range(v):
        for t in neighbors[offsets[u]:offsets[u + 1]]:
            ins[int(t)].append(u)
    out = np.zeros((v, heads, f))
    for t in range(v):
        for k in range(heads):
            acc = np.zeros(f)
            if ins[t]:
                er = float(ar[k] @ z[t, k])
                es = [leaky(float(al[k] @ z[u, k]) + er, slope)
                      for u in ins[t]]
                m = max(es)
                ws = [np.exp(x - m) for x in es]
                tot = sum(ws)
                for u, w in zip(ins[t], ws):
                    acc += (w / tot) * z[u, k]
            out[t, k] = acc + b[k]
    return out.reshape(v, hf) if concat else out.mean(axis=1)


def gat_per_layer(offsets, neighbors, features, layers, slope=0.2):
    """layers: list of (weight, attn_l, attn_r, bias, heads). Hidden layers
    concatenate heads and apply ReLU; the last averages heads. Returns the
    list of every layer's float64 output."""
    h = np.asarray(features, np.float64)
    outs = []
    for i, (w, al, ar, b, heads) in enumerate(layers):
        last = i == len(layers) - 1
        h = gat_layer(offsets, neighbors, h, w, al, ar, b, heads,
                      concat=not last, slope=slope)
        if not last:
            h = np.maximum(h, 0.0)
        outs.append(h)
    return outs


def gat_layer_at(dests, in_offsets, in_sources, h_src, h_dst, weight, attn_l,
                 attn_r, bias, heads, concat, slope=0.2):
    """The same layer for a SUBSET of destinations (float64), for checks at
    scales where whole layers do not fit the host: ``dests`` (n,) sampled
    destinations, ``in_offsets`` (n+1,) / ``in_sources`` their in-edges as
    row indices into ``h_src`` (the source rows the sample needs), ``h_dst``
    (n, in) the destinations' own rows (for er). Returns (n, H*F) or (n, F)
    -- ``gat_layer``'s rows for ``dests`` when h_src/h_dst are the layer
    input's rows."""
    w = np.asarray(weight, np.float64)
    hf = w.shape[0]
    f = hf // heads
    al, ar = np.asarray(attn_l, np.float64), np.asarray(attn_r, np.float64)
    zs = (np.asarray(h_src, np.float64) @ w.T).reshape(-1, heads, f)
    zd = (np.asarray(h_dst, np.float64) @ w.T).reshape(-1, heads, f)
    el = np.einsum("vhf,hf->vh", zs, al)
    er = np.einsum("vhf,hf->vh", zd, ar)
    n = len(dests)
    deg = np.diff(in_offsets)
    dst = np.repeat(np.arange(n), deg)
    src = np.asarray(in_sources, np.int64)
    e = leaky(el[src] + er[dst], slope)
    emax = np.full((n, heads), -np.inf)
    np.maximum.at(emax, dst, e)
    p = np.exp(e - emax[dst])
    s = np.zeros((n, heads))
    np.add.at(s, dst, p)
    out = np.zeros((n, heads, f))
    np.add.at(out, dst, (p / s[dst])[:, :, None] * zs[src])
    out += np.asarray(bias, np.float64).reshape(heads, f)
    return out.reshape(n, hf) if concat else out.mean(axis=1)
