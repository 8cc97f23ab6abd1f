"""The sweep formulation of the exact control machine (csrc/sweep.cu),
restated in Python and checked against the oracle machine (oracle/engine.py,
itself pinned to the reference's MemoryManager, oocgnn/memstore.py:305-497)
on random graphs with tight slot budgets: every eviction event's victims in
pop order, reloads per chunk, unique reloads and the hot peak.

The sweep never tracks per-vertex state. Its claims (sweep.cu header):
the delivery stream, each delivery's post-delivery pending count and each
vertex's next delivery are static; the bucket heap is the static list of
deliveries per pending value read from a forward-only head; an entry is in
the heap at sub-batch s iff sub(e) < s <= next(e) and no earlier pop took it.
"""

import numpy as np
import pytest

from oracle import engine as OE

GCN, SAGE, GIN = OE.GCN, OE.SAGE, OE.GIN


def static_stream(offsets, neighbors, indeg, model, chunk_rows, sub_batch,
                  lo, hi):
    """Elements (v, cnt, sub) in stream order, the chunk of every
    sub-batch and touched counts per chunk (oocgnn/orchestrator.py:216-299)."""
    V = len(indeg)
    els, sub_chunk, touched = [], [], []
    for c, start in enumerate(range(0, V, chunk_rows)):
        end = min(start + chunk_rows, V)
        src = np.arange(start, end)
        mine = src[(src >= lo) & (src < hi)]
        passes = []
        if model == GCN:
            passes.append([(v, 0) for v in mine if indeg[v] == 0])
        if model == SAGE:
            passes.append([(v, 1) for v in mine])
        else:
            passes.append([])
        first, count, order = {}, {}, 0
        for u in range(start, end):
            if model == GIN:
                if u not in first:
                    first[u] = order
                count[u] = count.get(u, 0) + 1
                order += 1
            for j in range(offsets[u], offsets[u + 1]):
                d = int(neighbors[j])
                if d not in first:
                    first[d] = order
                count[d] = count.get(d, 0) + 1
                order += 1
        edge = sorted((d for d in first if lo <= d < hi), key=first.get)
        passes.append([(d, count[d]) for d in edge])
        t = (len(mine) if model == SAGE else 0) + len(edge)
        touched.append(t)
        for p in passes:
            for i in range(0, len(p), sub_batch):
                s = len(sub_chunk)
                sub_chunk.append(c)
                els.extend((v, cnt, s) for v, cnt in p[i:i + sub_batch])
    return els, sub_chunk, touched


def sweep(els, sub_chunk, touched, indeg, model, slots, evict_batch, lru):
    pend0 = indeg.astype(np.int64) + (0 if model == GCN else 1)
    S = len(sub_chunk)
    by_v = {}
    for i, (v, cnt, s) in enumerate(els):
        by_v.setdefault(v, []).append(i)
    newp = [0] * len(els)
    nxt = [0] * len(els)
    fresh = [0] * S
    grad = [0] * S
    for v, idx in by_v.items():
        left = int(pend0[v])
        for q, i in enumerate(idx):
            left -= els[i][1]
            newp[i] = left
            nxt[i] = els[idx[q + 1]][2] if q + 1 < len(idx) else 0
        assert left == 0
        fresh[els[idx[0]][2]] += 1
    for i, (v, cnt, s) in enumerate(els):
        grad[s] += newp[i] == 0
    # heap lists: stable by pending value (MINPEND) or the stream (LRU)
    if lru:
        order = list(range(len(els)))
        keys = [0] * len(els)
        b0, nb = 0, 1
    else:
        order = sorted(range(len(els)), key=lambda i: newp[i])
        keys = [newp[i] for i in order]
        b0, nb = 1, max(newp, default=0) + 1
    boff = [0] * (nb + 1)
    for b in range(nb + 1):
        boff[b] = sum(1 for k in keys if k < b) if not lru else (
            0 if b == 0 else len(els))
    head = boff[:nb]
    ent_sub = [els[i][2] for i in order]
    ent_next = [nxt[i] if (lru and newp[i] > 0) or (not lru and newp[i] > 0)
                else 0 for i in order]
    cold = [0] * S
    hot = peak = evictions = reloads = 0
    events = []
    for s in range(S):
        mode_need = None
        while True:
            need = fresh[s] + cold[s]
            if need <= slots - hot:
                break
            assert need <= slots
            mode_need = need
            while slots - hot < mode_need:
                k = min(max(evict_batch, mode_need - (slots - hot)), hot)
                assert k > 0
                got = []
                b = b0
                while len(got) < k:
                    assert b < nb, "heap underflow"
                    h = head[b]
                    while h < boff[b + 1] and len(got) < k:
                        if ent_sub[h] >= s:
                            break
                        if ent_next[h] >= s:
                            got.append(h)
                        h += 1
                    head[b] = h
                    if len(got) < k:
                        b += 1
                for e in got:
                    cold[ent_next[e]] += 1
                events.append([els[order[e]][0] for e in got])
                hot -= k
                evictions += k
        hot += need
        peak = max(peak, hot)
        reloads += cold[s]
        hot -= grad[s]
    chunk_rel = [0] * len(touched)
    for s in range(S):
        chunk_rel[sub_chunk[s]] += cold[s]
    uniq = len({v for ev in events for v in ev})
    return dict(evictions=evictions, reloads=reloads, hot_peak=peak,
                unique=uniq, events=events, chunk_reloads=chunk_rel)


def random_graph(rng, V, avg, power):
    E = V * avg
    if power:
        w = 1.0 / np.arange(1, V + 1) ** 0.9
        dst = rng.choice(V, size=E, p=w / w.sum())
    else:
        dst = rng.integers(0, V, E)
    src = np.sort(rng.integers(0, V, E))
    offsets = np.zeros(V + 1, dtype=np.int64)
    np.add.at(offsets, src + 1, 1)
    offsets = np.cumsum(offsets)
    nbrs = dst[np.argsort(src, kind="stable")].astype(np.int64)
    indeg = np.bincount(nbrs, minlength=V).astype(np.int64)
    return offsets, nbrs, indeg


CASES = [
    # (seed, V, avg, power, model, chunk_rows, slots, policy, dst_range)
    (1, 300, 4, False, GCN, 17, 40, "minpend", None),
    (2, 300, 6, True, SAGE, 23, 32, "minpend", None),
    (3, 400, 5, False, GIN, 31, 60, "minpend", None),
    (4, 300, 4, True, GCN, 9, 25, "lru", None),
    (5, 350, 6, False, SAGE, 40, 50, "lru", None),
    (6, 300, 5, False, GIN, 13, 30, "lru", None),
    (7, 500, 8, True, SAGE, 50, 45, "minpend", (120, 330)),
    (8, 500, 3, False, GCN, 7, 12, "minpend", (0, 250)),
    (9, 200, 2, True, GCN, 11, 3, "minpend", None),
    (10, 200, 5, False, SAGE, 200, 20, "lru", (50, 150)),
]


@pytest.mark.parametrize("case", CASES, ids=[str(c[0]) for c in CASES])
def test_sweep_equals_machine(case):
    seed, V, avg, power, model, rows, slots, pol, rng_ = case
    rng = np.random.default_rng(seed)
    offsets, nbrs, indeg = random_graph(rng, V, avg, power)
    lo, hi = rng_ if rng_ else (0, V)
    feats = rng.standard_normal((V, 4)).astype(np.float32)
    agg_dim = 8 if model == SAGE else 4
    W = np.zeros((3, agg_dim), np.float32)
    _, m, log = OE.run_layer(offsets, nbrs, indeg, feats, model, W,
                             np.zeros(3, np.float32), False, embed_dim=4,
                             agg_dim=agg_dim, chunk_rows=rows,
                             slot_count=slots, eviction=pol,
                             dst_range=rng_)
    assert m.evictions > 0, "case must evict"
    sub_batch = max(1, slots // 2)
    evict_batch = max(1, slots // 100)
    els, sub_chunk, touched = static_stream(offsets, nbrs, indeg, model,
                                            rows, sub_batch, lo, hi)
    got = sweep(els, sub_chunk, touched, indeg, model, slots, evict_batch,
                pol == "lru")
    assert got["events"] == [list(ev) for ev in log.victims]
    assert got["evictions"] == m.evictions
    assert got["reloads"] == m.reloads
    assert got["unique"] == m.unique_reloads
    assert got["hot_peak"] == m.hot_peak
    pcts = [100.0 * r / max(1, t) for r, t in
            zip(got["chunk_reloads"], touched)]
    assert pcts == log.chunk_reload_pcts
