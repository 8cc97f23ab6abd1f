"""CPU restatement of the reference's broadcast layer engine.

TEST INFRASTRUCTURE ONLY. Nothing in the product package imports this
module; it is used by tests/, by ``__graft_entry__.smoke()`` as the
checker, and by ``bench.py`` as the timed CPU baseline (``cpu_baseline``
and ``--impl reference``). It restates, in numpy, the algorithm of:

* ``init_layer``      oocgnn/orchestrator.py:93-145
* ``process_chunk``   oocgnn/orchestrator.py:216-299
* ``_deliver``        oocgnn/orchestrator.py:165-213
* ``finalize_layer``  oocgnn/orchestrator.py:302-323
* ``MemoryManager``   oocgnn/memstore.py:305-497 (cold store kept in a dict
  instead of a file; same byte accounting)
* ``PendingBucketHeap``/``MinPendingPolicy`` oocgnn/memstore.py:103-214,
  ``LruPolicy`` :217-237, ``RandomPolicy`` :240-273
* ``MatmulBackend.apply`` (fixed k-order f32) oocgnn/compute.py:39-47 and
  ``transform`` :76-97

It additionally records the integer event log the GPU engine must
reproduce bit-exactly: the victim list of every
eviction, the reload list of every admission batch, and the graduation
order with its sub-batch grouping.

Pinned against the reference: tests/test_cpu_boundary.py
(``test_oracle_pinned_to_reference_goldens``) compares every output, metric
and event log of this module with the committed fixtures under
tests/golden/, which tests/golden/make_golden.py produced by running the
unmodified reference.
"""

from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

NOT_STARTED, HOT, COLD, COMPLETED = 0, 1, 2, 3
GCN, SAGE, GIN = 0, 1, 2


class OracleError(Exception):
    pass


# -- policies (oocgnn/memstore.py:103-283) ----------------------------------


class BucketHeap:
    """FIFO buckets keyed by pending count (oocgnn/memstore.py:103-193).

    Restated with one OrderedDict per key: insertion order is FIFO and
    pop_min walks keys upward from the cached minimum."""

    def __init__(self, max_key: int):
        self.max_key = max_key
        self.buckets = [OrderedDict() for _ in range(max_key + 1)]
        self.key = {}
        self.low = max_key + 1

    def __len__(self):
        return len(self.key)

    def insert(self, v: int, k: int) -> None:
        if v in self.key or not 0 <= k <= self.max_key:
            raise OracleError(f"bad insert {v} {k}")
        self.key[v] = k
        self.buckets[k][v] = None
        self.low = min(self.low, k)

    def move(self, v: int, k: int) -> None:
        old = self.key[v]
        if k == old:
            return
        if k > old:
            raise OracleError("key may only decrease")
        del self.buckets[old][v]
        self.key[v] = k
        self.buckets[k][v] = None
        self.low = min(self.low, k)

    def remove(self, v: int) -> None:
        del self.buckets[self.key.pop(v)][v]

    def pop_min(self, k: int) -> list:
        out = []
        b = self.low
        while len(out) < k and b <= self.max_key:
            bucket = self.buckets[b]
            if not bucket:
                b += 1
                continue
            v, _ = bucket.popitem(last=False)
            del self.key[v]
            out.append(v)
        self.low = b
        return out


class MinPending:
    name = "minpend"

    def __init__(self, max_pending: int):
        self.heap = BucketHeap(max_pending)

    def on_admit(self, v, p):
        self.heap.insert(v, p)

    def on_message(self, v, p):
        self.heap.move(v, p)

    def on_remove(self, v):
        self.heap.remove(v)

    def choose_victims(self, k):
        return self.heap.pop_min(k)


class Lru:
    name = "lru"

    def __init__(self):
        self.order = OrderedDict()

    def on_admit(self, v, p):
        self.order[v] = None

    def on_message(self, v, p):
        self.order.move_to_end(v)

    def on_remove(self, v):
        del self.order[v]

    def choose_victims(self, k):
        return [self.order.popitem(last=False)[0] for _ in range(k)]


class Rnd:
    name = "rnd"

    def __init__(self, seed: int):
        self.rng = np.random.default_rng(seed)
        self.members = []
        self.pos = {}

    def on_admit(self, v, p):
        self.pos[v] = len(self.members)
        self.members.append(v)

    def on_message(self, v, p):
        pass

    def _take(self, i: int) -> int:
        last = self.members.pop()
        if i == len(self.members):
            victim = last
        else:
            victim = self.members[i]
            self.members[i] = last
            self.pos[last] = i
        del self.pos[victim]
        return victim

    def on_remove(self, v):
        self._take(self.pos[v])

    def choose_victims(self, k):
        return [self._take(int(self.rng.integers(len(self.members))))
                for _ in range(k)]


def make_policy(name: str, max_pending: int, seed: int):
    if name == "minpend":
        return MinPending(max_pending)
    if name == "lru":
        return Lru()
    if name == "rnd":
        return Rnd(seed)
    raise OracleError(f"unknown eviction policy {name!r}")


# -- layer state ---------------------------------------------------------------


@dataclass
class Log:
    """Integer event log."""

    victims: list = field(default_factory=list)      # per eviction event
    reloads: list = field(default_factory=list)      # per reload batch
    graduated: list = field(default_factory=list)    # per release batch
    chunk_reload_pcts: list = field(default_factory=list)


@dataclass
class Metrics:
    messages: int = 0
    evictions: int = 0
    reloads: int = 0
    unique_reloads: int = 0
    mean_span: float = 0.0
    p99_span: float = 0.0
    mean_reload_pct: float = 0.0
    hot_peak: int = 0
    hot_slot_count: int = 0
    cold_bytes_read: int = 0
    cold_bytes_written: int = 0


class Layer:
    """One layer pass: LayerContext + MemoryManager of the reference."""

    def __init__(self, in_degrees, model: int, embed_dim: int, agg_dim: int,
                 slot_count: int, *, gin_epsilon: float = 0.0,
                 eviction: str = "minpend", seed: int = 0,
                 evict_batch=None, sink=None, dst_range=None):
        v = len(in_degrees)
        # one GPU rank = the same machine restricted to the
        # destinations [lo, hi); stream positions stay global
        self.lo, self.hi = dst_range if dst_range else (0, v)
        self.model = model
        self.in_degrees = np.asarray(in_degrees, dtype=np.int64)
        self.embed_dim = embed_dim
        self.agg_dim = agg_dim
        self.eps = gin_epsilon
        self.pending = self.in_degrees.astype(np.uint32)
        if model in (SAGE, GIN):
            self.pending = self.pending + np.uint32(1)
        self.state = np.zeros(v, dtype=np.uint8)
        if slot_count < 1:
            raise OracleError("slot_count must be >= 1")
        self.slot_count = slot_count
        self.slots = np.zeros((slot_count, agg_dim), dtype=np.float32)
        self.slot_of = {}
        self.free = list(range(slot_count - 1, -1, -1))
        self.cold = {}
        max_pending = int(self.pending.max()) if v else 1
        self.policy = make_policy(eviction, max_pending, seed)
        self.evict_batch = evict_batch or max(1, slot_count // 100)
        self.sub_batch = max(1, slot_count // 2)
        self.unique_reloaded = np.zeros(v, dtype=bool)
        self.first = np.full(v, -1, dtype=np.int64)
        self.last = np.full(v, -1, dtype=np.int64)
        self.step = 0
        self.m = Metrics(hot_slot_count=slot_count)
        self.log = Log()
        self.sink = sink

    # memstore.py:335-342
    def _check_budget(self):
        if len(self.slot_of) > self.slot_count:
            raise OracleError("budget exceeded")
        self.m.hot_peak = max(self.m.hot_peak, len(self.slot_of))

    # memstore.py:397-411
    def _evict(self, k: int):
        k = min(k, len(self.slot_of))
        if k == 0:
            return
        victims = self.policy.choose_victims(k)
        self.log.victims.append(list(victims))
        for v in victims:
            s = self.slot_of.pop(v)
            if self.state[v] != HOT:
                raise OracleError("evicting a non-hot vertex")
            self.cold[v] = self.slots[s].copy()
            self.state[v] = COLD
            self.free.append(s)
        self.m.evictions += k
        self.m.cold_bytes_written += k * self.agg_dim * 4

    # memstore.py:415-421
    def _make_room(self, n: int):
        if n > self.slot_count:
            raise OracleError(f"batch of {n} cannot fit in "
                              f"{self.slot_count} slots")
        while len(self.free) < n:
            self._evict(max(self.evict_batch, n - len(self.free)))

    # memstore.py:423-445
    def _admit(self, vs, rows):
        n = len(vs)
        self._make_room(n)
        taken = self.free[-n:]
        del self.free[-n:]
        self.slots[taken] = 0.0 if rows is None else rows
        for v, s in zip(vs.tolist(), taken):
            self.state[v] = HOT
            self.slot_of[v] = s
            self.policy.on_admit(v, int(self.pending[v]))
        self._check_budget()

    def _reload(self, vs):
        rows = np.stack([self.cold.pop(v) for v in vs.tolist()])
        self.m.cold_bytes_read += len(vs) * self.agg_dim * 4
        self._admit(vs, rows)
        self.m.reloads += len(vs)
        self.unique_reloaded[vs] = True
        self.log.reloads.append(vs.tolist())

    # memstore.py:447-477
    def ensure_hot(self, vs):
        while True:
            st = self.state[vs]
            if st.max(initial=0) > COLD:
                raise OracleError("completed vertex offered messages")
            need = int(np.count_nonzero(st != HOT))
            if need <= len(self.free):
                break
            self._make_room(need)
        fresh = vs[st == NOT_STARTED]
        cold = vs[st == COLD]
        if fresh.size:
            self._admit(fresh, None)
        if cold.size:
            self._reload(cold)
        return np.array([self.slot_of[v] for v in vs.tolist()],
                        dtype=np.int64)

    # memstore.py:479-494 + orchestrator.py:148-150
    def graduate(self, vs):
        if np.any(self.pending[vs] != 0):
            raise OracleError("release with pending messages")
        idx = [self.slot_of.pop(v) for v in vs.tolist()]
        rows = self.slots[idx].copy()
        for v, s in zip(vs.tolist(), idx):
            self.state[v] = COMPLETED
            self.free.append(s)
            self.policy.on_remove(v)
        self.log.graduated.append(vs.tolist())
        if self.sink is not None:
            self.sink(vs, rows)

    # orchestrator.py:165-213
    def _deliver(self, dests, starts, counts, firsts, lasts, msgs,
                 self_half=False):
        touched = 0
        for lo in range(0, len(dests), self.sub_batch):
            hi = min(lo + self.sub_batch, len(dests))
            vs = dests[lo:hi]
            slot_idx = self.ensure_hot(vs)
            cnt = counts[lo:hi]
            if self_half:
                self.slots[slot_idx, self.embed_dim:] = msgs[starts[lo:hi]]
            else:
                pick = np.concatenate(
                    [np.arange(s, s + c) for s, c in zip(starts[lo:hi], cnt)])
                np.add.at(self.slots[:, :msgs.shape[1]],
                          np.repeat(slot_idx, cnt), msgs[pick])
            pend = self.pending[vs]
            if np.any(pend < cnt):
                raise OracleError("more deliveries than pending")
            self.pending[vs] = pend - cnt.astype(np.uint32)
            newp = self.pending[vs]
            for v, p in zip(vs.tolist(), newp.tolist()):
                self.policy.on_message(v, int(p))
            self.m.messages += int(cnt.sum())
            f = self.first[vs]
            self.first[vs] = np.where(f < 0, firsts[lo:hi], f)
            self.last[vs] = lasts[lo:hi]
            done = vs[newp == 0]
            if done.size:
                self.graduate(done)
            touched += len(vs)
        return touched

    # orchestrator.py:216-299
    def process_chunk(self, start: int, end: int, features, local_offsets,
                      neighbors):
        n = end - start
        reloads0 = self.m.reloads
        touched = 0
        src = np.arange(start, end, dtype=np.int64)
        feats = np.asarray(features, dtype=np.float32)
        mine = (src >= self.lo) & (src < self.hi)
        if self.model == SAGE:
            sv = src[mine]
            steps = self.step + (sv - start)
            self.step += n
            touched += self._deliver(sv, sv - start, np.ones(len(sv), np.int64),
                                     steps, steps, feats, self_half=True)
        elif self.model == GCN:
            zeros = src[mine & (self.state[src] == NOT_STARTED)
                        & (self.pending[src] == 0)]
            for lo in range(0, len(zeros), self.sub_batch):
                vs = zeros[lo:lo + self.sub_batch]
                self.ensure_hot(vs)
                self.graduate(vs)
        fanout = np.diff(local_offsets)
        nbrs = np.asarray(neighbors, dtype=np.int64)
        if self.model == GIN:
            per = fanout + 1
            m = int(per.sum())
            stream_src = np.repeat(np.arange(n), per)
            is_self = np.zeros(m, dtype=bool)
            if n:
                is_self[np.concatenate(([0], np.cumsum(per)[:-1]))] = True
            stream_dst = np.empty(m, dtype=np.int64)
            stream_dst[is_self] = src
            stream_dst[~is_self] = nbrs
        else:
            m = len(nbrs)
            stream_src = np.repeat(np.arange(n), fanout)
            stream_dst = nbrs
            is_self = None
        if m:
            msgs = feats[stream_src]
            if is_self is not None:
                msgs[is_self] *= np.float32(1.0) + np.float32(self.eps)
            if self.model in (GCN, SAGE):
                norm = np.maximum(self.in_degrees[stream_dst], 1)
                msgs /= norm.astype(np.float32)[:, None]
            order = np.argsort(stream_dst, kind="stable")
            sdst = stream_dst[order]
            uniq, seg = np.unique(sdst, return_index=True)
            counts = np.diff(np.append(seg, m))
            pos = order + self.step
            self.step += m
            firsts = pos[seg]
            lasts = pos[seg + counts - 1]
            keep = (uniq >= self.lo) & (uniq < self.hi)
            uniq, seg, counts = uniq[keep], seg[keep], counts[keep]
            firsts, lasts = firsts[keep], lasts[keep]
            app = np.argsort(firsts, kind="stable")
            touched += self._deliver(uniq[app], seg[app], counts[app],
                                     firsts[app], lasts[app], msgs[order])
        pct = 100.0 * (self.m.reloads - reloads0) / max(1, touched)
        self.log.chunk_reload_pcts.append(pct)

    # orchestrator.py:302-323
    def finalize(self) -> Metrics:
        missing = np.flatnonzero(self.state[self.lo:self.hi] != COMPLETED)
        if missing.size:
            raise OracleError(f"{missing.size} vertices never completed")
        got = self.first >= 0
        if got.any():
            spans = (self.last[got] - self.first[got]).astype(np.float64)
            self.m.mean_span = float(spans.mean())
            self.m.p99_span = float(np.percentile(spans, 99))
        if self.log.chunk_reload_pcts:
            self.m.mean_reload_pct = float(np.mean(self.log.chunk_reload_pcts))
        self.m.unique_reloads = int(self.unique_reloaded.sum())
        return self.m


def plan_chunks(num_vertices: int, dim: int, dtype: str, budget: int):
    """oocgnn/chunks.py:36-48."""
    rows = max(1, budget // max(1, dim * (2 if dtype == "f16" else 4)))
    return [(s, min(s + rows, num_vertices))
            for s in range(0, num_vertices, rows)]


def stable_transform(batch, weight, bias, relu: bool):
    """MatmulBackend.apply + ReLU (oocgnn/compute.py:39-47, :94-96):
    out = bias; out += batch[:, k] * W[:, k] for k in order, all f32."""
    batch = np.asarray(batch, dtype=np.float32)
    out = np.empty((len(batch), weight.shape[0]), dtype=np.float32)
    out[:] = bias
    tmp = np.empty_like(out)
    for k in range(weight.shape[1]):
        np.multiply(batch[:, k, None], weight[None, :, k], out=tmp)
        out += tmp
    if relu:
        np.maximum(out, 0.0, out=out)
    return out


def run_layer(offsets, neighbors, in_degrees, features, model: int,
              weight, bias, relu: bool, *, embed_dim, agg_dim, chunk_rows,
              slot_count, gin_epsilon=0.0, eviction="minpend", seed=0,
              evict_batch=None, chunk_limit=None, dst_range=None):
    """One whole layer through the engine; returns (out, metrics, log).

    ``chunk_limit`` stops after that many chunks (bounded CPU-baseline
    samples); the returned output is then None. With ``dst_range`` the
    output holds the rows of [lo, hi) only (one GPU rank)."""
    v = len(in_degrees)
    agg = np.zeros((v, agg_dim), dtype=np.float32)

    def sink(vs, rows):
        agg[vs] = rows

    layer = Layer(in_degrees, model, embed_dim, agg_dim, slot_count,
                  gin_epsilon=gin_epsilon, eviction=eviction, seed=seed,
                  evict_batch=evict_batch, sink=sink, dst_range=dst_range)
    agg_rows = slice(layer.lo, layer.hi)
    feats = np.asarray(features)
    done = 0
    for start in range(0, v, chunk_rows):
        if chunk_limit is not None and done >= chunk_limit:
            return None, layer.m, layer.log
        end = min(start + chunk_rows, v)
        lo, hi = int(offsets[start]), int(offsets[end])
        layer.process_chunk(start, end, feats[start:end].astype(np.float32),
                            offsets[start:end + 1] - lo, neighbors[lo:hi])
        done += 1
    metrics = layer.finalize()
    return (stable_transform(agg[agg_rows], weight, bias, relu), metrics,
            layer.log)
