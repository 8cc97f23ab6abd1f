"""Destination-range exchange between GPU ranks.

Rank g owns destinations ``partition_ranges(V, G)[g]`` (oocgnn/storage.py
:372-388) and produces the next layer's input rows for exactly that range.
Every rank needs every row of the next layer's input, so each layer ends
with an exchange. It is done in place:

* the next layer's full input is ONE buffer (V, width) per layer; the
  producing kernel (transform epilogue or tcgen05 GEMM) writes the rank's
  own rows straight into its slice ``[lo, hi)``;
* the buffer is then filled by broadcasts from the rows' owners, in
  ascending source order, each owner range cut into a few pieces
  (``ncclBroadcast`` over NVLink on GPUs, gloo on CPU): no padding, no
  concatenation, no second copy of the input;
* every piece gets a CUDA event on a side stream, so the next layer's
  aggregation folds piece t in as soon as it lands
  (``atlas_layer_run_pieces``) -- the exchange overlaps the aggregation
  instead of preceding it. Pieces arrive in ascending source order, which is
  what keeps each destination's fold in the reference's source order.

Each row crosses NVLink once per receiving rank, as with the per-chunk
broadcast SURVEY.md §8e describes; the pieces only set the overlap grain.
"""

from __future__ import annotations

import numpy as np


class RangeExchange:
    """In-place all-gather of destination-range rows by owner broadcasts."""

    def __init__(self, num_vertices: int, ranges, rank: int, group=None,
                 pieces_per_rank: int = 4, min_piece_bytes: int = 4 << 20):
        self.num_vertices = num_vertices
        self.ranges = [tuple(map(int, r)) for r in ranges]
        self.rank = rank
        self.group = group
        self.lo, self.hi = self.ranges[rank]
        self.pieces_per_rank = max(1, int(pieces_per_rank))
        self.min_piece_bytes = max(1, int(min_piece_bytes))
        self._buffers = {}
        self._comm_stream = None
        self.bytes_received = 0  # rows other ranks sent here, since reset

    # -- buffers -----------------------------------------------------------
    def buffer(self, key, width: int, dtype, device):
        """The cached (V, width) input buffer named ``key`` (one per layer
        and tensor kind, reused across steps: stream order makes a reuse
        safe because every writer and reader is queued on one stream)."""
        import torch

        buf = self._buffers.get(key)
        if buf is None or buf.shape[1] != width or buf.dtype != dtype \
                or buf.device != torch.device(device):
            buf = torch.empty((self.num_vertices, width), dtype=dtype,
                              device=device)
            self._buffers[key] = buf
        return buf

    def own(self, full):
        """The rank's slice of a full buffer (a view: write it in place)."""
        return full[self.lo:self.hi]

    # -- schedule ----------------------------------------------------------
    def schedule(self, row_bytes: int):
        """[(owner, r0, r1)] in ascending row order: each owner range cut
        into up to ``pieces_per_rank`` pieces of at least min_piece_bytes."""
        out = []
        for owner, (lo, hi) in enumerate(self.ranges):
            n = hi - lo
            if n <= 0:
                continue
            cap = max(1, (n * row_bytes) // self.min_piece_bytes)
            k = int(min(self.pieces_per_rank, cap, n))
            edges = [lo + (n * i) // k for i in range(k + 1)]
            out.extend((owner, a, b) for a, b in zip(edges, edges[1:]))
        return out

    def _src(self, owner: int) -> int:
        import torch.distributed as dist

        if self.group is None:
            return owner
        return dist.get_global_rank(self.group, owner)

    # -- exchange ----------------------------------------------------------
    def start(self, full):
        """Broadcast every piece of ``full`` from its owner; returns
        (bounds int64[P+1], events[P]) -- events are CUDA events recorded
        when each piece has landed (None on CPU, where the broadcasts
        complete before this returns). Own pieces get no event: they are
        ordered before everything queued after their producer."""
        import torch
        import torch.distributed as dist

        if full.shape[0] != self.num_vertices or not full.is_contiguous():
            raise ValueError("exchange buffers are contiguous (V, width)")
        row_bytes = full.stride(0) * full.element_size()
        sched = self.schedule(row_bytes)
        cuda = full.is_cuda
        if cuda and self._comm_stream is None:
            self._comm_stream = torch.cuda.Stream()
        bounds, events = [0], []
        for owner, r0, r1 in sched:
            work = dist.broadcast(full[r0:r1], src=self._src(owner),
                                  group=self.group, async_op=True)
            ev = None
            if cuda:
                # make the side stream wait for the broadcast, then mark it
                with torch.cuda.stream(self._comm_stream):
                    work.wait()
                    if owner != self.rank:
                        ev = torch.cuda.Event()
                        ev.record(self._comm_stream)
            else:
                work.wait()
            if owner != self.rank:
                self.bytes_received += (r1 - r0) * row_bytes
            bounds.append(r1)
            events.append(ev)
        if bounds[-1] != self.num_vertices:  # trailing empty ranges
            bounds.append(self.num_vertices)
            events.append(None)
        return np.asarray(bounds, dtype=np.int64), events

    @staticmethod
    def finish(events):
        """Make the current stream wait for every piece."""
        import torch

        cur = None
        for ev in events:
            if ev is None:
                continue
            cur = cur or torch.cuda.current_stream()
            cur.wait_event(ev)

    def gather(self, y_local, key="gather"):
        """Full (V, width) tensor from every rank's ``y_local`` rows; when
        y_local already is this rank's slice of the buffer, nothing is
        copied locally."""
        full = self.buffer(key, y_local.shape[1], y_local.dtype,
                           y_local.device)
        own = self.own(full)
        if own.data_ptr() != y_local.data_ptr() or \
                own.stride() != y_local.stride():
            own.copy_(y_local)
        _, events = self.start(full)
        self.finish(events)
        return full


def gather_ranges(y_local, ranges, group=None):
    """Reassemble a full (V, width) tensor from every rank's destination
    range (partition_ranges order) by owner broadcasts into one buffer."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    v = int(ranges[-1][1])
    ex = RangeExchange(v, ranges, rank, group)
    return ex.gather(y_local.contiguous(), key="once")
