// Sweep replay: the exact control machine of a whole layer (MINPEND and
// LRU, no event logs) as ONE sequential sweep over sub-batches whose only
// dynamic input is the eviction history.
//
// The reference machine (oocgnn/orchestrator.py:165-299 driving
// oocgnn/memstore.py:305-497) has much more structure than its per-vertex
// state suggests:
//   * the delivery stream is fixed by the chunk plan: chunk c runs the GCN
//     zero pre-pass, the SAGE self pass and the edge pass (runs in
//     first-appearance order), each cut into sub-batches of sub_batch
//     elements; a vertex appears at most once per sub-batch;
//   * pending counts only change through deliveries, so the pending value a
//     vertex holds after each of its deliveries (its heap key,
//     memstore.py:182-194) is static; so is its first delivery (a fresh
//     admission) and its last (graduation, pending 0);
//   * the PendingBucketHeap is one FIFO list per key, appended in delivery
//     order (memstore.py:128-194): bucket b's list is the static list of
//     deliveries that left pending == b, in stream order. An entry is in
//     the heap at sub-batch s iff it was delivered before s, its vertex's
//     next delivery is at or after s (not superseded), and no earlier
//     eviction popped it. pop_min (memstore.py:196-211) walks the lowest
//     bucket's list from a head pointer that only moves forward, skipping
//     superseded entries for good. LRU (memstore.py:214-235) is the same
//     walk over the whole delivery stream.
//   * ensure_hot_many's need (memstore.py:447-470) is the sub-batch's
//     fresh count (static) plus its cold count: the vertices an earlier
//     eviction popped whose next delivery lies in this sub-batch. Each
//     popped entry knows that sub-batch (its successor's), so an eviction
//     adds to the cold count of exactly one future sub-batch.
// So the machine is a scalar loop over sub-batches (hot population, peak,
// reloads) that stops only where need exceeds the free slots; there the
// CTA pops victims from the static bucket lists and scatters their reload
// sub-batches. Every integer the reference reports is reproduced:
// evictions, reloads (per chunk), unique reloads, admissions, graduations,
// hot peak. The per-delivery victim/reload/graduation logs and the RND
// policy stay on the per-element machine (engine.cu).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "internal.cuh"

namespace atlas {
namespace {

constexpr int kSwThreads = 1024;
constexpr int kSwBlock = 2048;   // sub-batches staged in shared memory
constexpr uint32_t kNone = 0xFFFFFFFFu;

unsigned grid_of(int64_t n, int block = 256) {
  int64_t g = ceil_div(n, block);
  if (g > num_sms() * 16) g = num_sms() * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

// ---- static stream --------------------------------------------------------

__global__ void zero_flags(const uint32_t* __restrict__ indeg, int64_t n,
                           uint32_t* __restrict__ f) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    f[v] = indeg[v] == 0 ? 1u : 0u;
}

struct ChunkMap {
  int64_t R, lo, hi, sb;
  const int64_t* eoff;  // [3C]: first element of (pre, self, edge) of chunk c
  const int64_t* soff;  // [3C]: first sub-batch of (pre, self, edge)
  __device__ __forceinline__ int64_t local_start(int64_t c) const {
    return max(c * R, lo) - lo;
  }
};

// edge pass elements: run r of chunk c (binary search over run_off)
__global__ void fill_edge(const uint64_t* __restrict__ runs,
                          const int64_t* __restrict__ run_off, int64_t nchunks,
                          int64_t nruns, ChunkMap M, uint32_t* __restrict__ el_v,
                          uint32_t* __restrict__ el_cnt,
                          uint32_t* __restrict__ el_sub) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nruns;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = 0, b = nchunks;  // last c with run_off[c] <= r
    while (b - a > 1) {
      const int64_t m = (a + b) >> 1;
      if (run_off[m] <= r) a = m;
      else b = m;
    }
    const int64_t k = r - run_off[a];
    const int64_t i = M.eoff[3 * a + 2] + k;
    const uint64_t x = runs[r];
    el_v[i] = (uint32_t)x;
    el_cnt[i] = (uint32_t)(x >> 32);
    el_sub[i] = (uint32_t)(M.soff[3 * a + 2] + k / M.sb);
  }
}

// SAGE self pass: every local vertex, in its own chunk
__global__ void fill_self(int64_t nloc, ChunkMap M, uint32_t* __restrict__ el_v,
                          uint32_t* __restrict__ el_cnt,
                          uint32_t* __restrict__ el_sub) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nloc;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = (v + M.lo) / M.R;
    const int64_t k = v - M.local_start(c);
    const int64_t i = M.eoff[3 * c + 1] + k;
    el_v[i] = (uint32_t)v;
    el_cnt[i] = 1u;
    el_sub[i] = (uint32_t)(M.soff[3 * c + 1] + k / M.sb);
  }
}

// GCN pre-pass: zero in-degree vertices of the chunk, ascending
__global__ void fill_pre(int64_t nloc, const uint32_t* __restrict__ zr,
                         ChunkMap M, uint32_t* __restrict__ el_v,
                         uint32_t* __restrict__ el_cnt,
                         uint32_t* __restrict__ el_sub) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nloc;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (zr[v + 1] == zr[v]) continue;  // in-degree > 0
    const int64_t c = (v + M.lo) / M.R;
    const int64_t k = (int64_t)zr[v] - zr[M.local_start(c)];
    const int64_t i = M.eoff[3 * c + 0] + k;
    el_v[i] = (uint32_t)v;
    el_cnt[i] = 0u;
    el_sub[i] = (uint32_t)(M.soff[3 * c + 0] + k / M.sb);
  }
}

// per-chunk zero counts from the exclusive scan zr (nloc + 1 entries)
__global__ void chunk_zero_counts(const uint32_t* __restrict__ zr,
                                  int64_t nchunks, ChunkMap M, int64_t nloc,
                                  int64_t* __restrict__ out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       c < nchunks; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = min(M.local_start(c), nloc);
    const int64_t b = min(max((c + 1) * M.R, M.lo) - M.lo, nloc);
    out[c] = b > a ? (int64_t)zr[b] - zr[a] : 0;
  }
}



// per vertex: the prefix at its last element (elements grouped by vertex)
__global__ void vertex_last(const uint32_t* __restrict__ sv,
                            const unsigned long long* __restrict__ P,
                            int64_t n, unsigned long long* __restrict__ lastP) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    if (j == n - 1 || sv[j + 1] != sv[j]) lastP[sv[j]] = P[j];
}





// values of the vertex sort: element index (high word) | count (low)
__global__ void pack_idx_cnt(const uint32_t* __restrict__ el_cnt, int64_t n,
                             unsigned long long* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ((unsigned long long)i << 32) | el_cnt[i];
}

__global__ void low_words(const unsigned long long* __restrict__ in, int64_t n,
                          unsigned long long* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = in[j] & 0xFFFFFFFFull;
}

// In vertex order (each vertex's deliveries in stream order): pending after
// each delivery, its successor's sub-batch, fresh / graduating counts per
// sub-batch, and the heap entry of the delivery keyed (pending << 32 |
// element) -- MINPEND's bucket FIFOs once sorted -- or (element) for LRU,
// with value (sub << 32 | successor's sub; 0 when it graduates: never in
// the heap). Only two random reads per delivery (its and its successor's
// sub-batch); everything else streams.
__global__ void chain_entries(const uint32_t* __restrict__ sv,
                              const unsigned long long* __restrict__ sval,
                              const unsigned long long* __restrict__ P,
                              const unsigned long long* __restrict__ lastP,
                              const uint32_t* __restrict__ el_sub,
                              const uint32_t* __restrict__ indeg,
                              int self_term, int lru, int64_t n,
                              unsigned long long* __restrict__ key_out,
                              unsigned long long* __restrict__ val_out,
                              uint32_t* __restrict__ fresh,
                              uint32_t* __restrict__ grad,
                              int* __restrict__ mismatch,
                              unsigned* __restrict__ maxp) {
  unsigned my_max = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = sv[j];
    const unsigned long long x = sval[j];
    const uint32_t i = (uint32_t)(x >> 32), cnt = (uint32_t)x;
    const bool first = j == 0 || sv[j - 1] != v;
    const bool last = j == n - 1 || sv[j + 1] != v;
    const unsigned long long left = lastP[v] - P[j];
    if (first) {
      const unsigned long long p0 = (unsigned long long)indeg[v] + self_term;
      if (left + cnt != p0) atomicExch(mismatch, 1);
    }
    const uint32_t np = left > 0xFFFFFFF0ull ? 0xFFFFFFF0u : (uint32_t)left;
    const uint32_t sub = el_sub[i];
    const uint32_t nsub =
        (last || np == 0) ? 0u : el_sub[(uint32_t)(sval[j + 1] >> 32)];
    if (first) atomicAdd(fresh + sub, 1u);
    if (np == 0) atomicAdd(grad + sub, 1u);
    key_out[j] = lru ? (unsigned long long)i
                     : (((unsigned long long)np << 32) | i);
    val_out[j] = ((unsigned long long)sub << 32) | nsub;
    my_max = max(my_max, np);
  }
  for (int o = 16; o > 0; o >>= 1)
    my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
  if ((threadIdx.x & 31) == 0 && my_max) atomicMax(maxp, my_max);
}

__global__ void entries_from_sorted(const unsigned long long* __restrict__ skey,
                                    const unsigned long long* __restrict__ sval,
                                    int64_t n, uint32_t* __restrict__ ent_sub,
                                    uint32_t* __restrict__ ent_next,
                                    uint32_t* __restrict__ ent_el) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = sval[k];
    ent_sub[k] = (uint32_t)(v >> 32);
    ent_next[k] = (uint32_t)v;
    ent_el[k] = (uint32_t)skey[k];
  }
}

// boff[b] = first entry with key >= b (key = high word), b in [0, nb]
__global__ void bucket_bounds64(const unsigned long long* __restrict__ skey,
                                int64_t n, int64_t nb,
                                uint32_t* __restrict__ boff) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t prev = k == 0 ? -1 : (int64_t)(skey[k - 1] >> 32);
    const int64_t cur = k == n ? nb : min((int64_t)(skey[k] >> 32), nb);
    for (int64_t b = prev + 1; b <= cur; b++) boff[b] = (uint32_t)k;
  }
}

__global__ void mark_unique(const uint32_t* __restrict__ victims, int64_t nv,
                            const uint32_t* __restrict__ ent_el,
                            const uint32_t* __restrict__ el_v,
                            uint8_t* __restrict__ flag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nv;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t e = victims[k];
    flag[el_v[ent_el ? ent_el[e] : e]] = 1;
  }
}

// unique reloads from the single-CTA sweep's pop marks: every popped entry
// has a successor delivery, where its vertex reloads
__global__ void mark_unique_popped(const uint8_t* __restrict__ popped,
                                   int64_t n, const uint32_t* __restrict__ ent_el,
                                   const uint32_t* __restrict__ el_v,
                                   uint8_t* __restrict__ flag) {
  const int64_t n4 = n >> 2;
  const uint32_t* p4 = reinterpret_cast<const uint32_t*>(popped);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n4 + 1;
       q += (int64_t)gridDim.x * blockDim.x) {
    uint32_t m;
    if (q < n4) {
      m = p4[q];
    } else {  // tail
      m = 0;
      for (int64_t e = q * 4; e < n; e++)
        m |= (uint32_t)popped[e] << (8 * (e - q * 4));
    }
    while (m) {
      const int b = __ffs(m) - 1;
      const int64_t e = q * 4 + (b >> 3);
      flag[el_v[ent_el ? ent_el[e] : e]] = 1;
      m &= ~(0xFFu << (b & ~7));
    }
  }
}

__global__ void count_flags(const uint8_t* __restrict__ f, int64_t n,
                            unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += f[i] != 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// ---- the sweep (one CTA) ------------------------------------------------

struct SweepArgs {
  int64_t S;                 // sub-batches
  const uint32_t* fresh;     // [S]
  const uint32_t* grad;      // [S]
  uint32_t* cold;            // [S] reloads scattered by evictions
  uint32_t* cold_out;        // [S] final reload count per sub-batch
  int64_t slots, evict_batch;
  int32_t b0, nb;            // buckets [b0, nb)
  const uint32_t* boff;      // [nb + 1]
  uint32_t* head;            // [nb]
  const uint32_t* ent_sub;   // [n + 4]
  const uint32_t* ent_next;  // [n + 4]
  uint32_t* victims;         // popped entries, in pop order (coop kernel)
  uint8_t* popped;           // [n] 1 = entry popped (single-CTA kernel)
  int64_t* out;              // evictions, reloads, hot_peak, nvict, err, info
  int32_t diag_no_far;       // diagnostics only: skip far reload atomics
};

// The walk reads each bucket list through register windows of kSwWin
// entries (8 per thread, four 16-B loads in flight per thread); victims go
// to the log in coalesced rounds (lane-consecutive slots). Measured and
// dropped (profiles/r2_sweep_variants.txt): 512 threads x 16 entries with
// the next window prefetched in registers (1.5x slower), an L2 bulk
// prefetch of the next windows and shared-memory window buffers filled by
// bulk copies (no gain / slower), warp match-aggregated reload atomics
// (1.7x slower). Per-bucket
// state lives in shared memory for the first kSwCache buckets: the head,
// the list end and the sub-batch of the entry at the head when known
// (head_sub). A list whose head entry is not delivered yet (head_sub >= s)
// has nothing in the heap at s, so it is skipped without touching memory;
// most of an event's lists are in that state (their live entries were
// popped or superseded), and reading their head windows anyway was what
// the walk spent its time on.
constexpr int kSwPerT = 8;
constexpr int kSwWin = kSwThreads * kSwPerT;
constexpr int kSwCache = 4096;
constexpr uint32_t kUnknown = 0;  // head_sub not known: read the list

struct SweepSm {
  uint32_t fresh[kSwBlock], grad[kSwBlock], cold[kSwBlock];
  uint32_t head[kSwCache], end[kSwCache], head_sub[kSwCache];
  int64_t hot, peak, evictions, reloads, need_old, k, nv;
  int32_t i, mode, err;
  int64_t err_info;
  uint32_t last_taken, hs_new;
  uint32_t first_na[2];
  int32_t wtotal[2], wlog[2];
  unsigned long long windows, visits, skipped;
};

__global__ void __launch_bounds__(kSwThreads, 1) sweep_kernel(SweepArgs A) {
  extern __shared__ __align__(16) unsigned char sw_raw[];
  SweepSm& sm = *reinterpret_cast<SweepSm*>(sw_raw);
  using Scan = cub::BlockScan<int, kSwThreads>;
  __shared__ typename Scan::TempStorage scan;
  const int tid = threadIdx.x;
  const int ncache = A.nb < kSwCache ? A.nb : kSwCache;
  for (int b = tid; b < ncache; b += kSwThreads) {
    sm.head[b] = A.boff[b];
    sm.end[b] = A.boff[b + 1];
    sm.head_sub[b] = sm.head[b] >= sm.end[b] ? kNone : kUnknown;
  }
  if (tid == 0) {
    sm.hot = sm.peak = sm.evictions = sm.reloads = sm.nv = 0;
    sm.err = 0;
    sm.err_info = 0;
    sm.windows = sm.visits = sm.skipped = 0;
  }
  __syncthreads();
  for (int64_t base = 0; base < A.S; base += kSwBlock) {
    const int cnt = (int)(A.S - base < kSwBlock ? A.S - base : kSwBlock);
    for (int t = tid; t < cnt; t += kSwThreads) {
      sm.fresh[t] = A.fresh[base + t];
      sm.grad[t] = A.grad[base + t];
      sm.cold[t] = __ldcg(A.cold + base + t);
    }
    if (tid == 0) {
      sm.i = 0;
      sm.mode = 0;
    }
    __syncthreads();
    while (true) {
      // ---- thread 0: the scalar machine until it needs victims --------
      if (tid == 0) {
        sm.k = 0;
        int i = sm.i;
        int64_t hot = sm.hot;
        while (i < cnt) {
          if (sm.mode == 0) {  // classify (memstore.py:456-466)
            const int64_t need = (int64_t)sm.fresh[i] + sm.cold[i];
            if (need <= A.slots - hot) {
              hot += need;  // admit fresh, then reload cold
              if (hot > sm.peak) sm.peak = hot;
              sm.reloads += sm.cold[i];
              hot -= sm.grad[i];  // release_batch of the finished ones
              i++;
              continue;
            }
            if (need > A.slots) {  // _make_room (memstore.py:413-418)
              sm.err = ATLAS_ECONFIG;
              sm.err_info = need;
              break;
            }
            sm.need_old = need;
            sm.mode = 1;
          }
          const int64_t free = A.slots - hot;
          if (free < sm.need_old) {  // evict(max(batch, n - free))
            int64_t k = sm.need_old - free;
            if (k < A.evict_batch) k = A.evict_batch;
            if (k > hot) k = hot;
            if (k <= 0) {
              sm.err = ATLAS_EINVARIANT;
              sm.err_info = -1;
              break;
            }
            sm.k = k;
            break;
          }
          sm.mode = 0;  // re-classify: victims may sit in this batch
        }
        sm.i = i;
        sm.hot = hot;
        sm.first_na[0] = sm.first_na[1] = kNone;
        sm.wtotal[0] = sm.wtotal[1] = 0;
        sm.wlog[0] = sm.wlog[1] = 0;
      }
      __syncthreads();
      const int64_t k = sm.k;
      if (k == 0 || sm.err) break;
      // ---- all threads: pop k entries (PendingBucketHeap.pop_min) ------
      const uint32_t s = (uint32_t)(base + sm.i);
      const int64_t win_hi = base + cnt;  // sub-batches staged in smem
      int64_t rem = k;
      int64_t nv = sm.nv;
      int b = A.b0;
      int w = 0;
      bool bad = false;
      while (rem > 0) {
        if (b >= A.nb) {
          bad = true;
          break;
        }
        const bool cached = b < kSwCache;
        uint32_t h, e_end;
        if (cached) {
          if (sm.head_sub[b] >= s && sm.head_sub[b] != kUnknown) {
            if (tid == 0) sm.skipped++;
            b++;  // nothing of this list is in the heap yet (or it is done)
            continue;
          }
          h = sm.head[b];
          e_end = sm.end[b];
        } else {
          h = __ldcg(A.head + b);
          e_end = A.boff[b + 1];
        }
        if (h >= e_end) {
          b++;
          continue;
        }
        const uint32_t w0 = h & ~3u;
        const uint32_t j0 = w0 + (uint32_t)tid * kSwPerT;
        uint32_t subs[kSwPerT], nxts[kSwPerT];
#pragma unroll
        for (int q = 0; q < kSwPerT; q += 4) {
          uint4 a4 = make_uint4(kNone, kNone, kNone, kNone);
          uint4 n4 = make_uint4(0, 0, 0, 0);
          if (j0 + q < e_end) {
            a4 = __ldcg(reinterpret_cast<const uint4*>(A.ent_sub + j0 + q));
            n4 = __ldcg(reinterpret_cast<const uint4*>(A.ent_next + j0 + q));
          }
          subs[q] = a4.x; subs[q + 1] = a4.y; subs[q + 2] = a4.z; subs[q + 3] = a4.w;
          nxts[q] = n4.x; nxts[q + 1] = n4.y; nxts[q + 2] = n4.z; nxts[q + 3] = n4.w;
        }
        int valid = 0, nvalid = 0;
        uint32_t first_na = kNone;
#pragma unroll
        for (int e = 0; e < kSwPerT; e++) {
          const uint32_t j = j0 + e;
          if (j < h || j >= e_end) continue;
          if (subs[e] < s) {
            if (nxts[e] >= s) {
              valid |= 1 << e;
              nvalid++;
            }
          } else if (first_na == kNone) {
            first_na = j;
          }
        }
        // window totals: valid entries and the first undelivered entry
        {
          const int wv = __reduce_add_sync(0xffffffffu, nvalid);
          const uint32_t wf = __reduce_min_sync(0xffffffffu, first_na);
          if ((tid & 31) == 0) {
            if (wv) atomicAdd(&sm.wtotal[w & 1], wv);
            if (wf != kNone) atomicMin(&sm.first_na[w & 1], wf);
          }
          // the other slot was last read before the previous window's end
          if (tid == 0) {
            sm.first_na[(w + 1) & 1] = kNone;
            sm.wtotal[(w + 1) & 1] = 0;
            sm.wlog[(w + 1) & 1] = 0;
          }
        }
        __syncthreads();
        const int64_t total = sm.wtotal[w & 1];
        const uint32_t fna = sm.first_na[w & 1];
        uint32_t run_nx = kNone, run_c = 0;
        auto cold_add = [&](uint32_t nx) {  // consecutive equal keys: one atomic
          if (nx == run_nx) {
            run_c++;
            return;
          }
          if (run_c) {
            if ((int64_t)run_nx < win_hi) {
              if (A.diag_no_far < 2) atomicAdd(&sm.cold[run_nx - base], run_c);
            } else if (!A.diag_no_far) {
              atomicAdd(A.cold + run_nx, run_c);
            }
          }
          run_nx = nx;
          run_c = 1;
        };

        if (total <= rem) {
          // the whole window's valid entries are victims: order within the
          // event is irrelevant here (no logs), so log slots come from one
          // atomic per warp
          // pop marks: one byte per entry, stored by the thread owning
          // it (no log offsets to agree on); entries before the head are
          // never rewritten, so earlier marks in the window survive
#pragma unroll
          for (int e = 0; e < kSwPerT; e++) {
            if (valid >> e & 1) {
              A.popped[j0 + e] = 1;
              cold_add(nxts[e]);
            }
          }
          if (fna != kNone && fna >= j0 && fna < j0 + kSwPerT)
            sm.hs_new = subs[fna - j0];
        } else {
          // the event ends inside this window: exact ranks
          int off, t2;
          Scan(scan).ExclusiveSum(nvalid, off, t2);
#pragma unroll
          for (int e = 0; e < kSwPerT; e++) {
            if (!(valid >> e & 1)) continue;
            const int64_t r = off++;
            if (r >= rem) break;
            const uint32_t j = j0 + e;
            A.popped[j] = 1;
            cold_add(nxts[e]);
            if (r == rem - 1) {
              sm.last_taken = j;
              // the new head's sub-batch, when it is in this thread's slice
              sm.hs_new = e + 1 < kSwPerT && j + 1 < e_end ? subs[e + 1]
                                                          : kUnknown;
            }
          }
        }
        cold_add(kNone);  // flush the last run (a kNone run is never added)
        __syncthreads();
        uint32_t h_new, hs;
        const int bcur = b;
        const uint32_t wend = min(e_end, w0 + (uint32_t)kSwWin);
        if (total > rem) {
          h_new = sm.last_taken + 1;
          nv += rem;
          rem = 0;
          hs = 1;
        } else {
          nv += total;
          rem -= total;
          if (fna != kNone) {
            h_new = fna;  // the rest of the list is not delivered yet
            hs = 2;
            b++;
          } else {
            h_new = wend;
            hs = wend >= e_end ? 3 : 0;
            if (wend >= e_end) b++;
          }
        }
        if (tid == 0) {
          uint32_t v = kUnknown;
          if (hs == 1 || hs == 2) v = sm.hs_new;
          if (hs == 3) v = kNone;
          if (h_new >= e_end) v = kNone;
          if (cached) {
            sm.head[bcur] = h_new;
            sm.head_sub[bcur] = v;
          } else {
            A.head[bcur] = h_new;
          }
          sm.windows++;
          sm.visits += 1;
        }
        w++;
        __syncthreads();
      }
      if (tid == 0) {
        if (bad) {
          sm.err = ATLAS_EINVARIANT;
          sm.err_info = rem;
        }
        sm.hot -= k - rem;
        sm.evictions += k - rem;
        sm.nv = nv;
      }
      __syncthreads();
      if (sm.err) break;
    }
    __syncthreads();
    for (int t = tid; t < cnt; t += kSwThreads) A.cold_out[base + t] = sm.cold[t];
    __syncthreads();
    if (sm.err) break;
  }
  if (tid == 0) {
    A.out[0] = sm.evictions;
    A.out[1] = sm.reloads;
    A.out[2] = sm.peak;
    A.out[3] = sm.nv;
    A.out[4] = sm.err;
    A.out[5] = sm.err_info;
    A.out[6] = (int64_t)sm.windows;
    A.out[7] = (int64_t)sm.skipped;
  }
}

// ---- the sweep on a cooperative grid (sweep_coop_kernel) ----------------
// Same machine; an event's walk over a list is split into rounds of up to
// G consecutive 8192-entry windows, one per CTA. Round = two grid jobs that
// CTA 0 posts through CoopSync: SCAN (every CTA counts the valid entries of
// its window and finds its first undelivered one) and, after CTA 0 turned
// the counts into the cut, COMMIT (windows before the cut take all their
// valid entries, the cut window takes the first rem_cut in list order;
// victims go to the log at their window's prefix offset, reload counts to
// the global counters). The window contents stay in registers between the
// two jobs. CTA 0 refreshes its staged reload counts after each event.
constexpr int kCoopMax = 64;

struct CoopSync {
  unsigned job, done;
  int32_t type;  // 1 scan, 2 commit, 3 exit
  uint32_t h, end, s, w0;
  int32_t nwin, cut;
  int64_t rem_cut, nv;
  uint32_t cnt[kCoopMax];
  uint32_t fna[kCoopMax];
  uint32_t fna_sub[kCoopMax];
  int64_t off[kCoopMax];
  uint32_t last_taken, hs_new;
};

__device__ __forceinline__ unsigned vld(const unsigned* p) {
  return *reinterpret_cast<const volatile unsigned*>(p);
}

// one CTA's part of a round: window i of the posted range. The window's
// entries, valid mask and first undelivered entry persist in the caller's
// registers (`subs`, `nxts`, `valid`) from SCAN to COMMIT.
struct CoopWin {
  uint32_t subs[kSwPerT], nxts[kSwPerT];
  int valid, nvalid;
  uint32_t j0;
};

__device__ void coop_scan(const SweepArgs& A, CoopSync* C, int i, CoopWin& W,
                          uint32_t* red) {
  const int tid = threadIdx.x;
  const uint32_t h = vld(&C->h), end = vld(&C->end), s = vld(&C->s);
  const uint32_t w0 = vld(&C->w0);
  W.j0 = w0 + (uint32_t)i * kSwWin + (uint32_t)tid * kSwPerT;
#pragma unroll
  for (int q = 0; q < kSwPerT; q += 4) {
    uint4 a4 = make_uint4(kNone, kNone, kNone, kNone);
    uint4 n4 = make_uint4(0, 0, 0, 0);
    if (W.j0 + q < end) {
      a4 = __ldcg(reinterpret_cast<const uint4*>(A.ent_sub + W.j0 + q));
      n4 = __ldcg(reinterpret_cast<const uint4*>(A.ent_next + W.j0 + q));
    }
    W.subs[q] = a4.x; W.subs[q + 1] = a4.y; W.subs[q + 2] = a4.z; W.subs[q + 3] = a4.w;
    W.nxts[q] = n4.x; W.nxts[q + 1] = n4.y; W.nxts[q + 2] = n4.z; W.nxts[q + 3] = n4.w;
  }
  W.valid = 0;
  W.nvalid = 0;
  uint32_t first_na = kNone, fsub = kNone;
#pragma unroll
  for (int e = 0; e < kSwPerT; e++) {
    const uint32_t j = W.j0 + e;
    if (j < h || j >= end) continue;
    if (W.subs[e] < s) {
      if (W.nxts[e] >= s) {
        W.valid |= 1 << e;
        W.nvalid++;
      }
    } else if (first_na == kNone) {
      first_na = j;
      fsub = W.subs[e];
    }
  }
  if (tid == 0) {
    red[0] = 0;
    red[1] = kNone;
  }
  __syncthreads();
  const unsigned wv = __reduce_add_sync(0xffffffffu, (unsigned)W.nvalid);
  const uint32_t wf = __reduce_min_sync(0xffffffffu, first_na);
  if ((tid & 31) == 0) {
    if (wv) atomicAdd(&red[0], wv);
    if (wf != kNone) atomicMin(&red[1], wf);
  }
  __syncthreads();
  // the first undelivered entry's sub-batch (its holder writes it)
  if (first_na != kNone && first_na == red[1]) C->fna_sub[i] = fsub;
  if (tid == 0) {
    C->cnt[i] = red[0];
    C->fna[i] = red[1];
  }
}

__device__ void coop_commit(const SweepArgs& A, CoopSync* C, int i,
                            CoopWin& W, uint32_t* red, void* scan_storage) {
  using Scan = cub::BlockScan<int, kSwThreads>;
  auto& scan = *reinterpret_cast<typename Scan::TempStorage*>(scan_storage);
  const int tid = threadIdx.x;
  const int cut = (int)vld(reinterpret_cast<const unsigned*>(&C->cut));
  if (i > cut) return;
  const int64_t nv = *reinterpret_cast<const volatile int64_t*>(&C->nv);
  const int64_t base_off = nv + *reinterpret_cast<const volatile int64_t*>(&C->off[i]);
  if (i < cut) {
    // every valid entry of the window: warp rounds, one slot counter per CTA
    if (tid == 0) red[2] = 0;
    __syncthreads();
    int incl = W.nvalid;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if ((tid & 31) >= o) incl += t;
    }
    int wbase = 0;
    if ((tid & 31) == 31 && incl) wbase = (int)atomicAdd(&red[2], (unsigned)incl);
    wbase = __shfl_sync(0xffffffffu, wbase, 31);
    const unsigned lt = (1u << (tid & 31)) - 1u;
    int run = 0;
#pragma unroll
    for (int e = 0; e < kSwPerT; e++) {
      const bool v = W.valid >> e & 1;
      const unsigned m = __ballot_sync(0xffffffffu, v);
      if (v) {
        A.victims[base_off + wbase + run + __popc(m & lt)] = W.j0 + e;
        atomicAdd(A.cold + W.nxts[e], 1u);
      }
      run += __popc(m);
    }
    return;
  }
  // the cut window: the first rem_cut valid entries in list order
  const int64_t rem_cut = *reinterpret_cast<const volatile int64_t*>(&C->rem_cut);
  int off, total;
  Scan(scan).ExclusiveSum(W.nvalid, off, total);
#pragma unroll
  for (int e = 0; e < kSwPerT; e++) {
    if (!(W.valid >> e & 1)) continue;
    const int64_t r = off++;
    if (r >= rem_cut) break;
    const uint32_t j = W.j0 + e;
    A.victims[base_off + r] = j;
    atomicAdd(A.cold + W.nxts[e], 1u);
    if (r == rem_cut - 1) {
      C->last_taken = j;
      C->hs_new = e + 1 < kSwPerT ? W.subs[e + 1] : kUnknown;
    }
  }
}

__global__ void __launch_bounds__(kSwThreads, 1)
    sweep_coop_kernel(SweepArgs A, CoopSync* C) {
  extern __shared__ __align__(16) unsigned char sw_raw[];
  using Scan = cub::BlockScan<int, kSwThreads>;
  __shared__ typename Scan::TempStorage scan;
  __shared__ uint32_t red[4];
  __shared__ unsigned posted;
  __shared__ int64_t bc_taken;
  __shared__ int bc_b;
  __shared__ uint32_t bc_fna, bc_fsub;
  const int tid = threadIdx.x;
  const int G = (int)gridDim.x;
  CoopWin W;
  if (blockIdx.x != 0) {  // helpers: run posted jobs on window blockIdx.x
    unsigned seen = 0;
    while (true) {
      if (tid == 0) {
        unsigned j;
        while ((j = vld(&C->job)) == seen) __nanosleep(32);
        __threadfence();
        posted = j;
      }
      __syncthreads();
      seen = posted;
      const int type = (int)vld(reinterpret_cast<const unsigned*>(&C->type));
      if (type == 3) return;
      const int nwin = (int)vld(reinterpret_cast<const unsigned*>(&C->nwin));
      if ((int)blockIdx.x < nwin) {
        if (type == 1) coop_scan(A, C, blockIdx.x, W, red);
        else coop_commit(A, C, blockIdx.x, W, red, &scan);
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(&C->done, 1u);
      }
    }
  }
  SweepSm& sm = *reinterpret_cast<SweepSm*>(sw_raw);
  unsigned jobs = 0;  // posted so far (CTA 0 is the only poster)
  auto run_job = [&](int type) {
    if (tid == 0) {
      C->type = type;
      __threadfence();
      atomicAdd(&C->job, 1u);
    }
    jobs++;
    const int nwin = C->nwin;
    if (0 < nwin) {
      if (type == 1) coop_scan(A, C, 0, W, red);
      else coop_commit(A, C, 0, W, red, &scan);
    }
    __syncthreads();
    if (tid == 0) {
      const unsigned want = (unsigned)(G - 1) * jobs;
      while (vld(&C->done) < want) __nanosleep(32);
      __threadfence();
    }
    __syncthreads();
  };
  const int ncache = A.nb < kSwCache ? A.nb : kSwCache;
  for (int b = tid; b < ncache; b += kSwThreads) {
    sm.head[b] = A.boff[b];
    sm.end[b] = A.boff[b + 1];
    sm.head_sub[b] = sm.head[b] >= sm.end[b] ? kNone : kUnknown;
  }
  if (tid == 0) {
    sm.hot = sm.peak = sm.evictions = sm.reloads = sm.nv = 0;
    sm.err = 0;
    sm.err_info = 0;
    sm.windows = sm.visits = sm.skipped = 0;
  }
  __syncthreads();
  for (int64_t base = 0; base < A.S; base += kSwBlock) {
    const int cnt = (int)(A.S - base < kSwBlock ? A.S - base : kSwBlock);
    for (int t = tid; t < cnt; t += kSwThreads) {
      sm.fresh[t] = A.fresh[base + t];
      sm.grad[t] = A.grad[base + t];
      sm.cold[t] = __ldcg(A.cold + base + t);
    }
    if (tid == 0) {
      sm.i = 0;
      sm.mode = 0;
    }
    __syncthreads();
    while (true) {
      if (tid == 0) {  // the scalar machine (as in sweep_kernel)
        sm.k = 0;
        int i = sm.i;
        int64_t hot = sm.hot;
        while (i < cnt) {
          if (sm.mode == 0) {
            const int64_t need = (int64_t)sm.fresh[i] + sm.cold[i];
            if (need <= A.slots - hot) {
              hot += need;
              if (hot > sm.peak) sm.peak = hot;
              sm.reloads += sm.cold[i];
              hot -= sm.grad[i];
              i++;
              continue;
            }
            if (need > A.slots) {
              sm.err = ATLAS_ECONFIG;
              sm.err_info = need;
              break;
            }
            sm.need_old = need;
            sm.mode = 1;
          }
          const int64_t free = A.slots - hot;
          if (free < sm.need_old) {
            int64_t k = sm.need_old - free;
            if (k < A.evict_batch) k = A.evict_batch;
            if (k > hot) k = hot;
            if (k <= 0) {
              sm.err = ATLAS_EINVARIANT;
              sm.err_info = -1;
              break;
            }
            sm.k = k;
            break;
          }
          sm.mode = 0;
        }
        sm.i = i;
        sm.hot = hot;
      }
      __syncthreads();
      const int64_t k = sm.k;
      if (k == 0 || sm.err) break;
      // ---- pop k entries in rounds over the grid ---------------------
      const uint32_t s = (uint32_t)(base + sm.i);
      int64_t rem = k;
      int64_t nv = sm.nv;
      int b = A.b0;
      bool bad = false;
      while (rem > 0) {
        if (b >= A.nb) {
          bad = true;
          break;
        }
        const bool cached = b < kSwCache;
        uint32_t h, e_end;
        if (cached) {
          if (sm.head_sub[b] >= s && sm.head_sub[b] != kUnknown) {
            if (tid == 0) sm.skipped++;
            b++;
            continue;
          }
          h = sm.head[b];
          e_end = sm.end[b];
        } else {
          h = __ldcg(A.head + b);
          e_end = A.boff[b + 1];
        }
        if (h >= e_end) {
          b++;
          continue;
        }
        const uint32_t w0 = h & ~3u;
        const int64_t nw_all = ((int64_t)e_end - w0 + kSwWin - 1) / kSwWin;
        const int nwin = (int)(nw_all < G ? nw_all : G);
        if (tid == 0) {
          C->h = h;
          C->end = e_end;
          C->s = s;
          C->w0 = w0;
          C->nwin = nwin;
        }
        __syncthreads();
        run_job(1);
        // the cut: first window whose running count reaches rem; windows
        // past the first undelivered entry hold nothing (lists are sorted
        // by delivery sub-batch)
        if (tid == 0) {
          int64_t cum = 0;
          int cut = nwin;
          uint32_t fna = kNone, fsub = kUnknown;
          for (int w = 0; w < nwin; w++) {
            const int64_t c = (int64_t)vld(&C->cnt[w]);
            C->off[w] = cum;
            if (cut == nwin && cum + c >= rem) {
              cut = w;
              C->rem_cut = rem - cum;
            }
            if (cut == nwin) cum += c;
            if (fna == kNone && vld(&C->fna[w]) != kNone) {
              fna = vld(&C->fna[w]);
              fsub = vld(&C->fna_sub[w]);
            }
          }
          C->cut = cut;
          C->nv = nv;
          bc_fna = fna;
          bc_fsub = fsub;
          bc_taken = cum;
        }
        __syncthreads();
        run_job(2);
        if (tid == 0) {
          const int cut = C->cut;
          uint32_t h_new, v;
          const int bcur = b;
          if (cut < nwin) {  // satisfied inside window `cut`
            h_new = *reinterpret_cast<volatile uint32_t*>(&C->last_taken) + 1;
            v = *reinterpret_cast<volatile uint32_t*>(&C->hs_new);
            nv += rem;
            rem = 0;
          } else {
            const int64_t taken = bc_taken;
            nv += taken;
            rem -= taken;
            const uint32_t fna = bc_fna;
            const uint32_t wend = min(e_end, w0 + (uint32_t)(nwin * kSwWin));
            if (fna != kNone) {
              h_new = fna;
              v = bc_fsub;
              b++;
            } else {
              h_new = wend;
              v = wend >= e_end ? kNone : kUnknown;
              if (wend >= e_end) b++;
            }
          }
          if (h_new >= e_end) v = kNone;
          if (cached) {
            sm.head[bcur] = h_new;
            sm.head_sub[bcur] = v;
          } else {
            A.head[bcur] = h_new;
          }
          sm.windows += nwin;
          sm.visits++;
          bc_taken = rem;  // broadcast the walk state
          bc_b = b;
          sm.nv = nv;
        }
        __syncthreads();
        rem = bc_taken;
        nv = sm.nv;
        b = bc_b;
        __syncthreads();
      }
      if (tid == 0) {
        if (bad) {
          sm.err = ATLAS_EINVARIANT;
          sm.err_info = rem;
        }
        sm.hot -= k - rem;
        sm.evictions += k - rem;
        sm.nv = nv;
      }
      __syncthreads();
      // the helpers added reload counts in global memory: restage ours
      for (int t = sm.i + tid; t < cnt; t += kSwThreads)
        sm.cold[t] = __ldcg(A.cold + base + t);
      __syncthreads();
      if (sm.err) break;
    }
    __syncthreads();
    for (int t = tid; t < cnt; t += kSwThreads) A.cold_out[base + t] = sm.cold[t];
    __syncthreads();
    if (sm.err) break;
  }
  if (tid == 0) {
    C->type = 3;
    __threadfence();
    atomicAdd(&C->job, 1u);
    A.out[0] = sm.evictions;
    A.out[1] = sm.reloads;
    A.out[2] = sm.peak;
    A.out[3] = sm.nv;
    A.out[4] = sm.err;
    A.out[5] = sm.err_info;
    A.out[6] = (int64_t)sm.windows;
    A.out[7] = (int64_t)sm.skipped;
  }
}

template <typename T>
void fill_zero(DevBuf<T>& b, size_t n, cudaStream_t s) {
  b.reserve(std::max<size_t>(n, 1));
  ATLAS_CUDA(cudaMemsetAsync(b.ptr, 0, std::max<size_t>(n, 1) * sizeof(T), s));
}

int bits_for(uint64_t x) {  // bits needed to hold values <= x
  int b = 1;
  while (b < 64 && (x >> b) != 0) b++;
  return b;
}

}  // namespace

// ATLAS_SWEEP_PROFILE=1: per-phase device times of each replay on stderr
struct PhaseTimer {
  cudaStream_t s;
  bool on;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  explicit PhaseTimer(cudaStream_t st) : s(st) {
    const char* e = getenv("ATLAS_SWEEP_PROFILE");
    on = e && e[0] == '1';
    mark("start");
  }
  void mark(const char* name) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.emplace_back(name, e);
  }
  ~PhaseTimer() {
    if (!on) return;
    cudaEventSynchronize(ev.back().second);
    std::string line = "[sweep]";
    for (size_t i = 1; i < ev.size(); i++) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
      line += " " + std::string(ev[i].first) + "=" + std::to_string(ms);
    }
    fprintf(stderr, "%s\n", line.c_str());
    for (auto& e : ev) cudaEventDestroy(e.second);
  }
};

// ATLAS_SWEEP=0 (tests, A/B probes): replay on the per-element machine
void free_sweep_ws(SweepWs* w) { delete w; }

bool sweep_enabled() {
  const char* e = getenv("ATLAS_SWEEP");
  return !(e && e[0] == '0');
}

// Returns false (nothing changed) when the layer must take the per-element
// machine instead: inconsistent deliveries (it raises the reference's
// error) or a stream too long for 32-bit element indices.
static bool run_sweep(atlas_layer* L, SweepWs& W, PhaseTimer& T,
                      cudaStream_t s);

static bool key_matches(const SweepWs& W, const atlas_layer* L,
                        const atlas_graph* g, int64_t R) {
  return W.valid && W.key_gen == g->generation && W.key_R == R &&
         W.key_sb == L->sub_batch && W.key_model == L->desc.model &&
         W.key_policy == L->desc.policy;
}

// the layer's replay straight from a cached static schedule (no run
// materialisation); false when the cache does not hold this key
bool sweep_try_cached(atlas_layer* L, const atlas_graph* g, int64_t R,
                      cudaStream_t s) {
  if (!sweep_enabled() || L->desc.policy == ATLAS_RND || L->desc.record_log)
    return false;
  SweepWs& W = sweep_ws_of(g);
  if (!key_matches(W, L, g, R)) return false;
  ATLAS_NVTX("sweep_replay_cached");
  PhaseTimer T(s);
  return run_sweep(L, W, T, s);
}

bool sweep_replay(atlas_layer* L, const atlas_graph* g, int64_t R,
                  const uint64_t* runs, const int64_t* run_off_dev,
                  const std::vector<int64_t>& run_off, cudaStream_t s) {
  ATLAS_NVTX("sweep_replay");
  const int model = L->desc.model;
  const int64_t V = g->V, lo = g->lo, hi = g->hi, nloc = L->nloc;
  const int64_t nchunks = ceil_div(V, R);
  const int64_t sb = L->sub_batch;
  SweepWs& W = sweep_ws_of(g);
  W.valid = false;
  PhaseTimer T(s);

  // ---- per-chunk pass sizes and the element / sub-batch layout ----------
  std::vector<int64_t> npre(nchunks, 0);
  if (model == ATLAS_GCN && nloc > 0) {
    W.zr.reserve(nloc + 1);
    W.tmp_u32.reserve(nloc + 1);
    zero_flags<<<grid_of(nloc), 256, 0, s>>>(L->indeg.ptr, nloc, W.tmp_u32.ptr);
    ATLAS_CUDA(cudaMemsetAsync(W.tmp_u32.ptr + nloc, 0, sizeof(uint32_t), s));
    size_t tb = 0;
    ATLAS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, W.tmp_u32.ptr,
                                             W.zr.ptr, nloc + 1, s));
    W.cub_tmp.reserve(tb);
    ATLAS_CUDA(cub::DeviceScan::ExclusiveSum(W.cub_tmp.ptr, tb, W.tmp_u32.ptr,
                                             W.zr.ptr, nloc + 1, s));
    W.chunk64.reserve(nchunks);
    ChunkMap M0{R, lo, hi, sb, nullptr, nullptr};
    chunk_zero_counts<<<grid_of(nchunks), 256, 0, s>>>(W.zr.ptr, nchunks, M0,
                                                      nloc, W.chunk64.ptr);
    count_launch(3);
    ATLAS_LAUNCH_CHECK();
    ATLAS_CUDA(cudaMemcpyAsync(npre.data(), W.chunk64.ptr,
                               nchunks * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, s));
    ATLAS_CUDA(cudaStreamSynchronize(s));
  }
  T.mark("zeros");
  std::vector<int64_t> eoff(3 * nchunks), soff(3 * nchunks);
  std::vector<int64_t> touched(nchunks);
  int64_t NE = 0, S = 0;
  for (int64_t c = 0; c < nchunks; c++) {
    const int64_t self_n =
        model == ATLAS_SAGE
            ? std::max<int64_t>(0, std::min((c + 1) * R, hi) -
                                       std::max(c * R, lo))
            : 0;
    const int64_t sizes[3] = {npre[c], self_n, run_off[c + 1] - run_off[c]};
    for (int k = 0; k < 3; k++) {
      eoff[3 * c + k] = NE;
      soff[3 * c + k] = S;
      NE += sizes[k];
      S += ceil_div(sizes[k], sb);
    }
    touched[c] = sizes[1] + sizes[2];
  }
  if (NE >= (int64_t)0xFFFFFF00ll || S >= (int64_t)0xFFFFFF00ll) return false;
  if (NE == 0) return false;
  W.eoff.reserve(3 * nchunks);
  W.soff.reserve(3 * nchunks);
  ATLAS_CUDA(cudaMemcpyAsync(W.eoff.ptr, eoff.data(), eoff.size() * 8,
                             cudaMemcpyHostToDevice, s));
  ATLAS_CUDA(cudaMemcpyAsync(W.soff.ptr, soff.data(), soff.size() * 8,
                             cudaMemcpyHostToDevice, s));
  ChunkMap M{R, lo, hi, sb, W.eoff.ptr, W.soff.ptr};

  // ---- static per-element data ---------------------------------------
  W.el_v.reserve(NE);
  W.el_cnt.reserve(NE);
  W.el_sub.reserve(NE);
  const int64_t nruns = run_off[nchunks];
  if (nruns > 0) {
    fill_edge<<<grid_of(nruns), 256, 0, s>>>(runs, run_off_dev, nchunks, nruns,
                                             M, W.el_v.ptr, W.el_cnt.ptr,
                                             W.el_sub.ptr);
    count_launch();
  }
  if (model == ATLAS_SAGE && nloc > 0) {
    fill_self<<<grid_of(nloc), 256, 0, s>>>(nloc, M, W.el_v.ptr, W.el_cnt.ptr,
                                            W.el_sub.ptr);
    count_launch();
  }
  if (model == ATLAS_GCN && nloc > 0) {
    fill_pre<<<grid_of(nloc), 256, 0, s>>>(nloc, W.zr.ptr, M, W.el_v.ptr,
                                           W.el_cnt.ptr, W.el_sub.ptr);
    count_launch();
  }
  ATLAS_LAUNCH_CHECK();
  T.mark("fill");
  // group by vertex (stable: each vertex's deliveries in stream order);
  // the values carry (element, count) so the chain below streams
  W.sv.reserve(NE);
  W.se.reserve(NE);
  W.pk.reserve(NE);
  W.svk.reserve(NE);
  pack_idx_cnt<<<grid_of(NE), 256, 0, s>>>(W.el_cnt.ptr, NE, W.pk.ptr);
  count_launch();
  {
    size_t tb = 0;
    const int vb = bits_for((uint64_t)std::max<int64_t>(nloc - 1, 1));
    ATLAS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, W.el_v.ptr,
                                               W.sv.ptr, W.pk.ptr, W.svk.ptr,
                                               NE, 0, vb, s));
    W.cub_tmp.reserve(tb);
    ATLAS_CUDA(cub::DeviceRadixSort::SortPairs(W.cub_tmp.ptr, tb, W.el_v.ptr,
                                               W.sv.ptr, W.pk.ptr, W.svk.ptr,
                                               NE, 0, vb, s));
    count_launch();
  }
  T.mark("sort_v");
  W.cs.reserve(NE);
  W.P.reserve(NE);
  low_words<<<grid_of(NE), 256, 0, s>>>(W.svk.ptr, NE, W.cs.ptr);
  count_launch();
  {
    size_t tb = 0;
    ATLAS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, W.cs.ptr, W.P.ptr,
                                             NE, s));
    W.cub_tmp.reserve(tb);
    ATLAS_CUDA(cub::DeviceScan::InclusiveSum(W.cub_tmp.ptr, tb, W.cs.ptr,
                                             W.P.ptr, NE, s));
    count_launch();
  }
  T.mark("scan");
  W.lastP.reserve(std::max<int64_t>(nloc, 1));
  vertex_last<<<grid_of(NE), 256, 0, s>>>(W.sv.ptr, W.P.ptr, NE, W.lastP.ptr);
  fill_zero(W.flags, 4, s);  // mismatch, max pending
  fill_zero(W.fresh, S, s);
  fill_zero(W.grad, S, s);
  fill_zero(W.cold, S, s);
  W.cold_out.reserve(std::max<int64_t>(S, 1));
  const bool lru = L->desc.policy == ATLAS_LRU;
  // keys into pk (free after the vertex sort), values into cs (free after
  // the scan)
  chain_entries<<<grid_of(NE), 256, 0, s>>>(
      W.sv.ptr, W.svk.ptr, W.P.ptr, W.lastP.ptr, W.el_sub.ptr, L->indeg.ptr,
      model == ATLAS_GCN ? 0 : 1, lru ? 1 : 0, NE, W.pk.ptr, W.cs.ptr,
      W.fresh.ptr, W.grad.ptr, reinterpret_cast<int*>(W.flags.ptr),
      W.flags.ptr + 1);
  count_launch(2);
  ATLAS_LAUNCH_CHECK();
  T.mark("chain");
  uint32_t hflags[2] = {0, 0};
  unsigned long long total_msgs = 0;
  ATLAS_CUDA(cudaMemcpyAsync(hflags, W.flags.ptr, sizeof(hflags),
                             cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaMemcpyAsync(&total_msgs, W.P.ptr + NE - 1, sizeof(total_msgs),
                             cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
  if (hflags[0]) return false;  // deliveries != pending: exact errors
  const uint32_t maxp = hflags[1];
  T.mark("sub_stats");

  // ---- heap lists: MINPEND = one FIFO per pending value, i.e. the entries
  // sorted by (pending, element); LRU = the stream (sorted by element) ----
  const int64_t nb = lru ? 1 : (int64_t)maxp + 1;
  W.ent_sub.reserve(NE + 4);
  W.ent_next.reserve(NE + 4);
  W.boff.reserve(nb + 1);
  W.head.reserve(nb);
  W.sk64.reserve(NE);
  {
    size_t tb = 0;
    const int kb = lru ? 32 : 32 + bits_for(maxp);
    ATLAS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, W.pk.ptr,
                                               W.sk64.ptr, W.cs.ptr,
                                               W.svk.ptr, NE, 0, kb, s));
    W.cub_tmp.reserve(tb);
    ATLAS_CUDA(cub::DeviceRadixSort::SortPairs(W.cub_tmp.ptr, tb, W.pk.ptr,
                                               W.sk64.ptr, W.cs.ptr,
                                               W.svk.ptr, NE, 0, kb, s));
    count_launch();
  }
  entries_from_sorted<<<grid_of(NE), 256, 0, s>>>(W.sk64.ptr, W.svk.ptr, NE,
                                                  W.ent_sub.ptr,
                                                  W.ent_next.ptr, W.se.ptr);
  count_launch();
  if (lru) {
    const uint32_t hb[2] = {0u, (uint32_t)NE};
    ATLAS_CUDA(cudaMemcpyAsync(W.boff.ptr, hb, sizeof(hb),
                               cudaMemcpyHostToDevice, s));
  } else {
    bucket_bounds64<<<grid_of(NE + 1), 256, 0, s>>>(W.sk64.ptr, NE, nb,
                                                    W.boff.ptr);
    count_launch();
  }
  ATLAS_CUDA(cudaMemsetAsync(W.ent_sub.ptr + NE, 0xFF, 4 * sizeof(uint32_t), s));
  ATLAS_CUDA(cudaMemsetAsync(W.ent_next.ptr + NE, 0, 4 * sizeof(uint32_t), s));
  ATLAS_LAUNCH_CHECK();

  T.mark("buckets");
  W.valid = true;
  W.key_gen = g->generation;
  W.key_R = R;
  W.key_sb = sb;
  W.key_model = model;
  W.key_policy = L->desc.policy;
  W.NE = NE;
  W.S = S;
  W.nchunks = nchunks;
  W.nb = nb;
  W.b0 = lru ? 0 : 1;
  W.lru = lru;
  W.total_msgs = total_msgs;
  W.h_soff = soff;
  W.h_touched = touched;
  return run_sweep(L, W, T, s);
}

// the dynamic part: the sweep over sub-batches from fresh heads and zero
// reload counts, then unique reloads and per-chunk reloads
static bool run_sweep(atlas_layer* L, SweepWs& W, PhaseTimer& T,
                      cudaStream_t s) {
  const int64_t NE = W.NE, S = W.S, nchunks = W.nchunks, nb = W.nb;
  const int64_t nloc = L->nloc;
  const uint32_t* ent_el = W.se.ptr;  // element of each heap entry
  ATLAS_CUDA(cudaMemsetAsync(W.cold.ptr, 0, std::max<int64_t>(S, 1) * 4, s));
  ATLAS_CUDA(cudaMemcpyAsync(W.head.ptr, W.boff.ptr, nb * sizeof(uint32_t),
                             cudaMemcpyDeviceToDevice, s));
  // ---- the sweep ------------------------------------------------------
  W.victims.reserve(NE);
  W.out.reserve(8);
  SweepArgs A{};
  A.S = S;
  A.fresh = W.fresh.ptr;
  A.grad = W.grad.ptr;
  A.cold = W.cold.ptr;
  A.cold_out = W.cold_out.ptr;
  A.slots = L->desc.slot_count;
  A.evict_batch = L->evict_batch;
  A.b0 = W.b0;
  A.nb = (int32_t)nb;
  A.boff = W.boff.ptr;
  A.head = W.head.ptr;
  A.ent_sub = W.ent_sub.ptr;
  A.ent_next = W.ent_next.ptr;
  A.victims = W.victims.ptr;
  W.flags8.reserve(NE + 4);
  ATLAS_CUDA(cudaMemsetAsync(W.flags8.ptr, 0, NE + 4, s));
  A.popped = W.flags8.ptr;
  A.out = W.out.ptr;
  {
    const char* e = getenv("ATLAS_SWEEP_DIAG_NO_FAR");  // wrong results!
    A.diag_no_far = e ? atoi(e) : 0;  // 1: no far atomics, 2: none
  }
  const int smem = (int)sizeof(SweepSm);
  static bool attr = false;
  if (!attr) {
    ATLAS_CUDA(cudaFuncSetAttribute(
        sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  // ATLAS_SWEEP_COOP=1: the cooperative-grid sweep (measured 5-8x slower:
  // its two grid jobs per round cost ~14 us each, profiles/
  // r2_sweep_variants.txt), otherwise the single-CTA sweep
  const char* ce = getenv("ATLAS_SWEEP_COOP");
  int coop_grid = 0;
  if (ce && ce[0] == '1') {
    int dev = 0, coop = 0, per_sm = 0;
    ATLAS_CUDA(cudaGetDevice(&dev));
    ATLAS_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    static bool cattr = false;
    if (!cattr) {
      ATLAS_CUDA(cudaFuncSetAttribute(
          sweep_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
          smem));
      cattr = true;
    }
    ATLAS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, sweep_coop_kernel, kSwThreads, smem));
    if (coop && per_sm > 0)
      coop_grid = std::min<int>(kCoopMax, num_sms() * per_sm);
  }
  if (coop_grid > 1) {
    W.coop.reserve(sizeof(CoopSync));
    ATLAS_CUDA(cudaMemsetAsync(W.coop.ptr, 0, sizeof(CoopSync), s));
    CoopSync* C = reinterpret_cast<CoopSync*>(W.coop.ptr);
    void* args[] = {&A, &C};
    ATLAS_CUDA(cudaLaunchCooperativeKernel((const void*)sweep_coop_kernel,
                                           dim3(coop_grid), dim3(kSwThreads),
                                           args, smem, s));
  } else {
    sweep_kernel<<<1, kSwThreads, smem, s>>>(A);
  }
  count_launch();
  ATLAS_LAUNCH_CHECK();
  T.mark("sweep");
  int64_t out[8];
  ATLAS_CUDA(cudaMemcpyAsync(out, W.out.ptr, sizeof(out),
                             cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
  if (T.on)
    fprintf(stderr, "[sweep] S=%lld NE=%lld evictions=%lld windows=%lld "
                    "skipped_lists=%lld\n",
            (long long)S, (long long)NE, (long long)out[0], (long long)out[6],
            (long long)out[7]);
  if (out[4] == ATLAS_ECONFIG)
    fail(ATLAS_ECONFIG, "batch of " + std::to_string(out[5]) +
                            " cannot fit in " +
                            std::to_string(L->desc.slot_count) + " slots");
  if (out[4])
    fail(ATLAS_EINVARIANT, "sweep replay: heap underflow (" +
                               std::to_string(out[5]) + " victims missing)");
  const int64_t evictions = out[0], reloads = out[1], peak = out[2],
                nvict = out[3];

  // ---- unique reloads, per-chunk reloads -----------------------------
  ATLAS_CUDA(cudaMemsetAsync(L->unique_reloaded.ptr, 0,
                             std::max<int64_t>(nloc, 1), s));
  fill_zero(W.count, 1, s);
  if (nvict > 0 && coop_grid > 1) {
    mark_unique<<<grid_of(nvict), 256, 0, s>>>(W.victims.ptr, nvict, ent_el,
                                               W.el_v.ptr,
                                               L->unique_reloaded.ptr);
    count_launch();
  } else if (nvict > 0) {
    mark_unique_popped<<<grid_of(NE / 4 + 1), 256, 0, s>>>(
        W.flags8.ptr, NE, ent_el, W.el_v.ptr, L->unique_reloaded.ptr);
    count_launch();
  }
  count_flags<<<grid_of(nloc), 256, 0, s>>>(L->unique_reloaded.ptr, nloc,
                                            W.count.ptr);
  count_launch();
  T.mark("unique");
  std::vector<uint32_t> cold(S);
  unsigned long long uniq = 0;
  ATLAS_CUDA(cudaMemcpyAsync(cold.data(), W.cold_out.ptr, S * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaMemcpyAsync(&uniq, W.count.ptr, sizeof(uniq),
                             cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
  for (int64_t c = 0; c < nchunks; c++) {
    const int64_t s0 = W.h_soff[3 * c],
                  s1 = c + 1 < nchunks ? W.h_soff[3 * c + 3] : S;
    int64_t r = 0;
    for (int64_t q = s0; q < s1; q++) r += cold[q];
    L->chunk_reloads.push_back(r);
    L->chunk_touched.push_back(W.h_touched[c]);
  }
  L->sweep_path = true;
  L->sw_messages = (int64_t)W.total_msgs;
  L->sw_evictions = evictions;
  L->sw_reloads = reloads;
  L->sw_hot_peak = peak;
  L->sw_unique = (int64_t)uniq;
  L->sw_admissions = nloc + reloads;
  return true;
}

}  // namespace atlas
