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

__global__ void iota_u32(uint32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (uint32_t)i;
}

__global__ void gather_cnt(const uint32_t* __restrict__ se,
                           const uint32_t* __restrict__ el_cnt, int64_t n,
                           unsigned long long* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = el_cnt[se[j]];
}

// per vertex: the prefix at its last element (elements grouped by vertex)
__global__ void vertex_last(const uint32_t* __restrict__ sv,
                            const unsigned long long* __restrict__ P,
                            int64_t n, unsigned long long* __restrict__ lastP) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    if (j == n - 1 || sv[j + 1] != sv[j]) lastP[sv[j]] = P[j];
}

// pending after each delivery, successor's sub-batch, first-delivery flag;
// a vertex whose deliveries do not add up to its pending count is flagged
// (the per-element machine then reproduces the reference's error)
__global__ void chain_links(const uint32_t* __restrict__ sv,
                            const uint32_t* __restrict__ se,
                            const unsigned long long* __restrict__ P,
                            const unsigned long long* __restrict__ lastP,
                            const uint32_t* __restrict__ el_cnt,
                            const uint32_t* __restrict__ el_sub,
                            const uint32_t* __restrict__ indeg, int self_term,
                            int64_t n, uint32_t* __restrict__ el_newp,
                            uint32_t* __restrict__ el_nsub,
                            uint8_t* __restrict__ el_fresh,
                            int* __restrict__ mismatch,
                            unsigned* __restrict__ maxp) {
  unsigned my_max = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = sv[j], i = se[j];
    const bool first = j == 0 || sv[j - 1] != v;
    const bool last = j == n - 1 || sv[j + 1] != v;
    const unsigned long long left = lastP[v] - P[j];
    if (first) {
      const unsigned long long p0 = (unsigned long long)indeg[v] + self_term;
      if (left + el_cnt[i] != p0) atomicExch(mismatch, 1);
    }
    const uint32_t np = left > 0xFFFFFFF0ull ? 0xFFFFFFF0u : (uint32_t)left;
    el_newp[i] = np;
    el_nsub[i] = last ? 0u : el_sub[se[j + 1]];
    el_fresh[i] = first ? 1 : 0;
    my_max = max(my_max, np);
  }
  for (int o = 16; o > 0; o >>= 1)
    my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
  if ((threadIdx.x & 31) == 0 && my_max) atomicMax(maxp, my_max);
}

// per sub-batch fresh and graduating counts (elements in stream order, so
// a warp's elements mostly share one sub-batch)
__global__ void sub_stats(const uint32_t* __restrict__ el_sub,
                          const uint8_t* __restrict__ el_fresh,
                          const uint32_t* __restrict__ el_newp, int64_t n,
                          uint32_t* __restrict__ fresh,
                          uint32_t* __restrict__ grad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    const bool in = i < n;
    const uint32_t s = in ? el_sub[i] : kNone;
    const unsigned f = in ? el_fresh[i] : 0u;
    const unsigned g = (in && el_newp[i] == 0) ? 1u : 0u;
    const unsigned peers = __match_any_sync(0xffffffffu, s);
    const unsigned fsum = __reduce_add_sync(peers, f);
    const unsigned gsum = __reduce_add_sync(peers, g);
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1 && in) {
      if (fsum) atomicAdd(fresh + s, fsum);
      if (gsum) atomicAdd(grad + s, gsum);
    }
  }
}

// bucket list entries (sorted by key, stream order within a key)
__global__ void make_entries(const uint32_t* __restrict__ be,
                             const uint32_t* __restrict__ bk,
                             const uint32_t* __restrict__ el_sub,
                             const uint32_t* __restrict__ el_nsub, int64_t n,
                             uint32_t* __restrict__ ent_sub,
                             uint32_t* __restrict__ ent_next) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t i = be ? be[k] : (uint32_t)k;
    const uint32_t key = bk[be ? k : i];
    ent_sub[k] = el_sub[i];
    ent_next[k] = key > 0 ? el_nsub[i] : 0u;  // pending 0: never in the heap
  }
}

// boff[b] = first entry with key >= b, for b in [0, nb]
__global__ void bucket_bounds(const uint32_t* __restrict__ bk, int64_t n,
                              int64_t nb, uint32_t* __restrict__ boff) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t prev = k == 0 ? -1 : (int64_t)bk[k - 1];
    const int64_t cur = k == n ? nb : min((int64_t)bk[k], nb);
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
  uint32_t* victims;         // popped entries, in pop order
  int64_t* out;              // evictions, reloads, hot_peak, nvict, err, info
};

// Bucket entries reach the CTA through two shared-memory window buffers
// filled by bulk async copies (cp.async.bulk, one thread, mbarrier
// completion): the entry lists are static, so a buffer is a cache of the
// range [start, start + len) and the walk keeps the next window of the
// same list in flight while it scans the current one.
constexpr int kSwWin = 8192;                  // entries per window buffer
constexpr int kSwPerT = kSwWin / kSwThreads;  // 8 entries per thread

struct SweepSm {
  uint32_t sub[2][kSwWin];   // window buffers: ent_sub
  uint32_t nxt[2][kSwWin];   //                 ent_next
  uint32_t fresh[kSwBlock], grad[kSwBlock], cold[kSwBlock];
  uint64_t bar[2];
  uint32_t buf_start[2], buf_len[2], buf_phase[2];
  int32_t buf_busy[2];       // a copy is in flight (not yet waited on)
  int64_t hot, peak, evictions, reloads, need_old, k, nv;
  int32_t i, mode, err;
  int64_t err_info;
  uint32_t last_taken;
  uint32_t first_na[2];
};

__device__ __forceinline__ uint32_t sw_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// thread 0: start filling buffer q with entries [start, start + len)
__device__ void sw_fetch(SweepSm& sm, const SweepArgs& A, int q,
                         uint32_t start, uint32_t len) {
  const uint32_t bytes = ((len + 3u) & ~3u) * 4u;  // arrays padded by 4
  const uint32_t bar = sw_smem(&sm.bar[q]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
      "r"(2u * bytes)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(sw_smem(sm.sub[q])),
      "l"(A.ent_sub + start), "r"(bytes), "r"(bar)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(sw_smem(sm.nxt[q])),
      "l"(A.ent_next + start), "r"(bytes), "r"(bar)
      : "memory");
  sm.buf_start[q] = start;
  sm.buf_len[q] = len;
  sm.buf_busy[q] = 1;
}

__device__ __forceinline__ void sw_wait(SweepSm& sm, int q) {
  const uint32_t bar = sw_smem(&sm.bar[q]), ph = sm.buf_phase[q];
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "SW_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SW_WAIT_%=;\n}" ::"r"(bar),
      "r"(ph)
      : "memory");
}

__global__ void __launch_bounds__(kSwThreads, 1) sweep_kernel(SweepArgs A) {
  extern __shared__ __align__(128) unsigned char sw_raw[];
  SweepSm& sm = *reinterpret_cast<SweepSm*>(sw_raw);
  using Scan = cub::BlockScan<int, kSwThreads>;
  __shared__ typename Scan::TempStorage scan;
  const int tid = threadIdx.x;
  if (tid == 0) {
    sm.hot = sm.peak = sm.evictions = sm.reloads = sm.nv = 0;
    sm.err = 0;
    sm.err_info = 0;
    for (int q = 0; q < 2; q++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
          sw_smem(&sm.bar[q])));
      sm.buf_start[q] = sm.buf_len[q] = 0;
      sm.buf_phase[q] = 0;
      sm.buf_busy[q] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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
        const uint32_t h = __ldcg(A.head + b);
        const uint32_t e_end = A.boff[b + 1];
        if (h >= e_end) {
          b++;
          continue;
        }
        // a buffer holding h, else fetch [h & ~3, +kSwWin) into the idle one
        if (tid == 0) {
          int q = -1;
          for (int c = 0; c < 2; c++)
            if (h >= sm.buf_start[c] && h < sm.buf_start[c] + sm.buf_len[c])
              q = c;
          if (q < 0) {
            q = (sm.buf_busy[0] && !sm.buf_busy[1]) ? 1 : 0;
            if (sm.buf_busy[q]) {  // drain a stale prefetch first
              sw_wait(sm, q);
              sm.buf_phase[q] ^= 1;
              sm.buf_busy[q] = 0;
            }
            const uint32_t w0 = h & ~3u;
            sw_fetch(sm, A, q, w0, min((uint32_t)kSwWin, e_end - w0));
          }
          // keep the list's next window in flight in the other buffer
          const int o = q ^ 1;
          const uint32_t nx = sm.buf_start[q] + sm.buf_len[q];
          if (nx < e_end && !sm.buf_busy[o] &&
              !(nx >= sm.buf_start[o] && nx < sm.buf_start[o] + sm.buf_len[o]))
            sw_fetch(sm, A, o, nx, min((uint32_t)kSwWin, e_end - nx));
          sm.first_na[(w + 1) & 1] = (uint32_t)q;  // scratch: buffer index
        }
        __syncthreads();
        const int q = (int)sm.first_na[(w + 1) & 1];
        if (sm.buf_busy[q]) sw_wait(sm, q);
        const uint32_t bs = sm.buf_start[q];
        const uint32_t be = bs + sm.buf_len[q];
        __syncthreads();
        if (tid == 0) {
          if (sm.buf_busy[q]) {
            sm.buf_phase[q] ^= 1;
            sm.buf_busy[q] = 0;
          }
          sm.first_na[(w + 1) & 1] = kNone;
        }
        // scan [max(h, bs), be): thread t takes 8 consecutive entries
        const uint32_t j0 = bs + (uint32_t)tid * kSwPerT;
        uint32_t subs[kSwPerT], nxts[kSwPerT];
        {
          const uint4* ps = reinterpret_cast<const uint4*>(sm.sub[q]) + tid * 2;
          const uint4* pn = reinterpret_cast<const uint4*>(sm.nxt[q]) + tid * 2;
          const uint4 s0 = ps[0], s1 = ps[1], n0 = pn[0], n1 = pn[1];
          subs[0] = s0.x; subs[1] = s0.y; subs[2] = s0.z; subs[3] = s0.w;
          subs[4] = s1.x; subs[5] = s1.y; subs[6] = s1.z; subs[7] = s1.w;
          nxts[0] = n0.x; nxts[1] = n0.y; nxts[2] = n0.z; nxts[3] = n0.w;
          nxts[4] = n1.x; nxts[5] = n1.y; nxts[6] = n1.z; nxts[7] = n1.w;
        }
        int valid = 0, nvalid = 0;
        uint32_t first_na = kNone;
#pragma unroll
        for (int e = 0; e < kSwPerT; e++) {
          const uint32_t j = j0 + e;
          if (j < h || j >= be) continue;
          if (subs[e] < s) {
            if (nxts[e] >= s) {
              valid |= 1 << e;
              nvalid++;
            }
          } else if (first_na == kNone) {
            first_na = j;
          }
        }
        int off, total;
        Scan(scan).ExclusiveSum(nvalid, off, total);
        if (first_na != kNone) atomicMin(&sm.first_na[w & 1], first_na);
#pragma unroll
        for (int e = 0; e < kSwPerT; e++) {
          if (!(valid >> e & 1)) continue;
          const int64_t r = off++;
          if (r >= rem) break;
          const uint32_t j = j0 + e;
          A.victims[nv + r] = j;
          const uint32_t nx = nxts[e];
          if ((int64_t)nx < win_hi) atomicAdd(&sm.cold[nx - base], 1u);
          else atomicAdd(A.cold + nx, 1u);
          if (r == rem - 1) sm.last_taken = j;
        }
        __syncthreads();
        uint32_t h_new;
        const int bcur = b;
        if (total >= rem) {
          h_new = sm.last_taken + 1;
          nv += rem;
          rem = 0;
        } else {
          nv += total;
          rem -= total;
          const uint32_t fna = sm.first_na[w & 1];
          if (fna != kNone) {
            h_new = fna;  // the rest of the list is not delivered yet
            b++;
          } else {
            h_new = be;
            if (be >= e_end) b++;
          }
        }
        if (tid == 0) A.head[bcur] = h_new;
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
  // no copy may outlive the CTA
  if (tid == 0)
    for (int q = 0; q < 2; q++)
      if (sm.buf_busy[q]) sw_wait(sm, q);
  __syncthreads();
  if (tid == 0) {
    A.out[0] = sm.evictions;
    A.out[1] = sm.reloads;
    A.out[2] = sm.peak;
    A.out[3] = sm.nv;
    A.out[4] = sm.err;
    A.out[5] = sm.err_info;
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
bool sweep_replay(atlas_layer* L, const atlas_graph* g, int64_t R,
                  const uint64_t* runs, const int64_t* run_off_dev,
                  const std::vector<int64_t>& run_off, cudaStream_t s) {
  ATLAS_NVTX("sweep_replay");
  const int model = L->desc.model;
  const int64_t V = g->V, lo = g->lo, hi = g->hi, nloc = L->nloc;
  const int64_t nchunks = ceil_div(V, R);
  const int64_t sb = L->sub_batch;
  SweepWs& W = sweep_ws_of(g);
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
  // group by vertex (stable: each vertex's deliveries in stream order)
  W.iota.reserve(NE);
  W.sv.reserve(NE);
  W.se.reserve(NE);
  iota_u32<<<grid_of(NE), 256, 0, s>>>(W.iota.ptr, NE);
  count_launch();
  {
    size_t tb = 0;
    const int vb = bits_for((uint64_t)std::max<int64_t>(nloc - 1, 1));
    ATLAS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, W.el_v.ptr,
                                               W.sv.ptr, W.iota.ptr, W.se.ptr,
                                               NE, 0, vb, s));
    W.cub_tmp.reserve(tb);
    ATLAS_CUDA(cub::DeviceRadixSort::SortPairs(W.cub_tmp.ptr, tb, W.el_v.ptr,
                                               W.sv.ptr, W.iota.ptr, W.se.ptr,
                                               NE, 0, vb, s));
    count_launch();
  }
  T.mark("sort_v");
  W.cs.reserve(NE);
  W.P.reserve(NE);
  gather_cnt<<<grid_of(NE), 256, 0, s>>>(W.se.ptr, W.el_cnt.ptr, NE, W.cs.ptr);
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
  W.el_newp.reserve(NE);
  W.el_nsub.reserve(NE);
  W.el_fresh.reserve(NE);
  fill_zero(W.flags, 4, s);  // mismatch, max pending
  chain_links<<<grid_of(NE), 256, 0, s>>>(
      W.sv.ptr, W.se.ptr, W.P.ptr, W.lastP.ptr, W.el_cnt.ptr, W.el_sub.ptr,
      L->indeg.ptr, model == ATLAS_GCN ? 0 : 1, NE, W.el_newp.ptr,
      W.el_nsub.ptr, W.el_fresh.ptr, reinterpret_cast<int*>(W.flags.ptr),
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

  // ---- per sub-batch statics ------------------------------------------
  fill_zero(W.fresh, S, s);
  fill_zero(W.grad, S, s);
  fill_zero(W.cold, S, s);
  W.cold_out.reserve(std::max<int64_t>(S, 1));
  sub_stats<<<grid_of(NE), 256, 0, s>>>(W.el_sub.ptr, W.el_fresh.ptr,
                                        W.el_newp.ptr, NE, W.fresh.ptr,
                                        W.grad.ptr);
  count_launch();

  T.mark("sub_stats");
  // ---- heap lists: MINPEND = one per pending value; LRU = the stream --
  const bool lru = L->desc.policy == ATLAS_LRU;
  const int64_t nb = lru ? 1 : (int64_t)maxp + 1;
  W.ent_sub.reserve(NE + 4);
  W.ent_next.reserve(NE + 4);
  W.boff.reserve(nb + 1);
  W.head.reserve(nb);
  const uint32_t* ent_el = nullptr;
  if (lru) {
    make_entries<<<grid_of(NE), 256, 0, s>>>(nullptr, W.el_newp.ptr,
                                             W.el_sub.ptr, W.el_nsub.ptr, NE,
                                             W.ent_sub.ptr, W.ent_next.ptr);
    const uint32_t hb[2] = {0u, (uint32_t)NE};
    ATLAS_CUDA(cudaMemcpyAsync(W.boff.ptr, hb, sizeof(hb),
                               cudaMemcpyHostToDevice, s));
    count_launch();
  } else {
    // stable by key: stream order within each pending value (the FIFO)
    size_t tb = 0;
    const int kb = bits_for(maxp);
    ATLAS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, W.el_newp.ptr,
                                               W.sv.ptr, W.iota.ptr, W.se.ptr,
                                               NE, 0, kb, s));
    W.cub_tmp.reserve(tb);
    ATLAS_CUDA(cub::DeviceRadixSort::SortPairs(W.cub_tmp.ptr, tb,
                                               W.el_newp.ptr, W.sv.ptr,
                                               W.iota.ptr, W.se.ptr, NE, 0,
                                               kb, s));
    make_entries<<<grid_of(NE), 256, 0, s>>>(W.se.ptr, W.sv.ptr, W.el_sub.ptr,
                                             W.el_nsub.ptr, NE, W.ent_sub.ptr,
                                             W.ent_next.ptr);
    bucket_bounds<<<grid_of(NE + 1), 256, 0, s>>>(W.sv.ptr, NE, nb,
                                                  W.boff.ptr);
    count_launch(3);
    ent_el = W.se.ptr;
  }
  ATLAS_CUDA(cudaMemsetAsync(W.ent_sub.ptr + NE, 0xFF, 4 * sizeof(uint32_t), s));
  ATLAS_CUDA(cudaMemsetAsync(W.ent_next.ptr + NE, 0, 4 * sizeof(uint32_t), s));
  ATLAS_CUDA(cudaMemcpyAsync(W.head.ptr, W.boff.ptr, nb * sizeof(uint32_t),
                             cudaMemcpyDeviceToDevice, s));
  ATLAS_LAUNCH_CHECK();

  T.mark("buckets");
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
  A.b0 = lru ? 0 : 1;
  A.nb = (int32_t)nb;
  A.boff = W.boff.ptr;
  A.head = W.head.ptr;
  A.ent_sub = W.ent_sub.ptr;
  A.ent_next = W.ent_next.ptr;
  A.victims = W.victims.ptr;
  A.out = W.out.ptr;
  const int smem = (int)sizeof(SweepSm);
  static bool attr = false;
  if (!attr) {
    ATLAS_CUDA(cudaFuncSetAttribute(
        sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  sweep_kernel<<<1, kSwThreads, smem, s>>>(A);
  count_launch();
  ATLAS_LAUNCH_CHECK();
  T.mark("sweep");
  int64_t out[6];
  ATLAS_CUDA(cudaMemcpyAsync(out, W.out.ptr, sizeof(out),
                             cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
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
  if (nvict > 0) {
    mark_unique<<<grid_of(nvict), 256, 0, s>>>(W.victims.ptr, nvict, ent_el,
                                               W.el_v.ptr,
                                               L->unique_reloaded.ptr);
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
    const int64_t s0 = soff[3 * c], s1 = c + 1 < nchunks ? soff[3 * c + 3] : S;
    int64_t r = 0;
    for (int64_t q = s0; q < s1; q++) r += cold[q];
    L->chunk_reloads.push_back(r);
    L->chunk_touched.push_back(touched[c]);
  }
  L->sweep_path = true;
  L->sw_messages = (int64_t)total_msgs;
  L->sw_evictions = evictions;
  L->sw_reloads = reloads;
  L->sw_hot_peak = peak;
  L->sw_unique = (int64_t)uniq;
  L->sw_admissions = nloc + reloads;
  return true;
}

}  // namespace atlas
