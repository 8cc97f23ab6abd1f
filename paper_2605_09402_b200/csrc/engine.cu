// Exact control plane: pending counters, admission, min-pending eviction,
// reloads and graduation, replayed bit-exactly on the GPU (kernel plan
// K5/K6 of SURVEY.md §2.1).
//
// The reference's MemoryManager + policies (oocgnn/memstore.py:305-497,
// :103-283) are a sequential state machine driven by _deliver's
// sub-batches (oocgnn/orchestrator.py:165-213). Its observable integer
// results are fixed by:
//   * sub-batches of sub_batch = max(1, slots // 2) over each pass's
//     destination list (GCN zero-degree pre-pass, SAGE self pass, edge
//     pass in first-appearance order);
//   * ensure_hot_many: while need > free: evict max(evict_batch,
//     need - free) until free >= need, re-classify (victims may be in the
//     batch); then admit fresh, then reload cold, both in batch order;
//   * PendingBucketHeap.pop_min(k) == the k smallest (pending, seq) over
//     the HOT set, where seq orders the latest key change. Every HOT vertex
//     got its last key change from a message (an admission is always
//     followed by a message in the same sub-batch), so seq = index of the
//     vertex's latest message; LruPolicy picks the k smallest seq.
//   * RandomPolicy draws numpy PCG64 + Lemire bounded integers over a
//     swap-remove member list (reproduced here, pinned in tests).
// One CTA of 1024 threads runs the machine; every per-sub-batch step is a
// block-parallel pass (classification, ordered compaction with block
// scans, radix-select of victims over the hot list). Physical slot indices
// are not observable (A.2) and the accumulator records stay resident, so
// evict/reload only move state and byte counters (A.3).
#include <cub/cub.cuh>

#include "internal.cuh"

namespace atlas {
namespace {

constexpr int kThreads = 1024;
constexpr uint8_t NOT_STARTED = 0, HOT = 1, COLD = 2, COMPLETED = 3;
enum PassKind { PREPASS = 0, SELFPASS = 1, EDGEPASS = 2 };

using BlockScan = cub::BlockScan<int64_t, kThreads>;
using BlockReduce = cub::BlockReduce<int64_t, kThreads>;

struct EngineArgs {
  EngineState st;
  EngineScalars* sc;
  EngineConfig cfg;
  const uint64_t* runs;         // (cnt << 32) | local vertex, appearance order
  const int64_t* run_off;       // per chunk [c] .. [c+1]
  const int64_t* chunk_bounds;  // per chunk: start, end (global source ids)
  int64_t nchunks;
  int64_t* chunk_reloads;
  int64_t* chunk_touched;
  int64_t phys_slots;
  int32_t keep_chunk_grad;
  GridSync* gs;  // victim-selection jobs shared with the helper CTAs
  int64_t grid_min;  // sub-batches of at least this many elements run as
                     // grid jobs (when the launch has helper CTAs)
};

struct Smem {
  BlockScan::TempStorage scan;
  BlockReduce::TempStorage reduce;
  EngineScalars sc;
  uint32_t hist[256];
  int64_t bcast[4];
  int32_t err;
};

// ---- numpy PCG64 + Lemire bounded ints (Generator.integers(n)) ----------

__device__ __forceinline__ void pcg_step(EngineScalars& s) {
  const uint64_t MH = 2549297995355413924ull, ML = 4865540595714422341ull;
  // state = state * M + inc (mod 2^128)
  uint64_t lo = s.rng_state_lo * ML;
  uint64_t hi = __umul64hi(s.rng_state_lo, ML) + s.rng_state_lo * MH +
                s.rng_state_hi * ML;
  uint64_t nlo = lo + s.rng_inc_lo;
  hi += s.rng_inc_hi + (nlo < lo ? 1ull : 0ull);
  s.rng_state_lo = nlo;
  s.rng_state_hi = hi;
}

__device__ __forceinline__ uint64_t pcg_next64(EngineScalars& s) {
  pcg_step(s);
  uint64_t x = s.rng_state_hi ^ s.rng_state_lo;
  unsigned rot = (unsigned)(s.rng_state_hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__device__ __forceinline__ uint32_t pcg_next32(EngineScalars& s) {
  if (s.rng_has32) {
    s.rng_has32 = 0;
    return s.rng_u32;
  }
  uint64_t n = pcg_next64(s);
  s.rng_has32 = 1;
  s.rng_u32 = (uint32_t)(n >> 32);
  return (uint32_t)n;
}

__device__ uint64_t bounded_int(EngineScalars& s, uint64_t n) {
  const uint64_t rng = n - 1;
  if (rng == 0) return 0;
  const uint32_t excl = (uint32_t)n;
  uint64_t m = (uint64_t)pcg_next32(s) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    const uint32_t thr = (uint32_t)((0xFFFFFFFFull - rng) % excl);
    while (left < thr) {
      m = (uint64_t)pcg_next32(s) * excl;
      left = (uint32_t)m;
    }
  }
  return m >> 32;
}

// ---- helpers ------------------------------------------------------------

__device__ __forceinline__ uint64_t vkey(const EngineArgs& A, int32_t v) {
  const uint64_t sq = A.st.seq[v];
  if (A.cfg.policy == ATLAS_LRU) return sq;
  return ((uint64_t)A.st.pending[v] << 32) | sq;
}

__device__ void set_err(Smem& sm, int code, int64_t a, int64_t b) {
  if (atomicCAS(&sm.err, 0, code) == 0) {
    sm.sc.err = code;
    sm.sc.err_info[0] = a;
    sm.sc.err_info[1] = b;
  }
}

// Element accessors of a pass.
struct PassView {
  int kind;
  const uint64_t* runs;  // EDGEPASS
  const int32_t* list;   // PREPASS (explicit zeros list)
  int64_t first;         // SELFPASS: first local vertex
  __device__ __forceinline__ int32_t v(int64_t i) const {
    if (kind == EDGEPASS) return (int32_t)(uint32_t)runs[i];
    if (kind == PREPASS) return list[i];
    return (int32_t)(first + i);
  }
  __device__ __forceinline__ uint32_t cnt(int64_t i) const {
    if (kind == EDGEPASS) return (uint32_t)(runs[i] >> 32);
    return kind == SELFPASS ? 1u : 0u;
  }
};

// Ordered compaction of pass elements [0, n) satisfying pred into out[];
// returns the count (uniform across the block).
template <typename Pred>
__device__ int64_t compact(Smem& sm, int64_t n, Pred pred, int32_t* out) {
  int64_t base = 0;
  for (int64_t t0 = 0; t0 < n; t0 += kThreads) {
    const int64_t i = t0 + threadIdx.x;
    int32_t v = -1;
    int64_t f = 0;
    if (i < n) {
      v = pred(i);
      f = v >= 0 ? 1 : 0;
    }
    int64_t pos, total;
    BlockScan(sm.scan).ExclusiveSum(f, pos, total);
    if (f) out[base + pos] = v;
    base += total;
    __syncthreads();
  }
  return base;
}

__device__ int64_t block_sum(Smem& sm, int64_t x) {
  int64_t r = BlockReduce(sm.reduce).Sum(x);
  if (threadIdx.x == 0) sm.bcast[0] = r;
  __syncthreads();
  r = sm.bcast[0];
  __syncthreads();
  return r;
}

__device__ void log_push(int64_t* log, int64_t& n, int64_t cap, int64_t x,
                         int32_t& overflow) {
  if (n < cap) log[n] = x;
  else overflow = 1;
  n++;
}

// ---- grid jobs: scans of the hot list shared by all CTAs -------------

constexpr int kJobOr = 1, kJobHist = 2, kJobCollect = 3, kJobExit = 4;
// sub-batch jobs (large sub-batches only; the element order of every
// compaction is kept by per-CTA contiguous slices placed by their counts)
constexpr int kJobClassify = 5, kJobCount2 = 6, kJobWrite2 = 7,
              kJobAdmit = 8, kJobDeliver = 9, kJobCount0 = 10,
              kJobWrite0 = 11, kJobRelease = 12;

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}

__device__ __forceinline__ void warp_add(unsigned long long* dst, int64_t x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if ((threadIdx.x & 31) == 0 && x)
    atomicAdd(dst, (unsigned long long)x);
}

// this CTA's part of a sub-batch job (see GridSync)
__device__ void pass_slice(const EngineArgs& A, int type) {
  GridSync* gs = A.gs;
  const PassView P{gs->pkind, static_cast<const uint64_t*>(gs->pptr),
                   static_cast<const int32_t*>(gs->pptr), gs->pfirst};
  const int64_t lo = gs->lo, n = gs->n;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t first = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (type == kJobClassify) {
    int64_t need = 0, bad = 0;
    for (int64_t i = first; i < n; i += stride) {
      const uint8_t st = A.st.state[P.v(lo + i)];
      need += st != HOT;
      bad += st > COLD;
    }
    warp_add(&gs->sum[0], need);
    warp_add(&gs->sum[1], bad);
  } else if (type == kJobAdmit) {
    const int64_t ftop0 = gs->base;
    for (int64_t i = first; i < n; i += stride) {
      const int32_t v = gs->list[i];
      const int32_t slot = A.st.free_stack[ftop0 - 1 - i];
      A.st.state[v] = HOT;
      A.st.slot_of[v] = slot;
      A.st.hot_list[slot] = v;
      A.st.slot_key[slot] = vkey(A, v);
      if (gs->flag) A.st.unique_reloaded[v] = 1;
    }
  } else if (type == kJobDeliver) {
    int64_t msgs = 0, bad = 0;
    const uint64_t seq0 = (uint64_t)gs->base;
    for (int64_t i = first; i < n; i += stride) {
      const int32_t v = P.v(lo + i);
      const uint32_t c = P.cnt(lo + i);
      const uint32_t p = A.st.pending[v];
      if (p < c) {
        bad++;
        continue;
      }
      A.st.pending[v] = p - c;
      A.st.seq[v] = (uint32_t)(seq0 + (uint64_t)i);
      A.st.slot_key[A.st.slot_of[v]] = vkey(A, v);
      msgs += c;
    }
    warp_add(&gs->sum[0], msgs);
    warp_add(&gs->sum[1], bad);
  } else if (type == kJobRelease) {
    const int64_t ftop0 = gs->base;
    for (int64_t i = first; i < n; i += stride) {
      const int32_t v = gs->list[i];
      const int32_t slot = A.st.slot_of[v];
      A.st.state[v] = COMPLETED;
      A.st.slot_of[v] = -1;
      A.st.hot_list[slot] = -1;
      A.st.slot_key[slot] = ~0ull;
      A.st.free_stack[ftop0 + i] = slot;
      if (A.keep_chunk_grad) A.st.chunk_grad[gs->base2 + i] = v;
    }
  } else {
    // ordered compactions: CTA b owns elements [b*slice, (b+1)*slice)
    __shared__ BlockScan::TempStorage scan;
    __shared__ int64_t tot[2];
    const int64_t s0 = (int64_t)blockIdx.x * gs->slice;
    const int64_t s1 = min(n, s0 + gs->slice);
    const bool two = type == kJobCount2 || type == kJobWrite2;
    // predicate q of element i: 0 = fresh / done, 1 = cold
    auto pred = [&](int64_t i, int q) -> bool {
      const int32_t v = P.v(lo + i);
      if (!two) return A.st.pending[v] == 0;
      const uint8_t st = A.st.state[v];
      return q == 0 ? st == NOT_STARTED : st == COLD;
    };
    if (type == kJobCount2 || type == kJobCount0) {
      int64_t c[2] = {0, 0};
      for (int64_t i = s0 + threadIdx.x; i < s1; i += kThreads) {
        c[0] += pred(i, 0);
        if (two) c[1] += pred(i, 1);
      }
      if (threadIdx.x == 0) tot[0] = tot[1] = 0;
      __syncthreads();
      for (int q = 0; q < (two ? 2 : 1); q++) {
        int64_t x = c[q];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0 && x)
          atomicAdd(reinterpret_cast<unsigned long long*>(&tot[q]),
                    (unsigned long long)x);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        gs->cnt[blockIdx.x][0] = tot[0];
        gs->cnt[blockIdx.x][1] = tot[1];
      }
    } else {  // kJobWrite2 / kJobWrite0: place this slice's matches
      int64_t off[2] = {0, 0}, all0 = 0;
      for (int b = 0; b < (int)gridDim.x; b++) {
        const int64_t c0 = *reinterpret_cast<volatile int64_t*>(&gs->cnt[b][0]);
        const int64_t c1 = *reinterpret_cast<volatile int64_t*>(&gs->cnt[b][1]);
        if (b < (int)blockIdx.x) {
          off[0] += c0;
          off[1] += c1;
        }
        all0 += c0;
      }
      off[1] += all0;  // cold entries follow all fresh ones
      for (int q = 0; q < (two ? 2 : 1); q++) {
        int64_t base = off[q];
        for (int64_t t0 = s0; t0 < s1; t0 += kThreads) {
          const int64_t i = t0 + threadIdx.x;
          const int64_t f = (i < s1 && pred(i, q)) ? 1 : 0;
          int64_t pos, total;
          BlockScan(scan).ExclusiveSum(f, pos, total);
          if (f) gs->out[base + pos] = P.v(lo + i);
          base += total;
          __syncthreads();
        }
      }
    }
  }
  __syncthreads();
}

// this CTA's slices of the hot list (1024-entry blocks, round robin over
// the grid); OR of keys, 256-bin histogram of the masked-prefix keys, or
// the victims (keys <= prefix) appended through gs->nv
__device__ void job_slice(const EngineArgs& A, int type, int byte,
                          uint64_t prefix, uint64_t mask, int32_t* victims,
                          uint32_t* shist) {
  GridSync* gs = A.gs;
  if (type >= kJobClassify) {
    pass_slice(A, type);
    return;
  }
  if (type == kJobHist) {
    for (int j = threadIdx.x; j < 256; j += kThreads) shist[j] = 0;
    __syncthreads();
  }
  uint64_t o = 0;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  // keys by slot: a coalesced 8-byte read per slot (free slots hold ~0,
  // which no real key reaches: seq < 2^32, pending < 2^32)
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x;
       j < A.phys_slots; j += stride) {
    const uint64_t key = A.st.slot_key[j];
    if (key == ~0ull) continue;
    if (type == kJobOr) {
      o |= key;
    } else if (type == kJobHist) {
      if ((key & mask) == prefix)
        atomicAdd(&shist[(key >> (8 * byte)) & 255u], 1u);
    } else if (key <= prefix) {
      victims[atomicAdd(&gs->nv, 1)] = A.st.hot_list[j];
    }
  }
  if (type == kJobOr) {
    for (int s2 = 16; s2 > 0; s2 >>= 1) o |= __shfl_xor_sync(0xffffffffu, o, s2);
    if ((threadIdx.x & 31) == 0 && o)
      atomicOr(reinterpret_cast<unsigned long long*>(&gs->anybits),
               (unsigned long long)o);
  } else if (type == kJobHist) {
    __syncthreads();
    for (int j = threadIdx.x; j < 256; j += kThreads)
      if (shist[j]) atomicAdd(&gs->hist[j], shist[j]);
  }
  __syncthreads();
}

// CTA 0: post a job, take its own slice, wait for the helpers; returns
// the OR of keys (kJobOr) or the victim count (kJobCollect)
__device__ uint64_t grid_job(const EngineArgs& A, Smem& sm, int type,
                             int byte, uint64_t prefix, uint64_t mask,
                             int32_t* victims) {
  GridSync* gs = A.gs;
  const unsigned helpers = gridDim.x - 1;
  if (threadIdx.x == 0) {
    if (type == kJobOr) gs->anybits = 0;
    if (type == kJobCollect) gs->nv = 0;
    gs->type = type;
    gs->byte = byte;
    gs->prefix = prefix;
    gs->mask = mask;
  }
  if (type == kJobHist)
    for (int j = threadIdx.x; j < 256; j += kThreads) gs->hist[j] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&gs->job, 1u);  // publish
  }
  job_slice(A, type, byte, prefix, mask, victims, sm.hist);
  if (threadIdx.x == 0) {
    const unsigned want = helpers * ld_volatile(&gs->job);
    while (ld_volatile(&gs->done) < want) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
  uint64_t r = 0;
  if (type == kJobOr)
    r = *reinterpret_cast<const volatile uint64_t*>(&gs->anybits);
  else if (type == kJobCollect)
    r = (uint64_t)*reinterpret_cast<const volatile int32_t*>(&gs->nv);
  __syncthreads();
  return r;
}

// CTA 0: run a sub-batch job whose GridSync fields thread 0 has set
__device__ void pass_job(const EngineArgs& A, Smem& sm, int type) {
  GridSync* gs = A.gs;
  if (threadIdx.x == 0) {
    gs->type = type;
    if (type == kJobClassify || type == kJobDeliver)
      gs->sum[0] = gs->sum[1] = 0;
    __threadfence();
    atomicAdd(&gs->job, 1u);  // publish
  }
  __syncthreads();
  job_slice(A, type, 0, 0, 0, nullptr, sm.hist);
  if (threadIdx.x == 0) {
    const unsigned want = (gridDim.x - 1) * ld_volatile(&gs->job);
    while (ld_volatile(&gs->done) < want) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ int64_t gs_sum(const GridSync* gs, int k) {
  return (int64_t)*reinterpret_cast<const volatile unsigned long long*>(
      &gs->sum[k]);
}

// helper CTAs: run every posted job on their slices until kJobExit
__device__ void helper_loop(const EngineArgs& A) {
  __shared__ uint32_t shist[256];
  __shared__ unsigned posted;
  GridSync* gs = A.gs;
  unsigned seen = 0;
  while (true) {
    if (threadIdx.x == 0) {
      unsigned j;
      while ((j = ld_volatile(&gs->job)) == seen) __nanosleep(64);
      __threadfence();
      posted = j;
    }
    __syncthreads();
    seen = posted;
    const int type = *reinterpret_cast<const volatile int32_t*>(&gs->type);
    if (type == kJobExit) return;
    const int byte = *reinterpret_cast<const volatile int32_t*>(&gs->byte);
    const uint64_t prefix =
        *reinterpret_cast<const volatile uint64_t*>(&gs->prefix);
    const uint64_t mask = *reinterpret_cast<const volatile uint64_t*>(&gs->mask);
    job_slice(A, type, byte, prefix, mask, A.st.scratch_b, shist);
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&gs->done, 1u);
    }
  }
}

// evict(k) (oocgnn/memstore.py:397-411)
__device__ void evict(const EngineArgs& A, Smem& sm, int64_t k) {
  EngineScalars& s = sm.sc;
  if (k > s.hot_pop) k = s.hot_pop;
  if (k <= 0) return;
  int32_t* victims = A.st.scratch_b;
  if (A.cfg.policy == ATLAS_RND) {
    if (threadIdx.x == 0) {
      for (int64_t i = 0; i < k; i++) {
        const uint64_t idx = bounded_int(s, (uint64_t)s.rnd_n);
        // swap-remove (oocgnn/memstore.py:257-264)
        const int32_t last = A.st.rnd_members[s.rnd_n - 1];
        s.rnd_n--;
        int32_t victim;
        if ((int64_t)idx == s.rnd_n) {
          victim = last;
        } else {
          victim = A.st.rnd_members[idx];
          A.st.rnd_members[idx] = last;
          A.st.rnd_pos[last] = (int32_t)idx;
        }
        victims[i] = victim;
      }
    }
    __syncthreads();
  } else {
    // radix-select the k-th smallest key over the hot list; every scan
    // of the hot list is a grid job (all CTAs of the launch take slices)
    const uint64_t anybits = grid_job(A, sm, kJobOr, 0, 0, 0, victims);
    int top = 0;
    while (top < 7 && (anybits >> (8 * (top + 1))) != 0) top++;
    uint64_t prefix = 0, mask = 0;
    int64_t remaining = k;
    for (int byte = top; byte >= 0; byte--) {
      grid_job(A, sm, kJobHist, byte, prefix, mask, victims);
      if (threadIdx.x == 0) {
        int64_t cum = 0;
        int dd = 0;
        for (; dd < 256; dd++) {
          const uint32_t h = ld_volatile(&A.gs->hist[dd]);
          if (cum + h >= remaining) break;
          cum += h;
        }
        sm.bcast[2] = dd;
        sm.bcast[3] = remaining - cum;
      }
      __syncthreads();
      const uint64_t dd = (uint64_t)sm.bcast[2];
      remaining = sm.bcast[3];
      prefix |= dd << (8 * byte);
      mask |= 255ull << (8 * byte);
      __syncthreads();
    }
    // keys are unique: the victims are exactly the keys <= prefix
    const int64_t nv = (int64_t)grid_job(A, sm, kJobCollect, 0, prefix, 0,
                                         victims);
    if (threadIdx.x == 0 && nv != k) set_err(sm, ATLAS_EINVARIANT, nv, k);
    __syncthreads();
    if (sm.err) return;
  }
  // apply: HOT -> COLD, free the slot
  const int64_t ftop0 = s.free_top;
  for (int64_t i = threadIdx.x; i < k; i += kThreads) {
    const int32_t v = victims[i];
    const int32_t slot = A.st.slot_of[v];
    A.st.state[v] = COLD;
    A.st.slot_of[v] = -1;
    A.st.hot_list[slot] = -1;
    A.st.slot_key[slot] = ~0ull;
    A.st.free_stack[ftop0 + i] = slot;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s.free_top += k;
    s.hot_pop -= k;
    s.evictions += k;
    if (A.cfg.record_log) {
      int32_t of = 0;
      log_push(A.st.log_victims, s.log_victims_n, A.st.log_cap, -k, of);
      for (int64_t i = 0; i < k; i++) {
        const int32_t v = victims[i];
        log_push(A.st.log_victims, s.log_victims_n, A.st.log_cap, v, of);
        log_push(A.st.log_victims, s.log_victims_n, A.st.log_cap,
                 (int64_t)vkey(A, v), of);
      }
    }
  }
  __syncthreads();
}

// admit a compacted list (fresh or cold) in order (memstore.py:423-445)
__device__ void admit(const EngineArgs& A, Smem& sm, const int32_t* list,
                      int64_t n, bool reload) {
  if (n == 0) return;
  EngineScalars& s = sm.sc;
  const int64_t ftop0 = s.free_top;
  const int64_t rnd0 = s.rnd_n;
  for (int64_t i = threadIdx.x; i < n; i += kThreads) {
    const int32_t v = list[i];
    const int32_t slot = A.st.free_stack[ftop0 - 1 - i];
    A.st.state[v] = HOT;
    A.st.slot_of[v] = slot;
    A.st.hot_list[slot] = v;
    A.st.slot_key[slot] = vkey(A, v);
    if (reload) A.st.unique_reloaded[v] = 1;
    if (A.cfg.policy == ATLAS_RND) {
      A.st.rnd_members[rnd0 + i] = v;
      A.st.rnd_pos[v] = (int32_t)(rnd0 + i);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s.free_top -= n;
    s.hot_pop += n;
    s.admissions += n;
    if (A.cfg.policy == ATLAS_RND) s.rnd_n += n;
    if (s.hot_pop > s.hot_peak) s.hot_peak = s.hot_pop;
    if (s.hot_pop > A.cfg.slot_count) set_err(sm, ATLAS_EBUDGET, s.hot_pop, 0);
    if (reload) {
      s.reloads += n;
      if (A.cfg.record_log) {
        int32_t of = 0;
        log_push(A.st.log_reloads, s.log_reloads_n, A.st.log_cap, n, of);
        for (int64_t i = 0; i < n; i++)
          log_push(A.st.log_reloads, s.log_reloads_n, A.st.log_cap, list[i],
                   of);
      }
    }
  }
  __syncthreads();
}

// release a compacted list in order (memstore.py:479-494)
__device__ void release(const EngineArgs& A, Smem& sm, const int32_t* list,
                        int64_t n) {
  if (n == 0) return;
  EngineScalars& s = sm.sc;
  const int64_t ftop0 = s.free_top;
  for (int64_t i = threadIdx.x; i < n; i += kThreads) {
    const int32_t v = list[i];
    const int32_t slot = A.st.slot_of[v];
    A.st.state[v] = COMPLETED;
    A.st.slot_of[v] = -1;
    A.st.hot_list[slot] = -1;
    A.st.slot_key[slot] = ~0ull;
    A.st.free_stack[ftop0 + i] = slot;
    if (A.keep_chunk_grad) A.st.chunk_grad[s.chunk_grad_n + i] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (A.cfg.policy == ATLAS_RND) {
      for (int64_t i = 0; i < n; i++) {  // on_remove: swap-remove in order
        const int32_t v = list[i];
        const int32_t idx = A.st.rnd_pos[v];
        const int32_t last = A.st.rnd_members[s.rnd_n - 1];
        s.rnd_n--;
        if (idx != s.rnd_n) {
          A.st.rnd_members[idx] = last;
          A.st.rnd_pos[last] = idx;
        }
      }
    }
    s.free_top += n;
    s.hot_pop -= n;
    s.graduations += n;
    if (A.keep_chunk_grad) {
      s.chunk_grad_n += n;
      A.st.chunk_grad_batches[s.chunk_grad_batches_n++] = n;
    }
    if (A.cfg.record_log) {
      int32_t of = 0;
      log_push(A.st.log_grad, s.log_grad_n, A.st.log_cap, n, of);
      for (int64_t i = 0; i < n; i++)
        log_push(A.st.log_grad, s.log_grad_n, A.st.log_cap, list[i], of);
    }
  }
  __syncthreads();
}

// one sub-batch of a pass: ensure_hot_many + deliveries + graduation
// (orchestrator.py:177-212, memstore.py:447-477)
__device__ void sub_batch(const EngineArgs& A, Smem& sm, const PassView& P,
                          int64_t lo, int64_t n) {
  EngineScalars& s = sm.sc;
  // classify; evict until the non-hot part fits
  while (true) {
    int64_t need = 0, bad = 0;
    for (int64_t i = threadIdx.x; i < n; i += kThreads) {
      const uint8_t st = A.st.state[P.v(lo + i)];
      need += st != HOT;
      bad += st > COLD;
    }
    need = block_sum(sm, need);
    bad = block_sum(sm, bad);
    if (bad) {
      if (threadIdx.x == 0) set_err(sm, ATLAS_ESTATE, bad, 0);
      __syncthreads();
      return;
    }
    const int64_t free = A.cfg.slot_count - s.hot_pop;
    if (need <= free) break;
    if (need > A.cfg.slot_count) {
      if (threadIdx.x == 0) set_err(sm, ATLAS_ECONFIG, need, A.cfg.slot_count);
      __syncthreads();
      return;
    }
    while (A.cfg.slot_count - s.hot_pop < need) {
      const int64_t deficit = need - (A.cfg.slot_count - s.hot_pop);
      evict(A, sm, deficit > A.cfg.evict_batch ? deficit : A.cfg.evict_batch);
      if (sm.err) return;
    }
  }
  // admit fresh then reload cold, each in batch order
  const int64_t nf = compact(
      sm, n,
      [&](int64_t i) {
        const int32_t v = P.v(lo + i);
        return A.st.state[v] == NOT_STARTED ? v : -1;
      },
      A.st.scratch_a);
  const int64_t nc = compact(
      sm, n,
      [&](int64_t i) {
        const int32_t v = P.v(lo + i);
        return A.st.state[v] == COLD ? v : -1;
      },
      A.st.scratch_a + nf);
  admit(A, sm, A.st.scratch_a, nf, false);
  admit(A, sm, A.st.scratch_a + nf, nc, true);
  if (sm.err) return;
  if (P.kind == PREPASS) {
    release(A, sm, A.st.scratch_a, nf);  // zero-degree: straight out
    return;
  }
  // deliveries: pending -= cnt, seq = message index
  int64_t msgs = 0, bad = 0;
  for (int64_t i = threadIdx.x; i < n; i += kThreads) {
    const int32_t v = P.v(lo + i);
    const uint32_t c = P.cnt(lo + i);
    const uint32_t p = A.st.pending[v];
    if (p < c) {
      bad++;
      continue;
    }
    A.st.pending[v] = p - c;
    A.st.seq[v] = (uint32_t)(s.seq_ctr + (uint64_t)i);
    A.st.slot_key[A.st.slot_of[v]] = vkey(A, v);
    msgs += c;
  }
  msgs = block_sum(sm, msgs);
  bad = block_sum(sm, bad);
  if (bad) {
    if (threadIdx.x == 0) set_err(sm, ATLAS_ECONSISTENCY, bad, 0);
    __syncthreads();
    return;
  }
  if (threadIdx.x == 0) {
    s.messages += msgs;
    s.seq_ctr += (uint64_t)n;
  }
  __syncthreads();
  const int64_t nd = compact(
      sm, n,
      [&](int64_t i) {
        const int32_t v = P.v(lo + i);
        return A.st.pending[v] == 0 ? v : -1;
      },
      A.st.scratch_a);
  release(A, sm, A.st.scratch_a, nd);
}

// sub_batch() with every pass over the batch as a grid job (large
// sub-batches, MINPEND/LRU without logs): the same steps in the same order;
// compactions keep element order through per-CTA contiguous slices
__device__ void sub_batch_grid(const EngineArgs& A, Smem& sm,
                               const PassView& P, int64_t lo, int64_t n) {
  EngineScalars& s = sm.sc;
  GridSync* gs = A.gs;
  auto pass_fields = [&]() {
    if (threadIdx.x == 0) {
      gs->pkind = P.kind;
      gs->pptr = P.kind == EDGEPASS ? static_cast<const void*>(P.runs)
                                    : static_cast<const void*>(P.list);
      gs->pfirst = P.first;
      gs->lo = lo;
      gs->n = n;
      gs->slice = ((n + gridDim.x - 1) / gridDim.x + kThreads - 1) /
                  kThreads * kThreads;
      gs->out = A.st.scratch_a;
    }
  };
  auto counts = [&](int64_t& c0, int64_t& c1) {
    if (threadIdx.x == 0) {
      int64_t a = 0, b = 0;
      for (int k = 0; k < (int)gridDim.x; k++) {
        a += *reinterpret_cast<volatile int64_t*>(&gs->cnt[k][0]);
        b += *reinterpret_cast<volatile int64_t*>(&gs->cnt[k][1]);
      }
      sm.bcast[2] = a;
      sm.bcast[3] = b;
    }
    __syncthreads();
    c0 = sm.bcast[2];
    c1 = sm.bcast[3];
    __syncthreads();
  };
  // classify; evict until the non-hot part fits
  while (true) {
    pass_fields();
    pass_job(A, sm, kJobClassify);
    const int64_t need = gs_sum(gs, 0), bad = gs_sum(gs, 1);
    if (bad) {
      if (threadIdx.x == 0) set_err(sm, ATLAS_ESTATE, bad, 0);
      __syncthreads();
      return;
    }
    const int64_t free = A.cfg.slot_count - s.hot_pop;
    if (need <= free) break;
    if (need > A.cfg.slot_count) {
      if (threadIdx.x == 0) set_err(sm, ATLAS_ECONFIG, need, A.cfg.slot_count);
      __syncthreads();
      return;
    }
    while (A.cfg.slot_count - s.hot_pop < need) {
      const int64_t deficit = need - (A.cfg.slot_count - s.hot_pop);
      evict(A, sm, deficit > A.cfg.evict_batch ? deficit : A.cfg.evict_batch);
      if (sm.err) return;
    }
  }
  // fresh then cold, each in batch order, into scratch_a
  pass_fields();
  pass_job(A, sm, kJobCount2);
  int64_t nf, nc;
  counts(nf, nc);
  pass_job(A, sm, kJobWrite2);
  for (int r = 0; r < 2; r++) {
    const int64_t m = r ? nc : nf;
    if (m == 0) continue;
    if (threadIdx.x == 0) {
      gs->list = A.st.scratch_a + (r ? nf : 0);
      gs->n = m;
      gs->base = s.free_top;
      gs->flag = r;
    }
    pass_job(A, sm, kJobAdmit);
    if (threadIdx.x == 0) {
      s.free_top -= m;
      s.hot_pop += m;
      s.admissions += m;
      if (s.hot_pop > s.hot_peak) s.hot_peak = s.hot_pop;
      if (s.hot_pop > A.cfg.slot_count) set_err(sm, ATLAS_EBUDGET, s.hot_pop, 0);
      if (r) s.reloads += m;
    }
    __syncthreads();
    if (sm.err) return;
  }
  // deliveries: pending -= cnt, seq = message index
  pass_fields();
  if (threadIdx.x == 0) gs->base = (int64_t)s.seq_ctr;
  pass_job(A, sm, kJobDeliver);
  const int64_t msgs = gs_sum(gs, 0), bad = gs_sum(gs, 1);
  if (bad) {
    if (threadIdx.x == 0) set_err(sm, ATLAS_ECONSISTENCY, bad, 0);
    __syncthreads();
    return;
  }
  if (threadIdx.x == 0) {
    s.messages += msgs;
    s.seq_ctr += (uint64_t)n;
  }
  __syncthreads();
  // graduation: pending == 0 in batch order
  pass_fields();
  pass_job(A, sm, kJobCount0);
  int64_t nd, unused;
  counts(nd, unused);
  pass_job(A, sm, kJobWrite0);
  if (nd == 0) return;
  if (threadIdx.x == 0) {
    gs->list = A.st.scratch_a;
    gs->n = nd;
    gs->base = s.free_top;
    gs->base2 = s.chunk_grad_n;
  }
  pass_job(A, sm, kJobRelease);
  if (threadIdx.x == 0) {
    s.free_top += nd;
    s.hot_pop -= nd;
    s.graduations += nd;
    if (A.keep_chunk_grad) {
      s.chunk_grad_n += nd;
      A.st.chunk_grad_batches[s.chunk_grad_batches_n++] = nd;
    }
  }
  __syncthreads();
}

__device__ int64_t run_pass(const EngineArgs& A, Smem& sm, const PassView& P,
                            int64_t n) {
  const bool grid_ok = gridDim.x > 1 && P.kind != PREPASS &&
                       A.cfg.policy != ATLAS_RND && !A.cfg.record_log;
  for (int64_t lo = 0; lo < n && !sm.err; lo += A.cfg.sub_batch) {
    const int64_t m = min(A.cfg.sub_batch, n - lo);
    if (grid_ok && m >= A.grid_min) sub_batch_grid(A, sm, P, lo, m);
    else sub_batch(A, sm, P, lo, m);
  }
  return n;
}

__global__ void __launch_bounds__(kThreads, 1) engine_kernel(EngineArgs A) {
  if (blockIdx.x != 0) {
    helper_loop(A);
    return;
  }
  __shared__ Smem sm;
  if (threadIdx.x == 0) {
    sm.sc = *A.sc;
    sm.err = 0;
    sm.sc.chunk_grad_n = 0;
    sm.sc.chunk_grad_batches_n = 0;
  }
  __syncthreads();
  if (sm.sc.err) return;
  EngineScalars& s = sm.sc;
  for (int64_t c = 0; c < A.nchunks && !sm.err; c++) {
    const int64_t start = A.chunk_bounds[2 * c], end = A.chunk_bounds[2 * c + 1];
    const int64_t a = max(start, A.cfg.lo) - A.cfg.lo;
    const int64_t b = min(end, A.cfg.hi) - A.cfg.lo;
    const int64_t reloads0 = s.reloads;
    int64_t touched = 0;
    if (A.cfg.model == ATLAS_GCN && b > a) {
      // sources nobody points at graduate as zeros (orchestrator.py:234-241);
      // the list lives past the victim area of scratch_b (evict() reuses
      // scratch_b[0, hot_pop))
      int32_t* zl = A.st.scratch_b + A.phys_slots + kThreads;
      const int64_t nz = compact(
          sm, b - a,
          [&](int64_t i) {
            const int32_t v = (int32_t)(a + i);
            return (A.st.state[v] == NOT_STARTED && A.st.pending[v] == 0)
                       ? v
                       : -1;
          },
          zl);
      PassView P{PREPASS, nullptr, zl, 0};
      run_pass(A, sm, P, nz);
    }
    if (A.cfg.model == ATLAS_SAGE && b > a && !sm.err) {
      PassView P{SELFPASS, nullptr, nullptr, a};
      touched += run_pass(A, sm, P, b - a);
    }
    if (!sm.err) {
      const int64_t r0 = A.run_off[c], r1 = A.run_off[c + 1];
      PassView P{EDGEPASS, A.runs + r0, nullptr, 0};
      touched += run_pass(A, sm, P, r1 - r0);
    }
    if (threadIdx.x == 0) {
      A.chunk_reloads[c] = s.reloads - reloads0;
      A.chunk_touched[c] = touched;
      s.chunk_index++;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (sm.err) s.err = sm.err;
    *A.sc = s;
    if (gridDim.x > 1) {  // release the helpers
      A.gs->type = kJobExit;
      __threadfence();
      atomicAdd(&A.gs->job, 1u);
    }
  }
}

__global__ void init_state(uint32_t* pending, uint8_t* state, uint32_t* seq,
                           int32_t* slot_of, uint8_t* unique_reloaded,
                           const uint32_t* indeg, int64_t nloc, int self_term,
                           int64_t* first_pos, int64_t* last_pos) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i < nloc; i += (int64_t)gridDim.x * blockDim.x) {
    pending[i] = indeg[i] + (self_term ? 1u : 0u);
    state[i] = NOT_STARTED;
    seq[i] = 0;
    slot_of[i] = -1;
    unique_reloaded[i] = 0;
    first_pos[i] = -1;
    last_pos[i] = -1;
  }
}

__global__ void init_slots(int32_t* hot_list, uint64_t* slot_key,
                           int32_t* free_stack, int64_t phys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i < phys; i += (int64_t)gridDim.x * blockDim.x) {
    hot_list[i] = -1;
    slot_key[i] = ~0ull;
    free_stack[i] = (int32_t)(phys - 1 - i);
  }
}

unsigned grid_of(int64_t n) {
  int64_t g = ceil_div(n, 256);
  if (g > num_sms() * 8) g = num_sms() * 8;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

int64_t phys_slots_of(const atlas_layer* L) {
  return std::max<int64_t>(1, std::min<int64_t>(L->desc.slot_count, L->nloc));
}

__global__ void set_scalars(EngineScalars* dst, EngineScalars v) { *dst = v; }

void engine_init(atlas_layer* L, cudaStream_t s) {
  L->spans_queued = false;
  const int64_t n = L->nloc;
  const int64_t phys = phys_slots_of(L);
  const int64_t nn = n > 0 ? n : 1;
  L->pending.alloc(nn);
  L->state.alloc(nn);
  L->seq.alloc(nn);
  L->slot_of.alloc(nn);
  L->unique_reloaded.alloc(nn);
  L->first_pos.alloc(nn);
  L->last_pos.alloc(nn);
  L->hot_list.alloc(phys);
  L->slot_key.alloc(phys);
  L->free_stack.alloc(phys);
  L->scratch_a.alloc(std::max(phys, nn) + kThreads);
  L->scratch_b.alloc(phys + kThreads + nn + kThreads);
  L->chunk_grad.alloc(nn);
  L->chunk_grad_batches.alloc(nn + 1);
  if (L->desc.policy == ATLAS_RND) {
    L->rnd_members.alloc(nn);
    L->rnd_pos.alloc(nn);
  }
  L->scalars.alloc(1);
  if (n > 0) {
    init_state<<<grid_of(n), 256, 0, s>>>(
        L->pending.ptr, L->state.ptr, L->seq.ptr, L->slot_of.ptr,
        L->unique_reloaded.ptr, L->indeg.ptr, n,
        L->desc.model != ATLAS_GCN, L->first_pos.ptr, L->last_pos.ptr);
    count_launch();
    ATLAS_LAUNCH_CHECK();
  }
  init_slots<<<grid_of(phys), 256, 0, s>>>(L->hot_list.ptr, L->slot_key.ptr,
                                           L->free_stack.ptr, phys);
  count_launch();
  ATLAS_LAUNCH_CHECK();
  EngineScalars sc{};
  sc.free_top = phys;
  sc.rng_state_hi = L->desc.rnd_state[0];
  sc.rng_state_lo = L->desc.rnd_state[1];
  sc.rng_inc_hi = L->desc.rnd_state[2];
  sc.rng_inc_lo = L->desc.rnd_state[3];
  // by value through the launch: no staging buffer, no host wait (a
  // topology refresh re-arms every layer while the device still works)
  set_scalars<<<1, 1, 0, s>>>(L->scalars.ptr, sc);
  count_launch();
  ATLAS_LAUNCH_CHECK();
  L->engine_initialized = true;
}

static void grow_log(DevBuf<int64_t>& buf, int64_t used, int64_t need,
                     cudaStream_t s) {
  if ((int64_t)buf.count >= need) return;
  DevBuf<int64_t> nb;
  nb.alloc(std::max<int64_t>(need, 2 * buf.count));
  if (used > 0)
    ATLAS_CUDA(cudaMemcpyAsync(nb.ptr, buf.ptr, used * sizeof(int64_t),
                               cudaMemcpyDeviceToDevice, s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
  std::swap(buf.ptr, nb.ptr);
  std::swap(buf.count, nb.count);
}

EngineScalars read_scalars(atlas_layer* L, cudaStream_t s) {
  L->pin_scalars.reserve(1);
  ATLAS_CUDA(cudaMemcpyAsync(L->pin_scalars.ptr, L->scalars.ptr,
                             sizeof(EngineScalars), cudaMemcpyDeviceToHost,
                             s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
  return *L->pin_scalars.ptr;
}

void engine_run_chunks(atlas_layer* L, const uint64_t* runs,
                       const int64_t* run_off, const int64_t* chunk_bounds,
                       int64_t nchunks, const int64_t* host_run_off,
                       cudaStream_t s) {
  if (!L->engine_initialized) engine_init(L, s);
  const int64_t nruns = host_run_off[nchunks] - host_run_off[0];
  // per-chunk counters land in a device buffer then append to the host copy
  DevBuf<int64_t> stats;
  stats.alloc(2 * std::max<int64_t>(nchunks, 1));
  if (L->desc.record_log) {
    EngineScalars cur = read_scalars(L, s);
    // every delivery can cost at most one eviction and one reload record
    const int64_t extra = 4 * (nruns + L->nloc) + 64;
    grow_log(L->log_victims, cur.log_victims_n, cur.log_victims_n + 2 * extra, s);
    grow_log(L->log_reloads, cur.log_reloads_n, cur.log_reloads_n + extra, s);
    grow_log(L->log_grad, cur.log_grad_n, cur.log_grad_n + extra, s);
  }
  EngineArgs A{};
  A.st.pending = L->pending.ptr;
  A.st.state = L->state.ptr;
  A.st.seq = L->seq.ptr;
  A.st.slot_of = L->slot_of.ptr;
  A.st.unique_reloaded = L->unique_reloaded.ptr;
  A.st.hot_list = L->hot_list.ptr;
  A.st.slot_key = L->slot_key.ptr;
  A.st.free_stack = L->free_stack.ptr;
  A.st.scratch_a = L->scratch_a.ptr;
  A.st.scratch_b = L->scratch_b.ptr;
  A.st.rnd_members = L->rnd_members.ptr;
  A.st.rnd_pos = L->rnd_pos.ptr;
  A.st.log_victims = L->log_victims.ptr;
  A.st.log_reloads = L->log_reloads.ptr;
  A.st.log_grad = L->log_grad.ptr;
  A.st.log_cap = (int64_t)std::min(
      L->log_victims.count, std::min(L->log_reloads.count, L->log_grad.count));
  A.st.chunk_grad = L->chunk_grad.ptr;
  A.st.chunk_grad_batches = L->chunk_grad_batches.ptr;
  A.sc = L->scalars.ptr;
  A.cfg.lo = L->desc.dst_lo;
  A.cfg.hi = L->desc.dst_hi;
  A.cfg.nloc = L->nloc;
  A.cfg.slot_count = L->desc.slot_count;
  A.cfg.evict_batch = L->evict_batch;
  A.cfg.sub_batch = L->sub_batch;
  A.cfg.model = L->desc.model;
  A.cfg.policy = L->desc.policy;
  A.cfg.record_log = L->desc.record_log;
  A.runs = runs;
  A.run_off = run_off;
  A.chunk_bounds = chunk_bounds;
  A.nchunks = nchunks;
  A.chunk_reloads = stats.ptr;
  A.chunk_touched = stats.ptr + std::max<int64_t>(nchunks, 1);
  A.phys_slots = phys_slots_of(L);
  A.keep_chunk_grad = nchunks == 1 ? 1 : 0;
  // helper CTAs share the victim scans; a cooperative launch guarantees
  // they are co-resident with CTA 0 (which spins on them). Scans of a
  // small hot list stay on CTA 0.
  L->grid_sync.reserve(1);
  ATLAS_CUDA(cudaMemsetAsync(L->grid_sync.ptr, 0, sizeof(GridSync), s));
  A.gs = L->grid_sync.ptr;
  // ATLAS_ENGINE_GRID_MIN (tests): smallest sub-batch run as grid jobs
  static const int64_t grid_min = [] {
    const char* e = getenv("ATLAS_ENGINE_GRID_MIN");
    return e ? std::max<int64_t>(1, atoll(e)) : (int64_t)16384;
  }();
  A.grid_min = grid_min;
  int grid = 1;
  if ((A.phys_slots > 8 * kThreads || grid_min < 16384) &&
      L->desc.policy != ATLAS_RND) {
    int dev = 0, sms = 0, coop = 0, per_sm = 0;
    ATLAS_CUDA(cudaGetDevice(&dev));
    ATLAS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount,
                                      dev));
    ATLAS_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch,
                                      dev));
    ATLAS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, engine_kernel, kThreads, 0));
    const int64_t want = std::max<int64_t>(
        ceil_div(A.phys_slots, 4 * kThreads), grid_min < 16384 ? 8 : 1);
    if (coop && per_sm > 0)
      grid = (int)std::max<int64_t>(
          1, std::min<int64_t>(std::min<int64_t>(want, (int64_t)sms * per_sm),
                               64));
  }
  if (grid > 1) {
    void* args[] = {&A};
    ATLAS_CUDA(cudaLaunchCooperativeKernel((const void*)engine_kernel,
                                           dim3(grid), dim3(kThreads), args,
                                           0, s));
  } else {
    engine_kernel<<<1, kThreads, 0, s>>>(A);
  }
  count_launch();
  ATLAS_LAUNCH_CHECK();
  std::vector<int64_t> h(2 * std::max<int64_t>(nchunks, 1));
  ATLAS_CUDA(cudaMemcpyAsync(h.data(), stats.ptr, h.size() * sizeof(int64_t),
                             cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
  for (int64_t c = 0; c < nchunks; c++) {
    L->chunk_reloads.push_back(h[c]);
    L->chunk_touched.push_back(h[std::max<int64_t>(nchunks, 1) + c]);
  }
  check_engine_error(L, s);
}

void check_engine_error(atlas_layer* L, cudaStream_t s) {
  EngineScalars sc = read_scalars(L, s);
  if (!sc.err) return;
  switch (sc.err) {
    case ATLAS_ESTATE:
      fail(ATLAS_ESTATE, "completed vertices offered messages (" +
                             std::to_string(sc.err_info[0]) + ")");
    case ATLAS_ECONSISTENCY:
      fail(ATLAS_ECONSISTENCY, "more deliveries than pending for " +
                                   std::to_string(sc.err_info[0]) +
                                   " vertices");
    case ATLAS_ECONFIG:
      fail(ATLAS_ECONFIG, "batch of " + std::to_string(sc.err_info[0]) +
                              " cannot fit in " +
                              std::to_string(sc.err_info[1]) + " slots");
    case ATLAS_EBUDGET:
      fail(ATLAS_EBUDGET, "hot population " + std::to_string(sc.err_info[0]) +
                              " exceeds the slot budget");
    default:
      fail(sc.err, "control engine invariant broken (" +
                       std::to_string(sc.err_info[0]) + ", " +
                       std::to_string(sc.err_info[1]) + ")");
  }
}

}  // namespace atlas
