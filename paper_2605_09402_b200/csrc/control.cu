// Whole-layer control plane over the resident CSC view.
//
// Stream positions (the reference's ctx.step, oocgnn/orchestrator.py:
// 224-277) are closed-form in CSR coordinates for a chunk plan of R rows
// (chunk c = [s_c, e_c), s_c = cR, e_c = min(s_c + R, V)):
//   GCN : edge j (source u)  -> j
//   SAGE: self term of v     -> off[s_c(v)] + v ;  edge j -> j + e_c(u)
//   GIN : self term of v     -> off[v] + v      ;  edge j -> j + u + 1
// so first/last steps (spans), per-chunk destination runs (P_c) and the
// (chunk, pass) at which each destination is first admitted and finally
// graduated all come from ONE parallel walk of every destination's
// ascending source list. If no pass is split into sub-batches and the
// eviction-free hot-population trajectory never exceeds the slot budget,
// the reference machine provably never evicts; its integer results are
// then exactly these closed forms (the "fast path"). Otherwise the
// per-chunk destination runs are materialised in first-appearance order
// (flag at the run's first stream position + ordered compaction) and the
// exact engine (engine.cu) replays the machine.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>

#include "internal.cuh"

namespace atlas {

EngineScalars read_scalars(atlas_layer* L, cudaStream_t s);
int64_t phys_slots_of(const atlas_layer* L);

namespace {

constexpr uint64_t kNoRun = ~0ull;

struct Plan {
  int64_t R, V, nchunks;
  __device__ __forceinline__ int64_t chunk(int64_t u) const { return u / R; }
  __device__ __forceinline__ int64_t start(int64_t c) const { return c * R; }
  __device__ __forceinline__ int64_t end(int64_t c) const {
    return min((c + 1) * R, V);
  }
};

// position of an edge (CSR index j, source u) in the reference stream
__device__ __forceinline__ int64_t edge_pos(int model, const Plan& p,
                                            int64_t j, int64_t u) {
  if (model == ATLAS_GCN) return j;
  if (model == ATLAS_SAGE) return j + p.end(p.chunk(u));
  return j + u + 1;
}

__device__ __forceinline__ int64_t self_pos(int model, const Plan& p,
                                            const int64_t* off, int64_t v) {
  if (model == ATLAS_SAGE) return off[p.start(p.chunk(v))] + v;
  return off[v] + v;  // GIN
}

// Histogram [admit 3C | grad 3C | runs C]: per-block shared-memory copy
// when it fits (keys concentrate on few chunks, so global atomics would
// serialise), flushed once per block.
struct Hist {
  unsigned long long* g;
  unsigned int* s;  // nullptr -> global atomics
  __device__ __forceinline__ void add(int64_t i, unsigned n) const {
    if (s) atomicAdd(s + i, n);
    else atomicAdd(g + i, (unsigned long long)n);
  }
};

// warp-aggregated add of 1 to h[base + key] for lanes with pred
__device__ __forceinline__ void agg_inc(const Hist& h, int64_t base,
                                        int64_t key, bool pred) {
  const unsigned act = __ballot_sync(0xffffffffu, pred);
  if (!pred) return;
  const unsigned peers = __match_any_sync(act, (unsigned long long)key);
  const int leader = __ffs(peers) - 1;
  if ((int)(threadIdx.x & 31) == leader) h.add(base + key, __popc(peers));
}

// first/last stream step of v and the (chunk * 3 + pass) keys of its
// first admission and its graduation
__device__ __forceinline__ void dest_summary(
    int model, const Plan& p, const int64_t* __restrict__ off,
    const uint32_t* __restrict__ csc_src, const uint32_t* __restrict__ csc_eid,
    int64_t v, int64_t vg, int64_t beg, int64_t end,
    int64_t* __restrict__ first_pos, int64_t* __restrict__ last_pos,
    const Hist& h, int64_t A0, int64_t G0) {
  const int64_t cv = p.chunk(vg);
  int64_t first = -1, last = -1;
  int64_t a_key = 0, g_key = 0;
  if (end > beg) {
    const int64_t u0 = csc_src[beg], u1 = csc_src[end - 1];
    first = edge_pos(model, p, csc_eid[beg], u0);
    last = edge_pos(model, p, csc_eid[end - 1], u1);
    a_key = p.chunk(u0) * 3 + 2;
    g_key = p.chunk(u1) * 3 + 2;
  }
  if (model != ATLAS_GCN) {
    const int64_t sp = self_pos(model, p, off, vg);
    const int64_t sk = cv * 3 + (model == ATLAS_SAGE ? 1 : 2);
    if (end > beg) {
      first = min(first, sp);
      last = max(last, sp);
      a_key = min(a_key, sk);
      g_key = max(g_key, sk);
    } else {
      first = last = sp;
      a_key = g_key = sk;
    }
  } else if (end == beg) {
    a_key = g_key = cv * 3 + 0;  // GCN zero in-degree pre-pass
  }
  first_pos[v] = first;
  last_pos[v] = last;
  h.add(A0 + a_key, 1u);
  h.add(G0 + g_key, 1u);
}

// thread per destination when no run counting is needed
__global__ void __launch_bounds__(256)
    walk_light(int model, Plan p, const int64_t* __restrict__ off,
               const int64_t* __restrict__ csc_ptr,
               const uint32_t* __restrict__ csc_src,
               const uint32_t* __restrict__ csc_eid, int64_t lo, int64_t nloc,
               int64_t* __restrict__ first_pos, int64_t* __restrict__ last_pos,
               unsigned long long* __restrict__ ghist, int use_smem) {
  extern __shared__ unsigned int shist[];
  const int64_t hn = 7 * p.nchunks;
  Hist h{ghist, use_smem ? shist : nullptr};
  if (use_smem) {
    for (int64_t i = threadIdx.x; i < hn; i += blockDim.x) shist[i] = 0;
    __syncthreads();
  }
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nloc;
       v += (int64_t)gridDim.x * blockDim.x)
    dest_summary(model, p, off, csc_src, csc_eid, v, v + lo, csc_ptr[v],
                 csc_ptr[v + 1], first_pos, last_pos, h, 0, 3 * p.nchunks);
  if (use_smem) {
    __syncthreads();
    for (int64_t i = threadIdx.x; i < hn; i += blockDim.x)
      if (shist[i]) atomicAdd(ghist + i, (unsigned long long)shist[i]);
  }
}

// One warp per local destination: spans, admission / graduation
// (chunk, pass), per-chunk run counts and (optionally) run records.
__global__ void __launch_bounds__(256)
    walk_destinations(int model, Plan p, const int64_t* __restrict__ off,
                      const int64_t* __restrict__ csc_ptr,
                      const uint32_t* __restrict__ csc_src,
                      const uint32_t* __restrict__ csc_eid, int64_t lo,
                      int64_t nloc, int64_t* __restrict__ first_pos,
                      int64_t* __restrict__ last_pos,
                      unsigned long long* __restrict__ ghist, int use_smem,
                      uint64_t* __restrict__ run_at_pos, int count_runs) {
  extern __shared__ unsigned int shist[];
  const int64_t hn = 7 * p.nchunks;
  Hist h{ghist, use_smem ? shist : nullptr};
  if (use_smem) {
    for (int64_t i = threadIdx.x; i < hn; i += blockDim.x) shist[i] = 0;
    __syncthreads();
  }
  const int64_t A0 = 0, G0 = 3 * p.nchunks, R0 = 6 * p.nchunks;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
       v < nloc; v += nwarps) {
  const int64_t vg = v + lo;
  const int64_t beg = csc_ptr[v], end = csc_ptr[v + 1];

  const int64_t cv = p.chunk(vg);
  // ---- spans and admit/grad (chunk, pass) --------------------------------
  if (lane == 0)
    dest_summary(model, p, off, csc_src, csc_eid, v, vg, beg, end, first_pos,
                 last_pos, h, A0, G0);
  // ---- runs: maximal same-chunk stretches of the ascending source list ---
  bool self_merged = false;  // GIN self term joins the run of chunk cv
  for (int64_t base = beg; count_runs && base < end; base += 32) {
    const int64_t i = base + lane;
    const bool in = i < end;
    int64_t u = 0, c = -1;
    if (in) {
      u = csc_src[i];
      c = p.chunk(u);
    }
    int64_t prev_c = __shfl_up_sync(0xffffffffu, c, 1);
    const int64_t carry = (base > beg) ? p.chunk((int64_t)csc_src[base - 1]) : -2;
    if (lane == 0) prev_c = carry;
    const bool starts = in && c != prev_c;
    if (model == ATLAS_GIN && __any_sync(0xffffffffu, in && c == cv))
      self_merged = true;
    agg_inc(h, R0, c, starts);
    if (run_at_pos && starts) {
      // run [i, j): count its entries; GIN adds the self term
      int64_t j = i + 1;
      while (j < end && p.chunk((int64_t)csc_src[j]) == c) j++;
      uint64_t cnt = (uint64_t)(j - i);
      int64_t pos = edge_pos(model, p, csc_eid[i], u);
      if (model == ATLAS_GIN && c == cv) {
        cnt += 1;
        pos = min(pos, self_pos(model, p, off, vg));
      }
      run_at_pos[pos] = (cnt << 32) | (uint64_t)(uint32_t)v;
    }
  }
  if (model == ATLAS_GIN && !self_merged && lane == 0) {
    h.add(R0 + cv, 1u);
    if (run_at_pos)
      run_at_pos[self_pos(model, p, off, vg)] =
          (1ull << 32) | (uint64_t)(uint32_t)v;
  }
  }  // destinations
  if (use_smem) {
    __syncthreads();
    for (int64_t i = threadIdx.x; i < hn; i += blockDim.x)
      if (shist[i]) atomicAdd(ghist + i, (unsigned long long)shist[i]);
  }
}

// m_c = edges of reference chunk c (whole graph, CSR offsets)
__global__ void chunk_edges(const int64_t* __restrict__ off, Plan p,
                            int64_t* __restrict__ m) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; c < p.nchunks; c += (int64_t)gridDim.x * blockDim.x)
    m[c] = off[p.end(c)] - off[p.start(c)];
}

__global__ void fill_u64(uint64_t* p, int64_t n, uint64_t val) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = val;
}

__global__ void span_values(const int64_t* first, const int64_t* last,
                            int64_t n, int64_t* spans,
                            unsigned long long* sum_count,
                            int64_t sentinel = INT64_MAX) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t my_sum = 0, my_cnt = 0;
  for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool got = first[i] >= 0;
    spans[i] = got ? last[i] - first[i] : sentinel;
    if (got) {
      my_sum += last[i] - first[i];
      my_cnt++;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    my_sum += __shfl_xor_sync(0xffffffffu, my_sum, o);
    my_cnt += __shfl_xor_sync(0xffffffffu, my_cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(sum_count, (unsigned long long)my_sum);
    atomicAdd(sum_count + 1, (unsigned long long)my_cnt);
  }
}

struct NotNoRun {
  __device__ bool operator()(const uint64_t& x) const { return x != kNoRun; }
};

unsigned grid_of(int64_t n, int block = 256) {
  int64_t g = ceil_div(n, block);
  if (g > num_sms() * 16) g = num_sms() * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

// spans -> exact integer sum, count and the two order statistics that
// np.percentile(spans, 99) interpolates between.
// sum, count and the two order statistics np.percentile(spans, 99)
// interpolates between (numpy 'linear': virtual index (count - 1) * 0.99)
__global__ void span_pick(const unsigned long long* sum_count,
                          const int64_t* sorted, int64_t* out) {
  const int64_t cnt = (int64_t)sum_count[1];
  out[0] = (int64_t)sum_count[0];
  out[1] = cnt;
  out[2] = out[3] = 0;
  if (cnt > 0) {
    const double vi = (double)(cnt - 1) * 0.99;
    const int64_t lo_i = (int64_t)floor(vi);
    const int64_t hi_i = min(lo_i + 1, cnt - 1);
    out[2] = sorted[lo_i];
    out[3] = sorted[hi_i];
  }
}

// The two order statistics by MSB-first radix select instead of a sort:
// per digit (<= 10 bits) one histogram pass over the spans whose higher
// digits match each rank's prefix, then one block turns the histograms
// into the next digit and the rank within it. The kernels hold 8 KB of
// shared memory and a few registers, so they co-reside with the
// persistent aggregation grid on the data stream (a device radix sort's
// passes could not, and queued behind it as the layer's control tail).
struct SpanSel {
  long long pre[2];  // selected high digits of rank lo_i / hi_i
  long long k[2];    // rank within the current prefix
};
constexpr int kSelMaxBits = 10;

__global__ void span_sel_init(const unsigned long long* __restrict__ sc,
                              SpanSel* __restrict__ st,
                              unsigned* __restrict__ hist) {
  const long long cnt = (long long)sc[1];
  if (threadIdx.x == 0) {
    long long lo_i = 0, hi_i = 0;
    if (cnt > 0) {
      const double vi = (double)(cnt - 1) * 0.99;
      lo_i = (long long)floor(vi);
      hi_i = lo_i + 1 < cnt ? lo_i + 1 : cnt - 1;
    }
    st->pre[0] = st->pre[1] = 0;
    st->k[0] = lo_i;
    st->k[1] = hi_i;
  }
  for (int i = threadIdx.x; i < 2 << kSelMaxBits; i += blockDim.x) hist[i] = 0;
}

__global__ void __launch_bounds__(256)
    span_sel_hist(const int64_t* __restrict__ spans, int64_t n,
                  int64_t sentinel, const SpanSel* __restrict__ st, int shift,
                  int width, unsigned* __restrict__ hist) {
  __shared__ unsigned h[2 << kSelMaxBits];
  const int nb = 1 << width;
  for (int i = threadIdx.x; i < 2 * nb; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const long long p0 = st->pre[0], p1 = st->pre[1];
  const int hs = shift + width;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const long long key = spans[i];
    if (key == sentinel) continue;
    const long long top = hs >= 63 ? 0 : key >> hs;
    const int bin = (int)((key >> shift) & (nb - 1));
    if (top == p0) atomicAdd(&h[bin], 1u);
    if (top == p1) atomicAdd(&h[nb + bin], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * nb; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// one block of 1024 threads: bin t of each rank's histogram
__global__ void __launch_bounds__(1024)
    span_sel_pick(SpanSel* __restrict__ st, unsigned* __restrict__ hist,
                  int width) {
  __shared__ unsigned long long part[32];
  const int nb = 1 << width, t = threadIdx.x;
  for (int r = 0; r < 2; r++) {
    const unsigned c = t < nb ? hist[r * nb + t] : 0u;
    // block exclusive scan of the bin counts
    unsigned long long x = c;
    const int lane = t & 31, w = t >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) part[w] = x;
    __syncthreads();
    if (w == 0) {
      unsigned long long q = part[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, q, o);
        if (lane >= o) q += y;
      }
      part[lane] = q;  // inclusive over warps
    }
    __syncthreads();
    const unsigned long long excl = x - c + (w ? part[w - 1] : 0ull);
    const long long k = st->k[r];
    if (c && (long long)excl <= k && k < (long long)(excl + c)) {
      st->pre[r] = (st->pre[r] << width) | t;
      st->k[r] = k - (long long)excl;
    }
    __syncthreads();
  }
  for (int i = t; i < 2 * nb; i += blockDim.x) hist[i] = 0;
}

__global__ void span_sel_out(const unsigned long long* __restrict__ sc,
                             const SpanSel* __restrict__ st,
                             int64_t* __restrict__ out) {
  const int64_t cnt = (int64_t)sc[1];
  out[0] = (int64_t)sc[0];
  out[1] = cnt;
  out[2] = cnt > 0 ? st->pre[0] : 0;
  out[3] = cnt > 0 ? st->pre[1] : 0;
}

// Whole-layer passes: the spans' reductions are queued on the control
// stream right behind the walk that produced first/last positions, so
// finalize_layer only reads four pinned integers.
// ATLAS_SPAN_SORT=1: order statistics through a device radix sort (A/B)
static bool span_sort_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("ATLAS_SPAN_SORT");
    return e && e[0] == '1';
  }();
  return on;
}

void queue_spans(atlas_layer* L, const atlas_graph* g, cudaStream_t s) {
  const int64_t n = L->nloc;
  L->span_pin.reserve(4);
  L->span_dev.reserve(4);
  if (!L->span_ev)
    ATLAS_CUDA(cudaEventCreateWithFlags(&L->span_ev, cudaEventDisableTiming));
  if (n == 0) {
    ATLAS_CUDA(cudaMemsetAsync(L->span_dev.ptr, 0, 4 * sizeof(int64_t), s));
  } else {
    // spans are < E + V + 1 stream positions; the sentinel of vertices
    // without a step sorts last within the same bit width
    int bits = 1;
    while (bits < 62 && (int64_t(1) << bits) <= g->E + g->V + 2) bits++;
    bits++;
    const int64_t sentinel = (int64_t(1) << bits) - 1;
    DevBuf<int64_t>& spans = L->span_buf;
    DevBuf<int64_t>& sorted = L->span_sorted;
    DevBuf<unsigned long long>& sc = L->span_acc;
    spans.reserve(n);
    sorted.reserve(n);
    sc.reserve(2);
    ATLAS_CUDA(cudaMemsetAsync(sc.ptr, 0, 2 * sizeof(unsigned long long), s));
    span_values<<<grid_of(n), 256, 0, s>>>(L->first_pos.ptr, L->last_pos.ptr,
                                           n, spans.ptr, sc.ptr, sentinel);
    count_launch();
    ATLAS_LAUNCH_CHECK();
    if (span_sort_enabled()) {  // A/B: the device radix sort
      size_t tmp_bytes = 0;
      ATLAS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, spans.ptr,
                                                sorted.ptr, n, 0, bits, s));
      DevBuf<uint8_t>& tmp = L->span_tmp;
      tmp.reserve(tmp_bytes);
      ATLAS_CUDA(cub::DeviceRadixSort::SortKeys(tmp.ptr, tmp_bytes, spans.ptr,
                                                sorted.ptr, n, 0, bits, s));
      count_launch();
      span_pick<<<1, 1, 0, s>>>(sc.ptr, sorted.ptr, L->span_dev.ptr);
      count_launch();
      ATLAS_LAUNCH_CHECK();
    } else {
      // valid spans < 2^(bits - 1): digits of <= kSelMaxBits from the top
      const int vbits = bits - 1;
      const int passes = (vbits + kSelMaxBits - 1) / kSelMaxBits;
      const int width = (vbits + passes - 1) / passes;
      // scratch: SpanSel (32 B) + 2 x 1024 histogram words
      sorted.reserve(4 + (2 << kSelMaxBits) / 2);
      SpanSel* st = reinterpret_cast<SpanSel*>(sorted.ptr);
      unsigned* hist = reinterpret_cast<unsigned*>(sorted.ptr + 4);
      span_sel_init<<<1, 256, 0, s>>>(sc.ptr, st, hist);
      count_launch();
      const unsigned hgrid = (unsigned)std::min<int64_t>(
          ceil_div(n, 256), (int64_t)num_sms() * 2);
      for (int hi_bit = vbits; hi_bit > 0; hi_bit -= width) {
        const int lo_bit = std::max(0, hi_bit - width);
        span_sel_hist<<<hgrid, 256, 0, s>>>(spans.ptr, n, sentinel, st,
                                            lo_bit, hi_bit - lo_bit, hist);
        span_sel_pick<<<1, 1024, 0, s>>>(st, hist, hi_bit - lo_bit);
        count_launch();
        count_launch();
      }
      span_sel_out<<<1, 1, 0, s>>>(sc.ptr, st, L->span_dev.ptr);
      count_launch();
      ATLAS_LAUNCH_CHECK();
    }
  }
  ATLAS_CUDA(cudaMemcpyAsync(L->span_pin.ptr, L->span_dev.ptr,
                             4 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaEventRecord(L->span_ev, s));
  L->spans_queued = true;
}

void finish_spans(atlas_layer* L, cudaStream_t s) {
  const int64_t n = L->nloc;
  L->span_count = L->span_sum = L->span_q_lo = L->span_q_hi = 0;
  if (L->spans_queued) {
    L->spans_queued = false;
    ATLAS_CUDA(cudaEventSynchronize(L->span_ev));
    L->span_sum = L->span_pin.ptr[0];
    L->span_count = L->span_pin.ptr[1];
    L->span_q_lo = L->span_pin.ptr[2];
    L->span_q_hi = L->span_pin.ptr[3];
    return;
  }
  if (n == 0) return;
  DevBuf<int64_t>& spans = L->span_buf;
  DevBuf<int64_t>& sorted = L->span_sorted;
  DevBuf<unsigned long long>& sc = L->span_acc;
  spans.reserve(n);
  sorted.reserve(n);
  sc.reserve(2);
  ATLAS_CUDA(cudaMemsetAsync(sc.ptr, 0, 2 * sizeof(unsigned long long), s));
  span_values<<<grid_of(n), 256, 0, s>>>(L->first_pos.ptr, L->last_pos.ptr, n,
                                         spans.ptr, sc.ptr);
  count_launch();
  ATLAS_LAUNCH_CHECK();
  unsigned long long h[2];
  ATLAS_CUDA(cudaMemcpyAsync(h, sc.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
  L->span_sum = (int64_t)h[0];
  L->span_count = (int64_t)h[1];
  if (L->span_count == 0) return;
  size_t tmp_bytes = 0;
  ATLAS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, spans.ptr,
                                            sorted.ptr, n, 0, 64, s));
  DevBuf<uint8_t>& tmp = L->span_tmp;
  tmp.reserve(tmp_bytes);
  ATLAS_CUDA(cub::DeviceRadixSort::SortKeys(tmp.ptr, tmp_bytes, spans.ptr,
                                            sorted.ptr, n, 0, 64, s));
  count_launch();
  // numpy 'linear': virtual index (n - 1) * 0.99
  const double vi = (double)(L->span_count - 1) * 0.99;
  int64_t lo_i = (int64_t)std::floor(vi);
  int64_t hi_i = std::min<int64_t>(lo_i + 1, L->span_count - 1);
  ATLAS_CUDA(cudaMemcpyAsync(&L->span_q_lo, sorted.ptr + lo_i, sizeof(int64_t),
                             cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaMemcpyAsync(&L->span_q_hi, sorted.ptr + hi_i, sizeof(int64_t),
                             cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
}

// Largest edge pass of any chunk under plan R (GIN adds the chunk's self
// terms): topology-only, so cached per (graph generation, R).
static int64_t max_pass_of(atlas_layer* L, const atlas_graph* g, const Plan& p,
                           cudaStream_t s) {
  for (const auto& e : g->maxpass_cache)
    if (e.first == p.R * 4 + L->desc.model) return e.second;
  const int64_t nchunks = p.nchunks;
  if ((int64_t)g->offsets_host.size() == p.V + 1) {
    // from the host copy of the offsets: no device round trip, so queueing
    // a layer never waits for the layers queued before it
    const int64_t* off = g->offsets_host.data();
    int64_t max_pass = 0;
    for (int64_t c = 0; c < nchunks; c++) {
      const int64_t a = c * p.R, b = std::min((c + 1) * p.R, p.V);
      max_pass = std::max(max_pass, off[b] - off[a] +
                                        (L->desc.model == ATLAS_GIN ? b - a : 0));
    }
    g->maxpass_cache.emplace_back(p.R * 4 + L->desc.model, max_pass);
    return max_pass;
  }
  DevBuf<int64_t>& mc = L->span_buf;  // reused scratch (>= nchunks)
  mc.reserve(std::max<int64_t>(nchunks, 1));
  chunk_edges<<<grid_of(nchunks), 256, 0, s>>>(g->offsets.ptr, p, mc.ptr);
  count_launch();
  ATLAS_LAUNCH_CHECK();
  std::vector<int64_t> m(nchunks);
  ATLAS_CUDA(cudaMemcpyAsync(m.data(), mc.ptr, nchunks * sizeof(int64_t),
                             cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
  int64_t max_pass = 0;
  for (int64_t c = 0; c < nchunks; c++) {
    const int64_t n_c = std::min((c + 1) * p.R, p.V) - c * p.R;
    max_pass = std::max(max_pass,
                        m[c] + (L->desc.model == ATLAS_GIN ? n_c : 0));
  }
  g->maxpass_cache.emplace_back(p.R * 4 + L->desc.model, max_pass);
  return max_pass;
}

// Eviction-free verdict from the (chunk, pass) admission / graduation
// histogram h (7C entries). Returns true and fills the fast-path metrics
// when the reference provably never evicts.
static bool fast_verdict(atlas_layer* L, const atlas_graph* g, int64_t R,
                         const unsigned long long* h) {
  const int64_t V = g->V;
  const int model = L->desc.model;
  const int64_t nchunks = ceil_div(V, R);
  bool single = true;
  int64_t hot = 0, peak = 0;
  std::vector<int64_t> touched(nchunks, 0);
  for (int64_t c = 0; c < nchunks; c++) {
    const int64_t cs = c * R, ce = std::min(cs + R, V);
    const int64_t self_n = std::max<int64_t>(
        0, std::min(ce, g->hi) - std::max(cs, g->lo));
    const int64_t sizes[3] = {(int64_t)h[3 * c + 0],
                              model == ATLAS_SAGE ? self_n : 0,
                              (int64_t)h[6 * nchunks + c]};
    for (int ph = 0; ph < 3; ph++) {
      if (sizes[ph] > L->sub_batch) single = false;
      const int64_t a = (int64_t)h[3 * c + ph];
      if (a > 0) {
        hot += a;
        peak = std::max(peak, hot);
      }
      hot -= (int64_t)h[3 * nchunks + 3 * c + ph];
    }
    touched[c] = sizes[1] + sizes[2];
  }
  const bool fast = single && peak <= L->desc.slot_count &&
                    !L->desc.record_log && !L->desc.force_exact;
  if (!fast) return false;
  L->fast_path = true;
  L->fp_hot_peak = peak;
  L->fp_messages = g->eloc + (model == ATLAS_GCN ? 0 : L->nloc);
  for (int64_t c = 0; c < nchunks; c++) {
    L->chunk_reloads.push_back(0);
    L->chunk_touched.push_back(touched[c]);
  }
  return true;
}

// exact replay: materialise runs in first-appearance order and run the
// single-CTA engine over them (synchronous)
static void exact_replay(atlas_layer* L, const atlas_graph* g, int64_t R,
                         cudaStream_t s) {
  const char* prof = getenv("ATLAS_SWEEP_PROFILE");
  const bool timed = prof && prof[0] == '1';
  auto now = [&]() {
    if (timed) cudaStreamSynchronize(s);
    return std::chrono::steady_clock::now();
  };
  const auto t0 = now();
  const int64_t V = g->V;
  const int model = L->desc.model;
  Plan p{R, V, ceil_div(V, R)};
  const int64_t nchunks = p.nchunks;
  DevBuf<unsigned long long>& hist = L->ctl_hist;
  const size_t hbytes = 7 * (size_t)nchunks * 4;
  const int use_smem = hbytes <= 48 * 1024 ? 1 : 0;
  const unsigned blocks = (unsigned)std::min<int64_t>(
      num_sms() * 8, std::max<int64_t>(1, ceil_div(L->nloc, 8)));
  L->fast_path = false;
  L->sweep_path = false;
  // a cached static schedule of the same (topology, plan, model, sub-batch,
  // policy) skips the run materialisation entirely
  if (sweep_try_cached(L, g, R, s)) return;
  const int64_t npos = g->E + (model == ATLAS_GCN ? 0 : V) + 1;
  SweepWs& W = sweep_ws_of(g);  // grow-only, shared by the graph's layers
  DevBuf<uint64_t>& at_pos = W.at_pos;
  DevBuf<uint64_t>& runs = W.runs;
  DevBuf<int64_t>& nsel = W.nsel;
  at_pos.reserve(npos);
  nsel.reserve(1);
  fill_u64<<<grid_of(npos), 256, 0, s>>>(at_pos.ptr, npos, kNoRun);
  count_launch();
  ATLAS_CUDA(cudaMemsetAsync(hist.ptr, 0, hist.bytes(), s));
  walk_destinations<<<blocks, 256, use_smem ? hbytes : 0, s>>>(
      model, p, g->offsets.ptr, g->csc_ptr.ptr, g->csc_src.ptr,
      g->csc_eid.ptr, g->lo, L->nloc, L->first_pos.ptr, L->last_pos.ptr,
      hist.ptr, use_smem, at_pos.ptr, 1);
  count_launch();
  ATLAS_LAUNCH_CHECK();
  std::vector<unsigned long long> h(7 * nchunks);
  ATLAS_CUDA(cudaMemcpyAsync(h.data(), hist.ptr, h.size() * sizeof(h[0]),
                             cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
  int64_t total_runs = 0;
  std::vector<int64_t> run_off(nchunks + 1, 0);
  for (int64_t c = 0; c < nchunks; c++) {
    run_off[c + 1] = run_off[c] + (int64_t)h[6 * nchunks + c];
  }
  total_runs = run_off[nchunks];
  runs.reserve(std::max<int64_t>(total_runs, 1));
  size_t tmp_bytes = 0;
  NotNoRun pred;
  ATLAS_CUDA(cub::DeviceSelect::If(nullptr, tmp_bytes, at_pos.ptr, runs.ptr,
                                   nsel.ptr, npos, pred, s));
  DevBuf<uint8_t>& tmp = W.sel_tmp;
  tmp.reserve(tmp_bytes);
  ATLAS_CUDA(cub::DeviceSelect::If(tmp.ptr, tmp_bytes, at_pos.ptr, runs.ptr,
                                   nsel.ptr, npos, pred, s));
  count_launch();
  int64_t got = 0;
  ATLAS_CUDA(cudaMemcpyAsync(&got, nsel.ptr, sizeof(got),
                             cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
  if (got != total_runs)
    fail(ATLAS_EINVARIANT, "run materialisation mismatch " +
                               std::to_string(got) + " vs " +
                               std::to_string(total_runs));
  DevBuf<int64_t>& d_off = W.d_off;
  DevBuf<int64_t>& d_bounds = W.d_bounds;
  d_off.reserve(nchunks + 1);
  d_bounds.reserve(2 * nchunks);
  std::vector<int64_t> bounds(2 * nchunks);
  for (int64_t c = 0; c < nchunks; c++) {
    bounds[2 * c] = c * R;
    bounds[2 * c + 1] = std::min((c + 1) * R, V);
  }
  ATLAS_CUDA(cudaMemcpyAsync(d_off.ptr, run_off.data(),
                             (nchunks + 1) * sizeof(int64_t),
                             cudaMemcpyHostToDevice, s));
  ATLAS_CUDA(cudaMemcpyAsync(d_bounds.ptr, bounds.data(),
                             2 * nchunks * sizeof(int64_t),
                             cudaMemcpyHostToDevice, s));
  if (timed) {
    const auto t1 = now();
    fprintf(stderr, "[replay] runs materialised in %.3f ms (%lld runs)\n",
            std::chrono::duration<double, std::milli>(t1 - t0).count(),
            (long long)total_runs);
  }
  // MINPEND / LRU without logs: the sweep over sub-batches (sweep.cu);
  // RND, logs and inconsistent inputs: the per-element machine
  if (L->desc.policy != ATLAS_RND && !L->desc.record_log && sweep_enabled() &&
      sweep_replay(L, g, R, runs.ptr, d_off.ptr, run_off, s))
    return;
  engine_run_chunks(L, runs.ptr, d_off.ptr, d_bounds.ptr, nchunks,
                    run_off.data(), s);
}

// Control plane of a whole-layer pass on the reference chunk plan R.
// When no chunk pass can split into sub-batches (topology-only bound,
// cached) and no logs are requested, the parallel walk and the readback of
// its histogram are only QUEUED on s, and the verdict is taken later by
// settle_control(): the host never waits for the data plane here. A
// negative verdict then runs the exact replay (which only touches control
// state, never the records).
// true when resident_control(L, g, R) only queues device work (the
// eviction-free walk with a deferred verdict): it never waits on the host
bool control_is_async(atlas_layer* L, const atlas_graph* g, int64_t R) {
  if (L->desc.record_log || L->desc.force_exact) return false;
  const int64_t V = g->V;
  Plan p{R, V, ceil_div(V, R)};
  bool cached = (int64_t)g->offsets_host.size() == V + 1;
  for (const auto& e : g->maxpass_cache)
    if (e.first == p.R * 4 + L->desc.model) cached = true;
  if (!cached) return false;
  const int64_t max_pass = std::min(max_pass_of(L, g, p, nullptr), L->nloc);
  return L->sub_batch >= max_pass;
}

void resident_control(atlas_layer* L, const atlas_graph* g, int64_t R,
                      cudaStream_t s) {
  const int64_t V = g->V;
  const int model = L->desc.model;
  Plan p{R, V, ceil_div(V, R)};
  const int64_t nchunks = p.nchunks;
  DevBuf<unsigned long long>& hist = L->ctl_hist;  // admit 3C|grad 3C|runs C
  hist.reserve(7 * std::max<int64_t>(nchunks, 1));
  // An edge pass holds at most min(nloc, m_c (+ n_c for GIN)) destinations,
  // so when that bound is <= sub_batch for every chunk each pass is one
  // sub-batch and the per-chunk run counts (an E-wide walk) are not needed
  // to prove it; they only feed reload-% denominators, whose numerators are
  // zero on the eviction-free path.
  const int64_t max_pass = std::min(max_pass_of(L, g, p, s), L->nloc);
  const bool need_runs = L->sub_batch < max_pass || L->desc.record_log ||
                         L->desc.force_exact;
  ATLAS_CUDA(cudaMemsetAsync(hist.ptr, 0,
                             7 * std::max<int64_t>(nchunks, 1) * 8, s));
  // grid-stride warps; per-block shared histogram when 7C u32 fit in 48 KB
  const size_t hbytes = 7 * (size_t)nchunks * 4;
  const int use_smem = hbytes <= 48 * 1024 ? 1 : 0;
  const unsigned blocks = (unsigned)std::min<int64_t>(
      num_sms() * 8, std::max<int64_t>(1, ceil_div(L->nloc, 8)));
  L->chunks_seen += nchunks;
  if (need_runs) {
    walk_destinations<<<blocks, 256, use_smem ? hbytes : 0, s>>>(
        model, p, g->offsets.ptr, g->csc_ptr.ptr, g->csc_src.ptr,
        g->csc_eid.ptr, g->lo, L->nloc, L->first_pos.ptr, L->last_pos.ptr,
        hist.ptr, use_smem, nullptr, 1);
    count_launch();
    ATLAS_LAUNCH_CHECK();
    std::vector<unsigned long long> h(7 * nchunks);
    ATLAS_CUDA(cudaMemcpyAsync(h.data(), hist.ptr, h.size() * sizeof(h[0]),
                               cudaMemcpyDeviceToHost, s));
    ATLAS_CUDA(cudaStreamSynchronize(s));
    queue_spans(L, g, s);
    if (!fast_verdict(L, g, R, h.data())) exact_replay(L, g, R, s);
    return;
  }
  walk_light<<<blocks, 256, use_smem ? hbytes : 0, s>>>(
      model, p, g->offsets.ptr, g->csc_ptr.ptr, g->csc_src.ptr,
      g->csc_eid.ptr, g->lo, L->nloc, L->first_pos.ptr, L->last_pos.ptr,
      hist.ptr, use_smem);
  count_launch();
  ATLAS_LAUNCH_CHECK();
  L->pin_hist.reserve(7 * std::max<int64_t>(nchunks, 1));
  ATLAS_CUDA(cudaMemcpyAsync(L->pin_hist.ptr, hist.ptr,
                             7 * nchunks * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s));
  queue_spans(L, g, s);
  L->ctl_deferred = true;
  L->ctl_graph = g;
  L->ctl_R = R;
}

// Take a deferred verdict (waits for the control stream only).
void settle_control(atlas_layer* L) {
  if (!L->ctl_deferred) return;
  L->ctl_deferred = false;
  ATLAS_CUDA(cudaStreamSynchronize(L->ctl_stream));
  if (!fast_verdict(L, L->ctl_graph, L->ctl_R, L->pin_hist.ptr))
    exact_replay(L, L->ctl_graph, L->ctl_R, L->ctl_stream);
}

}  // namespace atlas
