// process_chunk for one caller-supplied source chunk (operator path).
//
// Mirrors oocgnn/orchestrator.py:216-299 for a chunk handed in by the
// caller (tests/test_orchestrator.py:61-84 drive the reference this way):
//   1. stage rows + CSR slice to HBM;
//   2. build the addend stream (GIN interleaves each source's self term
//      before its out-edges) and stable-sort it by destination
//      (oocgnn/orchestrator.py:270) -> destination runs in stream order;
//   3. data plane: SAGE self half + bit-exact run aggregation (aggregate.cu);
//   4. first/last steps of every touched destination;
//   5. runs in first-appearance order (oocgnn/orchestrator.py:285) ->
//      exact control engine (engine.cu) -> graduation list.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace atlas {

namespace {

constexpr uint32_t kInvalid = 0xFFFFFFFFu;
constexpr uint32_t kSelfBit = 0x80000000u;

// stream entries: key = local dst (or kInvalid), srcrow = source row | self
__global__ void build_stream(const int64_t* __restrict__ off,
                             const int64_t* __restrict__ nbrs, int64_t n,
                             int64_t start, int64_t lo, int64_t hi, int gin,
                             uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ vals,
                             uint32_t* __restrict__ srcrow) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const int64_t b = off[i], e = off[i + 1];
  const int64_t shift = gin ? i + 1 : 0;
  if (gin && lane == 0) {
    const int64_t t = b + i;
    const int64_t v = start + i;
    keys[t] = (v >= lo && v < hi) ? (uint32_t)(v - lo) : kInvalid;
    vals[t] = (uint32_t)t;
    srcrow[t] = (uint32_t)i | kSelfBit;
  }
  for (int64_t j = b + lane; j < e; j += 32) {
    const int64_t t = j + shift;
    const int64_t v = nbrs[j];
    keys[t] = (v >= lo && v < hi) ? (uint32_t)(v - lo) : kInvalid;
    vals[t] = (uint32_t)t;
    srcrow[t] = (uint32_t)i;
  }
}

__global__ void gather_src(const uint32_t* __restrict__ srcrow,
                           const uint32_t* __restrict__ order, int64_t n,
                           uint32_t* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i < n; i += (int64_t)gridDim.x * blockDim.x) out[i] = srcrow[order[i]];
}

// per run: appearance record + first/last step update
__global__ void runs_finish(const uint32_t* __restrict__ run_dst,
                            const int64_t* __restrict__ run_beg,
                            int64_t nruns,
                            const uint32_t* __restrict__ order,
                            int64_t pos_base, uint64_t* __restrict__ at_first,
                            int64_t* __restrict__ first_pos,
                            int64_t* __restrict__ last_pos) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; r < nruns; r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = run_dst[r];
    const int64_t b = run_beg[r], e = run_beg[r + 1];
    const uint32_t t0 = order[b], t1 = order[e - 1];
    at_first[t0] = ((uint64_t)(e - b) << 32) | v;
    if (first_pos[v] < 0) first_pos[v] = pos_base + t0;
    last_pos[v] = pos_base + t1;
  }
}

__global__ void self_steps(int64_t a, int64_t b, int64_t pos_base,
                           int64_t src0, int64_t* first_pos,
                           int64_t* last_pos) {
  int64_t v = a + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; v < b; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pos_base + (v - src0);
    if (first_pos[v] < 0) first_pos[v] = p;
    last_pos[v] = p;
  }
}

__global__ void fill_u64(uint64_t* p, int64_t n, uint64_t val) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = val;
}

struct IsRun {
  __device__ bool operator()(const uint64_t& x) const { return x != ~0ull; }
};

unsigned grid_of(int64_t n, int block = 256) {
  int64_t g = ceil_div(n, block);
  if (g > num_sms() * 16) g = num_sms() * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

template <typename F>
void cub_call(DevBuf<uint8_t>& tmp, F f) {
  size_t bytes = 0;
  ATLAS_CUDA(f(nullptr, bytes));
  tmp.reserve(bytes + 256);
  bytes = tmp.count;
  ATLAS_CUDA(f(tmp.ptr, bytes));
  count_launch();
}

}  // namespace

void submit_chunk(atlas_layer* L, int64_t start, int64_t end,
                  const void* rows_host, int dtype,
                  const int64_t* off_host, const int64_t* nbrs_host,
                  int64_t m, cudaStream_t s) {
  const atlas_layer_desc& D = L->desc;
  if (start < 0 || end < start || end > D.num_vertices)
    fail(ATLAS_ECONFIG, "chunk interval out of range");
  if (!L->engine_initialized) engine_init(L, s);
  const int64_t n = end - start;
  const int64_t d = D.embed_dim;
  const size_t item = dtype == ATLAS_F32 ? 4 : 2;
  const bool gin = D.model == ATLAS_GIN;
  const int64_t mm = m + (gin ? n : 0);
  if (mm >= (int64_t)0x7FFFFFFF) fail(ATLAS_ECONFIG, "chunk too large");

  // 1. stage
  L->tile.reserve(std::max<int64_t>(n * d, 1) * item);
  L->ch_offsets.reserve(n + 1);
  L->ch_nbrs.reserve(std::max<int64_t>(m, 1));
  if (n > 0)
    ATLAS_CUDA(cudaMemcpyAsync(L->tile.ptr, rows_host, n * d * item,
                               cudaMemcpyHostToDevice, s));
  ATLAS_CUDA(cudaMemcpyAsync(L->ch_offsets.ptr, off_host,
                             (n + 1) * sizeof(int64_t),
                             cudaMemcpyHostToDevice, s));
  if (m > 0)
    ATLAS_CUDA(cudaMemcpyAsync(L->ch_nbrs.ptr, nbrs_host, m * sizeof(int64_t),
                               cudaMemcpyHostToDevice, s));

  // 2. stream + stable sort by destination
  const int64_t mmx = std::max<int64_t>(mm, 1);
  L->keys_a.reserve(mmx);
  L->keys_b.reserve(mmx);
  L->vals_a.reserve(mmx);
  L->vals_b.reserve(mmx);
  L->ent_src.reserve(mmx);
  DevBuf<uint32_t>& srcrow = L->op_srcrow;
  srcrow.reserve(mmx);
  int64_t nruns = 0;
  const int64_t lo = D.dst_lo, hi = D.dst_hi;
  if (mm > 0 && n > 0) {
    build_stream<<<(unsigned)ceil_div(n, 8), 256, 0, s>>>(
        L->ch_offsets.ptr, L->ch_nbrs.ptr, n, start, lo, hi, gin,
        L->keys_a.ptr, L->vals_a.ptr, srcrow.ptr);
    count_launch();
    ATLAS_LAUNCH_CHECK();
    cub_call(L->sort_tmp, [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, L->keys_a.ptr,
                                             L->keys_b.ptr, L->vals_a.ptr,
                                             L->vals_b.ptr, mm, 0, 32, s);
    });
    // runs = equal-key segments of the sorted keys
    L->run_dst.reserve(mmx + 1);
    L->run_beg.reserve(mmx + 2);
    L->misc64.reserve(2);
    DevBuf<int64_t>& counts = L->op_counts;
    counts.reserve(mmx + 1);
    cub_call(L->sort_tmp, [&](void* t, size_t& b) {
      return cub::DeviceRunLengthEncode::Encode(t, b, L->keys_b.ptr,
                                                L->run_dst.ptr, counts.ptr,
                                                L->misc64.ptr, mm, s);
    });
    int64_t nr = 0;
    ATLAS_CUDA(cudaMemcpyAsync(&nr, L->misc64.ptr, sizeof(int64_t),
                               cudaMemcpyDeviceToHost, s));
    uint32_t last_key = 0;
    ATLAS_CUDA(cudaStreamSynchronize(s));
    if (nr > 0) {
      ATLAS_CUDA(cudaMemcpy(&last_key, L->run_dst.ptr + nr - 1,
                            sizeof(uint32_t), cudaMemcpyDeviceToHost));
      if (last_key == kInvalid) nr--;  // out-of-range destinations
    }
    nruns = nr;
    ATLAS_CUDA(cudaMemsetAsync(L->run_beg.ptr, 0, sizeof(int64_t), s));
    if (nruns > 0) {
      cub_call(L->sort_tmp, [&](void* t, size_t& b) {
        return cub::DeviceScan::InclusiveSum(t, b, counts.ptr,
                                             L->run_beg.ptr + 1, nruns, s);
      });
    }
    gather_src<<<grid_of(mm), 256, 0, s>>>(srcrow.ptr, L->vals_b.ptr, mm,
                                           L->ent_src.ptr);
    count_launch();
    ATLAS_LAUNCH_CHECK();
  }

  // 3. data plane
  const int64_t a = std::max(start, lo), b = std::min(end, hi);
  if (D.model == ATLAS_SAGE && b > a)
    launch_sage_self(L->tile.ptr, dtype, d, a - start, b - a, (int)d,
                     L->acc.ptr + (a - lo) * D.agg_dim + d, D.agg_dim, s);
  if (nruns > 0)
    launch_agg_runs(L->tile.ptr, dtype, d, start, L->run_dst.ptr,
                    L->run_beg.ptr, nruns, L->ent_src.ptr, L->indeg.ptr,
                    D.model, D.gin_epsilon, (int)d, L->acc.ptr, D.agg_dim,
                    L->touched.ptr, s);

  // 4. steps
  int64_t edge_base = L->stream_step;
  if (D.model == ATLAS_SAGE) {
    if (b > a) {
      self_steps<<<grid_of(b - a), 256, 0, s>>>(
          a - lo, b - lo, L->stream_step, start - lo, L->first_pos.ptr,
          L->last_pos.ptr);
      count_launch();
    }
    edge_base += n;
  }
  L->stream_step = edge_base + mm;

  // 5. appearance order + engine
  DevBuf<uint64_t>& at_first = L->op_at_first;
  DevBuf<uint64_t>& ordered = L->op_ordered;
  DevBuf<int64_t>& nsel = L->op_nsel;
  at_first.reserve(mmx);
  ordered.reserve(std::max<int64_t>(nruns, 1));
  nsel.reserve(1);
  if (nruns > 0) {
    fill_u64<<<grid_of(mm), 256, 0, s>>>(at_first.ptr, mm, ~0ull);
    count_launch();
    runs_finish<<<grid_of(nruns), 256, 0, s>>>(
        L->run_dst.ptr, L->run_beg.ptr, nruns, L->vals_b.ptr, edge_base,
        at_first.ptr, L->first_pos.ptr, L->last_pos.ptr);
    count_launch();
    ATLAS_LAUNCH_CHECK();
    IsRun pred;
    cub_call(L->sort_tmp, [&](void* t, size_t& bb) {
      return cub::DeviceSelect::If(t, bb, at_first.ptr, ordered.ptr, nsel.ptr,
                                   mm, pred, s);
    });
  }
  int64_t h_off[2] = {0, nruns};
  int64_t h_bounds[2] = {start, end};
  DevBuf<int64_t>& dv = L->op_dv;
  dv.reserve(4);
  ATLAS_CUDA(cudaMemcpyAsync(dv.ptr, h_off, sizeof(h_off),
                             cudaMemcpyHostToDevice, s));
  ATLAS_CUDA(cudaMemcpyAsync(dv.ptr + 2, h_bounds, sizeof(h_bounds),
                             cudaMemcpyHostToDevice, s));
  engine_run_chunks(L, ordered.ptr, dv.ptr, dv.ptr + 2, 1, h_off, s);
  L->chunks_seen += 1;
}

}  // namespace atlas
