// Destination-major topology for one GPU's destination range.
//
// The reference streams sources and pushes each out-edge to its
// destination (oocgnn/orchestrator.py:243-295). Because a stable sort of a
// chunk's edges by destination (oocgnn/orchestrator.py:270) keeps sources
// ascending inside each destination group, every chunk's destination runs
// are contiguous sub-ranges of ONE global destination-major (CSC) view
// whose per-destination sources ascend. This file builds that view once
// per graph and rank: a stable radix sort of (dst, csr_edge_index) pairs.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "internal.cuh"

namespace atlas {

namespace {

// src_of_edge[j] = u for j in [off[u], off[u+1]); warp per source row.
__global__ void expand_sources(const int64_t* __restrict__ off, int64_t V,
                               uint32_t* __restrict__ src_of_edge) {
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned lane = threadIdx.x & 31u;
  for (int64_t u = warp; u < V; u += nwarps) {
    int64_t b = off[u], e = off[u + 1];
    for (int64_t j = b + lane; j < e; j += 32) src_of_edge[j] = (uint32_t)u;
  }
}

// keys = dst - lo for in-range edges, in CSR order; vals = edge index.
__global__ void make_pairs(const uint32_t* __restrict__ nbrs, int64_t E,
                           int64_t lo, const uint32_t* __restrict__ sel,
                           int64_t nsel, uint32_t* __restrict__ keys,
                           uint32_t* __restrict__ vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (sel == nullptr) {
    for (; i < E; i += stride) {
      keys[i] = nbrs[i] - (uint32_t)lo;
      vals[i] = (uint32_t)i;
    }
  } else {
    for (; i < nsel; i += stride) {
      uint32_t j = sel[i];
      keys[i] = nbrs[j] - (uint32_t)lo;
      vals[i] = j;
    }
  }
}

__global__ void gather_u32(const uint32_t* __restrict__ table,
                           const uint32_t* __restrict__ idx, int64_t n,
                           uint32_t* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = table[idx[i]];
}

struct InRange {
  const uint32_t* nbrs;
  uint32_t lo, hi;
  __device__ bool operator()(const uint32_t& j) const {
    uint32_t d = nbrs[j];
    return d >= lo && d < hi;
  }
};

int grid_for(int64_t n, int block) {
  int64_t g = ceil_div(n, block);
  if (g > num_sms() * 16) g = num_sms() * 16;
  return (int)(g < 1 ? 1 : g);
}

int bits_for(int64_t n) {
  int b = 1;
  while (b < 32 && (int64_t(1) << b) < n) b++;
  return b;
}

}  // namespace

void build_csc(atlas_graph* g, DevBuf<uint32_t>& nbrs,
               const uint32_t* indeg_host, cudaStream_t s) {
  const int64_t V = g->V, E = g->E;
  const int64_t e1 = E > 0 ? E : 1;
  // workspaces live in the graph handle: a refresh of the same shape
  // (atlas_graph_update) allocates nothing
  DevBuf<uint32_t>& src_of_edge = g->ws_src;
  DevBuf<uint32_t>& keys = g->ws_keys;
  DevBuf<uint32_t>& vals = g->ws_vals;
  DevBuf<uint32_t>& keys_out = g->ws_keys_out;
  DevBuf<uint8_t>& tmp = g->ws_tmp;
  src_of_edge.reserve(e1);
  // every host->device copy goes first: one queued behind the sort would
  // wait in the copy engine behind whatever input copies the next layer
  // queues meanwhile
  g->indeg.reserve(g->nloc > 0 ? g->nloc : 1);
  if (g->nloc > 0)
    ATLAS_CUDA(cudaMemcpyAsync(g->indeg.ptr, indeg_host + g->lo,
                               g->nloc * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, s));
  if (E > 0) {
    expand_sources<<<grid_for(V * 32, 256), 256, 0, s>>>(g->offsets.ptr, V,
                                                        src_of_edge.ptr);
    count_launch();
    ATLAS_LAUNCH_CHECK();
  }

  // select in-range edges (order preserved) when this rank owns a sub-range
  const bool full = (g->lo == 0 && g->hi == V);
  int64_t nsel = E;
  if (!full && E > 0) {
    g->ws_sel.reserve(e1);
    g->ws_nsel.reserve(1);
    thrust::counting_iterator<uint32_t> it(0);
    size_t tmp_bytes = 0;
    InRange pred{nbrs.ptr, (uint32_t)g->lo, (uint32_t)g->hi};
    ATLAS_CUDA(cub::DeviceSelect::If(nullptr, tmp_bytes, it, g->ws_sel.ptr,
                                     g->ws_nsel.ptr, E, pred, s));
    tmp.reserve(tmp_bytes);
    ATLAS_CUDA(cub::DeviceSelect::If(tmp.ptr, tmp_bytes, it, g->ws_sel.ptr,
                                     g->ws_nsel.ptr, E, pred, s));
    count_launch();
    ATLAS_CUDA(cudaMemcpyAsync(&nsel, g->ws_nsel.ptr, sizeof(int64_t),
                               cudaMemcpyDeviceToHost, s));
    ATLAS_CUDA(cudaStreamSynchronize(s));
  }
  g->eloc = nsel;
  const int64_t n = nsel;
  const int64_t n1 = n > 0 ? n : 1;
  keys.reserve(n1);
  vals.reserve(n1);
  keys_out.reserve(n1);
  g->csc_eid.reserve(n1);
  if (n > 0) {
    make_pairs<<<grid_for(n, 256), 256, 0, s>>>(
        nbrs.ptr, E, g->lo, full ? nullptr : g->ws_sel.ptr, n, keys.ptr,
        vals.ptr);
    count_launch();
    ATLAS_LAUNCH_CHECK();
    size_t tmp_bytes = 0;
    int end_bit = bits_for(g->nloc);
    ATLAS_CUDA(cub::DeviceRadixSort::SortPairs(
        nullptr, tmp_bytes, keys.ptr, keys_out.ptr, vals.ptr,
        g->csc_eid.ptr, n, 0, end_bit, s));
    tmp.reserve(tmp_bytes);
    ATLAS_CUDA(cub::DeviceRadixSort::SortPairs(
        tmp.ptr, tmp_bytes, keys.ptr, keys_out.ptr, vals.ptr,
        g->csc_eid.ptr, n, 0, end_bit, s));
    count_launch();
  }
  g->csc_src.reserve(n1);
  if (n > 0) {
    gather_u32<<<grid_for(n, 256), 256, 0, s>>>(src_of_edge.ptr,
                                                g->csc_eid.ptr, n,
                                                g->csc_src.ptr);
    count_launch();
    ATLAS_LAUNCH_CHECK();
  }
  // csc_ptr = exclusive scan of local in-degrees
  g->csc_ptr.reserve(g->nloc + 1);
  ATLAS_CUDA(cudaMemsetAsync(g->csc_ptr.ptr, 0, sizeof(int64_t), s));
  if (g->nloc > 0) {
    size_t tmp_bytes = 0;
    ATLAS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, g->indeg.ptr,
                                             g->csc_ptr.ptr + 1, g->nloc, s));
    tmp.reserve(tmp_bytes);
    ATLAS_CUDA(cub::DeviceScan::InclusiveSum(tmp.ptr, tmp_bytes, g->indeg.ptr,
                                             g->csc_ptr.ptr + 1, g->nloc, s));
    count_launch();
  }
  // the consistency total is read back without stalling the host: the
  // next layer can be queued (and its input copies start) right away
  g->chk.reserve(1);
  if (!g->chk_ev)
    ATLAS_CUDA(cudaEventCreateWithFlags(&g->chk_ev, cudaEventDisableTiming));
  ATLAS_CUDA(cudaMemcpyAsync(g->chk.ptr, g->csc_ptr.ptr + g->nloc,
                             sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaEventRecord(g->chk_ev, s));
  g->chk_pending = true;
  g->chk_expect = n;
}

void verify_graph(const atlas_graph* g) {
  if (!g || !g->chk_pending) return;
  ATLAS_CUDA(cudaEventSynchronize(g->chk_ev));
  g->chk_pending = false;
  const int64_t total = g->chk.ptr[0];
  if (total != g->chk_expect)
    fail(ATLAS_EINVARIANT, "in-degrees disagree with adjacency (" +
                               std::to_string(total) + " vs " +
                               std::to_string(g->chk_expect) +
                               " in-range edges)");
}

}  // namespace atlas
