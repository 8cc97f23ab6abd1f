// Greedy vertex reordering on the GPU.
//
// Reference: oocgnn/reorder.py:30-88.
//   score(u) = (sum over u's out-edges, in CSR order, of 1/max(1, d_in(v)))
//              / d_out(u)            (float64; 0 when d_out(u) == 0)
//   new order = stable argsort of -score   (ties: ascending old id)
//   relabel: row r of the new CSR is old row new_to_old[r], neighbours
//            mapped through old_to_new and sorted ascending.
// np.add.at folds each source's gains left to right in f64, so one thread
// per source walking its row in order reproduces the sums bit-for-bit;
// the divisions are IEEE f64. The argsort is a stable radix sort of the
// negated f64 keys (cub), which orders every non-negative score like
// numpy's comparison sort (all zero scores negate to the same -0.0 key).
#include <cub/cub.cuh>

#include "internal.cuh"

namespace atlas {
namespace {

__global__ void inv_in_degrees(const uint32_t* __restrict__ indeg, int64_t v,
                               double* __restrict__ inv) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i < v; i += (int64_t)gridDim.x * blockDim.x)
    inv[i] = 1.0 / (double)max(1u, indeg[i]);
}

__global__ void neg_scores(const int64_t* __restrict__ off,
                           const uint32_t* __restrict__ nbrs,
                           const double* __restrict__ inv, int64_t v,
                           double* __restrict__ key,
                           uint32_t* __restrict__ ids) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; u < v; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = off[u], e = off[u + 1];
    double s = 0.0;
    for (int64_t j = b; j < e; j++) s = __dadd_rn(s, inv[nbrs[j]]);
    const double score = e > b ? __ddiv_rn(s, (double)(e - b)) : 0.0;
    key[u] = -score;
    ids[u] = (uint32_t)u;
  }
}

__global__ void invert_perm(const uint32_t* __restrict__ new_to_old,
                            int64_t v, int64_t* __restrict__ old_to_new) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; r < v; r += (int64_t)gridDim.x * blockDim.x)
    old_to_new[new_to_old[r]] = r;
}

__global__ void new_degrees(const int64_t* __restrict__ off,
                            const uint32_t* __restrict__ indeg,
                            const uint32_t* __restrict__ new_to_old, int64_t v,
                            int64_t* __restrict__ new_out,
                            uint32_t* __restrict__ new_in) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; r < v; r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = new_to_old[r];
    new_out[r] = off[o + 1] - off[o];
    new_in[r] = indeg[o];
  }
}

// warp per new row: copy the old row's neighbours through old_to_new
__global__ void relabel_rows(const int64_t* __restrict__ off,
                             const uint32_t* __restrict__ nbrs,
                             const uint32_t* __restrict__ new_to_old,
                             const int64_t* __restrict__ old_to_new,
                             const int64_t* __restrict__ new_off, int64_t v,
                             uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
       r < v; r += nw) {
    const uint32_t o = new_to_old[r];
    const int64_t b = off[o], e = off[o + 1], d = new_off[r];
    for (int64_t j = b + lane; j < e; j += 32)
      out[d + (j - b)] = (uint32_t)old_to_new[nbrs[j]];
  }
}

unsigned grid_of(int64_t n) {
  int64_t g = ceil_div(n, 256);
  if (g > num_sms() * 16) g = num_sms() * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

void reorder_graph(int64_t V, int64_t E, const int64_t* off_h,
                   const uint32_t* nbrs_h, const uint32_t* indeg_h,
                   int64_t* old_to_new_h, int64_t* new_off_h,
                   uint32_t* new_nbrs_h, uint32_t* new_indeg_h,
                   double* scores_h, cudaStream_t s) {
  const int64_t v1 = std::max<int64_t>(V, 1), e1 = std::max<int64_t>(E, 1);
  DevBuf<int64_t> off, o2n, noff, nout;
  DevBuf<uint32_t> nbrs, indeg, ids, n2o, nin, nn, nn_sorted;
  DevBuf<double> inv, key, key_sorted;
  DevBuf<uint8_t> tmp;
  off.alloc(V + 1);
  nbrs.alloc(e1);
  indeg.alloc(v1);
  ATLAS_CUDA(cudaMemcpyAsync(off.ptr, off_h, (V + 1) * 8,
                             cudaMemcpyHostToDevice, s));
  if (E)
    ATLAS_CUDA(cudaMemcpyAsync(nbrs.ptr, nbrs_h, E * 4,
                               cudaMemcpyHostToDevice, s));
  if (V)
    ATLAS_CUDA(cudaMemcpyAsync(indeg.ptr, indeg_h, V * 4,
                               cudaMemcpyHostToDevice, s));
  inv.alloc(v1);
  key.alloc(v1);
  key_sorted.alloc(v1);
  ids.alloc(v1);
  n2o.alloc(v1);
  if (V) {
    inv_in_degrees<<<grid_of(V), 256, 0, s>>>(indeg.ptr, V, inv.ptr);
    neg_scores<<<grid_of(V), 256, 0, s>>>(off.ptr, nbrs.ptr, inv.ptr, V,
                                          key.ptr, ids.ptr);
    count_launch(2);
    ATLAS_LAUNCH_CHECK();
    size_t tb = 0;
    ATLAS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.ptr,
                                               key_sorted.ptr, ids.ptr,
                                               n2o.ptr, V, 0, 64, s));
    tmp.reserve(tb);
    ATLAS_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tb, key.ptr,
                                               key_sorted.ptr, ids.ptr,
                                               n2o.ptr, V, 0, 64, s));
    count_launch();
  }
  o2n.alloc(v1);
  noff.alloc(V + 1);
  nout.alloc(v1);
  nin.alloc(v1);
  ATLAS_CUDA(cudaMemsetAsync(noff.ptr, 0, sizeof(int64_t), s));
  if (V) {
    invert_perm<<<grid_of(V), 256, 0, s>>>(n2o.ptr, V, o2n.ptr);
    new_degrees<<<grid_of(V), 256, 0, s>>>(off.ptr, indeg.ptr, n2o.ptr, V,
                                           nout.ptr, nin.ptr);
    count_launch(2);
    ATLAS_LAUNCH_CHECK();
    size_t tb = 0;
    ATLAS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, nout.ptr,
                                             noff.ptr + 1, V, s));
    tmp.reserve(tb);
    ATLAS_CUDA(cub::DeviceScan::InclusiveSum(tmp.ptr, tb, nout.ptr,
                                             noff.ptr + 1, V, s));
    count_launch();
  }
  nn.alloc(e1);
  nn_sorted.alloc(e1);
  if (V && E) {
    relabel_rows<<<grid_of(V * 32), 256, 0, s>>>(off.ptr, nbrs.ptr, n2o.ptr,
                                                o2n.ptr, noff.ptr, V, nn.ptr);
    count_launch();
    ATLAS_LAUNCH_CHECK();
    // every new row ascending (oocgnn/reorder.py:84-86)
    size_t tb = 0;
    ATLAS_CUDA(cub::DeviceSegmentedSort::SortKeys(
        nullptr, tb, nn.ptr, nn_sorted.ptr, E, V, noff.ptr, noff.ptr + 1, s));
    tmp.reserve(tb);
    ATLAS_CUDA(cub::DeviceSegmentedSort::SortKeys(
        tmp.ptr, tb, nn.ptr, nn_sorted.ptr, E, V, noff.ptr, noff.ptr + 1, s));
    count_launch();
  }
  if (V) {
    ATLAS_CUDA(cudaMemcpyAsync(old_to_new_h, o2n.ptr, V * 8,
                               cudaMemcpyDeviceToHost, s));
    ATLAS_CUDA(cudaMemcpyAsync(new_indeg_h, nin.ptr, V * 4,
                               cudaMemcpyDeviceToHost, s));
    if (scores_h) {
      // scores = -key in old-id order
      ATLAS_CUDA(cudaMemcpyAsync(scores_h, key.ptr, V * 8,
                                 cudaMemcpyDeviceToHost, s));
    }
  }
  ATLAS_CUDA(cudaMemcpyAsync(new_off_h, noff.ptr, (V + 1) * 8,
                             cudaMemcpyDeviceToHost, s));
  if (E)
    ATLAS_CUDA(cudaMemcpyAsync(new_nbrs_h, nn_sorted.ptr, E * 4,
                               cudaMemcpyDeviceToHost, s));
  ATLAS_CUDA(cudaStreamSynchronize(s));
  if (scores_h)
    for (int64_t i = 0; i < V; i++) scores_h[i] = -scores_h[i];
}

}  // namespace atlas
