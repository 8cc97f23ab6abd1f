// GAT pass B: edge-softmax-weighted broadcast aggregation (kernel plan K10,
// SURVEY.md §2.1 and A.5). The reference has no GAT; the
// semantics are oracle/gat.py's (DGL GATConv style):
//
//   e_uv[h] = LeakyReLU(el_u[h] + er_v[h]),  alpha = softmax_{u in N(v)} e
//   out_v[h] = sum_u alpha_uv[h] z_u[h] + b[h]   (concat, or mean over h)
//
// Pass A (transform first) is the tcgen05 GEMM z_ext = x . W_ext^T whose
// extra output columns are el and er (W_ext rows a_l[h]^T W_h, a_r[h]^T W_h),
// so every source row streamed here carries [z | el | er] (heads of z
// padded to whole 16-byte chunks, gat.ZLayout).
//
// Mapping (like agg_bulk): persistent warps grab runs of consecutive
// destinations, whose in-edges are one contiguous CSC range; lane 0 moves
// every source's whole z_ext row (z | el | er) into a shared-memory ring
// with one cp.async.bulk per row (mbarrier per slot, kGatSlots in flight
// per warp). Lanes own 16-byte column chunks of z; per edge each lane reads
// its chunk and its heads' el from the staged row and runs an online
// softmax in f32 (one exp per edge and head). The head mean / bias / ReLU
// epilogue is fused, so no f32 record ever goes back to HBM: the kernel
// reads E z_ext rows and writes V output rows.
#include "bulk.cuh"

namespace atlas {
namespace {

constexpr int kGatWarps = 4;
constexpr int kGatSlots = 8;   // rows in flight per warp (<= 1.1 KB each)
constexpr int kGatGrab = 16;   // destinations per work grab
constexpr int kMaxHeads = 8;
constexpr int kMaxCols = 256;

template <typename OutT>
__device__ __forceinline__ OutT out_cvt(float v);
template <>
__device__ __forceinline__ float out_cvt<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half out_cvt<__half>(float v) {
  return __float2half_rn(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 out_cvt<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

template <typename ZT>
struct ZChunk {
  uint4 raw;
  __device__ __forceinline__ float get(int e) const {
    return to_f32(reinterpret_cast<const ZT*>(&raw)[e]);
  }
};

struct GatArgs {
  int64_t ldz, ldy, lo, nloc;
  int heads, head_dim, head_stride, hf, el_col, er_col, mean_heads, relu;
  float slope;
  const float* bias;
};

// The z part of a row stores head h at columns [h*stride, h*stride + F)
// with stride = F rounded up to a 16-byte chunk, so the EPC elements of a
// lane's chunk always share one head and one online-softmax state.
template <typename ZT, typename OutT, int CH>
__global__ void __launch_bounds__(kGatWarps * 32,
                                  (CH == 1 && sizeof(ZT) == 4) ? 6 : 4)
    gat_bulk(const ZT* __restrict__ z, const int64_t* __restrict__ csc_ptr,
             const uint32_t* __restrict__ csc_src, OutT* __restrict__ y,
             GatArgs a, unsigned long long* __restrict__ work) {
  constexpr int EPC = 16 / sizeof(ZT);
  extern __shared__ __align__(128) uint8_t gat_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t row_bytes = (uint32_t)(a.ldz * sizeof(ZT));
  uint64_t* bars = reinterpret_cast<uint64_t*>(gat_smem) + warp * kGatSlots;
  float* out_s = reinterpret_cast<float*>(gat_smem + kGatWarps * kGatSlots * 8) +
                 warp * (kMaxCols + kMaxHeads);
  float* er_s = out_s + kMaxCols;
  uint8_t* ring = gat_smem + kGatWarps * kGatSlots * 8 +
                  kGatWarps * (kMaxCols + kMaxHeads) * 4 +
                  (size_t)warp * kGatSlots * row_bytes;
  if (lane == 0) {
    for (int k = 0; k < kGatSlots; k++) mbar_init_cta(&bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // chunk j of lane l = 16-B chunk 32 j + l of the z part: its head, the
  // column of its first element inside the head, and its output column
  int head[CH], fcol[CH];
  bool act[CH];
#pragma unroll
  for (int j = 0; j < CH; j++) {
    const int c0 = (j * 32 + lane) * EPC;
    act[j] = c0 < a.heads * a.head_stride;
    head[j] = act[j] ? c0 / a.head_stride : 0;
    fcol[j] = c0 - head[j] * a.head_stride;
  }
  RowFeeder<kGatSlots, 4> feed{ring, bars, row_bytes, csc_src};
  while (true) {
    unsigned long long v0 = 0;
    if (lane == 0) v0 = atomicAdd(work, (unsigned long long)kGatGrab);
    v0 = __shfl_sync(0xffffffffu, v0, 0);
    if ((int64_t)v0 >= a.nloc) break;
    const int64_t v1 = min((int64_t)v0 + kGatGrab, a.nloc);
    const int64_t e0 = csc_ptr[v0], e1 = csc_ptr[v1];
    feed.begin(e0, e1, z, a.ldz);
    int64_t ce = e0;
    for (int64_t v = (int64_t)v0; v < v1; v++) {
      const int64_t dend = csc_ptr[v + 1];
      const int64_t vg = v + a.lo;
      __syncwarp();  // the previous destination's er_s readers are done
      if (lane < a.heads) er_s[lane] = to_f32(z[vg * a.ldz + a.er_col + lane]);
      __syncwarp();
      float m[CH], s[CH], acc[CH][EPC];
#pragma unroll
      for (int j = 0; j < CH; j++) {
        m[j] = -INFINITY;
        s[j] = 0.0f;
#pragma unroll
        for (int e = 0; e < EPC; e++) acc[j][e] = 0.0f;
      }
      for (; ce < dend; ce++) {
        const uint32_t row = feed.wait();
        const uint32_t rel = row + (uint32_t)(a.el_col * sizeof(ZT));
#pragma unroll
        for (int j = 0; j < CH; j++) {
          if (!act[j]) continue;
          ZChunk<ZT> f;
          f.raw = lds_v4(row + (uint32_t)(j * 32 + lane) * 16u);
          // online softmax, one exp per (edge, head): with d = x - m,
          // t = exp(-|d|) rescales the old state (d > 0) or weighs the new
          // edge (d <= 0)
          float x = lds_as_f32<ZT>(rel + (uint32_t)(head[j] * sizeof(ZT))) +
                    er_s[head[j]];
          x = x >= 0.0f ? x : a.slope * x;
          const float d = x - m[j];
          const float t = __expf(-fabsf(d));
          const bool up = d > 0.0f;
          const float sc = up ? t : 1.0f, p = up ? 1.0f : t;
          m[j] = up ? x : m[j];
          s[j] = fmaf(s[j], sc, p);
#pragma unroll
          for (int e = 0; e < EPC; e++)
            acc[j][e] = fmaf(acc[j][e], sc, p * f.get(e));
        }
        feed.release(z, a.ldz);
      }
      // epilogue: + bias, then concat (+ReLU) or mean over heads
      OutT* yrow = y + v * a.ldy;
#pragma unroll
      for (int j = 0; j < CH; j++) {
        if (!act[j]) continue;
        const float rs = s[j] > 0.0f ? 1.0f / s[j] : 0.0f;
#pragma unroll
        for (int e = 0; e < EPC; e++) {
          const int f = fcol[j] + e;
          if (f < a.head_dim) {
            const int c = head[j] * a.head_dim + f;
            float o = acc[j][e] * rs + a.bias[c];
            if (a.mean_heads) {
              out_s[c] = o;
            } else {
              if (a.relu) o = fmaxf(o, 0.0f);
              yrow[c] = out_cvt<OutT>(o);
            }
          }
        }
      }
      if (a.mean_heads) {
        __syncwarp();
        for (int f = lane; f < a.head_dim; f += 32) {
          float o = 0.0f;
          for (int h = 0; h < a.heads; h++) o += out_s[h * a.head_dim + f];
          o = o / (float)a.heads;
          if (a.relu) o = fmaxf(o, 0.0f);
          yrow[f] = out_cvt<OutT>(o);
        }
      }
    }
  }
}

template <typename ZT, typename OutT>
void gat_typed(const atlas_graph* g, const void* z, void* y, const GatArgs& a,
               cudaStream_t s) {
  constexpr int EPC = 16 / sizeof(ZT);
  g->work.reserve(1);
  ATLAS_CUDA(cudaMemsetAsync(g->work.ptr, 0, sizeof(unsigned long long), s));
  const int smem = kGatWarps * (kGatSlots * (8 + (int)(a.ldz * sizeof(ZT))) +
                                (kMaxCols + kMaxHeads) * 4);
  auto go = [&](auto kern) {
    ATLAS_CUDA(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    ATLAS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, kern, kGatWarps * 32, smem));
    kern<<<kNumSMs * std::max(1, per_sm), kGatWarps * 32, smem, s>>>(
        static_cast<const ZT*>(z), g->csc_ptr.ptr, g->csc_src.ptr,
        static_cast<OutT*>(y), a, g->work.ptr);
  };
  if (a.heads * a.head_stride <= 32 * EPC) go(gat_bulk<ZT, OutT, 1>);
  else go(gat_bulk<ZT, OutT, 2>);
  count_launch();
  ATLAS_LAUNCH_CHECK();
}

template <typename ZT>
void gat_by_out(const atlas_graph* g, const void* z, void* y, int y_dtype,
                const GatArgs& a, cudaStream_t s) {
  if (y_dtype == ATLAS_F32) gat_typed<ZT, float>(g, z, y, a, s);
  else if (y_dtype == ATLAS_F16) gat_typed<ZT, __half>(g, z, y, a, s);
  else gat_typed<ZT, __nv_bfloat16>(g, z, y, a, s);
}

}  // namespace

void launch_gat_aggregate(const atlas_graph* g, const void* z, int z_dtype,
                          int64_t ldz, int heads, int head_dim,
                          int head_stride, int el_col, int er_col,
                          const float* bias, int mean_heads, int relu,
                          float slope, void* y, int y_dtype, int64_t ldy,
                          cudaStream_t s) {
  const int zs = z_dtype == ATLAS_F32 ? 4 : 2;
  const int epc = 16 / zs;
  const int hf = heads * head_dim;
  const int zw = heads * head_stride;
  if (heads < 1 || heads > kMaxHeads || head_dim < 1 || hf > kMaxCols ||
      zw > 2 * 32 * epc)
    fail(ATLAS_ECONFIG, "gat: heads <= 8 and heads*head_dim <= 256 "
                        "(128 for f16/bf16 z)");
  if (head_stride < head_dim || head_stride % epc != 0)
    fail(ATLAS_ECONFIG, "gat: head stride must cover head_dim in whole "
                        "16-byte chunks");
  if ((ldz * zs) % 16 != 0 || (reinterpret_cast<uintptr_t>(z) & 15) != 0)
    fail(ATLAS_ECONFIG, "gat: z rows must be 16-byte aligned");
  if (el_col < zw || er_col < el_col + heads || er_col + heads > ldz)
    fail(ATLAS_ECONFIG, "gat: el/er columns must follow the z part");
  if (ldy < (mean_heads ? head_dim : hf))
    fail(ATLAS_ECONFIG, "gat: output leading dimension too small");
  if (g->nloc == 0) return;
  GatArgs a{ldz,        ldy,     g->lo,  g->nloc,    heads, head_dim,
            head_stride, hf,     el_col, er_col,     mean_heads, relu,
            slope,      bias};
  if (z_dtype == ATLAS_F32) gat_by_out<float>(g, z, y, y_dtype, a, s);
  else if (z_dtype == ATLAS_F16) gat_by_out<__half>(g, z, y, y_dtype, a, s);
  else gat_by_out<__nv_bfloat16>(g, z, y, y_dtype, a, s);
}

}  // namespace atlas
