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
  // a_l at the strided z columns (heads x head_stride, zero pads); set when
  // gat_ring recomputes el per edge (f32 z of <= 128 columns)
  const float* attn_l;
  int lph;  // lanes per head
};

// The z part of a row stores head h at columns [h*stride, h*stride + F)
// with stride = F rounded up to a 16-byte chunk, so the EPC elements of a
// lane's chunk always share one head and one online-softmax state.
// PAIR: a z row needs at most 16 lanes (f16/bf16 z of <= 128 columns), so
// the two half-warps take alternate in-edges of the destination and merge
// their online-softmax states at its end
template <typename ZT, typename OutT, int CH, bool PAIR>
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
  static_assert(!PAIR || CH == 1, "paired half-warps use one chunk");
  const int half = PAIR ? lane >> 4 : 0;      // which edge of a pair
  const int cl = PAIR ? (lane & 15) : lane;   // chunk lane within the row
  int head[CH], fcol[CH];
  bool act[CH];
#pragma unroll
  for (int j = 0; j < CH; j++) {
    const int c0 = (j * 32 + cl) * EPC;
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
      while (ce < dend) {
        // PAIR: half-warp h takes edge ce + h (when it exists)
        const bool two = PAIR && ce + 1 < dend;
        const bool mine = !PAIR || half == 0 || two;
        const uint32_t row = mine ? feed.wait_k(PAIR ? half : 0) : 0u;
        const uint32_t rel = row + (uint32_t)(a.el_col * sizeof(ZT));
#pragma unroll
        for (int j = 0; j < CH; j++) {
          if (!act[j] || !mine) continue;
          ZChunk<ZT> f;
          f.raw = lds_v4(row + (uint32_t)(j * 32 + cl) * 16u);
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
        feed.release_n(two ? 2u : 1u, z, a.ldz);
        ce += two ? 2 : 1;
      }
      if (PAIR) {  // merge the two half-warps' (m, s, acc) of each chunk
#pragma unroll
        for (int j = 0; j < CH; j++) {
          const float mo = __shfl_xor_sync(0xffffffffu, m[j], 16);
          const float so = __shfl_xor_sync(0xffffffffu, s[j], 16);
          const float mm = fmaxf(m[j], mo);
          const float f1 = m[j] == -INFINITY ? 0.0f : __expf(m[j] - mm);
          const float f2 = mo == -INFINITY ? 0.0f : __expf(mo - mm);
          s[j] = s[j] * f1 + so * f2;
          m[j] = mm;
#pragma unroll
          for (int e = 0; e < EPC; e++) {
            const float ao = __shfl_xor_sync(0xffffffffu, acc[j][e], 16);
            acc[j][e] = acc[j][e] * f1 + ao * f2;
          }
        }
      }
      // epilogue: + bias, then concat (+ReLU) or mean over heads
      OutT* yrow = y + v * a.ldy;
#pragma unroll
      for (int j = 0; j < CH; j++) {
        if (!act[j] || half != 0) continue;
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

// f32 z rows of <= 128 columns: the per-lane cp.async ring of agg_ring, moving ONLY the z part of
// each source row (line-aligned rows, gat.ZLayout), with el_u = a_l . z_u
// recomputed per edge by a reduction over the head's lanes (butterfly for
// power-of-two lane groups, else a segmented tree). DRAM moves
// whole 128-byte lines for these random rows, so a [z | el] row costs 5-6
// lines and a bare 512-byte z row exactly 4.
constexpr int kGatRing = 8;
constexpr int kGatRingWarps = 8;

// LPH > 0: lanes per head (power of two, butterfly); LPH <= 0: any lane
// count, reduced in -LPH segmented steps
template <typename OutT, int LPH>
__global__ void __launch_bounds__(kGatRingWarps * 32, 4)
    gat_ring(const float* __restrict__ z, const int64_t* __restrict__ csc_ptr,
             const uint32_t* __restrict__ csc_src, OutT* __restrict__ y,
             GatArgs a, unsigned long long* __restrict__ work) {
  extern __shared__ __align__(128) uint8_t gr_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per warp: z ring (kGatRing x 32 lanes x 16 B), output staging
  // (kMaxCols floats), er (kMaxHeads floats)
  uint8_t* wbase = gr_smem + (size_t)warp * (kGatRing * 512 +
                                              (kMaxCols + kMaxHeads) * 4);
  const uint32_t zring = (uint32_t)__cvta_generic_to_shared(wbase) +
                         (uint32_t)lane * 16u;
  float* out_s = reinterpret_cast<float*>(wbase + kGatRing * 512);
  float* er_s = out_s + kMaxCols;
  const int zw = a.heads * a.head_stride;  // z columns
  const int c0 = lane * 4;
  const bool act = c0 < zw;
  const int head = act ? c0 / a.head_stride : 0;
  const int fcol = c0 - head * a.head_stride;
  const int hlead = head * a.lph, hl = lane - hlead;  // lane within head
  uint32_t seg = 0;  // bit k: the lane 2^k further on is in this head
  for (int k = 0; k < 5; k++) seg |= (uint32_t)(hl + (1 << k) < a.lph) << k;
  const int colc = act ? c0 : zw - 4;  // clamped: branch-free copies
  // source row address = zbase + u * pitch (one IMAD.WIDE per edge)
  const uint64_t zbase = reinterpret_cast<uint64_t>(z + colc);
  const uint32_t pitch = (uint32_t)(a.ldz * 4);
  // scores in the log2 domain: leaky ReLU is positively homogeneous, so
  // scaling a_l and er by log2(e) lets ex2 stand in for exp
  constexpr float kLog2e = 1.4426950408889634f;
  float al[4];
#pragma unroll
  for (int e = 0; e < 4; e++) al[e] = act ? a.attn_l[c0 + e] * kLog2e : 0.0f;
  while (true) {
    unsigned long long v0 = 0;
    if (lane == 0) v0 = atomicAdd(work, (unsigned long long)kGatGrab);
    v0 = __shfl_sync(0xffffffffu, v0, 0);
    if ((int64_t)v0 >= a.nloc) break;
    const int64_t v1 = min((int64_t)v0 + kGatGrab, a.nloc);
    const int64_t e0 = csc_ptr[v0];
    const int ne = (int)(csc_ptr[v1] - e0);
    const uint32_t* __restrict__ src0 = csc_src + e0;
    int pe = 0;
    uint32_t isrc = lane < ne ? src0[lane] : 0u;
    auto issue = [&]() {
      if (pe < ne) {
        if ((pe & 31) == 0 && pe != 0)
          isrc = pe + lane < ne ? src0[pe + lane] : 0u;
        const uint32_t u = __shfl_sync(0xffffffffu, isrc, pe & 31);
        cp_async16_s(zring + ((uint32_t)(pe & (kGatRing - 1)) << 9),
                     reinterpret_cast<const void*>(
                         zbase + (uint64_t)u * pitch));
        pe++;
      }
      cp_async_commit();  // empty groups keep the wait count uniform
    };
#pragma unroll 1
    for (int k = 0; k < kGatRing; k++) issue();
    int ce = 0;
    for (int64_t v = (int64_t)v0; v < v1; v++) {
      const int dend = (int)(csc_ptr[v + 1] - e0);
      const int64_t vg = v + a.lo;
      if (lane < a.heads) er_s[lane] = z[vg * a.ldz + a.er_col + lane];
      __syncwarp();
      const float er = er_s[head] * kLog2e;
      float m = -INFINITY, sum = 0.0f, acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (; ce < dend; ce++) {
        cp_async_wait<kGatRing - 1>();  // this lane's chunk of edge ce
        const uint4 r = lds16(zring + ((uint32_t)(ce & (kGatRing - 1)) << 9));
        const float zf[4] = {__uint_as_float(r.x), __uint_as_float(r.y),
                             __uint_as_float(r.z), __uint_as_float(r.w)};
        // el_u[head] = a_l . z_u, reduced over the head's aligned lane group
        float x = al[0] * zf[0];
#pragma unroll
        for (int e = 1; e < 4; e++) x = fmaf(al[e], zf[e], x);
        if constexpr (LPH > 0) {
#pragma unroll
          for (int o = 1; o < LPH; o <<= 1)
            x += __shfl_xor_sync(0xffffffffu, x, o);
        } else {  // -LPH steps of a segmented tree to the head's first lane
#pragma unroll
          for (int k = 0; k < -LPH; k++) {
            const float y = __shfl_down_sync(0xffffffffu, x, 1 << k);
            if (seg >> k & 1) x += y;
          }
          x = __shfl_sync(0xffffffffu, x, hlead);
        }
        x += er;
        x = x >= 0.0f ? x : a.slope * x;
        // online softmax, one exp per edge (see gat_bulk)
        const float d = x - m;
        float t;  // 2^-|d| (ftz: underflow to 0 is the exp's own limit)
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(-fabsf(d)));
        const bool up = d > 0.0f;
        const float sc = up ? t : 1.0f, p = up ? 1.0f : t;
        m = up ? x : m;
        sum = fmaf(sum, sc, p);
#pragma unroll
        for (int e = 0; e < 4; e++) acc[e] = fmaf(acc[e], sc, p * zf[e]);
        issue();  // each lane refills only the slot it just read
      }
      // epilogue: + bias, then concat (+ReLU) or mean over heads
      OutT* yrow = y + v * a.ldy;
      const float rs = sum > 0.0f ? 1.0f / sum : 0.0f;
      if (act) {
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const int f = fcol + e;
          if (f < a.head_dim) {
            const int c = head * a.head_dim + f;
            float o = acc[e] * rs + a.bias[c];
            if (a.mean_heads) {
              out_s[c] = o;
            } else {
              if (a.relu) o = fmaxf(o, 0.0f);
              yrow[c] = out_cvt<OutT>(o);
            }
          }
        }
      }
      __syncwarp();
      if (a.mean_heads) {
        for (int f = lane; f < a.head_dim; f += 32) {
          float o = 0.0f;
          for (int h = 0; h < a.heads; h++) o += out_s[h * a.head_dim + f];
          o = o / (float)a.heads;
          if (a.relu) o = fmaxf(o, 0.0f);
          yrow[f] = out_cvt<OutT>(o);
        }
        __syncwarp();
      }
    }
    cp_async_wait<0>();
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
    kern<<<num_sms() * std::max(1, per_sm), kGatWarps * 32, smem, s>>>(
        static_cast<const ZT*>(z), g->csc_ptr.ptr, g->csc_src.ptr,
        static_cast<OutT*>(y), a, g->work.ptr);
  };
  if (std::is_same<ZT, float>::value && a.attn_l) {
    const int rsmem = kGatRingWarps * (kGatRing * 512 +
                                       (kMaxCols + kMaxHeads) * 4);
    auto kern = a.lph == 1    ? gat_ring<OutT, 1>
                : a.lph == 2  ? gat_ring<OutT, 2>
                : a.lph == 4  ? gat_ring<OutT, 4>
                : a.lph == 8  ? gat_ring<OutT, 8>
                : a.lph == 16 ? gat_ring<OutT, 16>
                : a.lph == 32 ? gat_ring<OutT, 32>
                : a.lph <= 4  ? gat_ring<OutT, -2>
                : a.lph <= 8  ? gat_ring<OutT, -3>
                : a.lph <= 16 ? gat_ring<OutT, -4>
                              : gat_ring<OutT, -5>;
    ATLAS_CUDA(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, rsmem));
    int per_sm = 0;
    ATLAS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, kern, kGatRingWarps * 32, rsmem));
    kern<<<num_sms() * std::max(1, per_sm), kGatRingWarps * 32, rsmem, s>>>(
        reinterpret_cast<const float*>(z), g->csc_ptr.ptr, g->csc_src.ptr,
        static_cast<OutT*>(y), a, g->work.ptr);
  } else if (a.heads * a.head_stride <= 16 * EPC)
    go(gat_bulk<ZT, OutT, 1, true>);
  else if (a.heads * a.head_stride <= 32 * EPC)
    go(gat_bulk<ZT, OutT, 1, false>);
  else go(gat_bulk<ZT, OutT, 2, false>);
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
                          const float* attn_l, cudaStream_t s) {
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
  const int lph = head_stride / epc;
  const bool ring = attn_l && z_dtype == ATLAS_F32 && zw <= 128;
  GatArgs a{ldz,        ldy,     g->lo,  g->nloc,    heads, head_dim,
            head_stride, hf,     el_col, er_col,     mean_heads, relu,
            slope,      bias,    ring ? attn_l : nullptr, lph};
  if (z_dtype == ATLAS_F32) gat_by_out<float>(g, z, y, y_dtype, a, s);
  else if (z_dtype == ATLAS_F16) gat_by_out<__half>(g, z, y, y_dtype, a, s);
  else gat_by_out<__nv_bfloat16>(g, z, y, y_dtype, a, s);
}

}  // namespace atlas
