// GAT pass B: edge-softmax-weighted broadcast aggregation (kernel plan K10,
// SURVEY.md §2.1 and A.5). The reference has no GAT; the
// semantics are oracle/gat.py's (DGL GATConv style):
//
//   e_uv[h] = LeakyReLU(el_u[h] + er_v[h]),  alpha = softmax_{u in N(v)} e
//   out_v[h] = sum_u alpha_uv[h] z_u[h] + b[h]   (concat, or mean over h)
//
// Pass A (transform first) is the tcgen05 GEMM z_ext = x . W_ext^T whose
// extra output columns are el and er (W_ext rows a_l[h]^T W_h, a_r[h]^T W_h),
// so every source row streamed here carries [z | el | er].
//
// Mapping: one warp per destination (CSC view of the rank's range). Lanes
// own 16-byte column chunks of z. Per 32-edge batch, lane i scores edge i
// for every head (warp max + online sum, exact two-pass softmax because the
// whole in-edge list is resident), writes alpha_i[h] to shared memory, then
// the warp streams the z rows with 8 independent 16-byte loads in flight per
// lane and accumulates alpha * z in f32. The head mean / bias / ReLU
// epilogue is fused, so no f32 record ever goes back to HBM: the kernel
// reads E x (z row) + E x (el) and writes V x out.
#include "internal.cuh"

namespace atlas {
namespace {

constexpr int kGatWarps = 8;
constexpr int kMaxHeads = 8;
constexpr int kMaxCols = 256;
constexpr int kGatUnroll = 8;

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

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct GatArgs {
  int64_t ldz, ldy, lo, nloc;
  int heads, head_dim, hf, el_col, er_col, mean_heads, relu;
  float slope;
  const float* bias;
};

template <typename ZT, typename OutT, int CH>
__global__ void __launch_bounds__(kGatWarps * 32, CH == 1 ? 3 : 2)
    gat_aggregate(const ZT* __restrict__ z, const int64_t* __restrict__ csc_ptr,
                  const uint32_t* __restrict__ csc_src, OutT* __restrict__ y,
                  GatArgs a) {
  constexpr int EPC = 16 / sizeof(ZT);
  __shared__ float alpha_s[kGatWarps][32][kMaxHeads];
  __shared__ float out_s[kGatWarps][kMaxCols];
  __shared__ float stat_s[kGatWarps][3][kMaxHeads];  // er, max, 1/sum
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t v = (int64_t)blockIdx.x * kGatWarps + warp;
  if (v >= a.nloc) return;
  const int64_t vg = v + a.lo;
  const int64_t beg = csc_ptr[v], end = csc_ptr[v + 1];
  const int H = a.heads;

  // head of every element this lane owns
  int hidx[CH][EPC];
  bool act[CH];
#pragma unroll
  for (int j = 0; j < CH; j++) {
    act[j] = (j * 32 + lane) * EPC < a.hf;
#pragma unroll
    for (int e = 0; e < EPC; e++) {
      const int c = (j * 32 + lane) * EPC + e;
      hidx[j][e] = c < a.hf ? c / a.head_dim : 0;
    }
  }
  float er[kMaxHeads], m[kMaxHeads], s[kMaxHeads];
#pragma unroll
  for (int h = 0; h < kMaxHeads; h++) {
    er[h] = h < H ? to_f32(z[vg * a.ldz + a.er_col + h]) : 0.0f;
    m[h] = -INFINITY;
    s[h] = 0.0f;
  }
  auto score = [&](uint32_t u, int h) {
    const float x = to_f32(z[(int64_t)u * a.ldz + a.el_col + h]) + er[h];
    return x >= 0.0f ? x : a.slope * x;
  };
  // phase 1: per-head max and normaliser over all in-edges
  for (int64_t base = beg; base < end; base += 32) {
    const bool ok = base + lane < end;
    const uint32_t u = ok ? csc_src[base + lane] : 0u;
#pragma unroll
    for (int h = 0; h < kMaxHeads; h++) {
      if (h >= H) break;
      const float e = ok ? score(u, h) : -INFINITY;
      const float mn = fmaxf(m[h], warp_max(e));
      const float p = ok ? __expf(e - mn) : 0.0f;
      s[h] = s[h] * __expf(m[h] - mn) + warp_sum(p);
      m[h] = mn;
    }
  }
  if (lane < H) {
    stat_s[warp][0][lane] = to_f32(z[vg * a.ldz + a.er_col + lane]);
    float mh = m[0], sh = s[0];
#pragma unroll
    for (int h = 1; h < kMaxHeads; h++)
      if (h == lane) mh = m[h], sh = s[h];
    stat_s[warp][1][lane] = mh;
    stat_s[warp][2][lane] = sh > 0.0f ? 1.0f / sh : 0.0f;
  }
  __syncwarp();

  float acc[CH][EPC];
#pragma unroll
  for (int j = 0; j < CH; j++)
#pragma unroll
    for (int e = 0; e < EPC; e++) acc[j][e] = 0.0f;

  // phase 2: alpha per edge, then the weighted row sum
  for (int64_t base = beg; base < end; base += 32) {
    const int cnt = (int)((end - base) < 32 ? (end - base) : 32);
    const bool ok = lane < cnt;
    const uint32_t u = ok ? csc_src[base + lane] : 0u;
#pragma unroll
    for (int h = 0; h < kMaxHeads; h++) {
      if (h >= H) break;
      if (ok) {
        float x = to_f32(z[(int64_t)u * a.ldz + a.el_col + h]) +
                  stat_s[warp][0][h];
        x = x >= 0.0f ? x : a.slope * x;
        alpha_s[warp][lane][h] =
            __expf(x - stat_s[warp][1][h]) * stat_s[warp][2][h];
      }
    }
    __syncwarp();
    for (int k = 0; k < cnt; k += kGatUnroll) {
      ZChunk<ZT> f[kGatUnroll][CH];
#pragma unroll
      for (int t = 0; t < kGatUnroll; t++) {
        const uint32_t ut = __shfl_sync(0xffffffffu, u, (k + t) & 31);
        if (k + t < cnt) {
#pragma unroll
          for (int j = 0; j < CH; j++)
            if (act[j])
              f[t][j].raw = __ldg(reinterpret_cast<const uint4*>(
                  z + (int64_t)ut * a.ldz + (j * 32 + lane) * EPC));
        }
      }
#pragma unroll
      for (int t = 0; t < kGatUnroll; t++) {
        if (k + t < cnt) {
#pragma unroll
          for (int j = 0; j < CH; j++)
            if (act[j]) {
#pragma unroll
              for (int e = 0; e < EPC; e++)
                acc[j][e] = fmaf(alpha_s[warp][k + t][hidx[j][e]],
                                 f[t][j].get(e), acc[j][e]);
            }
        }
      }
    }
    __syncwarp();
  }

  // epilogue: + bias, then concat (+ReLU) or mean over heads
  OutT* yrow = y + v * a.ldy;
  if (!a.mean_heads) {
#pragma unroll
    for (int j = 0; j < CH; j++)
#pragma unroll
      for (int e = 0; e < EPC; e++) {
        const int c = (j * 32 + lane) * EPC + e;
        if (c < a.hf) {
          float o = acc[j][e] + a.bias[c];
          if (a.relu) o = fmaxf(o, 0.0f);
          yrow[c] = out_cvt<OutT>(o);
        }
      }
    return;
  }
#pragma unroll
  for (int j = 0; j < CH; j++)
#pragma unroll
    for (int e = 0; e < EPC; e++) {
      const int c = (j * 32 + lane) * EPC + e;
      if (c < a.hf) out_s[warp][c] = acc[j][e] + a.bias[c];
    }
  __syncwarp();
  for (int f = lane; f < a.head_dim; f += 32) {
    float o = 0.0f;
    for (int h = 0; h < H; h++) o += out_s[warp][h * a.head_dim + f];
    o = o / (float)H;
    if (a.relu) o = fmaxf(o, 0.0f);
    yrow[f] = out_cvt<OutT>(o);
  }
}

template <typename ZT, typename OutT>
void gat_typed(const atlas_graph* g, const void* z, void* y, const GatArgs& a,
               cudaStream_t s) {
  constexpr int EPC = 16 / sizeof(ZT);
  const unsigned grid = (unsigned)ceil_div(a.nloc, kGatWarps);
  if (a.hf <= 32 * EPC)
    gat_aggregate<ZT, OutT, 1><<<grid, kGatWarps * 32, 0, s>>>(
        static_cast<const ZT*>(z), g->csc_ptr.ptr, g->csc_src.ptr,
        static_cast<OutT*>(y), a);
  else
    gat_aggregate<ZT, OutT, 2><<<grid, kGatWarps * 32, 0, s>>>(
        static_cast<const ZT*>(z), g->csc_ptr.ptr, g->csc_src.ptr,
        static_cast<OutT*>(y), a);
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
                          int64_t ldz, int heads, int head_dim, int el_col,
                          int er_col, const float* bias, int mean_heads,
                          int relu, float slope, void* y, int y_dtype,
                          int64_t ldy, cudaStream_t s) {
  const int zs = z_dtype == ATLAS_F32 ? 4 : 2;
  const int hf = heads * head_dim;
  if (heads < 1 || heads > kMaxHeads || head_dim < 1 || hf > kMaxCols ||
      hf > 2 * 32 * (16 / zs))
    fail(ATLAS_ECONFIG, "gat: heads <= 8 and heads*head_dim <= 256 "
                        "(128 for f16/bf16 z)");
  if ((ldz * zs) % 16 != 0 || (reinterpret_cast<uintptr_t>(z) & 15) != 0)
    fail(ATLAS_ECONFIG, "gat: z rows must be 16-byte aligned");
  const int epc = 16 / zs;
  if (el_col < ((hf + epc - 1) / epc) * epc || er_col < el_col + heads ||
      er_col + heads > ldz)
    fail(ATLAS_ECONFIG, "gat: el/er columns must follow the padded z part");
  if (ldy < (mean_heads ? head_dim : hf))
    fail(ATLAS_ECONFIG, "gat: output leading dimension too small");
  if (g->nloc == 0) return;
  GatArgs a{ldz, ldy, g->lo, g->nloc, heads, head_dim, hf, el_col, er_col,
            mean_heads, relu, slope, bias};
  if (z_dtype == ATLAS_F32) gat_by_out<float>(g, z, y, y_dtype, a, s);
  else if (z_dtype == ATLAS_F16) gat_by_out<__half>(g, z, y, y_dtype, a, s);
  else gat_by_out<__nv_bfloat16>(g, z, y, y_dtype, a, s);
}

}  // namespace atlas
