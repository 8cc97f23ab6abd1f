// Dense layer transform, "stable" backend (kernel plan K9, SIMT variant).
//
// The reference's default MatmulBackend (oocgnn/compute.py:25-47) computes
// out = bias; for k in 0..K-1: out += batch[:, k] * W[:, k], i.e. every
// output element is a fixed-order chain of separately rounded f32
// multiplies and adds, independent of how rows are batched. This kernel
// evaluates exactly that chain per output element (k ascending,
// __fmul_rn then __fadd_rn, no FMA contraction), so its output is
// bit-identical to the reference's default backend. ReLU follows
// np.maximum(out, 0.0): NaN and -0.0 pass through unchanged.
//
// The fast tensor-core backend (tcgen05, transform_tc.cu) trades this
// bit-identity for throughput under a stated tolerance.
#include "internal.cuh"

namespace atlas {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

__device__ __forceinline__ float relu_np(float v) {
  return (v >= 0.0f || v != v) ? v : 0.0f;
}

template <typename OutT>
__device__ __forceinline__ OutT cast_out(float v);
template <>
__device__ __forceinline__ float cast_out<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half cast_out<__half>(float v) {
  return __float2half_rn(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 cast_out<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

template <typename OutT>
__global__ void __launch_bounds__(256)
    transform_stable_kernel(const float* __restrict__ x, int64_t ldx,
                            int64_t M, int K, const float* __restrict__ w,
                            const float* __restrict__ b, int N, int relu,
                            OutT* __restrict__ y, int64_t ldy,
                            int32_t* __restrict__ flag) {
  __shared__ __align__(16) float As[BK][BM];
  __shared__ __align__(16) float Ws[BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  float acc[4][4];
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const int n = n0 + tx * 4 + j;
    const float bias = n < N ? b[n] : 0.0f;
#pragma unroll
    for (int i = 0; i < 4; i++) acc[i][j] = bias;
  }
  for (int k0 = 0; k0 < K; k0 += BK) {
    // 64x16 tiles of x and w, 4 elements per thread, transposed to [k][m]
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int e = tid + r * 256;
      const int row = e / BK, kk = e % BK;
      const int64_t gm = m0 + row;
      const int gk = k0 + kk;
      As[kk][row] = (gm < M && gk < K) ? x[gm * ldx + gk] : 0.0f;
      const int gn = n0 + row;
      Ws[kk][row] = (gn < N && gk < K) ? w[(int64_t)gn * K + gk] : 0.0f;
    }
    __syncthreads();
    const int kmax = min(BK, K - k0);
    for (int kk = 0; kk < kmax; kk++) {
      float a[4];
#pragma unroll
      for (int i = 0; i < 4; i++) a[i] = As[kk][ty * 4 + i];
      const float4 bw = *reinterpret_cast<const float4*>(&Ws[kk][tx * 4]);
      const float bv[4] = {bw.x, bw.y, bw.z, bw.w};
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++)
          acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], bv[j]));
    }
    __syncthreads();
  }
  int bad = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (relu) v = relu_np(v);
      const OutT o = cast_out<OutT>(v);
      y[m * ldy + n] = o;
      bad |= is_extreme(to_f32(o));
    }
  }
  if (__syncthreads_or(bad) && flag && threadIdx.x == 0) atomicOr(flag, 1);
}

}  // namespace

void launch_transform_stable(const float* x, int64_t rows, int64_t k,
                             int64_t ldx, const float* w, const float* b,
                             int64_t n, int relu, void* y, int y_dtype,
                             int64_t ldy, int32_t* flag, cudaStream_t s) {
  if (rows <= 0 || n <= 0) return;
  dim3 grid((unsigned)ceil_div(rows, BM), (unsigned)ceil_div(n, BN));
  if (y_dtype == ATLAS_F32)
    transform_stable_kernel<float><<<grid, 256, 0, s>>>(
        x, ldx, rows, (int)k, w, b, (int)n, relu, static_cast<float*>(y), ldy,
        flag);
  else if (y_dtype == ATLAS_F16)
    transform_stable_kernel<__half><<<grid, 256, 0, s>>>(
        x, ldx, rows, (int)k, w, b, (int)n, relu, static_cast<__half*>(y),
        ldy, flag);
  else
    transform_stable_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
        x, ldx, rows, (int)k, w, b, (int)n, relu,
        static_cast<__nv_bfloat16*>(y), ldy, flag);
  count_launch();
  ATLAS_LAUNCH_CHECK();
}

}  // namespace atlas
