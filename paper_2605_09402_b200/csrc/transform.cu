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


// ---------------------------------------------------------------------------
// Register-tiled persistent variant (the one normally taken). W^T lives in
// shared memory for the whole kernel (read from HBM/L2 once per CTA); x
// streams through two 128 x 16 shared tiles, staged through registers one
// tile ahead so the global loads overlap the previous tile's math. Each
// thread owns an 8 x TN block of outputs and still evaluates every element
// as the reference's sequential chain (k ascending, __fmul_rn then
// __fadd_rn): tiling changes which thread does the work, not the order of
// any element's operations, so the output stays bit-identical.
// The chain is FMUL + FADD per term, which makes this kernel FP32-issue
// bound: 2*M*K*N instructions. (The packed f32x2 pipe was tried: ptxas
// contracts mul.rn.f32x2 + add.rn.f32x2 into one FFMA2 even under
// `asm volatile` and -fmad=false; an fma with an opaque -0.0 addend avoids
// that and stays bit-exact, but measured 6% slower than scalar on B200.)

constexpr int kTM = 8, kRBM = 128, kRBK = 16, kAsLd = kRBM + 4;

template <typename OutT, int TN, bool VX>
__global__ void __launch_bounds__(256, 2)
    transform_stable_tiled(const float* __restrict__ x, int64_t ldx,
                           int64_t M, int K, const float* __restrict__ w,
                           const float* __restrict__ b, int N, int relu,
                           OutT* __restrict__ y, int64_t ldy,
                           int32_t* __restrict__ flag) {
  constexpr int BN = 16 * TN;
  extern __shared__ __align__(16) float tsm[];
  float* Ws = tsm;                              // [Kpad][BN]
  const int Kpad = (K + kRBK - 1) / kRBK * kRBK;
  float* As = tsm + (size_t)Kpad * BN;          // [2][kRBK][kAsLd]
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  for (int e = tid; e < Kpad * BN; e += 256) {
    const int n = e / Kpad, k = e % Kpad;  // W row-major (N, K): coalesced
    Ws[k * BN + n] = (n < N && k < K) ? w[(int64_t)n * K + k] : 0.0f;
  }
  float bias[TN];
#pragma unroll
  for (int j = 0; j < TN; j++) {
    const int n = tx * TN + j;
    bias[j] = n < N ? b[n] : 0.0f;
  }
  const int64_t ntiles = (M + kRBM - 1) / kRBM;
  const int nk = Kpad / kRBK;
  const int64_t my_tiles =
      blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t iters = my_tiles * nk;

  // staging: thread covers rows r = (tid + 256*q) >> 2, k quad (e & 3) * 4
  float stage[2][4];
  auto load = [&](int64_t it) {
    const int64_t t = blockIdx.x + (it / nk) * gridDim.x;
    const int k0 = (int)(it % nk) * kRBK;
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const int e = tid + 256 * q;
      const int row = e >> 2, kq = (e & 3) * 4;
      const int64_t gm = t * kRBM + row;
      const int gk = k0 + kq;
      if (VX) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (gm < M && gk < K)
          v = __ldg(reinterpret_cast<const float4*>(x + gm * ldx + gk));
        stage[q][0] = v.x; stage[q][1] = v.y; stage[q][2] = v.z;
        stage[q][3] = v.w;
      } else {
#pragma unroll
        for (int j = 0; j < 4; j++)
          stage[q][j] = (gm < M && gk + j < K) ? __ldg(x + gm * ldx + gk + j)
                                                : 0.0f;
      }
    }
  };
  auto store = [&](int buf) {
    float* A = As + buf * (kRBK * kAsLd);
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const int e = tid + 256 * q;
      const int row = e >> 2, kq = (e & 3) * 4;
#pragma unroll
      for (int j = 0; j < 4; j++) A[(kq + j) * kAsLd + row] = stage[q][j];
    }
  };

  float acc[kTM][TN];
  auto reset = [&]() {
#pragma unroll
    for (int i = 0; i < kTM; i++)
#pragma unroll
      for (int j = 0; j < TN; j++) acc[i][j] = bias[j];
  };
  reset();
  int bad = 0;
  if (iters > 0) {
    load(0);
    store(0);
  }
  __syncthreads();
  for (int64_t it = 0; it < iters; it++) {
    if (it + 1 < iters) load(it + 1);
    const float* A = As + (it & 1) * (kRBK * kAsLd);
    const int k0 = (int)(it % nk) * kRBK;
    auto step = [&](int kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&A[kk * kAsLd + ty * kTM]);
      const float4 a1 = *reinterpret_cast<const float4*>(&A[kk * kAsLd + ty * kTM + 4]);
      const float av[kTM] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float wv[TN];
      const float* wr = &Ws[(k0 + kk) * BN + tx * TN];
      if (TN % 4 == 0) {
#pragma unroll
        for (int j = 0; j < TN; j += 4) {
          const float4 q = *reinterpret_cast<const float4*>(wr + j);
          wv[j] = q.x; wv[j + 1] = q.y; wv[j + 2] = q.z; wv[j + 3] = q.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < TN; j++) wv[j] = wr[j];
      }
#pragma unroll
      for (int i = 0; i < kTM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++)
          acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], wv[j]));
    };
    if (k0 + kRBK <= K) {
#pragma unroll
      for (int kk = 0; kk < kRBK; kk++) step(kk);
    } else {
      for (int kk = 0; kk < K - k0; kk++) step(kk);
    }
    if ((it + 1) % nk == 0) {  // last k tile of this row tile: epilogue
      const int64_t t = blockIdx.x + (it / nk) * gridDim.x;
#pragma unroll
      for (int i = 0; i < kTM; i++) {
        const int64_t m = t * kRBM + ty * kTM + i;
        if (m < M) {
          OutT* yr = y + m * ldy + tx * TN;
#pragma unroll
          for (int j = 0; j < TN; j++) {
            if (tx * TN + j < N) {
              float v = acc[i][j];
              if (relu) v = relu_np(v);
              const OutT o = cast_out<OutT>(v);
              yr[j] = o;
              bad |= is_extreme(to_f32(o));
            }
          }
        }
      }
      reset();
    }
    if (it + 1 < iters) store((int)((it + 1) & 1));
    __syncthreads();
  }
  if (__syncthreads_or(bad) && flag && threadIdx.x == 0) atomicOr(flag, 1);
}

template <typename OutT, int TN>
bool tiled_go(const float* x, int64_t rows, int64_t k, int64_t ldx,
              const float* w, const float* b, int64_t n, int relu, OutT* y,
              int64_t ldy, int32_t* flag, cudaStream_t s) {
  const int64_t kpad = (k + kRBK - 1) / kRBK * kRBK;
  const size_t smem =
      sizeof(float) * ((size_t)kpad * 16 * TN + 2 * kRBK * kAsLd);
  if (smem > 200 * 1024) return false;
  const bool vx = ldx % 4 == 0 && k % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  auto kern = vx ? transform_stable_tiled<OutT, TN, true>
                 : transform_stable_tiled<OutT, TN, false>;
  ATLAS_CUDA(cudaFuncSetAttribute(
      kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  ATLAS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256,
                                                           smem));
  int dev = 0, sms = 0;
  ATLAS_CUDA(cudaGetDevice(&dev));
  ATLAS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t tiles = (rows + kRBM - 1) / kRBM;
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)sms * std::max(1, per_sm));
  kern<<<grid, 256, smem, s>>>(x, ldx, rows, (int)k, w, b, (int)n, relu, y,
                               ldy, flag);
  return true;
}

template <typename OutT>
bool tiled_typed(const float* x, int64_t rows, int64_t k, int64_t ldx,
                 const float* w, const float* b, int64_t n, int relu, OutT* y,
                 int64_t ldy, int32_t* flag, cudaStream_t s) {
  if (n > 128) return false;
  if (n > 64) return tiled_go<OutT, 8>(x, rows, k, ldx, w, b, n, relu, y, ldy, flag, s);
  if (n > 48) return tiled_go<OutT, 4>(x, rows, k, ldx, w, b, n, relu, y, ldy, flag, s);
  if (n > 32) return tiled_go<OutT, 3>(x, rows, k, ldx, w, b, n, relu, y, ldy, flag, s);
  return tiled_go<OutT, 2>(x, rows, k, ldx, w, b, n, relu, y, ldy, flag, s);
}

}  // namespace

void launch_transform_stable(const float* x, int64_t rows, int64_t k,
                             int64_t ldx, const float* w, const float* b,
                             int64_t n, int relu, void* y, int y_dtype,
                             int64_t ldy, int32_t* flag, cudaStream_t s) {
  if (rows <= 0 || n <= 0) return;
  bool done = false;
  if (y_dtype == ATLAS_F32)
    done = tiled_typed(x, rows, k, ldx, w, b, n, relu, static_cast<float*>(y),
                       ldy, flag, s);
  else if (y_dtype == ATLAS_F16)
    done = tiled_typed(x, rows, k, ldx, w, b, n, relu, static_cast<__half*>(y),
                       ldy, flag, s);
  else
    done = tiled_typed(x, rows, k, ldx, w, b, n, relu,
                       static_cast<__nv_bfloat16*>(y), ldy, flag, s);
  if (done) {
    count_launch();
    ATLAS_LAUNCH_CHECK();
    return;
  }
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
