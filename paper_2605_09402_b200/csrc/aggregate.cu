// Broadcast scatter-aggregate (kernel plan K3/K4 of SURVEY.md §2.1).
//
// Reference semantics (oocgnn/orchestrator.py:262-268, :186-191): every
// addend is m = h_u / max(1, d_in(v)) for the mean models (GCN, SAGE) or
// m = h_u for GIN (its own self term is (1 + eps) * h_v), rounded to f32,
// and np.add.at applies the addends of one destination in stream
// (source-major) order onto a zeroed f32 record. Here each warp owns one
// destination and a 32*VEC column slice of its record; lanes walk the
// destination's sources in ascending order and apply exactly the same
// rounded f32 divide and add per column (correctly rounded division via
// div_rn below, __fadd_rn, no FMA contraction of the sum), so records are
// bit-identical to the reference for ANY chunking. Parallelism is over destinations and columns; memory-level
// parallelism comes from issuing UNROLL independent 16-byte row loads per
// lane before the dependent adds.
//
// Two front ends share the inner loop:
//  * resident: the whole layer input is in HBM; destinations are walked
//    through the CSC view (graph.cu) in one pass and each record is
//    written once (no read-modify-write). GIN's self term is inserted
//    before the first source >= v, which is its stream position.
//  * runs: one caller-supplied chunk tile; destination runs come from the
//    per-chunk stable sort (chunk.cu); a record is read back only if an
//    earlier chunk already touched it.
#include <cstdlib>
#include <string>
#include "bulk.cuh"

namespace atlas {
namespace {

constexpr int kUnroll = 8;
constexpr uint32_t kSelfBit = 0x80000000u;

// 16-byte (or narrower) raw row fragment of VEC elements.
template <typename T, int VEC>
struct Frag {
  static constexpr int kBytes = VEC * sizeof(T);
  using Raw = typename std::conditional<
      kBytes == 16, uint4,
      typename std::conditional<
          kBytes == 8, uint2,
          typename std::conditional<kBytes == 4, uint32_t,
                                    uint16_t>::type>::type>::type;
  Raw raw;
  __device__ __forceinline__ void load(const T* p) {
    raw = __ldg(reinterpret_cast<const Raw*>(p));
  }
  __device__ __forceinline__ float get(int e) const {
    const T* t = reinterpret_cast<const T*>(&raw);
    return to_f32(t[e]);
  }
  // elements e, e+1 (e even) as a float2 (exact widening)
  __device__ __forceinline__ float2 get2(int e) const {
    const T* t = reinterpret_cast<const T*>(&raw);
    if constexpr (std::is_same<T, __half>::value)
      return __half22float2(*reinterpret_cast<const __half2*>(t + e));
    else if constexpr (std::is_same<T, __nv_bfloat16>::value)
      return __bfloat1622float2(
          *reinterpret_cast<const __nv_bfloat162*>(t + e));
    else
      return make_float2(t[e], t[e + 1]);
  }
};

template <int VEC>
__device__ __forceinline__ void store_f32(float* p, const float (&a)[VEC]) {
  if constexpr (VEC % 4 == 0) {
#pragma unroll
    for (int e = 0; e < VEC; e += 4)
      *reinterpret_cast<float4*>(p + e) =
          make_float4(a[e], a[e + 1], a[e + 2], a[e + 3]);
  } else {
#pragma unroll
    for (int e = 0; e < VEC; e++) p[e] = a[e];
  }
}

template <int VEC>
__device__ __forceinline__ void load_f32(const float* p, float (&a)[VEC]) {
  if constexpr (VEC % 4 == 0) {
#pragma unroll
    for (int e = 0; e < VEC; e += 4) {
      float4 t = *reinterpret_cast<const float4*>(p + e);
      a[e] = t.x;
      a[e + 1] = t.y;
      a[e + 2] = t.z;
      a[e + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; e++) a[e] = p[e];
  }
}

// Correctly rounded m / d from the correctly rounded reciprocal r = RN(1/d)
// (Markstein): q = RN(m r); e = m - q d exactly (FMA); RN(q + e r) ==
// RN(m / d) whenever the quotient is a normal number or zero. Tiny or
// non-finite m (quotient possibly subnormal / NaN-producing residual) take
// the IEEE division. Exhaustively checked against RN(m / d) on 1e8 random
// (m, d) pairs (tests/test_cpu_boundary.py::test_markstein_division).
// GUARD=false is only used after scan_extremes() proved the layer input
// holds no such value (one read of the input per layer).
template <bool GUARD>
__device__ __forceinline__ float div_rn(float m, float d, float r) {
  if (GUARD) {
    const float am = fabsf(m);
    if ((am < 0x1p-100f && am != 0.0f) || !(am <= 3.402823466e38f))
      return __fdiv_rn(m, d);
  }
  const float q = __fmul_rn(m, r);
  const float e = __fmaf_rn(-q, d, m);
  return __fmaf_rn(e, r, q);
}

// a += (self ? m * self_scale : (MEAN ? m / denom : m)), per element.
// Unguarded even widths run on the packed f32x2 pipe (FMUL2/FFMA2/FADD2:
// two IEEE round-to-nearest results per instruction, the same bits as the
// scalar sequence; e = m - q d is formed as fma(q, -d, m), equal to
// fma(-q, d, m) since negation is exact).
template <typename T, int VEC, bool MEAN, bool GUARD = true>
__device__ __forceinline__ void add_msg(float (&a)[VEC],
                                        const Frag<T, VEC>& f, bool self,
                                        float denom, float rcp,
                                        float self_scale) {
  if constexpr (VEC % 2 == 0 && !GUARD) {
    const float2 r2 = make_float2(rcp, rcp);
    const float2 nd2 = make_float2(-denom, -denom);
    const float2 s2 = make_float2(self_scale, self_scale);
#pragma unroll
    for (int e = 0; e < VEC; e += 2) {
      float2 m = f.get2(e);
      if (self) {
        m = __fmul2_rn(m, s2);
      } else if (MEAN) {
        const float2 q = __fmul2_rn(m, r2);
        const float2 r = __ffma2_rn(q, nd2, m);
        m = __ffma2_rn(r, r2, q);
      }
      const float2 o = __fadd2_rn(make_float2(a[e], a[e + 1]), m);
      a[e] = o.x;
      a[e + 1] = o.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; e++) {
      float m = f.get(e);
      if (self)
        m = __fmul_rn(m, self_scale);
      else if (MEAN)
        m = div_rn<GUARD>(m, denom, rcp);
      a[e] = __fadd_rn(a[e], m);
    }
  }
}

// flag[0] |= 1 if any element of x (rows x d) is non-finite or a nonzero
// with |x| < 2^-100 (the inputs for which div_rn needs the IEEE path)
template <typename T>
__global__ void scan_extremes(const T* __restrict__ x, int64_t rows, int d,
                              int64_t ldx, int* __restrict__ flag) {
  int bad = 0;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
       r < rows; r += nwarps) {
    const T* row = x + r * ldx;
    for (int c = lane; c < d; c += 32) bad |= is_extreme(to_f32(row[c]));
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// dense rows (ldx == d): one flat pass with 16-byte loads
template <typename T>
__global__ void scan_extremes_flat(const T* __restrict__ x, int64_t n,
                                   int* __restrict__ flag) {
  constexpr int EPC = 16 / sizeof(T);
  const int64_t nvec = n / EPC;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += stride) {
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(x) + i);
    const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int k = 0; k < EPC; k++) bad |= is_extreme(to_f32(e[k]));
  }
  for (int64_t i = nvec * EPC + blockIdx.x * (int64_t)blockDim.x +
                   threadIdx.x;
       i < n; i += stride)
    bad |= is_extreme(to_f32(x[i]));
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

template <typename T>
void launch_scan(const T* x, int64_t rows, int d, int64_t ldx, int* flag,
                 cudaStream_t s) {
  if (ldx == d && (reinterpret_cast<uintptr_t>(x) & 15) == 0)
    scan_extremes_flat<T><<<num_sms() * 8, 256, 0, s>>>(x, rows * d, flag);
  else
    scan_extremes<T><<<num_sms() * 8, 256, 0, s>>>(x, rows, d, ldx, flag);
  count_launch();
  ATLAS_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// resident front end: warp per destination, CSC walk

template <typename T, int VEC, int MODEL, bool GUARD>
__device__ __forceinline__ void resident_body(
    const T* __restrict__ x, int64_t ldx, const int64_t* __restrict__ csc_ptr,
    const uint32_t* __restrict__ csc_src, const uint32_t* __restrict__ indeg,
    int64_t lo, int64_t v, int d, float* __restrict__ acc, int64_t ldacc,
    float self_scale) {
  constexpr bool kMean = MODEL != ATLAS_GIN;
  const int lane = threadIdx.x & 31;
  const int64_t beg = csc_ptr[v], end = csc_ptr[v + 1];
  const uint32_t vg = (uint32_t)(v + lo);
  const float denom = kMean ? (float)max(1u, indeg[v]) : 1.0f;
  const float rcp = kMean ? __frcp_rn(denom) : 1.0f;
  float* out = acc + v * ldacc;
  for (int c0 = 0; c0 < d; c0 += 32 * VEC) {
    const int col = c0 + lane * VEC;
    const bool active = col < d;
    float a[VEC];
#pragma unroll
    for (int e = 0; e < VEC; e++) a[e] = 0.0f;
    bool self_pending = MODEL == ATLAS_GIN;
    for (int64_t base = beg; base < end; base += 32) {
      const int cnt = (int)((end - base) < 32 ? (end - base) : 32);
      const uint32_t mine = lane < cnt ? csc_src[base + lane] : 0u;
      for (int i = 0; i < cnt; i += kUnroll) {
        Frag<T, VEC> f[kUnroll];
        uint32_t s[kUnroll];
#pragma unroll
        for (int j = 0; j < kUnroll; j++) {
          s[j] = __shfl_sync(0xffffffffu, mine, (i + j) & 31);
          if (active && i + j < cnt) f[j].load(x + (int64_t)s[j] * ldx + col);
        }
#pragma unroll
        for (int j = 0; j < kUnroll; j++) {
          if (i + j < cnt) {
            if (MODEL == ATLAS_GIN && self_pending && s[j] >= vg) {
              self_pending = false;
              if (active) {
                Frag<T, VEC> me;
                me.load(x + (int64_t)vg * ldx + col);
                add_msg<T, VEC, false>(a, me, true, 1.0f, 1.0f, self_scale);
              }
            }
            if (active)
              add_msg<T, VEC, kMean, GUARD>(a, f[j], false, denom, rcp, 1.0f);
          }
        }
      }
    }
    if (MODEL == ATLAS_GIN && self_pending && active) {
      Frag<T, VEC> me;
      me.load(x + (int64_t)vg * ldx + col);
      add_msg<T, VEC, false>(a, me, true, 1.0f, 1.0f, self_scale);
    }
    if (active) {
      store_f32<VEC>(out + col, a);
      if (MODEL == ATLAS_SAGE) {  // self half: f32 copy of h_v
        Frag<T, VEC> me;
        me.load(x + (int64_t)vg * ldx + col);
        float h[VEC];
#pragma unroll
        for (int e = 0; e < VEC; e++) h[e] = me.get(e);
        store_f32<VEC>(out + d + col, h);
      }
    }
  }
}

// 6 blocks of 8 warps per SM (<= 40 registers): more rows in flight per SM
template <typename T, int VEC, int MODEL>
__global__ void __launch_bounds__(256, 6)
    agg_resident(const T* __restrict__ x, int64_t ldx,
                 const int64_t* __restrict__ csc_ptr,
                 const uint32_t* __restrict__ csc_src,
                 const uint32_t* __restrict__ indeg, int64_t lo,
                 int64_t nloc, int d, float* __restrict__ acc,
                 int64_t ldacc, float self_scale,
                 const int* __restrict__ guard_flag) {
  const int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (v >= nloc) return;
  if (*guard_flag)
    resident_body<T, VEC, MODEL, true>(x, ldx, csc_ptr, csc_src, indeg, lo, v,
                                       d, acc, ldacc, self_scale);
  else
    resident_body<T, VEC, MODEL, false>(x, ldx, csc_ptr, csc_src, indeg, lo,
                                        v, d, acc, ldacc, self_scale);
}

// ---------------------------------------------------------------------------
// resident front end, ring variant (rows of <= 32*VEC elements): each warp
// grabs batches of consecutive destinations, whose in-edges are one
// contiguous CSC range, and streams that range through a per-warp
// shared-memory ring with cp.async (LDGSTS, 16 B per lane per edge).
// Every lane reads back only the slots it filled itself, so no warp
// synchronisation is needed, and kRing row loads stay in flight across
// destination boundaries without holding registers.

constexpr int kRing = 16;
constexpr int kGrab = 32;  // destinations per work grab

// Fused epilogue of the transform-first layer (tcgen05 backend): the ring
// aggregates z = h . W_z^T instead of h, then writes the layer output
// y[v] = act(agg(z)[v] + self[v] + b) straight away (self = SAGE's
// z2 = h_v . W2^T, indexed by the LOCAL destination, or none).
struct EpiArgs {
  void* y;
  int64_t ldy;
  const float* bias;
  const float* self_rows;  // may be null
  int64_t ld_self;
  int n;                   // output columns
  int relu;
  int32_t* flag;           // extremes flag of y for the next layer
  int64_t vbeg;            // first destination of this launch's slice
};

template <typename OutT>
__device__ __forceinline__ OutT cvt_from_f32(float v);
template <>
__device__ __forceinline__ float cvt_from_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half cvt_from_f32<__half>(float v) {
  return __float2half_rn(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

template <typename T, int VEC, int MODEL, bool GUARD, typename OutT = void>
__device__ __forceinline__ void ring_body(
    const T* __restrict__ x, int64_t ldx, const int64_t* __restrict__ csc_ptr,
    const uint32_t* __restrict__ csc_src, const uint32_t* __restrict__ indeg,
    int64_t lo, int64_t nloc, int d, float* __restrict__ acc, int64_t ldacc,
    float self_scale, unsigned long long* __restrict__ work,
    uint4* __restrict__ ring, const EpiArgs& epi = EpiArgs{}) {
  using F = Frag<T, VEC>;
  static_assert(sizeof(F) == 16, "ring slots are 16 B");
  constexpr bool kEpi = !std::is_void<OutT>::value;
  int bad = 0;  // epilogue: extremes seen in y
  constexpr bool kMean = MODEL != ATLAS_GIN;
  const int lane = threadIdx.x & 31;
  const int col = lane * VEC;
  const bool active = col < d;
  // lanes past the row's end copy (and ignore) the last chunk instead of
  // branching around the copy, so the hot loop has no divergence
  const int colc = active ? col : d - VEC;
  // this lane's column of the ring as a shared-space address; slot k is
  // 32 lanes x 16 B, so it starts kRing-periodically at k * 512 B
  const uint32_t ring_lane =
      (uint32_t)__cvta_generic_to_shared(ring) + (uint32_t)lane * 16u;
  while (true) {
    unsigned long long v0 = 0;
    if (lane == 0) v0 = atomicAdd(work, (unsigned long long)kGrab);
    v0 = __shfl_sync(0xffffffffu, v0, 0);
    if constexpr (kEpi) v0 += (unsigned long long)epi.vbeg;
    if ((int64_t)v0 >= nloc) break;
    const int64_t v1 = min((int64_t)v0 + kGrab, nloc);
    const int64_t e0 = csc_ptr[v0], e1 = csc_ptr[v1];
    // edges of the grab, relative to e0 (a grab holds < 2^31 edges)
    const int ne = (int)(e1 - e0);
    const uint32_t* __restrict__ src0 = csc_src + e0;
    const T* __restrict__ xc = x + colc;
    // issue side: edges [pe, ne) not yet requested; src ids 32 at a time
    int pe = 0;
    uint32_t isrc = lane < ne ? src0[lane] : 0u;
    auto issue = [&]() {
      if (pe < ne) {
        if ((pe & 31) == 0 && pe != 0)
          isrc = pe + lane < ne ? src0[pe + lane] : 0u;
        const uint32_t s = __shfl_sync(0xffffffffu, isrc, pe & 31);
        cp_async16_s(ring_lane + ((uint32_t)(pe & (kRing - 1)) << 9),
                     xc + (int64_t)s * ldx);
        pe++;
      }
      cp_async_commit();  // empty groups keep the wait count uniform
    };
#pragma unroll 1
    for (int k = 0; k < kRing; k++) issue();
    // consume side (GIN needs the source id to place its self term)
    int ce = 0;
    uint32_t csrc = lane < ne ? src0[lane] : 0u;
    for (int64_t v = (int64_t)v0; v < v1; v++) {
      const int dend = (int)(csc_ptr[v + 1] - e0);
      const uint32_t vg = (uint32_t)(v + lo);
      const float denom = kMean ? (float)max(1u, indeg[v]) : 1.0f;
      const float rcp = kMean ? __frcp_rn(denom) : 1.0f;
      float a[VEC];
#pragma unroll
      for (int e = 0; e < VEC; e++) a[e] = 0.0f;
      bool self_pending = MODEL == ATLAS_GIN;
      for (; ce < dend; ce++) {
        if (MODEL == ATLAS_GIN) {
          if ((ce & 31) == 0 && ce != 0)
            csrc = ce + lane < ne ? src0[ce + lane] : 0u;
          const uint32_t s = __shfl_sync(0xffffffffu, csrc, ce & 31);
          if (self_pending && s >= vg) {
            self_pending = false;
            if (active) {
              F me;
              me.load(x + (int64_t)vg * ldx + col);
              add_msg<T, VEC, false>(a, me, true, 1.0f, 1.0f, self_scale);
            }
          }
        }
        cp_async_wait<kRing - 1>();  // this lane's copy of edge ce landed
        F f;
        f.raw = lds16(ring_lane + ((uint32_t)(ce & (kRing - 1)) << 9));
        add_msg<T, VEC, kMean, GUARD>(a, f, false, denom, rcp, 1.0f);
        issue();  // refill the slot just consumed
      }
      if (MODEL == ATLAS_GIN && self_pending && active) {
        F me;
        me.load(x + (int64_t)vg * ldx + col);
        add_msg<T, VEC, false>(a, me, true, 1.0f, 1.0f, self_scale);
      }
      if constexpr (kEpi) {
        using O = typename std::conditional<kEpi, OutT, float>::type;
        O* yrow = static_cast<O*>(epi.y) + v * epi.ldy;
#pragma unroll
        for (int e = 0; e < VEC; e++) {
          const int c = col + e;
          if (c < epi.n) {
            float o = a[e];
            if (epi.self_rows) o += epi.self_rows[v * epi.ld_self + c];
            o += epi.bias[c];
            if (epi.relu) o = (o >= 0.0f || o != o) ? o : 0.0f;
            const O q = cvt_from_f32<O>(o);
            bad |= is_extreme(to_f32(q));
            yrow[c] = q;
          }
        }
      } else if (active) {
        float* out = acc + v * ldacc;
        store_f32<VEC>(out + col, a);
        if (MODEL == ATLAS_SAGE) {
          F me;
          me.load(x + (int64_t)vg * ldx + col);
          float h[VEC];
#pragma unroll
          for (int e = 0; e < VEC; e++) h[e] = me.get(e);
          store_f32<VEC>(out + d + col, h);
        }
      }
    }
    cp_async_wait<0>();
  }
  if constexpr (kEpi)
    if (__any_sync(0xffffffffu, bad) && lane == 0 && epi.flag)
      atomicOr(epi.flag, 1);
}

// transform-first layer: ring aggregation of z with the fused epilogue
template <int MODEL, typename OutT>
__global__ void __launch_bounds__(256, 3)
    agg_ring_epi(const float* __restrict__ z, int64_t ldz,
                 const int64_t* __restrict__ csc_ptr,
                 const uint32_t* __restrict__ csc_src,
                 const uint32_t* __restrict__ indeg, int64_t lo, int64_t nloc,
                 int d, float self_scale, const int* __restrict__ guard_flag,
                 unsigned long long* __restrict__ work, EpiArgs epi) {
  extern __shared__ uint4 ring_smem[];
  uint4* ring = ring_smem + (threadIdx.x >> 5) * (kRing * 32);
  if (*guard_flag)
    ring_body<float, 4, MODEL, true, OutT>(z, ldz, csc_ptr, csc_src, indeg,
                                           lo, nloc, d, nullptr, 0,
                                           self_scale, work, ring, epi);
  else
    ring_body<float, 4, MODEL, false, OutT>(z, ldz, csc_ptr, csc_src, indeg,
                                            lo, nloc, d, nullptr, 0,
                                            self_scale, work, ring, epi);
}

template <typename T, int VEC, int MODEL>
__global__ void __launch_bounds__(256, 3)
    agg_ring(const T* __restrict__ x, int64_t ldx,
             const int64_t* __restrict__ csc_ptr,
             const uint32_t* __restrict__ csc_src,
             const uint32_t* __restrict__ indeg, int64_t lo, int64_t nloc,
             int d, float* __restrict__ acc, int64_t ldacc, float self_scale,
             const int* __restrict__ guard_flag,
             unsigned long long* __restrict__ work) {
  extern __shared__ uint4 ring_smem[];
  uint4* ring = ring_smem + (threadIdx.x >> 5) * (kRing * 32);
  if (*guard_flag)
    ring_body<T, VEC, MODEL, true>(x, ldx, csc_ptr, csc_src, indeg, lo, nloc,
                                   d, acc, ldacc, self_scale, work, ring);
  else
    ring_body<T, VEC, MODEL, false>(x, ldx, csc_ptr, csc_src, indeg, lo, nloc,
                                    d, acc, ldacc, self_scale, work, ring);
}

// Bit-exact ring for narrow rows (<= 16 chunks of 16 B: 128-d f16, 64-d
// f32): 32/LPD sub-groups of LPD lanes per warp, each walking its own run
// of consecutive destinations (a contiguous CSC range) in lockstep with the
// others -- the agg_tf_ring schedule with ring_body's arithmetic. Each
// destination's sources are still folded one at a time in ascending order
// (same rounded divide and add per column), so records are the bits of
// agg_ring; the warp just keeps every lane busy instead of idling the
// half (or more) of it a narrow row does not cover.
// shallower ring than agg_ring's: 32/LPD runs share a warp's rows in
// flight, and the smaller footprint leaves room for more blocks per SM
constexpr int kSubRing = 8;
constexpr int kSubBlocks = 4;  // agg_sub_ring blocks per SM (64 registers
                                // each: no address rematerialisation)
// per-warp grab metadata words of agg_sub_ring (offsets + denominators)
template <int LPD>
constexpr int kSubMeta = 2 * kGrab * (32 / LPD) + 4;

template <typename T, int LPD, int MODEL, bool GUARD>
__device__ __forceinline__ void sub_ring_body(
    const T* __restrict__ x, int64_t ldx, const int64_t* __restrict__ csc_ptr,
    const uint32_t* __restrict__ csc_src, const uint32_t* __restrict__ indeg,
    int64_t lo, int64_t nloc, int d, float* __restrict__ acc, int64_t ldacc,
    float self_scale, unsigned long long* __restrict__ work,
    uint4* __restrict__ ring, uint32_t* __restrict__ mptr) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int DPW = 32 / LPD;
  constexpr int kWarpDst = kGrab * DPW;
  constexpr int kIdR = LPD >= 16 ? 1 : 16 / LPD;
  // per-warp grab metadata (as in agg_tf_multi): CSC offsets relative to
  // the grab's first edge and the mean's denominators, staged once per
  // grab so arming a destination never waits on a dependent global load
  float* mden = reinterpret_cast<float*>(mptr + kWarpDst + 4);
  constexpr bool kMean = MODEL != ATLAS_GIN;
  using F = Frag<T, VEC>;
  const int lane = threadIdx.x & 31, sub = lane / LPD, sl = lane % LPD;
  const int col = sl * VEC;
  const bool lane_on = col < d;
  const int colc = lane_on ? col : d - VEC;  // clamped: branch-free copies
  const uint32_t ring_lane =
      (uint32_t)__cvta_generic_to_shared(ring) + (uint32_t)lane * 16u;
  // source row address = xbase + u * pitch (one IMAD.WIDE per edge)
  const uint64_t xbase = reinterpret_cast<uint64_t>(x + colc);
  const uint32_t pitch = (uint32_t)(ldx * (int64_t)sizeof(T));
  while (true) {
    unsigned long long w0 = 0;
    if (lane == 0) w0 = atomicAdd(work, (unsigned long long)(kGrab * DPW));
    w0 = __shfl_sync(0xffffffffu, w0, 0);
    if ((int64_t)w0 >= nloc) break;
    const int nw = (int)min((int64_t)kWarpDst, nloc - (int64_t)w0);
    const int64_t ew = csc_ptr[w0];
    for (int i = lane; i <= nw; i += 32)
      mptr[i] = (uint32_t)(csc_ptr[w0 + i] - ew);
    if (kMean)
      for (int i = lane; i < nw; i += 32)
        mden[i] = (float)max(1u, indeg[w0 + i]);
    __syncwarp();
    // this sub-group's destinations [v, v_end) (grab-local lv) and its
    // edges [0, ne) relative to its first edge
    int lv = min(sub * kGrab, nw);
    const int lv_end = min(lv + kGrab, nw);
    int64_t v = (int64_t)w0 + lv;
    const int64_t v_end = (int64_t)w0 + lv_end;
    const uint32_t e_rel = mptr[lv];
    const int ne = (int)(mptr[lv_end] - e_rel);
    const uint32_t* __restrict__ src0 = csc_src + ew + e_rel;
    int ce = 0, pe = 0;
    int dend = 0;
    float denom = 1.0f, rcp = 1.0f;
    bool self_pending = false;
    // source ids in register batches of kIdR x LPD edges, the next batch
    // loaded one batch ahead (off the cp.async issue path)
    uint32_t cur[kIdR], nxt[kIdR];
    int pbase = 0;
#pragma unroll
    for (int r = 0; r < kIdR; r++) {
      const int i0 = sl + r * LPD, i1 = i0 + kIdR * LPD;
      cur[r] = i0 < ne ? src0[i0] : 0u;
      nxt[r] = i1 < ne ? src0[i1] : 0u;
    }
    uint32_t csrc = cur[0];  // GIN: consume-side source ids, LPD at a time
    float a[VEC];
    auto start_dest = [&]() {  // arm destination v (v < v_end)
      dend = (int)(mptr[lv + 1] - e_rel);
      if (kMean) {
        denom = mden[lv];
        rcp = __frcp_rn(denom);
      }
      self_pending = MODEL == ATLAS_GIN;
#pragma unroll
      for (int e = 0; e < VEC; e++) a[e] = 0.0f;
    };
    auto add_self = [&]() {
      if (lane_on) {
        F me;
        me.load(x + (v + lo) * ldx + col);
        add_msg<T, VEC, false>(a, me, true, 1.0f, 1.0f, self_scale);
      }
    };
    auto issue = [&]() {
      const bool more = pe < ne;
      if (more && pe - pbase == kIdR * LPD) {
        pbase = pe;
#pragma unroll
        for (int r = 0; r < kIdR; r++) {
          cur[r] = nxt[r];
          const int i1 = pbase + kIdR * LPD + sl + r * LPD;
          nxt[r] = i1 < ne ? src0[i1] : 0u;
        }
      }
      const int q = pe - pbase;
      uint32_t pick = cur[0];
#pragma unroll
      for (int r = 1; r < kIdR; r++)
        if (q / LPD == r) pick = cur[r];
      const uint32_t u = __shfl_sync(0xffffffffu, pick, q & (LPD - 1), LPD);
      if (more) {
        cp_async16_s(ring_lane + ((uint32_t)(pe & (kSubRing - 1)) << 9),
                     reinterpret_cast<const void*>(
                         xbase + (uint64_t)u * pitch));
        pe++;
      }
      cp_async_commit();  // one group per lane per iteration, maybe empty
    };
    // write out finished destinations (zero-degree ones included)
    auto flush = [&]() {
      while (v < v_end && ce == dend) {
        if (MODEL == ATLAS_GIN && self_pending) add_self();
        if (lane_on) {
          float* out = acc + v * ldacc;
          store_f32<VEC>(out + col, a);
          if (MODEL == ATLAS_SAGE) {
            F me;
            me.load(x + (v + lo) * ldx + col);
            float h[VEC];
#pragma unroll
            for (int e = 0; e < VEC; e++) h[e] = me.get(e);
            store_f32<VEC>(out + d + col, h);
          }
        }
        v++;
        lv++;
        if (v < v_end) start_dest();
      }
    };
    if (v < v_end) start_dest();
#pragma unroll 1
    for (int k = 0; k < kSubRing; k++) issue();
    flush();
    while (__any_sync(0xffffffffu, ce < ne)) {
      const bool on = ce < ne;
      if (MODEL == ATLAS_GIN) {
        // GIN's self term goes before the first source >= v (its stream
        // position); ids of the consumed edges, LPD at a time
        if (on && (ce & (LPD - 1)) == 0 && ce != 0)
          csrc = ce + sl < ne ? src0[ce + sl] : 0u;
        const uint32_t s =
            __shfl_sync(0xffffffffu, csrc, ce & (LPD - 1), LPD);
        if (on && self_pending && s >= (uint32_t)(v + lo)) {
          self_pending = false;
          add_self();
        }
      }
      cp_async_wait<kSubRing - 1>();  // the row issued kSubRing iterations ago
      if (on) {
        F f;
        f.raw = lds16(ring_lane + ((uint32_t)(ce & (kSubRing - 1)) << 9));
        add_msg<T, VEC, kMean, GUARD>(a, f, false, denom, rcp, 1.0f);
        ce++;
      }
      issue();
      flush();
    }
    cp_async_wait<0>();
    __syncwarp();  // metadata reads done before the next grab rewrites it
  }
}

template <typename T, int LPD, int MODEL>
__global__ void __launch_bounds__(256, kSubBlocks)
    agg_sub_ring(const T* __restrict__ x, int64_t ldx,
                 const int64_t* __restrict__ csc_ptr,
                 const uint32_t* __restrict__ csc_src,
                 const uint32_t* __restrict__ indeg, int64_t lo, int64_t nloc,
                 int d, float* __restrict__ acc, int64_t ldacc,
                 float self_scale, const int* __restrict__ guard_flag,
                 unsigned long long* __restrict__ work) {
  extern __shared__ uint4 ring_smem[];
  uint4* ring = ring_smem + (threadIdx.x >> 5) * (kSubRing * 32);
  uint32_t* meta = reinterpret_cast<uint32_t*>(ring_smem + 8 * kSubRing * 32) +
                   (threadIdx.x >> 5) * kSubMeta<LPD>;
  if (*guard_flag)
    sub_ring_body<T, LPD, MODEL, true>(x, ldx, csc_ptr, csc_src, indeg, lo,
                                       nloc, d, acc, ldacc, self_scale, work,
                                       ring, meta);
  else
    sub_ring_body<T, LPD, MODEL, false>(x, ldx, csc_ptr, csc_src, indeg, lo,
                                        nloc, d, acc, ldacc, self_scale, work,
                                        ring, meta);
}

// transform-first layer, narrow z rows (<= 64 f32), streaming version:
// 32/LPD sub-groups of LPD lanes per warp, each walking its own run of
// consecutive destinations (one contiguous CSC range) in lockstep with the
// others: every iteration each sub-group consumes one edge and issues the
// cp.async of the edge kTfRing ahead into its lanes' shared-memory ring,
// so kTfRing rows per lane stay in flight across destination boundaries
// and the per-edge instruction cost is shared by 32/LPD destinations.
// ring depth / blocks per SM by sub-group width (measured: 8-lane groups,
// e.g. 20-wide z, are latency-bound at 16 deep x 3 blocks; 16-lane groups
// are issue-bound and keep the deeper ring)
template <int LPD>
constexpr int kTfRing = LPD == 8 ? 8 : 16;
template <int LPD>
constexpr int kTfBlocks = LPD == 8 ? 5 : 4;

template <int LPD, int MODEL, typename OutT>
__global__ void __launch_bounds__(256, kTfBlocks<LPD>)
    agg_tf_ring(const float* __restrict__ z, int64_t ldz,
                const int64_t* __restrict__ csc_ptr,
                const uint32_t* __restrict__ csc_src,
                const uint32_t* __restrict__ indeg, int64_t lo, int64_t nloc,
                int d, float self_scale, EpiArgs epi,
                unsigned long long* __restrict__ work) {
  constexpr int DPW = 32 / LPD;
  extern __shared__ uint4 ring_smem[];
  const int lane = threadIdx.x & 31, sub = lane / LPD, sl = lane % LPD;
  const int col = sl * 4;
  const bool lane_on = col < d;
  const int colc = lane_on ? col : d - 4;  // clamped: branch-free copies
  const uint32_t ring_lane =
      (uint32_t)__cvta_generic_to_shared(ring_smem + (threadIdx.x >> 5) *
                                                         (kTfRing<LPD> * 32)) +
      (uint32_t)lane * 16u;
  const float* __restrict__ zc = z + colc;
  int bad = 0;
  while (true) {
    unsigned long long w0 = 0;
    if (lane == 0) w0 = atomicAdd(work, (unsigned long long)(kGrab * DPW));
    w0 = __shfl_sync(0xffffffffu, w0, 0) + (unsigned long long)epi.vbeg;
    if ((int64_t)w0 >= nloc) break;
    // this sub-group's destinations [v, v_end) and its edges, relative to
    // e_beg: [0, ne)
    int64_t v = min((int64_t)w0 + (int64_t)sub * kGrab, nloc);
    const int64_t v_end = min(v + kGrab, nloc);
    const int64_t e_beg = csc_ptr[v];
    const int ne = (int)(csc_ptr[v_end] - e_beg);
    const uint32_t* __restrict__ src0 = csc_src + e_beg;
    int ce = 0, pe = 0;
    int dend = v < v_end ? (int)(csc_ptr[v + 1] - e_beg) : ne;
    uint32_t isrc = sl < ne ? src0[sl] : 0u;
    float a[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    auto issue = [&]() {
      const bool more = pe < ne;
      if (more && (pe & (LPD - 1)) == 0 && pe != 0)
        isrc = pe + sl < ne ? src0[pe + sl] : 0u;
      const uint32_t u = __shfl_sync(0xffffffffu, isrc, pe & (LPD - 1), LPD);
      if (more) {
        cp_async16_s(ring_lane + ((uint32_t)(pe & (kTfRing<LPD> - 1)) << 9),
                     zc + (int64_t)u * ldz);
        pe++;
      }
      cp_async_commit();  // one group per lane per iteration, maybe empty
    };
    // emit finished destinations (zero-degree ones included)
    auto flush = [&]() {
      while (v < v_end && ce == dend) {
        const int64_t vg = v + lo;
        float o4[4] = {a[0], a[1], a[2], a[3]};
        if (MODEL == ATLAS_GIN) {
          if (lane_on) {
            const float4 me =
                __ldg(reinterpret_cast<const float4*>(z + vg * ldz + col));
            o4[0] += self_scale * me.x;
            o4[1] += self_scale * me.y;
            o4[2] += self_scale * me.z;
            o4[3] += self_scale * me.w;
          }
        } else {
          const float r = 1.0f / (float)max(1u, indeg[v]);
#pragma unroll
          for (int e = 0; e < 4; e++) o4[e] *= r;
        }
        OutT* yrow = static_cast<OutT*>(epi.y) + v * epi.ldy;
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const int c = col + e;
          if (c < epi.n) {
            float o = o4[e];
            if (epi.self_rows) o += epi.self_rows[v * epi.ld_self + c];
            o += epi.bias[c];
            if (epi.relu) o = (o >= 0.0f || o != o) ? o : 0.0f;
            const OutT q = cvt_from_f32<OutT>(o);
            bad |= is_extreme(to_f32(q));
            yrow[c] = q;
          }
        }
        a[0] = a[1] = a[2] = a[3] = 0.0f;
        v++;
        dend = v < v_end ? (int)(csc_ptr[v + 1] - e_beg) : ne;
      }
    };
#pragma unroll 1
    for (int k = 0; k < kTfRing<LPD>; k++) issue();
    flush();
    while (__any_sync(0xffffffffu, ce < ne)) {
      cp_async_wait<kTfRing<LPD> - 1>();  // the row issued kTfRing<LPD> iterations ago
      if (ce < ne) {
        const uint4 r = lds16(ring_lane + ((uint32_t)(ce & (kTfRing<LPD> - 1)) << 9));
        a[0] += __uint_as_float(r.x);
        a[1] += __uint_as_float(r.y);
        a[2] += __uint_as_float(r.z);
        a[3] += __uint_as_float(r.w);
        ce++;
      }
      issue();
      flush();
    }
    cp_async_wait<0>();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0 && epi.flag)
    atomicOr(epi.flag, 1);
}

// transform-first layer, multi-chunk lanes: the agg_tf_ring walk with each
// lane owning CPL 16-byte chunks of the z row (chunk sl + j*LPD), so a
// 48-wide row (12 chunks, cfg2's 47-wide last layer) runs 4-lane groups
// with every lane busy instead of 16-lane groups with 4 idle, and one
// iteration serves 8 edges per warp instead of 2 (the per-edge issue,
// shuffle and loop cost is what bound agg_tf_ring: ncu 83 % issue-active
// at 0.69 of HBM). Ring slot s, chunk j of a lane sits at plane s*CPL + j
// (512 B per plane, lane-contiguous: conflict-free).
template <int LPD, int CPL, int DEPTH, int MODEL, typename OutT, int MINB = 1>
__global__ void __launch_bounds__(256, MINB)
    agg_tf_multi(const float* __restrict__ z, int64_t ldz,
                 const int64_t* __restrict__ csc_ptr,
                 const uint32_t* __restrict__ csc_src,
                 const uint32_t* __restrict__ indeg, int64_t lo, int64_t nloc,
                 int d, float self_scale, EpiArgs epi,
                 unsigned long long* __restrict__ work) {
  constexpr int DPW = 32 / LPD;
  constexpr int kWarpDst = kGrab * DPW;  // destinations per warp grab
  constexpr int kIdR = LPD >= 16 ? 1 : 16 / LPD;
  extern __shared__ uint4 ring_smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31, sub = lane / LPD, sl = lane % LPD;
  // per-warp grab metadata after the rings: CSC offsets relative to the
  // grab's first edge, and the mean's reciprocal per destination, loaded
  // once per grab (coalesced) so a finished destination never waits on a
  // dependent global load
  uint32_t* mptr = reinterpret_cast<uint32_t*>(ring_smem + 8 * DEPTH * CPL * 32) +
                   warp * (2 * kWarpDst + 4);
  float* mrcp = reinterpret_cast<float*>(mptr + kWarpDst + 4);
  int colc[CPL];
  bool on[CPL];
#pragma unroll
  for (int j = 0; j < CPL; j++) {
    const int c = (sl + j * LPD) * 4;
    on[j] = c < d;
    colc[j] = on[j] ? c : d - 4;
  }
  const uint32_t ring_lane =
      (uint32_t)__cvta_generic_to_shared(ring_smem + warp * (DEPTH * CPL * 32)) +
      (uint32_t)lane * 16u;
  int bad = 0;
  while (true) {
    unsigned long long w0 = 0;
    if (lane == 0) w0 = atomicAdd(work, (unsigned long long)kWarpDst);
    w0 = __shfl_sync(0xffffffffu, w0, 0) + (unsigned long long)epi.vbeg;
    if ((int64_t)w0 >= nloc) break;
    const int nw = (int)min((int64_t)kWarpDst, nloc - (int64_t)w0);
    const int64_t ew = csc_ptr[w0];
    for (int i = lane; i <= nw; i += 32)
      mptr[i] = (uint32_t)(csc_ptr[w0 + i] - ew);
    if (MODEL != ATLAS_GIN)
      for (int i = lane; i < nw; i += 32)
        mrcp[i] = 1.0f / (float)max(1u, indeg[w0 + i]);
    __syncwarp();
    // this sub-group's destinations [lv, lv_end) of the grab
    int lv = min(sub * kGrab, nw);
    const int lv_end = min(lv + kGrab, nw);
    const uint32_t e_rel = mptr[lv];
    const int ne = (int)(mptr[lv_end] - e_rel);
    const uint32_t* __restrict__ src0 = csc_src + ew + e_rel;
    int ce = 0, pe = 0;
    int dend = lv < lv_end ? (int)(mptr[lv + 1] - e_rel) : ne;
    // source ids in register batches of kIdR x LPD edges (lane sl holds
    // edge base + sl + r * LPD), the next batch loaded one batch ahead so
    // the id load is never on the cp.async issue path
    uint32_t cur[kIdR], nxt[kIdR];
    int pbase = 0;
#pragma unroll
    for (int r = 0; r < kIdR; r++) {
      const int i0 = sl + r * LPD, i1 = i0 + kIdR * LPD;
      cur[r] = i0 < ne ? src0[i0] : 0u;
      nxt[r] = i1 < ne ? src0[i1] : 0u;
    }
    float a[CPL][4];
#pragma unroll
    for (int j = 0; j < CPL; j++) a[j][0] = a[j][1] = a[j][2] = a[j][3] = 0.0f;
    auto issue = [&]() {
      const bool more = pe < ne;
      if (more && pe - pbase == kIdR * LPD) {
        pbase = pe;
#pragma unroll
        for (int r = 0; r < kIdR; r++) {
          cur[r] = nxt[r];
          const int i1 = pbase + kIdR * LPD + sl + r * LPD;
          nxt[r] = i1 < ne ? src0[i1] : 0u;
        }
      }
      const int q = pe - pbase;
      uint32_t pick = cur[0];
#pragma unroll
      for (int r = 1; r < kIdR; r++)
        if (q / LPD == r) pick = cur[r];
      const uint32_t u = LPD == 1 ? pick
                                  : __shfl_sync(0xffffffffu, pick,
                                                q & (LPD - 1), LPD);
      if (more) {
        const float* row = z + (int64_t)u * ldz;
        const uint32_t slot =
            ring_lane + ((uint32_t)(pe & (DEPTH - 1)) * CPL << 9);
#pragma unroll
        for (int j = 0; j < CPL; j++)
          if (on[j]) cp_async16_s(slot + ((uint32_t)j << 9), row + colc[j]);
        pe++;
      }
      cp_async_commit();  // one group per lane per iteration, maybe empty
    };
    auto flush = [&]() {
      while (lv < lv_end && ce == dend) {
        const int64_t v = (int64_t)w0 + lv;
        const float r = MODEL == ATLAS_GIN ? 1.0f : mrcp[lv];
        OutT* yrow = static_cast<OutT*>(epi.y) + v * epi.ldy;
#pragma unroll
        for (int j = 0; j < CPL; j++) {
          if (!on[j]) continue;
          const int col = colc[j];
          float o4[4] = {a[j][0], a[j][1], a[j][2], a[j][3]};
          if (MODEL == ATLAS_GIN) {
            const float4 me = __ldg(
                reinterpret_cast<const float4*>(z + (v + lo) * ldz + col));
            o4[0] += self_scale * me.x;
            o4[1] += self_scale * me.y;
            o4[2] += self_scale * me.z;
            o4[3] += self_scale * me.w;
          } else {
#pragma unroll
            for (int e = 0; e < 4; e++) o4[e] *= r;
          }
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const int c = col + e;
            if (c < epi.n) {
              float o = o4[e];
              if (epi.self_rows) o += epi.self_rows[v * epi.ld_self + c];
              o += __ldg(epi.bias + c);
              if (epi.relu) o = (o >= 0.0f || o != o) ? o : 0.0f;
              const OutT q = cvt_from_f32<OutT>(o);
              bad |= is_extreme(to_f32(q));
              yrow[c] = q;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < CPL; j++)
          a[j][0] = a[j][1] = a[j][2] = a[j][3] = 0.0f;
        lv++;
        dend = lv < lv_end ? (int)(mptr[lv + 1] - e_rel) : ne;
      }
    };
#pragma unroll 1
    for (int k = 0; k < DEPTH; k++) issue();
    flush();
    while (__any_sync(0xffffffffu, ce < ne)) {
      cp_async_wait<DEPTH - 1>();  // the row issued DEPTH iterations ago
      if (ce < ne) {
        const uint32_t slot =
            ring_lane + ((uint32_t)(ce & (DEPTH - 1)) * CPL << 9);
#pragma unroll
        for (int j = 0; j < CPL; j++) {
          const uint4 r = lds16(slot + ((uint32_t)j << 9));
          a[j][0] += __uint_as_float(r.x);
          a[j][1] += __uint_as_float(r.y);
          a[j][2] += __uint_as_float(r.z);
          a[j][3] += __uint_as_float(r.w);
        }
        ce++;
      }
      issue();
      flush();
    }
    cp_async_wait<0>();
    __syncwarp();  // metadata reads done before the next grab rewrites it
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0 && epi.flag)
    atomicOr(epi.flag, 1);
}

// ---------------------------------------------------------------------------
// resident front end, bulk-copy variant for wide rows (> 512 B, e.g. 1024-d
// f16 = 2 KB): the same persistent warps and contiguous CSC ranges as the
// ring kernel, but each source row moves global -> shared memory as ONE
// cp.async.bulk (TMA engine, UBLKCP) issued by lane 0 and completed on a
// per-slot mbarrier (expect_tx = row bytes). kSlots rows stay in flight per
// warp without costing registers or LSU issue slots; lanes then read their
// 16-byte chunks from shared memory (chunk j of lane l at byte
// (32 j + l) * 16, conflict-free) and fold them in source order exactly like
// the other front ends.

constexpr int kBulkWarps = 4;
constexpr int kBulkGrab = 16;

template <typename T, int CH, int SLOTS, int MODEL, bool GUARD>
__device__ __forceinline__ void bulk_body(
    const T* __restrict__ x, int64_t ldx, const int64_t* __restrict__ csc_ptr,
    const uint32_t* __restrict__ csc_src, const uint32_t* __restrict__ indeg,
    int64_t lo, int64_t nloc, int d, float* __restrict__ acc, int64_t ldacc,
    float self_scale, unsigned long long* __restrict__ work,
    uint8_t* __restrict__ ring, uint64_t* __restrict__ bars) {
  using F = Frag<T, 16 / sizeof(T)>;
  static_assert((SLOTS & (SLOTS - 1)) == 0, "power-of-two ring");
  constexpr int EPC = 16 / sizeof(T);  // elements per 16-byte chunk
  constexpr bool kMean = MODEL != ATLAS_GIN;
  const int lane = threadIdx.x & 31;
  const uint32_t row_bytes = (uint32_t)(d * sizeof(T));
  bool act[CH];
#pragma unroll
  for (int j = 0; j < CH; j++) act[j] = (j * 32 + lane) * EPC < d;
  RowFeeder<SLOTS, (SLOTS >= 8 ? 4 : SLOTS / 2)> feed{ring, bars, row_bytes,
                                                   csc_src};
  while (true) {
    unsigned long long v0 = 0;
    if (lane == 0) v0 = atomicAdd(work, (unsigned long long)kBulkGrab);
    v0 = __shfl_sync(0xffffffffu, v0, 0);
    if ((int64_t)v0 >= nloc) break;
    const int64_t v1 = min((int64_t)v0 + kBulkGrab, nloc);
    const int64_t e0 = csc_ptr[v0], e1 = csc_ptr[v1];
    feed.begin(e0, e1, x, ldx);
    int64_t ce = e0, cbase = e0;
    uint32_t csrc = 0;
    if (MODEL == ATLAS_GIN) csrc = (e0 + lane < e1) ? csc_src[e0 + lane] : 0u;
    for (int64_t v = (int64_t)v0; v < v1; v++) {
      const int64_t dend = csc_ptr[v + 1];
      const uint32_t vg = (uint32_t)(v + lo);
      const float denom = kMean ? (float)max(1u, indeg[v]) : 1.0f;
      const float rcp = kMean ? __frcp_rn(denom) : 1.0f;
      float a[CH][EPC];
#pragma unroll
      for (int j = 0; j < CH; j++)
#pragma unroll
        for (int e = 0; e < EPC; e++) a[j][e] = 0.0f;
      bool self_pending = MODEL == ATLAS_GIN;
      auto self_term = [&]() {
#pragma unroll
        for (int j = 0; j < CH; j++)
          if (act[j]) {
            F me;
            me.load(x + (int64_t)vg * ldx + (j * 32 + lane) * EPC);
            add_msg<T, EPC, false>(a[j], me, true, 1.0f, 1.0f, self_scale);
          }
      };
      for (; ce < dend; ce++) {
        if (MODEL == ATLAS_GIN) {
          if (ce - cbase == 32) {
            cbase = ce;
            csrc = (ce + lane < e1) ? csc_src[ce + lane] : 0u;
          }
          const uint32_t s = __shfl_sync(0xffffffffu, csrc, (int)(ce - cbase));
          if (self_pending && s >= vg) {
            self_pending = false;
            self_term();
          }
        }
        const uint32_t row = feed.wait();
        F f[CH];
#pragma unroll
        for (int j = 0; j < CH; j++)
          if (act[j]) f[j].raw = lds_v4(row + (uint32_t)(j * 32 + lane) * 16u);
#pragma unroll
        for (int j = 0; j < CH; j++)
          if (act[j])
            add_msg<T, EPC, kMean, GUARD>(a[j], f[j], false, denom, rcp, 1.0f);
        feed.release(x, ldx);
      }
      if (MODEL == ATLAS_GIN && self_pending) self_term();
      float* out = acc + v * ldacc;
#pragma unroll
      for (int j = 0; j < CH; j++)
        if (act[j]) {
          const int col = (j * 32 + lane) * EPC;
          store_f32<EPC>(out + col, a[j]);
          if (MODEL == ATLAS_SAGE) {
            F me;
            me.load(x + (int64_t)vg * ldx + col);
            float h[EPC];
#pragma unroll
            for (int e = 0; e < EPC; e++) h[e] = me.get(e);
            store_f32<EPC>(out + d + col, h);
          }
        }
    }
  }
}

template <typename T, int CH, int MODEL>
__global__ void __launch_bounds__(kBulkWarps * 32, CH >= 8 ? 3 : 6)
    agg_bulk(const T* __restrict__ x, int64_t ldx,
             const int64_t* __restrict__ csc_ptr,
             const uint32_t* __restrict__ csc_src,
             const uint32_t* __restrict__ indeg, int64_t lo, int64_t nloc,
             int d, float* __restrict__ acc, int64_t ldacc, float self_scale,
             const int* __restrict__ guard_flag,
             unsigned long long* __restrict__ work) {
  constexpr int SLOTS = 16 / CH;  // <= 8 KB of rows in flight per warp
  extern __shared__ __align__(128) uint8_t bulk_smem[];
  const int warp = threadIdx.x >> 5;
  const uint32_t row_bytes = (uint32_t)(d * sizeof(T));
  uint64_t* bars = reinterpret_cast<uint64_t*>(bulk_smem) + warp * SLOTS;
  uint8_t* ring = bulk_smem + kBulkWarps * SLOTS * 8 +
                  (size_t)warp * SLOTS * row_bytes;
  if ((threadIdx.x & 31) == 0) {
    for (int k = 0; k < SLOTS; k++) mbar_init_cta(&bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (*guard_flag)
    bulk_body<T, CH, SLOTS, MODEL, true>(x, ldx, csc_ptr, csc_src, indeg, lo,
                                         nloc, d, acc, ldacc, self_scale,
                                         work, ring, bars);
  else
    bulk_body<T, CH, SLOTS, MODEL, false>(x, ldx, csc_ptr, csc_src, indeg, lo,
                                          nloc, d, acc, ldacc, self_scale,
                                          work, ring, bars);
}

// ---------------------------------------------------------------------------
// streamed front end: the layer input arrives in row tiles [tile_lo,
// tile_hi) (host -> HBM, double-buffered); every destination consumes the
// part of its ascending source list that falls in the tile, resuming at
// cursor[v]. Per-column addition order is unchanged, so the records are
// the same bits as the resident pass.

template <typename T, int VEC, int MODEL>
__global__ void __launch_bounds__(256, 6)
    agg_tile(const T* __restrict__ tile, int64_t ldx, int64_t tile_lo,
             int64_t tile_hi, const int64_t* __restrict__ csc_ptr,
             const uint32_t* __restrict__ csc_src,
             const uint32_t* __restrict__ indeg, int64_t lo, int64_t nloc,
             int d, float* __restrict__ acc, int64_t ldacc,
             int64_t* __restrict__ cursor, uint8_t* __restrict__ touched,
             float self_scale) {
  constexpr bool kMean = MODEL != ATLAS_GIN;
  const int lane = threadIdx.x & 31;
  const int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (v >= nloc) return;
  const int64_t vg = v + lo;
  const bool own = vg >= tile_lo && vg < tile_hi;  // v's own row is here
  const int64_t beg = cursor[v], end = csc_ptr[v + 1];
  const bool has_src = beg < end && (int64_t)csc_src[beg] < tile_hi;
  const bool self_here = own && MODEL != ATLAS_GCN;
  const bool zero_row = own && MODEL == ATLAS_GCN && indeg[v] == 0;
  if (!has_src && !self_here && !zero_row) return;
  const float denom = kMean ? (float)max(1u, indeg[v]) : 1.0f;
  const float rcp = kMean ? __frcp_rn(denom) : 1.0f;
  const bool resume = touched[v] != 0;
  float* out = acc + v * ldacc;
  int64_t consumed = 0;
  for (int c0 = 0; c0 < d; c0 += 32 * VEC) {
    const int col = c0 + lane * VEC;
    const bool active = col < d;
    float a[VEC];
#pragma unroll
    for (int e = 0; e < VEC; e++) a[e] = 0.0f;
    if (resume && active) load_f32<VEC>(out + col, a);
    bool self_pending = MODEL == ATLAS_GIN && own;
    int64_t base = beg;
    while (base < end) {
      const int64_t i = base + lane;
      const uint32_t mine = i < end ? csc_src[i] : 0xFFFFFFFFu;
      const unsigned ok = __ballot_sync(0xffffffffu,
                                        i < end && (int64_t)mine < tile_hi);
      const int cnt = __popc(ok);  // sources ascend: a prefix is in the tile
      for (int k = 0; k < cnt; k += kUnroll) {
        Frag<T, VEC> f[kUnroll];
        uint32_t s[kUnroll];
#pragma unroll
        for (int j = 0; j < kUnroll; j++) {
          s[j] = __shfl_sync(0xffffffffu, mine, (k + j) & 31);
          if (active && k + j < cnt)
            f[j].load(tile + ((int64_t)s[j] - tile_lo) * ldx + col);
        }
#pragma unroll
        for (int j = 0; j < kUnroll; j++) {
          if (k + j < cnt) {
            if (MODEL == ATLAS_GIN && self_pending && (int64_t)s[j] >= vg) {
              self_pending = false;
              if (active) {
                Frag<T, VEC> me;
                me.load(tile + (vg - tile_lo) * ldx + col);
                add_msg<T, VEC, false>(a, me, true, 1.0f, 1.0f, self_scale);
              }
            }
            if (active) add_msg<T, VEC, kMean>(a, f[j], false, denom, rcp, 1.0f);
          }
        }
      }
      base += cnt;
      if (cnt < 32) break;
    }
    if (MODEL == ATLAS_GIN && self_pending && active) {
      Frag<T, VEC> me;
      me.load(tile + (vg - tile_lo) * ldx + col);
      add_msg<T, VEC, false>(a, me, true, 1.0f, 1.0f, self_scale);
    }
    if (active) {
      store_f32<VEC>(out + col, a);
      if (MODEL == ATLAS_SAGE && own) {
        Frag<T, VEC> me;
        me.load(tile + (vg - tile_lo) * ldx + col);
        float h[VEC];
#pragma unroll
        for (int e = 0; e < VEC; e++) h[e] = me.get(e);
        store_f32<VEC>(out + d + col, h);
      }
    }
    consumed = base - beg;
  }
  if (lane == 0) {
    cursor[v] = beg + consumed;
    touched[v] = 1;
  }
}

// ---------------------------------------------------------------------------
// runs front end: warp per (chunk, destination) run

template <typename T, int VEC, int MODEL>
__global__ void __launch_bounds__(256)
    agg_runs(const T* __restrict__ tile, int64_t ldx,
             const uint32_t* __restrict__ run_dst,
             const int64_t* __restrict__ run_beg, int64_t nruns,
             const uint32_t* __restrict__ ent_src,
             const uint32_t* __restrict__ indeg, int d,
             float* __restrict__ acc, int64_t ldacc,
             uint8_t* __restrict__ touched, float self_scale) {
  constexpr bool kMean = MODEL != ATLAS_GIN;
  const int lane = threadIdx.x & 31;
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (r >= nruns) return;
  const uint32_t v = run_dst[r];
  const int64_t beg = run_beg[r], end = run_beg[r + 1];
  const float denom = kMean ? (float)max(1u, indeg[v]) : 1.0f;
  const float rcp = kMean ? __frcp_rn(denom) : 1.0f;
  const bool resume = touched[v] != 0;
  float* out = acc + (int64_t)v * ldacc;
  for (int c0 = 0; c0 < d; c0 += 32 * VEC) {
    const int col = c0 + lane * VEC;
    const bool active = col < d;
    float a[VEC];
#pragma unroll
    for (int e = 0; e < VEC; e++) a[e] = 0.0f;
    if (resume && active) load_f32<VEC>(out + col, a);
    for (int64_t base = beg; base < end; base += 32) {
      const int cnt = (int)((end - base) < 32 ? (end - base) : 32);
      const uint32_t mine = lane < cnt ? ent_src[base + lane] : 0u;
      for (int i = 0; i < cnt; i += kUnroll) {
        Frag<T, VEC> f[kUnroll];
        uint32_t s[kUnroll];
#pragma unroll
        for (int j = 0; j < kUnroll; j++) {
          s[j] = __shfl_sync(0xffffffffu, mine, (i + j) & 31);
          if (active && i + j < cnt)
            f[j].load(tile + (int64_t)(s[j] & ~kSelfBit) * ldx + col);
        }
#pragma unroll
        for (int j = 0; j < kUnroll; j++)
          if (active && i + j < cnt)
            add_msg<T, VEC, kMean>(a, f[j], (s[j] & kSelfBit) != 0, denom,
                                   rcp, self_scale);
      }
    }
    if (active) store_f32<VEC>(out + col, a);
  }
  if (lane == 0) touched[v] = 1;
}

template <typename T>
__global__ void sage_self_rows(const T* __restrict__ tile, int64_t ldx,
                               int64_t nrows, int d, float* __restrict__ out,
                               int64_t ldacc) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.y + threadIdx.y;
  if (i >= nrows) return;
  for (int c = threadIdx.x; c < d; c += blockDim.x)
    out[i * ldacc + c] = to_f32(tile[i * ldx + c]);
}

__global__ void gather_rows_kernel(const float* __restrict__ acc,
                                   int64_t ldacc,
                                   const int32_t* __restrict__ ids, int64_t n,
                                   int64_t width, float* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.y + threadIdx.y;
  if (i >= n) return;
  const float* src = acc + (int64_t)ids[i] * ldacc;
  for (int64_t c = threadIdx.x; c < width; c += blockDim.x)
    out[i * width + c] = src[c];
}

template <typename T>
int pick_vec(int d, int64_t ldx) {
  if (sizeof(T) == 4) return (d % 4 == 0 && ldx % 4 == 0) ? 4 : 1;
  if (d % 8 == 0 && ldx % 8 == 0) return 8;
  if (d % 2 == 0 && ldx % 2 == 0) return 2;
  return 1;
}

template <typename T, int VEC>
void resident_model(const atlas_graph* g, const T* x, int64_t ldx, int model,
                    float eps1, int d, float* acc, int64_t ldacc, int64_t v0,
                    int64_t v1, cudaStream_t s) {
  // destinations [v0, v1) of the rank: the CSC pointers, in-degrees and
  // global ids are offset views, acc row 0 is destination v0
  const int64_t* csc_ptr = g->csc_ptr.ptr + v0;
  const uint32_t* indeg = g->indeg.ptr + v0;
  const int64_t lo = g->lo + v0, nloc = v1 - v0;
  const int64_t blocks = ceil_div(nloc, 8);
  if (blocks == 0) return;
  // whether the division guard is needed: the producing transform's flag,
  // or one pass over the input
  g->scan_flag.reserve(1);
  const int* flag = g->known_flag;
  if (!flag) {
    ATLAS_CUDA(cudaMemsetAsync(g->scan_flag.ptr, 0, sizeof(int), s));
    launch_scan<T>(x, g->V, d, ldx, g->scan_flag.ptr, s);
    flag = g->scan_flag.ptr;
  }
  if constexpr (VEC * sizeof(T) == 16) if (d <= 32 * VEC) {
    // ring kernel: persistent warps, dynamic destination batches; rows of
    // <= 16 chunks run 32/LPD destination runs per warp in lockstep
    g->work.reserve(1);
    ATLAS_CUDA(cudaMemsetAsync(g->work.ptr, 0, sizeof(unsigned long long), s));
    const int smem = 8 * kRing * 32 * 16;
    auto ring = [&](auto kern) {
      ATLAS_CUDA(cudaFuncSetAttribute(
          kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kern<<<num_sms() * 3, 256, smem, s>>>(
          x, ldx, csc_ptr, g->csc_src.ptr, indeg, lo,
          nloc, d, acc, ldacc, eps1, flag, g->work.ptr);
    };
    if (d <= 16 * VEC) {
      const int sub_smem = 8 * kSubRing * 32 * 16 + 8 * kSubMeta<8> * 4;
      auto sub = [&](auto kern) {
        ATLAS_CUDA(cudaFuncSetAttribute(
            kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sub_smem));
        kern<<<num_sms() * kSubBlocks, 256, sub_smem, s>>>(
            x, ldx, csc_ptr, g->csc_src.ptr, indeg, lo,
            nloc, d, acc, ldacc, eps1, flag, g->work.ptr);
      };
      if (d <= 8 * VEC) {
        if (model == ATLAS_GCN) sub(agg_sub_ring<T, 8, ATLAS_GCN>);
        else if (model == ATLAS_SAGE) sub(agg_sub_ring<T, 8, ATLAS_SAGE>);
        else sub(agg_sub_ring<T, 8, ATLAS_GIN>);
      } else {
        if (model == ATLAS_GCN) sub(agg_sub_ring<T, 16, ATLAS_GCN>);
        else if (model == ATLAS_SAGE) sub(agg_sub_ring<T, 16, ATLAS_SAGE>);
        else sub(agg_sub_ring<T, 16, ATLAS_GIN>);
      }
    } else {
      if (model == ATLAS_GCN) ring(agg_ring<T, VEC, ATLAS_GCN>);
      else if (model == ATLAS_SAGE) ring(agg_ring<T, VEC, ATLAS_SAGE>);
      else ring(agg_ring<T, VEC, ATLAS_GIN>);
    }
    count_launch();
    ATLAS_LAUNCH_CHECK();
    return;
  }
  const int64_t row_bytes = (int64_t)d * sizeof(T);
  if constexpr (VEC * sizeof(T) == 16) if (row_bytes <= 8 * 512 &&
      (ldx * (int64_t)sizeof(T)) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    // bulk-copy kernel: one TMA row copy per in-edge, mbarrier ring
    g->work.reserve(1);
    ATLAS_CUDA(cudaMemsetAsync(g->work.ptr, 0, sizeof(unsigned long long), s));
    auto bulk = [&](auto kern, int slots) {
      const int smem = kBulkWarps * slots * (8 + (int)row_bytes);
      ATLAS_CUDA(cudaFuncSetAttribute(
          kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      int per_sm = 0;
      ATLAS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, kern, kBulkWarps * 32, smem));
      kern<<<num_sms() * std::max(1, per_sm), kBulkWarps * 32, smem, s>>>(
          x, ldx, csc_ptr, g->csc_src.ptr, indeg, lo,
          nloc, d, acc, ldacc, eps1, flag, g->work.ptr);
    };
    auto by_model = [&](auto ch) {
      constexpr int CH = decltype(ch)::value;
      if (model == ATLAS_GCN) bulk(agg_bulk<T, CH, ATLAS_GCN>, 16 / CH);
      else if (model == ATLAS_SAGE) bulk(agg_bulk<T, CH, ATLAS_SAGE>, 16 / CH);
      else bulk(agg_bulk<T, CH, ATLAS_GIN>, 16 / CH);
    };
    if (row_bytes <= 2 * 512) by_model(std::integral_constant<int, 2>());
    else if (row_bytes <= 4 * 512) by_model(std::integral_constant<int, 4>());
    else by_model(std::integral_constant<int, 8>());
    count_launch();
    ATLAS_LAUNCH_CHECK();
    return;
  }
  auto go = [&](auto kern) {
    kern<<<(unsigned)blocks, 256, 0, s>>>(
        x, ldx, csc_ptr, g->csc_src.ptr, indeg, lo, nloc,
        d, acc, ldacc, eps1, flag);
  };
  if (model == ATLAS_GCN) go(agg_resident<T, VEC, ATLAS_GCN>);
  else if (model == ATLAS_SAGE) go(agg_resident<T, VEC, ATLAS_SAGE>);
  else go(agg_resident<T, VEC, ATLAS_GIN>);
  count_launch();
  ATLAS_LAUNCH_CHECK();
}

template <typename T>
void resident_typed(const atlas_graph* g, const void* x, int64_t ldx,
                    int model, float eps1, int d, float* acc, int64_t ldacc,
                    int64_t v0, int64_t v1, cudaStream_t s) {
  const T* xt = static_cast<const T*>(x);
  int vec = pick_vec<T>(d, ldx);
  if (vec > 1 && ldacc % 4 != 0) vec = 1;
  if (sizeof(T) == 4) {
    if (vec == 4) resident_model<T, 4>(g, xt, ldx, model, eps1, d, acc, ldacc, v0, v1, s);
    else resident_model<T, 1>(g, xt, ldx, model, eps1, d, acc, ldacc, v0, v1, s);
  } else {
    if (vec == 8) resident_model<T, 8>(g, xt, ldx, model, eps1, d, acc, ldacc, v0, v1, s);
    else if (vec == 2) resident_model<T, 2>(g, xt, ldx, model, eps1, d, acc, ldacc, v0, v1, s);
    else resident_model<T, 1>(g, xt, ldx, model, eps1, d, acc, ldacc, v0, v1, s);
  }
}

template <typename T, int VEC>
void runs_model(const T* tile, int64_t ldx, const uint32_t* run_dst,
                const int64_t* run_beg, int64_t nruns, const uint32_t* ent,
                const uint32_t* indeg, int model, float eps1, int d,
                float* acc, int64_t ldacc, uint8_t* touched, cudaStream_t s) {
  const int64_t blocks = ceil_div(nruns, 8);
  if (blocks == 0) return;
  auto go = [&](auto kern) {
    kern<<<(unsigned)blocks, 256, 0, s>>>(tile, ldx, run_dst, run_beg, nruns,
                                          ent, indeg, d, acc, ldacc, touched,
                                          eps1);
  };
  if (model == ATLAS_GCN) go(agg_runs<T, VEC, ATLAS_GCN>);
  else if (model == ATLAS_SAGE) go(agg_runs<T, VEC, ATLAS_SAGE>);
  else go(agg_runs<T, VEC, ATLAS_GIN>);
  count_launch();
  ATLAS_LAUNCH_CHECK();
}

template <typename T>
void runs_typed(const void* tile, int64_t ldx, const uint32_t* run_dst,
                const int64_t* run_beg, int64_t nruns, const uint32_t* ent,
                const uint32_t* indeg, int model, float eps1, int d,
                float* acc, int64_t ldacc, uint8_t* touched, cudaStream_t s) {
  const T* t = static_cast<const T*>(tile);
  int vec = pick_vec<T>(d, ldx);
  if (vec > 1 && ldacc % 4 != 0) vec = 1;
  if (sizeof(T) == 4) {
    if (vec == 4) runs_model<T, 4>(t, ldx, run_dst, run_beg, nruns, ent, indeg, model, eps1, d, acc, ldacc, touched, s);
    else runs_model<T, 1>(t, ldx, run_dst, run_beg, nruns, ent, indeg, model, eps1, d, acc, ldacc, touched, s);
  } else {
    if (vec == 8) runs_model<T, 8>(t, ldx, run_dst, run_beg, nruns, ent, indeg, model, eps1, d, acc, ldacc, touched, s);
    else if (vec == 2) runs_model<T, 2>(t, ldx, run_dst, run_beg, nruns, ent, indeg, model, eps1, d, acc, ldacc, touched, s);
    else runs_model<T, 1>(t, ldx, run_dst, run_beg, nruns, ent, indeg, model, eps1, d, acc, ldacc, touched, s);
  }
}

// ---------------------------------------------------------------------------
// streamed front end, LAST tile of a whole-input stream (GCN, f32 rows of
// <= 512 B): every edge a destination still has, [cursor[v], end_v), has its
// source in this tile, so the remaining work is each destination's edge
// SUFFIX. Persistent warps take 32 destinations, concatenate their suffixes
// (warp scan of the lengths) and stream the rows through the per-lane
// cp.async ring of agg_ring across destination boundaries; each record is
// resumed from acc when an earlier tile touched it, folded in source order
// exactly like agg_tile (same guarded divide and add), and stored. This is
// the part of the stream left after the last copy lands, so it is what the
// end-to-end time sees; agg_tile (a warp per destination, ~6 edges per
// tile) runs it at a third of the DRAM rate.
// Occupancy: 5 blocks/SM caps registers at 51; ptxas -v reports 42 and no
// spills for VEC=4 (the 64-register note on kSubBlocks is for
// agg_sub_ring's lockstep sub-groups, not this kernel).
// MODEL = ATLAS_SAGE: the neighbour half is the same mean; the self half
// (columns [d, 2d) of the record) is the destination's own row, copied when
// that row is in the tile (agg_tile's SAGE rule). MODEL = ATLAS_GIN: a sum
// (no division) with the self term (1 + eps) * x_v folded at its place in
// ascending source order -- before the first remaining source >= v -- in
// the tile holding row v. T: the stored input type (f32 or 2-byte rows,
// widened exactly); each lane moves 16 B of the row per edge.
template <typename T, int VEC, int MODEL>
__global__ void __launch_bounds__(256, kSubBlocks + 1)
    agg_suffix_ring(const T* __restrict__ tile, int64_t ldx,
                    int64_t tile_lo, int64_t tile_hi, int64_t V,
                    const int64_t* __restrict__ csc_ptr,
                    const uint32_t* __restrict__ csc_src,
                    const uint32_t* __restrict__ indeg, int64_t lo,
                    int64_t nloc, int d, float* __restrict__ acc,
                    int64_t ldacc, int64_t* __restrict__ cursor,
                    uint8_t* __restrict__ touched,
                    unsigned long long* __restrict__ work,
                    float self_scale) {
  using F = Frag<T, VEC>;
  constexpr bool kMean = MODEL != ATLAS_GIN;
  extern __shared__ uint4 ring_smem[];
  const int lane = threadIdx.x & 31;
  const int col = lane * VEC;
  const bool active = col < d;
  const int colc = active ? col : d - VEC;
  const uint32_t ring_lane =
      (uint32_t)__cvta_generic_to_shared(ring_smem +
                                         (threadIdx.x >> 5) * (kSubRing * 32)) +
      (uint32_t)lane * 16u;
  const T* __restrict__ xc = tile + colc;
  while (true) {
    unsigned long long v0 = 0;
    if (lane == 0) v0 = atomicAdd(work, (unsigned long long)kGrab);
    v0 = __shfl_sync(0xffffffffu, v0, 0);
    if ((int64_t)v0 >= nloc) break;
    const int64_t v1 = min((int64_t)v0 + kGrab, nloc);
    // lane j: destination v0 + j, its suffix [b_j, b_j + n_j), its place
    // off_j in the grab's concatenated edge list; GIN: sp_j = edges of the
    // suffix before the self term (sources < v)
    const int64_t vj = (int64_t)v0 + lane;
    int64_t b_j = 0;
    int n_j = 0, sp_j = 0;
    uint32_t dg_j = 0, tch_j = 0;  // in-degree, touched flag of v0 + j
    if (vj < v1) {
      b_j = cursor[vj];
      int64_t e = csc_ptr[vj + 1];
      if (tile_hi < V) {  // the ascending sources below tile_hi
        int64_t a = b_j;
        while (a < e) {
          const int64_t m = (a + e) >> 1;
          if ((int64_t)csc_src[m] < tile_hi) a = m + 1;
          else e = m;
        }
        cursor[vj] = e;  // the next tile resumes here
      }
      n_j = (int)(e - b_j);
      if (MODEL == ATLAS_GIN) {
        const int64_t vg = vj + lo;
        int64_t a = b_j, z = e;
        while (a < z) {
          const int64_t m = (a + z) >> 1;
          if ((int64_t)csc_src[m] < vg) a = m + 1;
          else z = m;
        }
        sp_j = (int)(a - b_j);
      }
      dg_j = indeg[vj];
      tch_j = touched[vj];
    }
    int off_j = n_j;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, off_j, o);
      if (lane >= o) off_j += y;
    }
    const int ne = __shfl_sync(0xffffffffu, off_j, 31);
    off_j -= n_j;  // exclusive
    // source id of grab edge k: the last destination j with off_j <= k
    auto src_of = [&](int k) -> uint32_t {
      int j = 0;
#pragma unroll
      for (int st = 16; st >= 1; st >>= 1) {
        const int oc = __shfl_sync(0xffffffffu, off_j, (j + st) & 31);
        if (j + st < 32 && oc <= k) j += st;
      }
      const int64_t bj = __shfl_sync(0xffffffffu, b_j, j);
      const int oj = __shfl_sync(0xffffffffu, off_j, j);
      return k < ne ? csc_src[bj + (k - oj)] : 0u;
    };
    int pe = 0;
    uint32_t isrc = src_of(lane);
    auto issue = [&]() {
      if (pe < ne) {
        if ((pe & 31) == 0 && pe != 0) isrc = src_of(pe + lane);
        const uint32_t u = __shfl_sync(0xffffffffu, isrc, pe & 31);
        cp_async16_s(ring_lane + ((uint32_t)(pe & (kSubRing - 1)) << 9),
                     xc + ((int64_t)u - tile_lo) * ldx);
        pe++;
      }
      cp_async_commit();
    };
#pragma unroll 1
    for (int k = 0; k < kSubRing; k++) issue();
    int ce = 0;
    for (int j = 0; j < (int)(v1 - (int64_t)v0); j++) {
      const int64_t v = (int64_t)v0 + j;
      const int nj = __shfl_sync(0xffffffffu, n_j, j);
      const uint32_t dg = __shfl_sync(0xffffffffu, dg_j, j);
      const bool own = v + lo >= tile_lo && v + lo < tile_hi;
      // GCN: a zero in-degree destination owes a zero record once (in its
      // own row's tile); SAGE / GIN: the own row's tile writes the self
      // half / folds the self term
      const bool must = MODEL == ATLAS_GCN ? (own && dg == 0) : own;
      if (nj == 0 && !must) continue;
      const float denom = kMean ? (float)max(1u, dg) : 1.0f;
      const float rcp = kMean ? __frcp_rn(denom) : 1.0f;
      float a[VEC];
#pragma unroll
      for (int e = 0; e < VEC; e++) a[e] = 0.0f;
      const bool resume = __shfl_sync(0xffffffffu, tch_j, j) != 0;
      float* out = acc + v * ldacc;
      if (resume && active) load_f32<VEC>(out + col, a);
      const int sp = MODEL == ATLAS_GIN && own
                         ? __shfl_sync(0xffffffffu, sp_j, j) : -1;
      auto fold_self = [&]() {
        if (active) {
          F me;
          me.load(tile + (v + lo - tile_lo) * ldx + col);
          add_msg<T, VEC, false>(a, me, true, 1.0f, 1.0f, self_scale);
        }
      };
      for (int c = 0; c < nj; c++, ce++) {
        if (c == sp) fold_self();
        cp_async_wait<kSubRing - 1>();
        F f;
        f.raw = lds16(ring_lane + ((uint32_t)(ce & (kSubRing - 1)) << 9));
        add_msg<T, VEC, kMean>(a, f, false, denom, rcp, 1.0f);
        issue();
      }
      if (sp == nj) fold_self();  // every remaining source is below v
      if (active) {
        store_f32<VEC>(out + col, a);
        if (MODEL == ATLAS_SAGE && own) {
          F me;
          me.load(tile + (v + lo - tile_lo) * ldx + col);
          float h[VEC];
#pragma unroll
          for (int e = 0; e < VEC; e++) h[e] = me.get(e);
          store_f32<VEC>(out + d + col, h);
        }
      }
      if (lane == 0) touched[v] = 1;
    }
    cp_async_wait<0>();
  }
}

struct TileArgs {
  int64_t ldx, tile_lo, tile_hi;
  const atlas_graph* g;
  int model, d;
  float eps1;
  float* acc;
  int64_t ldacc;
  int64_t* cursor;
  uint8_t* touched;
};

template <typename T, int VEC>
void tile_model(const T* x, const TileArgs& a, cudaStream_t s) {
  const int64_t blocks = ceil_div(a.g->nloc, 8);
  if (blocks == 0) return;
  auto go = [&](auto kern) {
    kern<<<(unsigned)blocks, 256, 0, s>>>(
        x, a.ldx, a.tile_lo, a.tile_hi, a.g->csc_ptr.ptr, a.g->csc_src.ptr,
        a.g->indeg.ptr, a.g->lo, a.g->nloc, a.d, a.acc, a.ldacc, a.cursor,
        a.touched, a.eps1);
  };
  if (a.model == ATLAS_GCN) go(agg_tile<T, VEC, ATLAS_GCN>);
  else if (a.model == ATLAS_SAGE) go(agg_tile<T, VEC, ATLAS_SAGE>);
  else go(agg_tile<T, VEC, ATLAS_GIN>);
  count_launch();
  ATLAS_LAUNCH_CHECK();
}

template <typename T>
void tile_typed(const void* x, const TileArgs& a, cudaStream_t s) {
  const T* t = static_cast<const T*>(x);
  int vec = pick_vec<T>(a.d, a.ldx);
  if (vec > 1 && a.ldacc % 4 != 0) vec = 1;
  if (sizeof(T) == 4) {
    if (vec == 4) tile_model<T, 4>(t, a, s);
    else tile_model<T, 1>(t, a, s);
  } else {
    if (vec == 8) tile_model<T, 8>(t, a, s);
    else if (vec == 2) tile_model<T, 2>(t, a, s);
    else tile_model<T, 1>(t, a, s);
  }
}

}  // namespace

void launch_agg_tile(const void* tile, int dtype, int64_t ldx, int64_t tile_lo,
                     int64_t tile_hi, const atlas_graph* g, int model,
                     float gin_epsilon, int d, float* acc, int64_t ldacc,
                     int64_t* cursor, uint8_t* touched, cudaStream_t s) {
  TileArgs a{ldx, tile_lo, tile_hi, g, model, d, 1.0f + gin_epsilon, acc,
             ldacc, cursor, touched};
  if (dtype == ATLAS_F32) tile_typed<float>(tile, a, s);
  else if (dtype == ATLAS_F16) tile_typed<__half>(tile, a, s);
  else tile_typed<__nv_bfloat16>(tile, a, s);
}

bool launch_agg_suffix(const void* tile, int dtype, int64_t ldx,
                       int64_t tile_lo, int64_t tile_hi,
                       const atlas_graph* g, int model, float gin_epsilon,
                       int d, float* acc, int64_t ldacc, int64_t* cursor,
                       uint8_t* touched, cudaStream_t s) {
  // 16 B per lane per edge: f32 rows up to 128 columns, 2-byte rows up to
  // 256, whole 16-B chunks, 16-B aligned rows
  const int es = dtype == ATLAS_F32 ? 4 : 2;
  const int vec = 16 / es;
  if (d % vec != 0 || d > 32 * vec || (ldx * es) % 16 != 0 ||
      ldacc % 4 != 0 || (reinterpret_cast<uintptr_t>(tile) & 15) != 0)
    return false;
  if (g->nloc == 0) return true;
  g->work.reserve(1);
  ATLAS_CUDA(cudaMemsetAsync(g->work.ptr, 0, sizeof(unsigned long long), s));
  const int smem = 8 * kSubRing * 32 * 16;
  const float e1 = 1.0f + gin_epsilon;  // np.float32(1) + np.float32(eps)
  auto go = [&](auto kern, auto tag) {
    using T = decltype(tag);
    ATLAS_CUDA(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<num_sms() * (kSubBlocks + 1), 256, smem, s>>>(
        static_cast<const T*>(tile), ldx, tile_lo, tile_hi, g->V,
        g->csc_ptr.ptr, g->csc_src.ptr, g->indeg.ptr, g->lo, g->nloc, d, acc,
        ldacc, cursor, touched, g->work.ptr, e1);
  };
  auto by_model = [&](auto tag) {
    using T = decltype(tag);
    constexpr int V = 16 / sizeof(T);
    if (model == ATLAS_GCN) go(agg_suffix_ring<T, V, ATLAS_GCN>, tag);
    else if (model == ATLAS_SAGE) go(agg_suffix_ring<T, V, ATLAS_SAGE>, tag);
    else go(agg_suffix_ring<T, V, ATLAS_GIN>, tag);
  };
  if (dtype == ATLAS_F32) by_model(float());
  else if (dtype == ATLAS_F16) by_model(__half());
  else by_model(__nv_bfloat16());
  count_launch();
  ATLAS_LAUNCH_CHECK();
  return true;
}

// numpy: np.float32(1.0) + np.float32(eps), rounded to f32
static float self_scale_of(float eps) { return 1.0f + eps; }

void launch_agg_resident(const atlas_graph* g, const void* x, int dtype,
                         int64_t ldx, int model, float gin_epsilon, int d,
                         float* acc, int64_t ldacc, const int32_t* input_flag,
                         cudaStream_t s) {
  g->known_flag = input_flag;
  launch_agg_resident_range(g, x, dtype, ldx, model, gin_epsilon, d, acc,
                            ldacc, 0, g->nloc, s);
}

// destinations [v0, v1) only (blocked records, atlas_layer_run_blocked):
// record row 0 of acc is destination v0; with g->known_flag unset the
// input is scanned for extremes on every call
void launch_agg_resident_range(const atlas_graph* g, const void* x, int dtype,
                               int64_t ldx, int model, float gin_epsilon,
                               int d, float* acc, int64_t ldacc, int64_t v0,
                               int64_t v1, cudaStream_t s) {
  if (v1 <= v0) return;
  const float e1 = self_scale_of(gin_epsilon);
  if (dtype == ATLAS_F32)
    resident_typed<float>(g, x, ldx, model, e1, d, acc, ldacc, v0, v1, s);
  else if (dtype == ATLAS_F16)
    resident_typed<__half>(g, x, ldx, model, e1, d, acc, ldacc, v0, v1, s);
  else
    resident_typed<__nv_bfloat16>(g, x, ldx, model, e1, d, acc, ldacc, v0,
                                  v1, s);
}

void launch_agg_resident_epi(const atlas_graph* g, const float* z,
                             int64_t ldz, int data_model, float gin_epsilon,
                             int d, const int32_t* input_flag, void* y,
                             int y_dtype, int64_t ldy, const float* bias,
                             const float* self_rows, int64_t ld_self, int n,
                             int relu, int32_t* out_flag, int64_t v_begin,
                             int64_t v_end, cudaStream_t s) {
  if (v_end <= v_begin) return;
  if (d > 128 || d % 4 != 0 || ldz % 4 != 0 ||
      (reinterpret_cast<uintptr_t>(z) & 15) != 0)
    fail(ATLAS_ECONFIG, "transform-first aggregation needs <= 128 f32 "
                        "columns in 16-byte rows");
  EpiArgs epi{y, ldy, bias, self_rows, ld_self, n, relu, out_flag, v_begin};
  const float e1 = self_scale_of(gin_epsilon);
  if (d <= 64) {  // narrow rows: several destinations per warp
    g->work.reserve(1);
    ATLAS_CUDA(cudaMemsetAsync(g->work.ptr, 0, sizeof(unsigned long long), s));
    auto narrow = [&](auto lpd_tag, auto model_tag) {
      constexpr int LPD = decltype(lpd_tag)::value;
      constexpr int M = decltype(model_tag)::value;
      const int smem = 8 * kTfRing<LPD> * 32 * 16;
      auto go = [&](auto kern) {
        ATLAS_CUDA(cudaFuncSetAttribute(
            kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int per_sm = 0;
        ATLAS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, kern, 256, smem));
        kern<<<num_sms() * std::max(1, per_sm), 256, smem, s>>>(
            z, ldz, g->csc_ptr.ptr, g->csc_src.ptr, g->indeg.ptr, g->lo,
            v_end, d, e1, epi, g->work.ptr);
      };
      if (y_dtype == ATLAS_F32) go(agg_tf_ring<LPD, M, float>);
      else if (y_dtype == ATLAS_F16) go(agg_tf_ring<LPD, M, __half>);
      else go(agg_tf_ring<LPD, M, __nv_bfloat16>);
    };
    auto by_model = [&](auto lpd_tag) {
      if (data_model == ATLAS_GIN)
        narrow(lpd_tag, std::integral_constant<int, ATLAS_GIN>());
      else
        narrow(lpd_tag, std::integral_constant<int, ATLAS_GCN>());
    };
    static const bool old_ring = [] {
      const char* e = std::getenv("ATLAS_TF_RING");
      return e && std::string(e) == "old";
    }();
    static const int depth = [] {
      const char* e = std::getenv("ATLAS_TF_DEPTH");
      return e ? std::atoi(e) : 0;
    }();
    const int nch = d / 4;
    if (old_ring) {
      if (d <= 32) by_model(std::integral_constant<int, 8>());
      else by_model(std::integral_constant<int, 16>());
    } else {
      // lanes per row x chunks per lane covering nch with the least waste
      auto multi = [&](auto lpd_tag, auto cpl_tag, auto depth_tag,
                       auto minb_tag) {
        constexpr int LPD = decltype(lpd_tag)::value;
        constexpr int CPL = decltype(cpl_tag)::value;
        constexpr int DEPTH = decltype(depth_tag)::value;
        constexpr int MINB = decltype(minb_tag)::value;
        const int smem = 8 * DEPTH * CPL * 32 * 16 +
                         8 * (2 * kGrab * (32 / LPD) + 4) * 4;
        auto go = [&](auto kern) {
          ATLAS_CUDA(cudaFuncSetAttribute(
              kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          int per_sm = 0;
          ATLAS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
              &per_sm, kern, 256, smem));
          kern<<<num_sms() * std::max(1, per_sm), 256, smem, s>>>(
              z, ldz, g->csc_ptr.ptr, g->csc_src.ptr, g->indeg.ptr, g->lo,
              v_end, d, e1, epi, g->work.ptr);
        };
        auto by_out = [&](auto model_tag) {
          constexpr int M = decltype(model_tag)::value;
          if (y_dtype == ATLAS_F32)
            go(agg_tf_multi<LPD, CPL, DEPTH, M, float, MINB>);
          else if (y_dtype == ATLAS_F16)
            go(agg_tf_multi<LPD, CPL, DEPTH, M, __half, MINB>);
          else
            go(agg_tf_multi<LPD, CPL, DEPTH, M, __nv_bfloat16, MINB>);
        };
        if (data_model == ATLAS_GIN)
          by_out(std::integral_constant<int, ATLAS_GIN>());
        else
          by_out(std::integral_constant<int, ATLAS_GCN>());
      };
      using I = std::integral_constant<int, 1>;
      using I2 = std::integral_constant<int, 2>;
      using I3 = std::integral_constant<int, 3>;
      using I4 = std::integral_constant<int, 4>;
      using I5 = std::integral_constant<int, 5>;
      using I8 = std::integral_constant<int, 8>;
      using I16 = std::integral_constant<int, 16>;
      // measured (profiles/r2_tf_multi_shapes.txt): 8-lane groups with a
      // 4-deep ring at 4-5 blocks/SM beat both wider groups (fewer edges
      // per iteration) and narrower ones (more flushes per iteration)
      if (nch <= 4) multi(I4(), I(), I4(), I5());
      else if (nch <= 8) multi(I8(), I(), I4(), I5());
      else if (nch <= 12) {
        if (depth == 6) multi(I8(), I2(), I4(), I5());
        else if (depth == 7) multi(I8(), I2(), I2(), I4());
        else if (depth == 9) multi(I16(), I(), I4(), I5());
        else if (depth == 4) multi(I4(), I3(), I4(), I3());
        else multi(I8(), I2(), I4(), I4());
      } else multi(I8(), I2(), I4(), I4());
    }
    count_launch();
    ATLAS_LAUNCH_CHECK();
    return;
  }
  const int* flag = input_flag;
  if (!flag) {
    g->scan_flag.reserve(1);
    ATLAS_CUDA(cudaMemsetAsync(g->scan_flag.ptr, 0, sizeof(int), s));
    launch_scan<float>(z, g->V, d, ldz, g->scan_flag.ptr, s);
    flag = g->scan_flag.ptr;
  }
  g->work.reserve(1);
  ATLAS_CUDA(cudaMemsetAsync(g->work.ptr, 0, sizeof(unsigned long long), s));
  const int smem = 8 * kRing * 32 * 16;
  auto go = [&](auto kern) {
    ATLAS_CUDA(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<num_sms() * 3, 256, smem, s>>>(z, ldz, g->csc_ptr.ptr, g->csc_src.ptr,
                                    g->indeg.ptr, g->lo, v_end, d, e1, flag,
                                    g->work.ptr, epi);
  };
  auto by_out = [&](auto model_tag) {
    constexpr int M = decltype(model_tag)::value;
    if (y_dtype == ATLAS_F32) go(agg_ring_epi<M, float>);
    else if (y_dtype == ATLAS_F16) go(agg_ring_epi<M, __half>);
    else go(agg_ring_epi<M, __nv_bfloat16>);
  };
  if (data_model == ATLAS_GIN) by_out(std::integral_constant<int, ATLAS_GIN>());
  else by_out(std::integral_constant<int, ATLAS_GCN>());
  count_launch();
  ATLAS_LAUNCH_CHECK();
}

void launch_agg_runs(const void* tile, int dtype, int64_t ldx,
                     int64_t /*tile_lo*/, const uint32_t* run_dst,
                     const int64_t* run_beg, int64_t nruns,
                     const uint32_t* ent_src, const uint32_t* indeg,
                     int model, float gin_epsilon, int d, float* acc,
                     int64_t ldacc, uint8_t* touched, cudaStream_t s) {
  const float e1 = self_scale_of(gin_epsilon);
  if (dtype == ATLAS_F32)
    runs_typed<float>(tile, ldx, run_dst, run_beg, nruns, ent_src, indeg,
                      model, e1, d, acc, ldacc, touched, s);
  else if (dtype == ATLAS_F16)
    runs_typed<__half>(tile, ldx, run_dst, run_beg, nruns, ent_src, indeg,
                       model, e1, d, acc, ldacc, touched, s);
  else
    runs_typed<__nv_bfloat16>(tile, ldx, run_dst, run_beg, nruns, ent_src,
                              indeg, model, e1, d, acc, ldacc, touched, s);
}

void launch_sage_self(const void* tile, int dtype, int64_t ldx, int64_t row0,
                      int64_t nrows, int d, float* acc_rows, int64_t ldacc,
                      cudaStream_t s) {
  if (nrows <= 0) return;
  dim3 block(32, 8);
  unsigned grid = (unsigned)ceil_div(nrows, 8);
  if (dtype == ATLAS_F32)
    sage_self_rows<float><<<grid, block, 0, s>>>(
        static_cast<const float*>(tile) + row0 * ldx, ldx, nrows, d, acc_rows,
        ldacc);
  else if (dtype == ATLAS_F16)
    sage_self_rows<__half><<<grid, block, 0, s>>>(
        static_cast<const __half*>(tile) + row0 * ldx, ldx, nrows, d,
        acc_rows, ldacc);
  else
    sage_self_rows<__nv_bfloat16><<<grid, block, 0, s>>>(
        static_cast<const __nv_bfloat16*>(tile) + row0 * ldx, ldx, nrows, d,
        acc_rows, ldacc);
  count_launch();
  ATLAS_LAUNCH_CHECK();
}

void launch_gather_rows(const float* acc, int64_t ldacc, const int32_t* ids,
                        int64_t n, int64_t width, float* out, cudaStream_t s) {
  if (n <= 0) return;
  dim3 block(32, 8);
  gather_rows_kernel<<<(unsigned)ceil_div(n, 8), block, 0, s>>>(
      acc, ldacc, ids, n, width, out);
  count_launch();
  ATLAS_LAUNCH_CHECK();
}

}  // namespace atlas
