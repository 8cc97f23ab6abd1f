// Dense layer transform on the 5th-gen tensor cores (kernel plan K9).
//
// y = act(x . W^T + b), x (M x K) f32 row-major, W (N x K) f32.
// The reference computes this in f32 (oocgnn/compute.py:39-47); tcgen05
// has no f32 kind, so we use the 3xTF32 split: a = a_hi + a_lo with a_hi
// = a truncated to tf32 and a_lo = a - a_hi (exact in f32), and
//   D = a_hi.w_hi + a_hi.w_lo + a_lo.w_hi       (f32 accumulate in TMEM)
// which keeps ~f32 accuracy (dropped a_lo.w_lo and the tf32 rounding of
// the lo parts are ~2^-22 relative). The tensor-core work is 3x a plain
// GEMM, which is free here: at N <= 256 the transform is HBM-bound.
//
// Structure (persistent, one CTA per SM, warp-specialised):
//   warp 0      TMA producer: x tile (128 x 32 f32, SWIZZLE_128B) and the
//               w_hi / w_lo tiles (BN x 32) per k-block, mbarrier tx count
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5   splitter: x tile -> x_hi (in place) + x_lo (generic proxy
//               writes, then fence.proxy.async before the MMA reads)
//   warps 6-13  epilogue: tcgen05.ld 32x32b -> per-warp smem transpose ->
//               +bias -> ReLU -> 16-B row-contiguous stores; warp 6+q and
//               10+q share TMEM lane quarter q and alternate 16-col blocks
// Two TMEM accumulators (2 x BN columns) let the epilogue of tile t
// overlap the MMAs of tile t+1.
#include <cuda.h>

#include <memory>
#include <mutex>
#include <vector>

#include "internal.cuh"

namespace atlas {
namespace {

constexpr int BM = 128, BK = 32;  // BK f32 = 128 B = one swizzle atom row
constexpr int kEpiWarps = 8;           // two per TMEM lane quarter
constexpr int kStageLd = 20;           // 32 x 16 staging block, padded
constexpr int kThreads = (6 + kEpiWarps) * 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map,
                                            uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx"
      "::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0),
      "r"(c1)
      : "memory");
}

// L2 prefetch of a tensor tile (no shared memory, no barrier): the
// producers run these a few k-blocks ahead of their shared-memory loads so
// the loads hit L2 instead of waiting a full DRAM latency; the x bytes in
// flight are then no longer bounded by the stages that fit next to W
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0,
                                                int c1) {
  asm volatile(
      "cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1)
      : "memory");
}

// the (tile, k-block) cursor of a producer's L2 prefetches
struct L2Ahead {
  int64_t t;
  int kb;
  __device__ __forceinline__ void run(const CUtensorMap* m, int64_t ntiles,
                                      int kblocks, int bk, int rows, int sub,
                                      int n) {
    for (int i = 0; i < n && t < ntiles; i++) {
      for (int u = 0; u < sub; u++)
        tma_prefetch_2d(m, kb * bk, (int)((t * sub + u) * rows));
      if (++kb == kblocks) {
        kb = 0;
        t += gridDim.x;
      }
    }
  }
};

// K-major, SWIZZLE_128B UMMA shared-memory descriptor (sm100 version 1):
// start >> 4, LBO = 1 (unused when swizzled), SBO = 1024 B (8 rows x 128 B)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // leading byte offset (16 B units)
  d |= (uint64_t)(1024 >> 4) << 32;  // stride byte offset
  d |= (uint64_t)1 << 46;            // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc,
                                         uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(
          tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 "
      "[%0];" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, "
      "%7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]),
        "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
        "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float relu_np(float v) {
  return (v >= 0.0f || v != v) ? v : 0.0f;
}

template <typename OutT>
__device__ __forceinline__ OutT cvt_out(float v);
template <>
__device__ __forceinline__ float cvt_out<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half cvt_out<__half>(float v) {
  return __float2half_rn(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

__device__ __forceinline__ void store4(float* d, const float (&q)[4]) {
  *reinterpret_cast<float4*>(d) = make_float4(q[0], q[1], q[2], q[3]);
}
template <typename H>
__device__ __forceinline__ void store4(H* d, const H (&q)[4]) {
  uint2 u;
  u.x = (uint32_t)__half_as_ushort(*reinterpret_cast<const __half*>(&q[0])) |
        ((uint32_t)__half_as_ushort(*reinterpret_cast<const __half*>(&q[1])) << 16);
  u.y = (uint32_t)__half_as_ushort(*reinterpret_cast<const __half*>(&q[2])) |
        ((uint32_t)__half_as_ushort(*reinterpret_cast<const __half*>(&q[3])) << 16);
  *reinterpret_cast<uint2*>(d) = u;
}

struct TcParams {
  int64_t M;
  int K, N, BN, stages, kblocks, relu;
  int nacc;  // TMEM accumulators in the ring: 2 (default, 0 = 2) or 1
  int64_t ldy;
  const float* bias;
  void* y;
  uint32_t tmem_cols;
  int32_t* flag;
  int l2ahead;  // x k-blocks prefetched into L2 ahead of the loads
  // GAT pass A: er[h] = sum over head h's columns of z * er_w (written at
  // column er_col + h of each output row; null = off)
  const float* er_w;
  int er_col, er_heads, er_hs;
};

// the er request of the current atlas_transform_er call (host thread)
struct ErSpec {
  const float* w = nullptr;
  int col = 0, heads = 0, hs = 0;
};
static thread_local ErSpec g_er;
constexpr int kErMaxHeads = 8;
// pair exchange of er partials: 2 parities x 4 lane quarters x heads x 32
constexpr int kErBytes = 2 * 4 * kErMaxHeads * 32 * 4;
static void apply_er(TcParams& p) {
  p.er_w = g_er.w;
  p.er_col = g_er.col;
  p.er_heads = g_er.heads;
  p.er_hs = g_er.hs;
}
static int er_smem() { return g_er.w ? kErBytes : 0; }

// ATLAS_TF_L2AHEAD: x k-blocks the producers prefetch into L2 ahead of
// their shared-memory loads (0 = off)
static int l2ahead_knob() {
  static const int v = [] {
    const char* e = std::getenv("ATLAS_TF_L2AHEAD");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

// Epilogue warps (8): thread = accumulator row (TMEM lane) for
// tcgen05.ld; each 32 x 16 block is transposed through a per-warp smem tile
// so that a warp store covers 8 rows x 64 B (4 lanes x 16 B per row).
// sscale (per output column, may be null) multiplies the accumulator
// before the bias (the power-of-two weight scales of the f16 kernel).
template <typename OutT>
__device__ __forceinline__ void epilogue_loop(
    const TcParams& p, int ew, int warp, int lane, int64_t ntiles,
    uint32_t tmem_base, uint64_t* tfull, uint64_t* tempty,
    const float* sbias, const float* sscale, float* stage_out, int sub = 1) {
  const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31
  const int cpar = ew >> 2;      // which 16-col blocks this warp takes
  float* stage = stage_out + ew * 32 * kStageLd;
  int acc = 0;
  uint32_t aph[2] = {0, 0};
  OutT* y = static_cast<OutT*>(p.y);
  const int rsub = lane >> 2, c4 = (lane & 3) * 4;
  const bool vec_ok = (p.ldy % 4) == 0 &&
                      (reinterpret_cast<uintptr_t>(p.y) % (4 * sizeof(OutT))) == 0;
  int bad = 0;
  // er: each thread (= row) folds its 16-column blocks into per-head
  // partials; the two warps sharing a lane quarter hold alternate blocks,
  // so the odd-block warp hands its partials over through shared memory
  // (named barrier per quarter) and the even-block warp stores er
  const bool er_on = p.er_w != nullptr;
  float* erx = stage_out + kEpiWarps * 32 * kStageLd;
  int xpar = 0;
  // a tile is `sub` 128-row halves (sub accumulators of BN columns each)
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(&tfull[acc], aph[acc]);
    aph[acc] ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int u = 0; u < sub; u++) {
    const int64_t row0 = (t * sub + u) * BM + quarter * 32;
    const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) +
                           (uint32_t)((acc * sub + u) * p.BN);
    float erp[kErMaxHeads];
#pragma unroll
    for (int hh = 0; hh < kErMaxHeads; hh++) erp[hh] = 0.0f;
    for (int c0 = cpar * 16; c0 < p.BN; c0 += 32) {
      float v[16];
      tmem_ld16(taddr + c0, v);
      if (er_on) {
        const int hd = c0 / p.er_hs;
        float sacc = 0.0f;
#pragma unroll
        for (int j = 0; j < 16; j++) {
          const float zj = sscale ? v[j] * sscale[c0 + j] : v[j];
          sacc = fmaf(zj, __ldg(p.er_w + c0 + j), sacc);
        }
#pragma unroll
        for (int hh = 0; hh < kErMaxHeads; hh++)
          if (hh == hd) erp[hh] += sacc;
      }
#pragma unroll
      for (int j = 0; j < 16; j += 4)
        *reinterpret_cast<float4*>(&stage[lane * kStageLd + j]) =
            make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      __syncwarp();
      const int c = c0 + c4;
      float bias4[4], scale4[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        bias4[j] = sbias[c + j];
        scale4[j] = sscale ? sscale[c + j] : 1.0f;
      }
#pragma unroll
      for (int rr = 0; rr < 32; rr += 8) {
        const int r = rr + rsub;
        const int64_t row = row0 + r;
        if (row < p.M) {
          const float4 a = *reinterpret_cast<const float4*>(&stage[r * kStageLd + c4]);
          const float av[4] = {a.x, a.y, a.z, a.w};
          OutT q[4];
#pragma unroll
          for (int j = 0; j < 4; j++) {
            float o = __fadd_rn(sscale ? av[j] * scale4[j] : av[j], bias4[j]);
            if (p.relu) o = relu_np(o);
            q[j] = cvt_out<OutT>(o);
            bad |= (c + j < p.N) ? is_extreme(to_f32(q[j])) : 0;
          }
          OutT* dst = y + row * p.ldy + c;
          if (vec_ok && c + 4 <= p.N) {
            store4(dst, q);
          } else {
#pragma unroll
            for (int j = 0; j < 4; j++)
              if (c + j < p.N) dst[j] = q[j];
          }
        }
      }
      __syncwarp();
    }
    if (er_on) {
      float* xb = erx + ((xpar & 1) * 4 + quarter) * kErMaxHeads * 32;
      if (cpar == 1)
        for (int hh = 0; hh < p.er_heads; hh++) xb[hh * 32 + lane] = erp[hh];
      asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
      const int64_t row = row0 + lane;
      if (cpar == 0 && row < p.M) {
        OutT* dst = y + row * p.ldy + p.er_col;
#pragma unroll
        for (int hh = 0; hh < kErMaxHeads; hh++)
          if (hh < p.er_heads) dst[hh] = cvt_out<OutT>(erp[hh] + xb[hh * 32 + lane]);
      }
      xpar++;
    }
    }  // halves
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    mbar_arrive(&tempty[acc]);
    acc = p.nacc == 1 ? 0 : acc ^ 1;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0 && p.flag)
    atomicOr(p.flag, 1);
}

template <typename TIn, typename OutT, bool RES_W>
__global__ void __launch_bounds__(kThreads, 1)
    transform_tc_kernel(const __grid_constant__ CUtensorMap map_x,
                        const __grid_constant__ CUtensorMap map_w,
                        TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B aligned carve-up (pointer arithmetic keeps the shared space):
  //   RES_W : [w_hi kb0..kbN | w_lo kb0..kbN] then per stage [x | x_lo]
  //   !RES_W: per stage [x | x_lo | w | w_lo]
  // f32 input: TMA lands in x and is split in place (x -> tf32 hi, x_lo).
  // f16/bf16 input (exact in tf32): TMA lands, unswizzled, in the x_lo
  // area and the splitter widens it into x in the SW128 f32 layout; the
  // MMA then needs only x.w_lo + x.w_hi.
  constexpr bool kExact = sizeof(TIn) == 2;
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t x_bytes = BM * BK * 4;
  const uint32_t w_bytes = p.BN * BK * 4;
  const uint32_t wres_bytes = RES_W ? 2u * w_bytes * p.kblocks : 0u;
  const uint32_t stage_bytes = 2 * x_bytes + (RES_W ? 0u : 2 * w_bytes);
  uint8_t* stages = base + wres_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + p.stages * stage_bytes);
  uint64_t* split = full + p.stages;
  uint64_t* empty = split + p.stages;
  uint64_t* tfull = empty + p.stages;  // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint64_t* wfull = tempty + 2;        // resident W landed
  uint64_t* wsplit = wfull + 1;        // resident W split
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wsplit + 1);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);
  float* stage_out = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(sbias + 256) + 15) & ~uintptr_t(15));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (p.M + BM - 1) / BM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], 128);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; a++) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * 32);
    }
    mbar_init(wfull, 1);
    mbar_init(wsplit, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = threadIdx.x; j < p.BN; j += kThreads)
    sbias[j] = j < p.N ? p.bias[j] : 0.0f;
  if (warp == 1) {
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::
            "r"(smem_u32(tmem_slot)),
        "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  // W tiles of k-block kb: resident area, or inside stage s
  auto w_hi_ptr = [&](int s, int kb) -> uint8_t* {
    return RES_W ? base + kb * w_bytes
                 : stages + s * stage_bytes + 2 * x_bytes;
  };
  auto w_lo_ptr = [&](int s, int kb) -> uint8_t* {
    return RES_W ? base + (p.kblocks + kb) * w_bytes
                 : stages + s * stage_bytes + 2 * x_bytes + w_bytes;
  };

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      if (RES_W) {  // W once per CTA
        mbar_expect_tx(wfull, w_bytes * p.kblocks);
        for (int kb = 0; kb < p.kblocks; kb++)
          tma_load_2d(base + kb * w_bytes, &map_w, wfull, kb * BK, 0);
      }
      int s = 0;
      uint32_t ph = 0;
      L2Ahead pf{(int64_t)blockIdx.x, 0};
      pf.run(&map_x, ntiles, p.kblocks, BK, BM, 1, p.l2ahead);
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kb = 0; kb < p.kblocks; kb++) {
          pf.run(&map_x, ntiles, p.kblocks, BK, BM, 1, p.l2ahead > 0 ? 1 : 0);
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = stages + s * stage_bytes;
          mbar_expect_tx(&full[s], BM * BK * (uint32_t)sizeof(TIn) +
                                       (RES_W ? 0u : w_bytes));
          tma_load_2d(kExact ? st + x_bytes : st, &map_x, &full[s], kb * BK,
                      (int)(t * BM));
          if (!RES_W)
            tma_load_2d(st + 2 * x_bytes, &map_w, &full[s], kb * BK, 0);
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = (1u << 4)                       // D = f32
                           | (2u << 7) | (2u << 10)        // A, B = tf32
                           | ((uint32_t)(p.BN >> 3) << 17)  // N
                           | ((uint32_t)(BM >> 4) << 24);   // M
    if (RES_W) mbar_wait(wsplit, 0);
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t aph[2] = {0, 0};
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], aph[acc] ^ 1);
      aph[acc] ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dt = tmem_base + (uint32_t)(acc * p.BN);
      for (int kb = 0; kb < p.kblocks; kb++) {
        mbar_wait(&split[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          uint8_t* st = stages + s * stage_bytes;
          const uint32_t a_hi = smem_u32(st), a_lo = smem_u32(st + x_bytes);
          const uint32_t b_hi = smem_u32(w_hi_ptr(s, kb));
          const uint32_t b_lo = smem_u32(w_lo_ptr(s, kb));
#pragma unroll
          for (int k = 0; k < BK / 8; k++) {  // UMMA_K = 8 tf32 = 32 B
            const uint32_t off = k * 32;
            const uint32_t first = (kb == 0 && k == 0) ? 0u : 1u;
            if (!kExact)
              mma_tf32(dt, sw128_desc(a_lo + off), sw128_desc(b_hi + off),
                       idesc, first);
            mma_tf32(dt, sw128_desc(a_hi + off), sw128_desc(b_lo + off),
                     idesc, kExact ? first : 1u);
            mma_tf32(dt, sw128_desc(a_hi + off), sw128_desc(b_hi + off),
                     idesc, 1u);
          }
          mma_commit(&empty[s]);
          if (kb == p.kblocks - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
      }
      acc ^= 1;
    }
  } else if (warp < 6) {
    // -------- splitter: tiles -> tf32 hi (in place) + lo ----------------
    const int tid = threadIdx.x - 64;  // 0..127
    auto split16 = [](float4* hi, float4* lo, int e) {
      const float4 v = hi[e];
      float4 h, l;
      h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
      h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
      h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
      h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
      l.x = v.x - h.x;
      l.y = v.y - h.y;
      l.z = v.z - h.z;
      l.w = v.w - h.w;
      hi[e] = h;
      lo[e] = l;
    };
    if (RES_W) {
      mbar_wait(wfull, 0);
      for (int kb = 0; kb < p.kblocks; kb++) {
        float4* wh = reinterpret_cast<float4*>(w_hi_ptr(0, kb));
        float4* wl = reinterpret_cast<float4*>(w_lo_ptr(0, kb));
        for (int e = tid; e < p.BN * BK / 4; e += 128) split16(wh, wl, e);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(wsplit);
    }
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kb = 0; kb < p.kblocks; kb++) {
        mbar_wait(&full[s], ph);
        uint8_t* st = stages + s * stage_bytes;
        float4* xs = reinterpret_cast<float4*>(st);
        float4* xl = reinterpret_cast<float4*>(st + x_bytes);
        if constexpr (kExact) {
          // raw [128 rows][32] 2-byte elements -> f32 row r, 16-B chunk c
          // at the SW128 position (c ^ (r & 7)) of the 128-B row
          const uint2* raw = reinterpret_cast<const uint2*>(st + x_bytes);
#pragma unroll
          for (int i = 0; i < (BM * BK / 4) / 128; i++) {
            const int g = tid + i * 128, r = g >> 3, c = g & 7;
            const uint2 h = raw[g];
            const TIn* e = reinterpret_cast<const TIn*>(&h);
            xs[r * 8 + (c ^ (r & 7))] =
                make_float4(to_f32(e[0]), to_f32(e[1]), to_f32(e[2]),
                            to_f32(e[3]));
          }
        } else {
#pragma unroll
          for (int i = 0; i < (BM * BK / 4) / 128; i++)
            split16(xs, xl, tid + i * 128);
        }
        if (!RES_W) {
          float4* ws = reinterpret_cast<float4*>(w_hi_ptr(s, kb));
          float4* wl = reinterpret_cast<float4*>(w_lo_ptr(s, kb));
          for (int e = tid; e < p.BN * BK / 4; e += 128) split16(ws, wl, e);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&split[s]);
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue ----------------
    epilogue_loop<OutT>(p, warp - 6, warp, lane, ntiles, tmem_base, tfull,
                        tempty, sbias, nullptr, stage_out);
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile(
        "tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(
            tmem_base),
        "r"(p.tmem_cols));
  }
}

// ---------------------------------------------------------------------------
// f16 inputs on kind::f16 (K = 16 per MMA, twice tf32's rate, no splitter):
// x is consumed as loaded by TMA; W is pre-split per output row n into
// f16 hi + lo of W[n,:] * 2^k_n (k_n puts the row maximum in [2^14, 2^15),
// so lo never loses bits to f16's range), both products accumulate in f32
// in TMEM and the epilogue multiplies by 2^-k_n (exact). W is carried to
// ~2^-22 relative, x exactly: the same accuracy class as 3xTF32.

constexpr int BKH = 64;                 // 64 f16 = 128 B = one swizzle row
constexpr int kThreadsH = (2 + kEpiWarps) * 32;

__global__ void split_w_f16(const float* __restrict__ w, int64_t k,
                            __half* __restrict__ hi, __half* __restrict__ lo,
                            float* __restrict__ scale) {
  const int64_t n = blockIdx.x;
  const float* row = w + n * k;
  float m = 0.0f;
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x)
    m = fmaxf(m, fabsf(row[i]));
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
#pragma unroll
    for (int o = 16; o; o >>= 1)
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  m = red[0];
  const int e = (m > 0.0f && m <= 3.402823466e38f) ? 14 - ilogbf(m) : 0;
  const float up = ldexpf(1.0f, e);
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {
    const float v = row[i] * up;  // exact: power-of-two scale
    const __half h = __float2half_rn(v);
    hi[n * k + i] = h;
    lo[n * k + i] = __float2half_rn(v - __half2float(h));
  }
  if (threadIdx.x == 0) scale[n] = ldexpf(1.0f, -e);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc,
                                        uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(
          tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// SUB = 2: 256-row tiles, two M=128 MMAs per k-step sharing one W stage,
// so each W byte fetched from L2 serves twice the rows (BN <= 128: two
// double-buffered accumulator pairs fill the 512 TMEM columns)
template <typename OutT, int SUB>
__global__ void __launch_bounds__(kThreadsH, 1)
    transform_h_kernel(const __grid_constant__ CUtensorMap map_x,
                       const __grid_constant__ CUtensorMap map_whi,
                       const __grid_constant__ CUtensorMap map_wlo,
                       TcParams p, const float* __restrict__ wscale) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t x_bytes = BM * BKH * 2;  // one 128-row half
  const uint32_t w_bytes = p.BN * BKH * 2;
  const uint32_t stage_bytes = SUB * x_bytes + 2 * w_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + p.stages * stage_bytes);
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;  // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);
  float* sscale = sbias + 256;
  float* stage_out = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(sscale + 256) + 15) & ~uintptr_t(15));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (p.M + BM * SUB - 1) / (BM * SUB);
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; a++) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = threadIdx.x; j < p.BN; j += kThreadsH) {
    sbias[j] = j < p.N ? p.bias[j] : 0.0f;
    sscale[j] = j < p.N ? wscale[j] : 0.0f;
  }
  if (warp == 1) {
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::
            "r"(smem_u32(tmem_slot)),
        "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      L2Ahead pf{(int64_t)blockIdx.x, 0};
      pf.run(&map_x, ntiles, p.kblocks, BKH, BM, SUB, p.l2ahead);
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kb = 0; kb < p.kblocks; kb++) {
          pf.run(&map_x, ntiles, p.kblocks, BKH, BM, SUB, p.l2ahead > 0 ? 1 : 0);
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = base + s * stage_bytes;
          mbar_expect_tx(&full[s], stage_bytes);
          for (int u = 0; u < SUB; u++)
            tma_load_2d(st + u * x_bytes, &map_x, &full[s], kb * BKH,
                        (int)((t * SUB + u) * BM));
          tma_load_2d(st + SUB * x_bytes, &map_whi, &full[s], kb * BKH, 0);
          tma_load_2d(st + SUB * x_bytes + w_bytes, &map_wlo, &full[s],
                      kb * BKH, 0);
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = (1u << 4)                       // D = f32
                           | (0u << 7) | (0u << 10)        // A, B = f16
                           | ((uint32_t)(p.BN >> 3) << 17)  // N
                           | ((uint32_t)(BM >> 4) << 24);   // M
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t aph[2] = {0, 0};
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], aph[acc] ^ 1);
      aph[acc] ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dt = tmem_base + (uint32_t)(acc * SUB * p.BN);
      for (int kb = 0; kb < p.kblocks; kb++) {
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          uint8_t* st = base + s * stage_bytes;
          const uint32_t bh = smem_u32(st + SUB * x_bytes);
          const uint32_t bl = smem_u32(st + SUB * x_bytes + w_bytes);
#pragma unroll
          for (int k = 0; k < BKH / 16; k++) {  // UMMA_K = 16 f16 = 32 B
            const uint32_t off = k * 32;
            const uint32_t first = (kb == 0 && k == 0) ? 0u : 1u;
#pragma unroll
            for (int u = 0; u < SUB; u++) {
              const uint32_t a = smem_u32(st + u * x_bytes);
              const uint32_t d = dt + (uint32_t)(u * p.BN);
              mma_f16(d, sw128_desc(a + off), sw128_desc(bl + off), idesc,
                      first);
              mma_f16(d, sw128_desc(a + off), sw128_desc(bh + off), idesc,
                      1u);
            }
          }
          mma_commit(&empty[s]);
          if (kb == p.kblocks - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
      }
      acc = p.nacc == 1 ? 0 : acc ^ 1;
    }
  } else {
    epilogue_loop<OutT>(p, warp - 2, warp, lane, ntiles, tmem_base, tfull,
                        tempty, sbias, sscale, stage_out, SUB);
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile(
        "tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(
            tmem_base),
        "r"(p.tmem_cols));
  }
}

// ---------------------------------------------------------------------------
// f32 x with K <= 128 and N <= 128: the transposed product on a TMEM-resident
// W. D^T (N x rows) = W (N x K, A operand from TMEM) . x^T (B operand: the
// x tile is rows x K, K-major, exactly the N x K K-major B layout). W hi/lo
// live in TMEM columns [0, 2Kp), so shared memory holds nothing but x
// stages (6 x 32 KB in flight instead of 2 next to a resident W in smem),
// and the epilogue needs no transpose: TMEM lane = output column, so each
// tcgen05.ld register is one row and a warp's store covers 32 consecutive
// columns of that row (one 128-B line for f32).
//   warp 0      TMA producer (x tiles, 128 rows x 32 f32, SWIZZLE_128B)
//   warp 1      TMEM allocator + MMA issuer
//   warps 2-5   splitter: x -> tf32 hi (in place) + lo
//   warps 6-13  W -> TMEM (hi/lo split, tcgen05.st) once, then epilogue:
//               warp 6+q / 10+q own TMEM lane quarter (warp & 3) and
//               alternate 64-row halves of the tile
constexpr int BR = 128;  // rows per tile = MMA N

__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a,
                                            uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(
          tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, "
      "%7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
      "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]),
      "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

struct TtParams {
  int64_t M;
  int K, Kp, N, stages, kblocks, relu;
  int64_t ldy;
  const float* w;     // N x K row-major
  const float* bias;
  void* y;
  int32_t* flag;
  int l2ahead;
};

template <typename OutT>
__global__ void __launch_bounds__(kThreads, 1)
    transform_t_kernel(const __grid_constant__ CUtensorMap map_x,
                       TtParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr uint32_t x_bytes = BR * BK * 4;
  constexpr uint32_t stage_bytes = 2 * x_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + p.stages * stage_bytes);
  uint64_t* split = full + p.stages;
  uint64_t* empty = split + p.stages;
  uint64_t* tfull = empty + p.stages;  // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint64_t* wready = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wready + 1);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (p.M + BR - 1) / BR;
  const uint32_t d_col0 = 2u * (uint32_t)p.Kp;  // D buffers after W hi/lo

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], 128);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; a++) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * 32);
    }
    mbar_init(wready, 4 * 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = threadIdx.x; j < 128; j += kThreads)
    sbias[j] = j < p.N ? p.bias[j] : 0.0f;
  if (warp == 1) {
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::
            "r"(smem_u32(tmem_slot)),
        "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      L2Ahead pf{(int64_t)blockIdx.x, 0};
      pf.run(&map_x, ntiles, p.kblocks, BK, BR, 1, p.l2ahead);
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kb = 0; kb < p.kblocks; kb++) {
          pf.run(&map_x, ntiles, p.kblocks, BK, BR, 1, p.l2ahead > 0 ? 1 : 0);
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], x_bytes);
          tma_load_2d(base + s * stage_bytes, &map_x, &full[s], kb * BK,
                      (int)(t * BR));
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // M = 128 (output columns, W rows zero-padded), N = 128 rows
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                           ((uint32_t)(BR >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);
    mbar_wait(wready, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t aph[2] = {0, 0};
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], aph[acc] ^ 1);
      aph[acc] ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dt = tmem_base + d_col0 + (uint32_t)(acc * BR);
      for (int kb = 0; kb < p.kblocks; kb++) {
        mbar_wait(&split[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          uint8_t* st = base + s * stage_bytes;
          const uint32_t b_hi = smem_u32(st), b_lo = smem_u32(st + x_bytes);
#pragma unroll
          for (int k = 0; k < BK / 8; k++) {  // UMMA_K = 8 tf32
            const uint32_t col = (uint32_t)(kb * BK + k * 8);
            const uint32_t a_hi = tmem_base + col;
            const uint32_t a_lo = tmem_base + (uint32_t)p.Kp + col;
            const uint32_t off = k * 32;
            const uint32_t first = (kb == 0 && k == 0) ? 0u : 1u;
            mma_tf32_ts(dt, a_lo, sw128_desc(b_hi + off), idesc, first);
            mma_tf32_ts(dt, a_hi, sw128_desc(b_lo + off), idesc, 1u);
            mma_tf32_ts(dt, a_hi, sw128_desc(b_hi + off), idesc, 1u);
          }
          mma_commit(&empty[s]);
          if (kb == p.kblocks - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
      }
      acc ^= 1;
    }
  } else if (warp < 6) {
    const int tid = threadIdx.x - 64;  // 0..127
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kb = 0; kb < p.kblocks; kb++) {
        mbar_wait(&full[s], ph);
        uint8_t* st = base + s * stage_bytes;
        float4* xs = reinterpret_cast<float4*>(st);
        float4* xl = reinterpret_cast<float4*>(st + x_bytes);
#pragma unroll
        for (int i = 0; i < (BR * BK / 4) / 128; i++) {
          const int e = tid + i * 128;
          const float4 v = xs[e];
          float4 h, l;
          h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          l.x = v.x - h.x;
          l.y = v.y - h.y;
          l.z = v.z - h.z;
          l.w = v.w - h.w;
          xs[e] = h;
          xl[e] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&split[s]);
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else {
    const int ew = warp - 6;
    const int quarter = warp & 3;
    const int n = quarter * 32 + lane;  // TMEM lane = output column
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    if (ew < 4) {  // W -> TMEM: row n, hi at [0, Kp), lo at [Kp, 2Kp)
      for (int c0 = 0; c0 < p.Kp; c0 += 16) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int j = 0; j < 16; j++) {
          const int c = c0 + j;
          const float v = (n < p.N && c < p.K) ? p.w[(int64_t)n * p.K + c] : 0.0f;
          const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
          hi[j] = __float_as_uint(h);
          lo[j] = __float_as_uint(v - h);
        }
        tmem_st16(tmem_base + lane_off + (uint32_t)c0, hi);
        tmem_st16(tmem_base + lane_off + (uint32_t)(p.Kp + c0), lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(wready);
    }
    const int half = ew >> 2;  // rows [64*half, 64*half + 64) of each tile
    const float bias = sbias[n];
    OutT* y = static_cast<OutT*>(p.y);
    int acc = 0;
    uint32_t aph[2] = {0, 0};
    int bad = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(&tfull[acc], aph[acc]);
      aph[acc] ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t taddr = tmem_base + lane_off + d_col0 + (uint32_t)(acc * BR);
      const int64_t row0 = t * BR;
      for (int c0 = half * 64; c0 < half * 64 + 64; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + c0, v);
        if (n < p.N) {
#pragma unroll
          for (int j = 0; j < 16; j++) {
            const int64_t row = row0 + c0 + j;
            if (row < p.M) {
              float o = __fadd_rn(v[j], bias);
              if (p.relu) o = relu_np(o);
              const OutT q = cvt_out<OutT>(o);
              bad |= is_extreme(to_f32(q));
              y[row * p.ldy + n] = q;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&tempty[acc]);
      acc ^= 1;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0 && p.flag)
      atomicOr(p.flag, 1);
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile(
        "tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(
            tmem_base),
        "r"(512));
  }
}

// ---------------------------------------------------------------------------
// f32 x, register split (the default f32 kernel when W fits resident): the
// splitter warps read each x row chunk once from the TMA stage, release the
// stage at once, and write hi / lo straight into TMEM, where they are the
// MMA's A operand. Shared memory then holds only W (hi + lo, resident) and
// 16-KB x landing stages that turn over as soon as they are split, so more
// x bytes are in flight per SM than when x_hi / x_lo occupy the stages
// until their MMAs retire (transform_tc_kernel, whose in-flight bytes cap
// it at ~0.6 of HBM). TMEM: D double buffer [0, 2 BN), then kAStages A
// stages of 64 columns (hi 32 | lo 32) from column 256.
//   warp 0      TMA producer (x tiles; W once)
//   warp 1      TMEM allocator + MMA issuer
//   warps 2-5   W split (once), then x split: warp w owns TMEM lane quarter
//               w & 3, thread = tile row
//   warps 6-13  epilogue (shared with transform_tc_kernel)
constexpr int kAStages = 4;
constexpr uint32_t kACol0 = 256;

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, "
      "%7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, "
      "%21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]),
      "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]),
      "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]),
      "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]),
      "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]),
      "f"(v[30]), "f"(v[31])
      : "memory");
}

template <typename OutT>
__global__ void __launch_bounds__(kThreads, 1)
    transform_r_kernel(const __grid_constant__ CUtensorMap map_x,
                       const __grid_constant__ CUtensorMap map_w,
                       TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t x_bytes = BM * BK * 4;
  const uint32_t w_bytes = p.BN * BK * 4;
  const uint32_t wres_bytes = 2u * w_bytes * p.kblocks;
  uint8_t* stages = base + wres_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + p.stages * x_bytes);
  uint64_t* sempty = full + p.stages;
  uint64_t* afull = sempty + p.stages;   // [kAStages]
  uint64_t* aempty = afull + kAStages;   // [kAStages]
  uint64_t* tfull = aempty + kAStages;   // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint64_t* wfull = tempty + 2;
  uint64_t* wsplit = wfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wsplit + 1);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);
  float* stage_out = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(sbias + 256) + 15) & ~uintptr_t(15));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (p.M + BM - 1) / BM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&sempty[s], 128);
    }
    for (int a = 0; a < kAStages; a++) {
      mbar_init(&afull[a], 128);
      mbar_init(&aempty[a], 1);
    }
    for (int a = 0; a < 2; a++) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * 32);
    }
    mbar_init(wfull, 1);
    mbar_init(wsplit, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = threadIdx.x; j < p.BN; j += kThreads)
    sbias[j] = j < p.N ? p.bias[j] : 0.0f;
  if (warp == 1) {
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::
            "r"(smem_u32(tmem_slot)),
        "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  auto w_hi_ptr = [&](int kb) -> uint8_t* { return base + kb * w_bytes; };
  auto w_lo_ptr = [&](int kb) -> uint8_t* {
    return base + (p.kblocks + kb) * w_bytes;
  };

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(wfull, w_bytes * p.kblocks);
      for (int kb = 0; kb < p.kblocks; kb++)
        tma_load_2d(w_hi_ptr(kb), &map_w, wfull, kb * BK, 0);
      int s = 0;
      uint32_t ph = 0;
      L2Ahead pf{(int64_t)blockIdx.x, 0};
      pf.run(&map_x, ntiles, p.kblocks, BK, BM, 1, p.l2ahead);
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kb = 0; kb < p.kblocks; kb++) {
          pf.run(&map_x, ntiles, p.kblocks, BK, BM, 1, p.l2ahead > 0 ? 1 : 0);
          mbar_wait(&sempty[s], ph ^ 1);
          mbar_expect_tx(&full[s], x_bytes);
          tma_load_2d(stages + s * x_bytes, &map_x, &full[s], kb * BK,
                      (int)(t * BM));
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                           ((uint32_t)(p.BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
    mbar_wait(wsplit, 0);
    int a = 0;
    uint32_t aph = 0;
    int acc = 0;
    uint32_t tph[2] = {0, 0};
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], tph[acc] ^ 1);
      tph[acc] ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dt = tmem_base + (uint32_t)(acc * p.BN);
      for (int kb = 0; kb < p.kblocks; kb++) {
        mbar_wait(&afull[a], aph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint32_t ahi = tmem_base + kACol0 + (uint32_t)(a * 64);
          const uint32_t b_hi = smem_u32(w_hi_ptr(kb));
          const uint32_t b_lo = smem_u32(w_lo_ptr(kb));
#pragma unroll
          for (int k = 0; k < BK / 8; k++) {
            const uint32_t off = k * 32;
            const uint32_t first = (kb == 0 && k == 0) ? 0u : 1u;
            mma_tf32_ts(dt, ahi + 32 + k * 8, sw128_desc(b_hi + off), idesc,
                        first);
            mma_tf32_ts(dt, ahi + k * 8, sw128_desc(b_lo + off), idesc, 1u);
            mma_tf32_ts(dt, ahi + k * 8, sw128_desc(b_hi + off), idesc, 1u);
          }
          mma_commit(&aempty[a]);
          if (kb == p.kblocks - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++a == kAStages) {
          a = 0;
          aph ^= 1;
        }
      }
      acc ^= 1;
    }
  } else if (warp < 6) {
    const int tid = threadIdx.x - 64;  // 0..127
    {  // W -> tf32 hi (in place) + lo, once
      mbar_wait(wfull, 0);
      for (int kb = 0; kb < p.kblocks; kb++) {
        float4* wh = reinterpret_cast<float4*>(w_hi_ptr(kb));
        float4* wl = reinterpret_cast<float4*>(w_lo_ptr(kb));
        for (int e = tid; e < p.BN * BK / 4; e += 128) {
          const float4 v = wh[e];
          float4 h, l;
          h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          l.x = v.x - h.x;
          l.y = v.y - h.y;
          l.z = v.z - h.z;
          l.w = v.w - h.w;
          wh[e] = h;
          wl[e] = l;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(wsplit);
    }
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // tile row = TMEM lane
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    int s = 0, a = 0;
    uint32_t ph = 0, aph = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kb = 0; kb < p.kblocks; kb++) {
        mbar_wait(&full[s], ph);
        // row r's 128-B chunk: 16-B unit c sits at SW128 slot c ^ (r & 7)
        const float4* xs =
            reinterpret_cast<const float4*>(stages + s * x_bytes) + r * 8;
        float hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; c++) {
          const float4 v = xs[c ^ (r & 7)];
          const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float h = __uint_as_float(__float_as_uint(e[q]) & 0xFFFFE000u);
            hi[c * 4 + q] = h;
            lo[c * 4 + q] = e[q] - h;
          }
        }
        // the stage is free once read (the TMA refilling it is an
        // async-proxy write after these generic-proxy reads)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&sempty[s]);
        mbar_wait(&aempty[a], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ta = tmem_base + lane_off + kACol0 + (uint32_t)(a * 64);
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(&afull[a]);
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
        if (++a == kAStages) {
          a = 0;
          aph ^= 1;
        }
      }
    }
  } else {
    epilogue_loop<OutT>(p, warp - 6, warp, lane, ntiles, tmem_base, tfull,
                        tempty, sbias, nullptr, stage_out);
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile(
        "tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(
            tmem_base),
        "r"(512));
  }
}

// ---------------------------------------------------------------------------
// f32 x, register split, W too large to stay resident (K x BN x 8 B > ~190
// KB, e.g. SAGE's K = 256 aggregate at BN = 128): W is pre-split once into
// tf32 hi / lo arrays in global memory and streamed through its own ring
// of (hi, lo) k-block stages next to the x landing ring; x is split into
// TMEM A stages exactly as in transform_r_kernel. Ring stages are released
// by the splitter (x) and by the MMA's commit (W).
__global__ void split_w_tf32(const float* __restrict__ w, int64_t n,
                             float* __restrict__ hi, float* __restrict__ lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = w[i];
    const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    hi[i] = h;
    lo[i] = v - h;
  }
}

template <typename OutT>
__global__ void __launch_bounds__(kThreads, 1)
    transform_rs_kernel(const __grid_constant__ CUtensorMap map_x,
                        const __grid_constant__ CUtensorMap map_whi,
                        const __grid_constant__ CUtensorMap map_wlo,
                        TcParams p, int wst) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t x_bytes = BM * BK * 4;
  const uint32_t w_bytes = p.BN * BK * 4;
  uint8_t* xring = base;
  uint8_t* wring = base + p.stages * x_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(wring + wst * 2 * w_bytes);
  uint64_t* sempty = full + p.stages;
  uint64_t* wfull = sempty + p.stages;   // [wst]
  uint64_t* wempty = wfull + wst;        // [wst]
  uint64_t* afull = wempty + wst;        // [kAStages]
  uint64_t* aempty = afull + kAStages;   // [kAStages]
  uint64_t* tfull = aempty + kAStages;   // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);
  float* stage_out = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(sbias + 256) + 15) & ~uintptr_t(15));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (p.M + BM - 1) / BM;
  // TMEM: the two accumulators take [0, 2 BN); A stages of 64 columns
  // follow (4 when BN <= 128, 2 for 128 < BN <= 192)
  const uint32_t acol0 = p.BN <= 128 ? kACol0 : (uint32_t)((2 * p.BN + 63) / 64 * 64);
  const int na = min(kAStages, (int)((512 - acol0) / 64));
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&sempty[s], 128);
    }
    for (int s = 0; s < wst; s++) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);
    }
    for (int a = 0; a < na; a++) {
      mbar_init(&afull[a], 128);
      mbar_init(&aempty[a], 1);
    }
    for (int a = 0; a < 2; a++) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = threadIdx.x; j < p.BN; j += kThreads)
    sbias[j] = j < p.N ? p.bias[j] : 0.0f;
  if (warp == 1) {
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::
            "r"(smem_u32(tmem_slot)),
        "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int xs = 0, ws = 0;
      uint32_t xph = 0, wph = 0;
      L2Ahead pf{(int64_t)blockIdx.x, 0};
      pf.run(&map_x, ntiles, p.kblocks, BK, BM, 1, p.l2ahead);
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kb = 0; kb < p.kblocks; kb++) {
          pf.run(&map_x, ntiles, p.kblocks, BK, BM, 1, p.l2ahead > 0 ? 1 : 0);
          mbar_wait(&sempty[xs], xph ^ 1);
          mbar_expect_tx(&full[xs], x_bytes);
          tma_load_2d(xring + xs * x_bytes, &map_x, &full[xs], kb * BK,
                      (int)(t * BM));
          mbar_wait(&wempty[ws], wph ^ 1);
          mbar_expect_tx(&wfull[ws], 2 * w_bytes);
          uint8_t* wst_ptr = wring + ws * 2 * w_bytes;
          tma_load_2d(wst_ptr, &map_whi, &wfull[ws], kb * BK, 0);
          tma_load_2d(wst_ptr + w_bytes, &map_wlo, &wfull[ws], kb * BK, 0);
          if (++xs == p.stages) {
            xs = 0;
            xph ^= 1;
          }
          if (++ws == wst) {
            ws = 0;
            wph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                           ((uint32_t)(p.BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
    int a = 0, ws = 0;
    uint32_t aph = 0, wph = 0;
    int acc = 0;
    uint32_t tph[2] = {0, 0};
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], tph[acc] ^ 1);
      tph[acc] ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dt = tmem_base + (uint32_t)(acc * p.BN);
      for (int kb = 0; kb < p.kblocks; kb++) {
        mbar_wait(&afull[a], aph);
        mbar_wait(&wfull[ws], wph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint32_t ahi = tmem_base + acol0 + (uint32_t)(a * 64);
          const uint32_t b_hi = smem_u32(wring + ws * 2 * w_bytes);
          const uint32_t b_lo = b_hi + w_bytes;
#pragma unroll
          for (int k = 0; k < BK / 8; k++) {
            const uint32_t off = k * 32;
            const uint32_t first = (kb == 0 && k == 0) ? 0u : 1u;
            mma_tf32_ts(dt, ahi + 32 + k * 8, sw128_desc(b_hi + off), idesc,
                        first);
            mma_tf32_ts(dt, ahi + k * 8, sw128_desc(b_lo + off), idesc, 1u);
            mma_tf32_ts(dt, ahi + k * 8, sw128_desc(b_hi + off), idesc, 1u);
          }
          mma_commit(&aempty[a]);
          mma_commit(&wempty[ws]);
          if (kb == p.kblocks - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++a == na) {
          a = 0;
          aph ^= 1;
        }
        if (++ws == wst) {
          ws = 0;
          wph ^= 1;
        }
      }
      acc ^= 1;
    }
  } else if (warp < 6) {
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // tile row = TMEM lane
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    int s = 0, a = 0;
    uint32_t ph = 0, aph = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kb = 0; kb < p.kblocks; kb++) {
        mbar_wait(&full[s], ph);
        const float4* xs =
            reinterpret_cast<const float4*>(xring + s * x_bytes) + r * 8;
        float hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; c++) {
          const float4 v = xs[c ^ (r & 7)];
          const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float h = __uint_as_float(__float_as_uint(e[q]) & 0xFFFFE000u);
            hi[c * 4 + q] = h;
            lo[c * 4 + q] = e[q] - h;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&sempty[s]);
        mbar_wait(&aempty[a], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ta = tmem_base + lane_off + acol0 + (uint32_t)(a * 64);
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(&afull[a]);
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
        if (++a == na) {
          a = 0;
          aph ^= 1;
        }
      }
    }
  } else {
    epilogue_loop<OutT>(p, warp - 6, warp, lane, ntiles, tmem_base, tfull,
                        tempty, sbias, nullptr, stage_out);
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile(
        "tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(
            tmem_base),
        "r"(512));
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t,
                              void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p,
                                cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2-D f32 map: inner dim `cols` (K), outer `rows`, row pitch `ld` elements,
// box = 32 x box_rows, 128-B swizzle, zero fill out of bounds
// 2-byte inputs use an unswizzled box (64-B rows), widened by the splitter
bool make_map(CUtensorMap* m, const void* ptr, int dtype, int64_t rows,
              int64_t cols, int64_t ld, int box_rows) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  const int es = dtype == ATLAS_F32 ? 4 : 2;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType t = dtype == ATLAS_F32
                                    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                : dtype == ATLAS_F16
                                    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                    : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  return enc(m, t, 2, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             es == 4 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

struct SplitScratch {
  int device;
  cudaStream_t stream;
  DevBuf<uint8_t> buf;
};

SplitScratch& split_scratch(cudaStream_t s) {
  static std::mutex mu;
  static std::vector<std::unique_ptr<SplitScratch>> all;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : all)
    if (e->device == dev && e->stream == s) return *e;
  all.emplace_back(new SplitScratch{dev, s, {}});
  return *all.back();
}

// 2-D f16 map, box = 64 x box_rows (128-B rows), 128-B swizzle
bool make_map_h(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols,
                int64_t ld, int box_rows) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BKH, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr),
             dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// f16 x on kind::f16; false if the shape does not fit (caller falls back)
bool launch_transform_h(const void* x, int64_t rows, int64_t k, int64_t ldx,
                        const float* w, const float* b, int64_t n, int relu,
                        void* y, int y_dtype, int64_t ldy, int32_t* flag,
                        cudaStream_t s) {
  if (n < 1 || n > 256 || k < 8 || k % 8 != 0 || ldx % 8 != 0 ||
      (reinterpret_cast<uintptr_t>(x) & 15) != 0)
    return false;
  const int BN = (int)((n + 15) / 16 * 16);
  const int kblocks = (int)((k + BKH - 1) / BKH);
  // 256-row tiles (two halves per W stage) unless ATLAS_TRANSFORM_H_SUB=1
  const char* sub_env = getenv("ATLAS_TRANSFORM_H_SUB");
  // BN <= 128: two accumulator pairs (the epilogue of tile t overlaps the
  // MMAs of t+1). Above, one pair would have to do (4 x BN TMEM columns do
  // not fit): measured slower than 128-row tiles at N = 136 (0.52 vs 0.56
  // of HBM, profiles/r2_transform_probe_v3.txt), so those keep sub = 1;
  // ATLAS_TRANSFORM_H_SUB=2 forces the single-pair variant
  const bool force2 = sub_env && sub_env[0] == '2';
  const int sub = ((BN <= 128 || (force2 && BN <= 256)) &&
                   !(sub_env && sub_env[0] == '1')) ? 2 : 1;
  const int nacc = (sub == 2 && BN > 128) ? 1 : 2;
  const int stage_bytes = sub * BM * BKH * 2 + 2 * BN * BKH * 2;
  const int fixed = 1024 + 8 * 16 + 16 + 2 * 4 * 256 + 16 +
                    kEpiWarps * 32 * kStageLd * 4;
  int stages = (227 * 1024 - fixed - er_smem()) / stage_bytes;
  if (stages > 6) stages = 6;
  if (stages < 2) return false;
  // pre-split W into the (device, stream)'s grow-only scratch: work on one
  // stream is ordered, so reusing it across calls is safe without syncs
  SplitScratch& ws = split_scratch(s);
  ws.buf.reserve((size_t)(2 * n * k * sizeof(__half) + n * sizeof(float) + 64));
  __half* whi = reinterpret_cast<__half*>(ws.buf.ptr);
  __half* wlo = whi + n * k;
  float* wsc = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(wlo + n * k) + 15) & ~uintptr_t(15));
  split_w_f16<<<(unsigned)n, 256, 0, s>>>(w, k, whi, wlo, wsc);
  count_launch();
  ATLAS_LAUNCH_CHECK();
  CUtensorMap mx, mhi, mlo;
  bool ok = make_map_h(&mx, x, rows, k, ldx, BM) &&
            make_map_h(&mhi, whi, n, k, k, BN) &&
            make_map_h(&mlo, wlo, n, k, k, BN);
  if (ok) {
    const int smem = fixed + stages * stage_bytes + er_smem();
    TcParams p{};
    apply_er(p);
    p.l2ahead = l2ahead_knob();
    p.M = rows;
    p.K = (int)k;
    p.N = (int)n;
    p.BN = BN;
    p.stages = stages;
    p.kblocks = kblocks;
    p.relu = relu;
    p.ldy = ldy;
    p.bias = b;
    p.y = y;
    p.flag = flag;
    p.nacc = nacc;
    uint32_t cols = 32;
    while (cols < (uint32_t)(nacc * sub * BN)) cols <<= 1;
    p.tmem_cols = cols;
    const int64_t ntiles = (rows + BM * sub - 1) / (BM * sub);
    const unsigned grid = (unsigned)std::min<int64_t>(ntiles, num_sms());
    auto launch = [&](auto kern) {
      ATLAS_CUDA(cudaFuncSetAttribute(
          kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kern<<<grid, kThreadsH, smem, s>>>(mx, mhi, mlo, p, wsc);
    };
    auto by_out = [&](auto sub_tag) {
      constexpr int S = decltype(sub_tag)::value;
      if (y_dtype == ATLAS_F32) launch(transform_h_kernel<float, S>);
      else if (y_dtype == ATLAS_F16) launch(transform_h_kernel<__half, S>);
      else launch(transform_h_kernel<__nv_bfloat16, S>);
    };
    if (sub == 2) by_out(std::integral_constant<int, 2>());
    else by_out(std::integral_constant<int, 1>());
    count_launch();
    ATLAS_LAUNCH_CHECK();
  }
  return ok;
}

// ATLAS_TRANSFORM_R=0 (A/B probes): x hi / lo in shared memory instead
bool regsplit_enabled() {
  const char* e = getenv("ATLAS_TRANSFORM_R");
  return !(e && e[0] == '0');
}

// false when W (hi + lo) cannot stay resident next to 3 x stages or the
// accumulators do not fit beside the A stages in TMEM
bool launch_transform_r(const void* x, int64_t rows, int64_t k, int64_t ldx,
                        const float* w, const float* b, int64_t n, int relu,
                        void* y, int y_dtype, int64_t ldy, int32_t* flag,
                        cudaStream_t s) {
  const int BN = (int)((n + 15) / 16 * 16);
  if (BN > 128) return false;
  const int kblocks = (int)((k + BK - 1) / BK);
  const int w_res = 2 * BN * BK * 4 * kblocks;
  const int x_stage = BM * BK * 4;
  const int fixed = 1024 + 8 * 64 + 16 + 4 * 256 + 16 +
                    kEpiWarps * 32 * kStageLd * 4;
  int stages = (227 * 1024 - fixed - w_res) / x_stage;
  if (stages > 8) stages = 8;
  if (const char* e = getenv("ATLAS_TRANSFORM_STAGES"))  // diagnostics
    stages = std::min(stages, std::max(3, atoi(e)));
  if (stages < 3) return false;
  CUtensorMap mx, mw;
  if (!make_map(&mx, x, ATLAS_F32, rows, k, ldx, BM) ||
      !make_map(&mw, w, ATLAS_F32, n, k, k, BN))
    return false;
  if (g_er.w && stages * x_stage + er_smem() > 227 * 1024 - fixed - w_res)
    stages--;
  if (stages < 3) return false;
  const int smem = fixed + w_res + stages * x_stage + er_smem();
  TcParams p{};
  apply_er(p);
    p.l2ahead = l2ahead_knob();
  p.M = rows;
  p.K = (int)k;
  p.N = (int)n;
  p.BN = BN;
  p.stages = stages;
  p.kblocks = kblocks;
  p.relu = relu;
  p.ldy = ldy;
  p.bias = b;
  p.y = y;
  p.flag = flag;
  p.tmem_cols = 512;
  const int64_t ntiles = (rows + BM - 1) / BM;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, num_sms());
  auto launch = [&](auto kern) {
    ATLAS_CUDA(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, kThreads, smem, s>>>(mx, mw, p);
  };
  if (y_dtype == ATLAS_F32) launch(transform_r_kernel<float>);
  else if (y_dtype == ATLAS_F16) launch(transform_r_kernel<__half>);
  else launch(transform_r_kernel<__nv_bfloat16>);
  count_launch();
  ATLAS_LAUNCH_CHECK();
  return true;
}

// ATLAS_TRANSFORM_RS_WIDE=0 (A/B): N in (128, 192] back on transform_tc
static bool wide_rs_enabled() {
  const char* e = getenv("ATLAS_TRANSFORM_RS_WIDE");
  return !(e && e[0] == '0');
}

// register split with W streamed (pre-split in global memory): false when
// BN > 128 or the rings do not fit
bool launch_transform_rs(const void* x, int64_t rows, int64_t k, int64_t ldx,
                         const float* w, const float* b, int64_t n, int relu,
                         void* y, int y_dtype, int64_t ldy, int32_t* flag,
                         cudaStream_t s) {
  const int BN = (int)((n + 15) / 16 * 16);
  // above 128 columns the accumulator pair leaves TMEM for 2 A stages
  // (BN <= 192; e.g. the papers100M SAGE head, K = 256 -> 172)
  if (BN > 192 || (BN > 128 && (k < 256 || !wide_rs_enabled()))) return false;
  const int kblocks = (int)((k + BK - 1) / BK);
  const int x_stage = BM * BK * 4;
  const int w_stage = 2 * BN * BK * 4;
  const int fixed = 1024 + 8 * 64 + 16 + 4 * 256 + 16 +
                    kEpiWarps * 32 * kStageLd * 4;
  const int xst = 4;
  int wst = (227 * 1024 - fixed - er_smem() - xst * x_stage) / w_stage;
  if (wst > 4) wst = 4;
  if (wst < 2) return false;
  // pre-split W into the (device, stream)'s grow-only scratch
  SplitScratch& ws = split_scratch(s);
  ws.buf.reserve((size_t)(2 * n * k * sizeof(float) + 64));
  float* whi = reinterpret_cast<float*>(ws.buf.ptr);
  float* wlo = whi + n * k;
  split_w_tf32<<<(unsigned)std::min<int64_t>(ceil_div(n * k, 256), 4096), 256,
                 0, s>>>(w, n * k, whi, wlo);
  count_launch();
  ATLAS_LAUNCH_CHECK();
  CUtensorMap mx, mhi, mlo;
  if (!make_map(&mx, x, ATLAS_F32, rows, k, ldx, BM) ||
      !make_map(&mhi, whi, ATLAS_F32, n, k, k, BN) ||
      !make_map(&mlo, wlo, ATLAS_F32, n, k, k, BN))
    return false;
  const int smem =
      fixed + xst * x_stage + wst * w_stage + 8 * 2 * wst + er_smem();
  TcParams p{};
  apply_er(p);
    p.l2ahead = l2ahead_knob();
  p.M = rows;
  p.K = (int)k;
  p.N = (int)n;
  p.BN = BN;
  p.stages = xst;
  p.kblocks = kblocks;
  p.relu = relu;
  p.ldy = ldy;
  p.bias = b;
  p.y = y;
  p.flag = flag;
  p.tmem_cols = 512;
  const int64_t ntiles = (rows + BM - 1) / BM;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, num_sms());
  auto launch = [&](auto kern) {
    ATLAS_CUDA(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, kThreads, smem, s>>>(mx, mhi, mlo, p, wst);
  };
  if (y_dtype == ATLAS_F32) launch(transform_rs_kernel<float>);
  else if (y_dtype == ATLAS_F16) launch(transform_rs_kernel<__half>);
  else launch(transform_rs_kernel<__nv_bfloat16>);
  count_launch();
  ATLAS_LAUNCH_CHECK();
  return true;
}

// ATLAS_TRANSFORM_T=1 (A/B probes): the TMEM-resident-W variant; measured
// slower than W in shared memory on every cfg2 shape
// (profiles/r2_transform_probe_v1.txt), so it is not the default
bool transposed_enabled() {
  const char* e = getenv("ATLAS_TRANSFORM_T");
  return e && e[0] == '1';
}

bool launch_transform_t(const void* x, int64_t rows, int64_t k, int64_t ldx,
                        const float* w, const float* b, int64_t n, int relu,
                        void* y, int y_dtype, int64_t ldy, int32_t* flag,
                        cudaStream_t s) {
  CUtensorMap mx;
  if (!make_map(&mx, x, ATLAS_F32, rows, k, ldx, BR)) return false;
  const int kblocks = (int)((k + BK - 1) / BK);
  const int stage_bytes = 2 * BR * BK * 4;
  const int fixed = 1024 + 8 * 64 + 16 + 4 * 128 + 64;
  int stages = (227 * 1024 - fixed) / stage_bytes;
  if (stages > 8) stages = 8;
  const int smem = fixed + stages * stage_bytes;
  TtParams p{};
  p.l2ahead = l2ahead_knob();
  p.M = rows;
  p.K = (int)k;
  p.Kp = kblocks * BK;
  p.N = (int)n;
  p.stages = stages;
  p.kblocks = kblocks;
  p.relu = relu;
  p.ldy = ldy;
  p.w = w;
  p.bias = b;
  p.y = y;
  p.flag = flag;
  const int64_t ntiles = (rows + BR - 1) / BR;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, num_sms());
  auto launch = [&](auto kern) {
    ATLAS_CUDA(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, kThreads, smem, s>>>(mx, p);
  };
  if (y_dtype == ATLAS_F32) launch(transform_t_kernel<float>);
  else if (y_dtype == ATLAS_F16) launch(transform_t_kernel<__half>);
  else launch(transform_t_kernel<__nv_bfloat16>);
  count_launch();
  ATLAS_LAUNCH_CHECK();
  return true;
}

bool launch_transform_tc(const void* x, int x_dtype, int64_t rows, int64_t k,
                         int64_t ldx, const float* w, const float* b,
                         int64_t n, int relu, void* y, int y_dtype,
                         int64_t ldy, int32_t* flag, cudaStream_t s) {
  if (rows <= 0) return true;
  if (x_dtype == ATLAS_F16 &&
      launch_transform_h(x, rows, k, ldx, w, b, n, relu, y, y_dtype, ldy,
                         flag, s))
    return true;
  const int xs = x_dtype == ATLAS_F32 ? 4 : 2;
  if (n < 1 || n > 256 || k < 1 || (ldx * xs) % 16 != 0 || k % 4 != 0 ||
      (reinterpret_cast<uintptr_t>(x) & 15) != 0)
    return false;
  if (g_er.w && x_dtype == ATLAS_F16) return false;  // er: h kernel only
  if (x_dtype == ATLAS_F32 && n <= 128 && k <= 128 && transposed_enabled() &&
      !g_er.w)
    return launch_transform_t(x, rows, k, ldx, w, b, n, relu, y, y_dtype, ldy,
                              flag, s);
  if (x_dtype == ATLAS_F32 && regsplit_enabled() &&
      (launch_transform_r(x, rows, k, ldx, w, b, n, relu, y, y_dtype, ldy,
                          flag, s) ||
       launch_transform_rs(x, rows, k, ldx, w, b, n, relu, y, y_dtype, ldy,
                           flag, s)))
    return true;
  if (g_er.w) return false;  // er: register-split kernels only
  const int BN = (int)((n + 15) / 16 * 16);
  const int kblocks = (int)((k + BK - 1) / BK);
  if ((reinterpret_cast<uintptr_t>(w) & 15) != 0) return false;
  CUtensorMap mx, mw;
  if (!make_map(&mx, x, x_dtype, rows, k, ldx, BM) ||
      !make_map(&mw, w, ATLAS_F32, n, k, k, BN))
    return false;
  // W (hi + lo, all k-blocks) stays resident when it leaves room for two
  // x stages; otherwise it streams through the stages with x
  const int budget = 220 * 1024 - 1024 - 2048 - kEpiWarps * 32 * kStageLd * 4;
  const int x_stage = 2 * BM * BK * 4;
  const int w_res = 2 * BN * BK * 4 * kblocks;
  const bool res_w = w_res + 2 * x_stage <= budget;
  const int stage_bytes = res_w ? x_stage : x_stage + 2 * BN * BK * 4;
  int stages = (budget - (res_w ? w_res : 0)) / stage_bytes;
  if (stages > 8) stages = 8;
  if (stages < 2) return false;
  const int smem = 1024 + (res_w ? w_res : 0) + stages * stage_bytes +
                   8 * (3 * stages + 6) + 16 + 4 * 256 + 16 +
                   kEpiWarps * 32 * kStageLd * 4;
  TcParams p{};
    p.l2ahead = l2ahead_knob();
  p.M = rows;
  p.K = (int)k;
  p.N = (int)n;
  p.BN = BN;
  p.stages = stages;
  p.kblocks = kblocks;
  p.relu = relu;
  p.ldy = ldy;
  p.bias = b;
  p.y = y;
  p.flag = flag;
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * BN)) cols <<= 1;
  p.tmem_cols = cols;
  const int64_t ntiles = (rows + BM - 1) / BM;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, num_sms());
  auto launch = [&](auto kern) {
    ATLAS_CUDA(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, kThreads, smem, s>>>(mx, mw, p);
  };
  auto by_out = [&](auto in_tag, auto res_tag) {
    using TIn = decltype(in_tag);
    constexpr bool R = decltype(res_tag)::value;
    if (y_dtype == ATLAS_F32) launch(transform_tc_kernel<TIn, float, R>);
    else if (y_dtype == ATLAS_F16) launch(transform_tc_kernel<TIn, __half, R>);
    else launch(transform_tc_kernel<TIn, __nv_bfloat16, R>);
  };
  auto by_in = [&](auto res_tag) {
    if (x_dtype == ATLAS_F32) by_out(float(), res_tag);
    else if (x_dtype == ATLAS_F16) by_out(__half(), res_tag);
    else by_out(__nv_bfloat16(), res_tag);
  };
  if (res_w) by_in(std::true_type());
  else by_in(std::false_type());
  count_launch();
  ATLAS_LAUNCH_CHECK();
  return true;
}

void set_transform_er(const float* w, int col, int heads, int hs) {
  g_er.w = w;
  g_er.col = col;
  g_er.heads = heads;
  g_er.hs = hs;
}

}  // namespace atlas
