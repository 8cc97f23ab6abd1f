// Staging primitives of the aggregation kernels: row-granular bulk copies
// (TMA engine, cp.async.bulk -> UBLKCP) completed on shared-memory
// mbarriers (aggregate.cu agg_bulk, gat.cu gat_bulk) and per-lane 16-byte
// cp.async copies (LDGSTS) waited on per lane (the ring kernels).
#pragma once

#include "internal.cuh"

namespace atlas {

__device__ __forceinline__ void mbar_init_cta(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)),
               "r"(n));
}

__device__ __forceinline__ void bulk_row(void* smem, const void* gmem,
                                         uint32_t bytes, uint64_t* bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
      "r"(bytes)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
      "l"(gmem), "r"(bytes), "r"(b)
      : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar,
                                                 uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "BW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra BW_%=;\n}" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_row_s(uint32_t smem, const void* gmem,
                                           uint32_t bytes, uint32_t bar) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
      "r"(bytes)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem),
      "l"(gmem), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void mbar_wait_parity_s(uint32_t bar,
                                                   uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "BWS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra BWS_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint4 lds_v4(uint32_t smem) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem)
               : "memory");
  return v;
}
template <typename T>
__device__ __forceinline__ float lds_as_f32(uint32_t smem);
template <>
__device__ __forceinline__ float lds_as_f32<float>(uint32_t smem) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem) : "memory");
  return v;
}
template <>
__device__ __forceinline__ float lds_as_f32<__half>(uint32_t smem) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(smem) : "memory");
  return __half2float(__ushort_as_half(v));
}
template <>
__device__ __forceinline__ float lds_as_f32<__nv_bfloat16>(uint32_t smem) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(smem) : "memory");
  return __bfloat162float(__ushort_as_bfloat16(v));
}

// per-lane 16-byte asynchronous copies (LDGSTS) into shared memory
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
// same, with a precomputed shared-space destination address
__device__ __forceinline__ void cp_async16_s(uint32_t smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ uint4 lds16(uint32_t smem) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem)
               : "memory");
  return v;
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}


// Feeds the rows of a contiguous edge range [e0, e1) of a CSC source list
// through a per-warp ring of SLOTS shared-memory row buffers. Refills go
// out in groups of G: lanes 0..G-1 each issue one row copy (source ids come
// from a 32-wide register batch by shuffle), so a warp spends one issue
// slot per G rows. Indices are relative to e0 (32-bit) and every shared
// address is precomputed. All lanes call every member uniformly.
template <int SLOTS, int G>
struct RowFeeder {
  static_assert((SLOTS & (SLOTS - 1)) == 0 && G <= SLOTS && 32 % G == 0,
                "power-of-two ring, group divides the warp");
  uint32_t ring;  // shared address of slot 0
  uint32_t bars;  // shared address of the slot-0 mbarrier (8 B apart)
  uint32_t row_bytes;
  const uint32_t* __restrict__ src;
  uint32_t n_issued = 0, n_used = 0;
  const uint32_t* __restrict__ src0 = nullptr;
  int pe = 0, ne = 0, ibase = 0;  // ids of edges [ibase, ibase + 32) held
  uint32_t isrc = 0;

  __device__ RowFeeder(uint8_t* ring_ptr, uint64_t* bar_ptr, uint32_t rb,
                       const uint32_t* s)
      : ring((uint32_t)__cvta_generic_to_shared(ring_ptr)),
        bars((uint32_t)__cvta_generic_to_shared(bar_ptr)),
        row_bytes(rb),
        src(s) {}

  template <typename T>
  __device__ __forceinline__ void issue_group(const T* base, int64_t ld) {
    if (pe >= ne) return;
    const int lane = threadIdx.x & 31;
    if (pe - ibase == 32) {  // pe steps by G, which divides 32
      ibase = pe;
      isrc = pe + lane < ne ? src0[pe + lane] : 0u;
    }
    const int k = ne - pe < G ? ne - pe : G;
    const uint32_t u =
        __shfl_sync(0xffffffffu, isrc, pe - ibase + (lane & (G - 1)));
    if (lane < k) {
      const uint32_t slot = (n_issued + lane) & (SLOTS - 1);
      bulk_row_s(ring + slot * row_bytes, base + (int64_t)u * ld, row_bytes,
                 bars + slot * 8u);
    }
    n_issued += k;
    pe += k;
  }
  // start a new edge range (rows of the previous one may still be queued)
  template <typename T>
  __device__ __forceinline__ void begin(int64_t e0, int64_t end, const T* base,
                                        int64_t ld) {
    const int lane = threadIdx.x & 31;
    src0 = src + e0;
    ne = (int)(end - e0);
    pe = ibase = 0;
    isrc = lane < ne ? src0[lane] : 0u;
    if (pe < ne && n_issued - n_used <= SLOTS - G) {
      __syncwarp();  // slots freed by release_n without a refill: order
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      do {
        issue_group(base, ld);
      } while (pe < ne && n_issued - n_used <= SLOTS - G);
    }
  }
  // wait for the next row in edge order; returns its shared address
  __device__ __forceinline__ uint32_t wait() {
    const uint32_t slot = n_used & (SLOTS - 1);
    mbar_wait_parity_s(bars + slot * 8u, (n_used / SLOTS) & 1u);
    return ring + slot * row_bytes;
  }
  // the row from wait() is consumed by every lane: refill when G are free
  template <typename T>
  __device__ __forceinline__ void release(const T* base, int64_t ld) {
    release_n(1, base, ld);
  }
  // the k-th row after the next one (k = 0: wait()), not consumed yet
  __device__ __forceinline__ uint32_t wait_k(uint32_t k) {
    const uint32_t n = n_used + k;
    const uint32_t slot = n & (SLOTS - 1);
    mbar_wait_parity_s(bars + slot * 8u, (n / SLOTS) & 1u);
    return ring + slot * row_bytes;
  }
  // n rows consumed by every lane; refill while whole groups are free
  template <typename T>
  __device__ __forceinline__ void release_n(uint32_t n, const T* base,
                                            int64_t ld) {
    n_used += n;
    if (pe < ne && n_issued - n_used <= SLOTS - G) {
      __syncwarp();  // every lane is done with the slots being refilled
      // ...and those generic-proxy reads are ordered before the
      // async-proxy bulk copies that overwrite the slots (compute-sanitizer
      // racecheck flags the WAR without it, profiles/r2_sanitize_*.txt)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      do {
        issue_group(base, ld);
      } while (pe < ne && n_issued - n_used <= SLOTS - G);
    }
  }
};

}  // namespace atlas
