// Row-granular bulk copies (TMA engine, cp.async.bulk -> UBLKCP) completed
// on shared-memory mbarriers: the staging primitive of the wide-row
// aggregation kernels (aggregate.cu agg_bulk, gat.cu gat_bulk).
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

// Feeds the rows of a contiguous edge range [e0, e1) of a CSC source list
// through a per-warp ring of SLOTS shared-memory row buffers. Refills go
// out in groups of G: lanes 0..G-1 each issue one row copy (source ids come
// from a 32-wide register batch by shuffle), so a warp spends one issue
// slot per G rows. All lanes call every member uniformly.
template <int SLOTS, int G>
struct RowFeeder {
  static_assert((SLOTS & (SLOTS - 1)) == 0 && G <= SLOTS && 32 % G == 0,
                "power-of-two ring, group divides the warp");
  uint8_t* ring;
  uint64_t* bars;
  uint32_t row_bytes;
  const uint32_t* __restrict__ src;
  uint32_t n_issued = 0, n_used = 0;
  int64_t pe = 0, e1 = 0, ibase = 0;
  uint32_t isrc = 0;

  template <typename T>
  __device__ __forceinline__ void issue_group(const T* base, int64_t ld) {
    if (pe >= e1) return;
    const int lane = threadIdx.x & 31;
    if (pe + G > ibase + 32) {
      ibase = pe;
      isrc = (pe + lane < e1) ? src[pe + lane] : 0u;
    }
    const int k = (int)((e1 - pe) < G ? (e1 - pe) : G);
    const uint32_t u =
        __shfl_sync(0xffffffffu, isrc, (int)(pe - ibase) + (lane & (G - 1)));
    if (lane < k) {
      const uint32_t slot = (n_issued + lane) & (SLOTS - 1);
      bulk_row(ring + (size_t)slot * row_bytes, base + (int64_t)u * ld,
               row_bytes, &bars[slot]);
    }
    n_issued += k;
    pe += k;
  }
  // start a new edge range (rows of the previous one may still be queued)
  template <typename T>
  __device__ __forceinline__ void begin(int64_t e0, int64_t end, const T* base,
                                        int64_t ld) {
    const int lane = threadIdx.x & 31;
    pe = e0;
    e1 = end;
    ibase = e0;
    isrc = (e0 + lane < end) ? src[e0 + lane] : 0u;
    while (pe < e1 && n_issued - n_used <= SLOTS - G) issue_group(base, ld);
  }
  // wait for the next row in edge order; returns its staging buffer
  __device__ __forceinline__ const uint8_t* wait() {
    const uint32_t slot = n_used & (SLOTS - 1);
    mbar_wait_parity(&bars[slot], (n_used / SLOTS) & 1u);
    return ring + (size_t)slot * row_bytes;
  }
  // the row from wait() is consumed by every lane: refill when G are free
  template <typename T>
  __device__ __forceinline__ void release(const T* base, int64_t ld) {
    n_used++;
    if (pe < e1 && n_issued - n_used <= SLOTS - G) {
      __syncwarp();  // every lane is done with the slots being refilled
      issue_group(base, ld);
    }
  }
};

}  // namespace atlas
