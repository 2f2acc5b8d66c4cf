// mp_radix.cuh -- K3r: 2048-key register/shared-memory block sort for bare
// 32-bit keys (u32, i32, f32 totalOrder), the first pass of the merge sort
// (replaces sort.hpp:59-67's 32-element insertion-sorted runs).
//
// Bare keys carry no payload, so equal keys are indistinguishable and any
// correct sort of a run produces the same bytes as the stable merge-based
// block sort (K3) -- which stays the path for values, elements and 64-bit
// keys.  This one is an LSD radix sort of the order-preserving u32 image:
// 4 passes of 8-bit digits, each pass stable:
//   * keys sit in smem in the current order and are read warp-striped
//     (warp w, item k, lane l  <->  position w*256 + k*32 + l), so "earlier
//     in the sequence" = (lower warp, then lower item, then lower lane);
//   * per item, __match_any_sync groups the warp's lanes by digit; a key's
//     warp-local rank = (keys of its digit in earlier items) + (lower lanes
//     in the same group); one leader per group bumps the warp's histogram;
//   * a 256-digit x 8-warp exclusive scan turns histograms into offsets;
//   * every key is scattered to offset[digit][warp] + its warp-local rank.
// ~16 instructions per key per pass instead of ~26 per key per merge pass.
#pragma once

#include "mp_common.cuh"

namespace mpb {

template <class KT> __device__ __forceinline__ uint32_t radix_image(typename KT::T x);
template <> __device__ __forceinline__ uint32_t radix_image<KeyU32>(uint32_t x) { return x; }
template <> __device__ __forceinline__ uint32_t radix_image<KeyI32>(int32_t x) {
  return static_cast<uint32_t>(x) ^ 0x80000000u;
}
template <> __device__ __forceinline__ uint32_t radix_image<KeyF32>(uint32_t x) {
  return f32_order(x);
}
template <class KT> __device__ __forceinline__ typename KT::T radix_key(uint32_t u);
template <> __device__ __forceinline__ uint32_t radix_key<KeyU32>(uint32_t u) { return u; }
template <> __device__ __forceinline__ int32_t radix_key<KeyI32>(uint32_t u) {
  return static_cast<int32_t>(u ^ 0x80000000u);
}
template <> __device__ __forceinline__ uint32_t radix_key<KeyF32>(uint32_t u) {
  return (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;  // inverse of f32_order
}

constexpr int kRadixNT = 256, kRadixVT = 8, kRadixNV = kRadixNT * kRadixVT;  // 2048
constexpr int kRadixWarps = kRadixNT / 32;

__host__ __device__ constexpr uint32_t radix_smem_bytes() {
  // two key buffers + per-warp 256-bin histograms + 256 digit totals
  return 2 * kRadixNV * 4 + kRadixWarps * 256 * 4 + 256 * 4 + 32 * 4;
}

template <class KT>
__global__ void __launch_bounds__(kRadixNT)
    block_radix_sort_kernel(const typename KT::T *__restrict__ in,
                            typename KT::T *__restrict__ out, uint64_t n) {
  extern __shared__ __align__(128) char smem[];
  uint32_t *buf0 = reinterpret_cast<uint32_t *>(smem);
  uint32_t *buf1 = buf0 + kRadixNV;
  uint32_t *hist = buf1 + kRadixNV;               // [warp][256]
  uint32_t *tot = hist + kRadixWarps * 256;       // [256] digit scan
  uint32_t *wsum = tot + 256;                     // [32] scan scratch
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t base = uint64_t(blockIdx.x) * kRadixNV;
  const int cnt = static_cast<int>((n - base) < kRadixNV ? (n - base) : kRadixNV);
  const unsigned lt_mask = (1u << lane) - 1u;

  // load (coalesced) as order images; pad with the maximum image
  for (int q = tid; q < kRadixNV; q += kRadixNT)
    buf0[q] = q < cnt ? radix_image<KT>(in[base + q]) : 0xFFFFFFFFu;

  uint32_t *src = buf0, *dst = buf1;
#pragma unroll 1
  for (int shift = 0; shift < 32; shift += 8) {
    for (int q = tid; q < kRadixWarps * 256; q += kRadixNT)
      hist[q] = 0;
    __syncthreads();
    uint32_t key[kRadixVT];
    uint32_t rank[kRadixVT];
    uint32_t *h = hist + warp * 256;
#pragma unroll
    for (int k = 0; k < kRadixVT; ++k) {
      key[k] = src[warp * 256 + k * 32 + lane];
      const uint32_t d = (key[k] >> shift) & 0xFFu;
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
      const uint32_t before = h[d];
      __syncwarp();
      rank[k] = before + __popc(peers & lt_mask);
      if ((peers & lt_mask) == 0)  // lowest lane of its group leads
        h[d] = before + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // offsets: thread t owns digit t; exclusive over warps, then over digits
    {
      const int d = tid;  // kRadixNT == 256 digits
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < kRadixWarps; ++w) {
        const uint32_t c = hist[w * 256 + d];
        hist[w * 256 + d] = run;
        run += c;
      }
      // block-wide exclusive scan of the 256 digit totals
      uint32_t x = run;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, off);
        if (lane >= off)
          x += y;
      }
      if (lane == 31)
        wsum[warp] = x;
      __syncthreads();
      if (warp == 0) {
        uint32_t s = lane < kRadixWarps ? wsum[lane] : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, off);
          if (lane >= off)
            s += y;
        }
        if (lane < kRadixWarps)
          wsum[lane] = s;  // inclusive over warps' digit blocks
      }
      __syncthreads();
      tot[d] = x - run + (warp ? wsum[warp - 1] : 0);  // exclusive digit start
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRadixVT; ++k) {
      const uint32_t d = (key[k] >> shift) & 0xFFu;
      dst[tot[d] + h[d] + rank[k]] = key[k];
    }
    __syncthreads();
    uint32_t *t = src;
    src = dst;
    dst = t;
  }
  for (int q = tid; q < cnt; q += kRadixNT)
    out[base + q] = radix_key<KT>(src[q]);
}

}  // namespace mpb
