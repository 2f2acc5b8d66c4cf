// mp_pieces.cuh -- merging sequences that are concatenations of pieces
// (shards that may live on other GPUs, mapped over NVLink / NVSwitch).
//
// A = A_0 ++ A_1 ++ ... and B = B_0 ++ B_1 ++ ... (virtual index spaces);
// the merge of (A, B) is the Merge Path over the virtual indices, exactly as
// if the pieces were one array (Theorem 14 does not care where bytes live).
//
// The merge itself needs no host round trip: pieces_partition_kernel
// searches every tile boundary of the requested output range in the
// virtual index space (each probe maps its index to a piece), and
// pieces_tiles_kernel stages each tile's A and B windows from the pieces --
// a window inside one local piece through the bulk-copy engine, inside one
// peer piece (another GPU's memory, mapped over NVLink) through LSU 16-byte
// loads, and a window that straddles piece boundaries (at most a few tiles
// per call) element by element -- then runs K2's merge half unchanged
// (merge_staged_window).  The NVLink pull is fused into the tile loads: no
// staging exchange, two launches, no host sync.
#pragma once

#include "mp_kernels.cuh"

namespace mpb {

constexpr int kMaxPieces = 16;

struct VPieces {
  const void *ptr[kMaxPieces];
  const uint32_t *vptr[kMaxPieces];  // values (NULL without values)
  uint64_t start[kMaxPieces + 1];    // start[n] = total length
  int n;
  uint32_t peer;  // bit k: piece k is another GPU's memory (LSU loads)
};

// piece holding virtual index i (i < total; empty pieces are skipped)
__device__ __forceinline__ int vpiece(const VPieces &v, uint64_t i) {
  int k = 0;
#pragma unroll 1
  while (k + 1 < v.n && i >= v.start[k + 1])
    ++k;
  return k;
}

template <class KT>
__device__ __forceinline__ typename KT::T vget(const VPieces &v, uint64_t i) {
  const int k = vpiece(v, i);
  return static_cast<const typename KT::T *>(v.ptr[k])[i - v.start[k]];
}

// a_off of the merge path on diagonal d (core.hpp:99-116 over pieces)
template <class KT>
__device__ uint64_t v_diag_search(const VPieces &A, const VPieces &B,
                                  uint64_t d) {
  const uint64_t na = A.start[A.n], nb = B.start[B.n];
  uint64_t lo = d > nb ? d - nb : 0;
  uint64_t hi = d < na ? d : na;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (take_b<KT>(vget<KT>(B, d - 1 - mid), vget<KT>(A, mid)))
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

// Split points of the tiles of output range [o0, o1): P[t] = a_off on
// diagonal min(o0 + t*nv, o1), t = 0..count-1 (core.hpp:99-132 semantics
// over the virtual index spaces).
template <class KT>
__global__ void pieces_partition_kernel(VPieces A, VPieces B, uint64_t o0, uint64_t o1,
                                        uint32_t nv, uint64_t count,
                                        uint64_t *__restrict__ P) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= count)
    return;
  const uint64_t d = o0 + t * nv < o1 ? o0 + t * nv : o1;
  P[t] = v_diag_search<KT>(A, B, d);
}

// Arbitrary diagonals over the pieces (mp_pieces_partition: split points of
// a sharded merge, e.g. for traffic accounting or a caller's own plan).
template <class KT>
__global__ void pieces_diagonals_kernel(VPieces A, VPieces B, const uint64_t *__restrict__ diags,
                                        uint64_t count, uint64_t *__restrict__ a_offs) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= count)
    return;
  const uint64_t n = A.start[A.n] + B.start[B.n];
  a_offs[t] = v_diag_search<KT>(A, B, diags[t] < n ? diags[t] : n);
}

// Copy `bytes` (a multiple of 16, 16-byte aligned ends) with SM vector loads
// -- the access pattern of the merge kernels' peer loader (LDG.128 of peer
// memory over NVLink).  Grid-stride, 4 loads in flight per thread.
__global__ void lsu_copy_kernel(uint4 *__restrict__ dst, const uint4 *__restrict__ src,
                                uint64_t n16) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  for (; q + 3 * stride < n16; q += 4 * stride) {
    const uint4 v0 = src[q], v1 = src[q + stride], v2 = src[q + 2 * stride],
                v3 = src[q + 3 * stride];
    dst[q] = v0;
    dst[q + stride] = v1;
    dst[q + 2 * stride] = v2;
    dst[q + 3 * stride] = v3;
  }
  for (; q < n16; q += stride)
    dst[q] = src[q];
}

// Stage virtual range [x0, x0 + cnt) of pieces V into smem at byte `off`
// element by element (all threads; windows that straddle piece boundaries).
template <class T, int NT>
__device__ __forceinline__ void stage_pieces_elems(char *smem, uint32_t off, uint32_t voff,
                                                   const VPieces &V, uint64_t x0,
                                                   uint32_t cnt, bool vals) {
  const uint64_t x1 = x0 + cnt;
  for (int k = vpiece(V, x0); k < V.n && V.start[k] < x1; ++k) {
    const uint64_t lo = V.start[k] > x0 ? V.start[k] : x0;
    const uint64_t hi = V.start[k + 1] < x1 ? V.start[k + 1] : x1;
    const T *src = static_cast<const T *>(V.ptr[k]) - V.start[k];
    for (uint64_t q = lo + threadIdx.x; q < hi; q += NT) {
      *reinterpret_cast<T *>(smem + off + (q - x0) * sizeof(T)) = src[q];
      if (vals)
        *reinterpret_cast<uint32_t *>(smem + voff + (q - x0) * 4) =
            (V.vptr[k] - V.start[k])[q];
    }
  }
}

// One CTA per tile of output range [o0, o1): window [P[t], P[t+1]) of A and
// the matching range of B, staged from the pieces, then K2's merge half.
template <class KT, bool VALS, int NT, int VT>
__global__ void __launch_bounds__(NT, (merge_min_blocks<KT, VALS, NT>()))
    pieces_tiles_kernel(VPieces A, VPieces B, const uint64_t *__restrict__ P, uint64_t o0,
                        uint64_t o1, typename KT::T *__restrict__ out,
                        uint32_t *__restrict__ outv, int force_lsu) {
  using T = typename KT::T;
  constexpr uint32_t KS = sizeof(T);
  constexpr uint32_t NV = NT * VT;
  constexpr bool SENT = merge_sentinels<KT, VALS>();
  extern __shared__ __align__(128) char smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  const int tid = threadIdx.x;
  const uint64_t t = blockIdx.x;
  const uint64_t d0 = o0 + t * NV, d1 = d0 + NV < o1 ? d0 + NV : o1;
  const uint64_t a0 = P[t], a1 = P[t + 1];
  const uint64_t b0 = d0 - a0, b1 = d1 - a1;
  TileWin win;
  win.a0 = a0;
  win.b0 = b0;
  win.o0 = d0 - o0;  // output index local to out
  win.na = static_cast<int>(a1 - a0);
  win.nb = static_cast<int>(b1 - b0);
  const int na_t = win.na, nb_t = win.nb;
  // source of each window: 0 = empty, 1 = one local piece (bulk copy),
  // 2 = one peer piece (LSU), 3 = straddles pieces (element copies)
  const int ka = na_t ? vpiece(A, a0) : 0, kb = nb_t ? vpiece(B, b0) : 0;
  const int mA = !na_t ? 0 : a1 > A.start[ka + 1] ? 3
                 : (force_lsu || ((A.peer >> ka) & 1)) ? 2 : 1;
  const int mB = !nb_t ? 0 : b1 > B.start[kb + 1] ? 3
                 : (force_lsu || ((B.peer >> kb) & 1)) ? 2 : 1;
  const char *gA = mA == 1 || mA == 2
                       ? static_cast<const char *>(A.ptr[ka]) + (a0 - A.start[ka]) * KS
                       : nullptr;
  const char *gB = mB == 1 || mB == 2
                       ? static_cast<const char *>(B.ptr[kb]) + (b0 - B.start[kb]) * KS
                       : nullptr;
  const char *gAv = nullptr, *gBv = nullptr;
  if constexpr (VALS) {
    gAv = gA ? reinterpret_cast<const char *>(A.vptr[ka] + (a0 - A.start[ka])) : nullptr;
    gBv = gB ? reinterpret_cast<const char *>(B.vptr[kb] + (b0 - B.start[kb])) : nullptr;
  }
  const uint32_t bA = na_t * KS, bB = nb_t * KS;
  const uint32_t oA = mirror_off(16, gA);
  const uint32_t oB = mirror_off(oA + bA + (SENT ? VT * KS : 0), gB);
  uint32_t oAv = 0, oBv = 0;
  if constexpr (VALS) {
    oAv = mirror_off(oB + bB, gAv);
    oBv = mirror_off(oAv + na_t * 4, gBv);
  }
  // bulk-copy interiors (local single-piece windows), issued by thread 0
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    uint32_t loA = 0, loB = 0, loAv = 0, loBv = 0, iA = 0, iB = 0, iAv = 0, iBv = 0;
    if (mA == 1) {
      iA = interior_bytes(gA, bA, &loA);
      if constexpr (VALS)
        iAv = interior_bytes(gAv, na_t * 4, &loAv);
    }
    if (mB == 1) {
      iB = interior_bytes(gB, bB, &loB);
      if constexpr (VALS)
        iBv = interior_bytes(gBv, nb_t * 4, &loBv);
    }
    mbar_arrive_expect_tx(bar, iA + iB + iAv + iBv);
    if (iA)
      bulk_g2s(smem + oA + loA, gA + loA, iA, bar);
    if (iB)
      bulk_g2s(smem + oB + loB, gB + loB, iB, bar);
    if (iAv)
      bulk_g2s(smem + oAv + loAv, gAv + loAv, iAv, bar);
    if (iBv)
      bulk_g2s(smem + oBv + loBv, gBv + loBv, iBv, bar);
  }
  // LSU interiors of peer windows (all threads)
  if (mA == 2) {
    uint32_t lo;
    uint32_t in = interior_bytes(gA, bA, &lo);
    lsu_copy16<NT>(smem + oA + lo, gA + lo, in, tid);
    if constexpr (VALS) {
      in = interior_bytes(gAv, na_t * 4, &lo);
      lsu_copy16<NT>(smem + oAv + lo, gAv + lo, in, tid);
    }
  }
  if (mB == 2) {
    uint32_t lo;
    uint32_t in = interior_bytes(gB, bB, &lo);
    lsu_copy16<NT>(smem + oB + lo, gB + lo, in, tid);
    if constexpr (VALS) {
      in = interior_bytes(gBv, nb_t * 4, &lo);
      lsu_copy16<NT>(smem + oBv + lo, gBv + lo, in, tid);
    }
  }
  // straddling windows, element by element
  if (mA == 3)
    stage_pieces_elems<T, NT>(smem, oA, oAv, A, a0, na_t, VALS);
  if (mB == 3)
    stage_pieces_elems<T, NT>(smem, oB, oBv, B, b0, nb_t, VALS);
  // unaligned heads/tails of the single-piece windows: warps 0/1 (keys),
  // 2/3 (values); warp 2 also writes the sentinels of bare keys
  {
    const int w = tid >> 5, l = tid & 31;
    static_assert(NT >= 128, "edge staging uses warps 0..3");
    if (w == 0 && (mA == 1 || mA == 2))
      stage_edges<KS>(smem, oA, gA, bA, l);
    else if (w == 1 && (mB == 1 || mB == 2))
      stage_edges<KS>(smem, oB, gB, bB, l);
    if constexpr (VALS) {
      if (w == 2 && (mA == 1 || mA == 2))
        stage_edges<4>(smem, oAv, gAv, na_t * 4, l);
      else if (w == 3 && (mB == 1 || mB == 2))
        stage_edges<4>(smem, oBv, gBv, nb_t * 4, l);
    }
    if constexpr (SENT) {
      static_assert(VT < 32, "one sentinel per lane");
      if (w == 2 && l <= VT)
        *reinterpret_cast<T *>(smem + (l < VT ? oA + bA + l * KS : oB + bB)) = KT::max_key();
    }
  }
  __syncthreads();
  mbar_wait(bar, 0);
  merge_staged_window<KT, VALS, NT, VT, false, SENT>(smem, win, oA, oB, oAv, oBv, out, outv,
                                                     nullptr);
}

}  // namespace mpb
