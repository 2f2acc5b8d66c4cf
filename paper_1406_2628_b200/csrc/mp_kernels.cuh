// mp_kernels.cuh -- the Merge Path kernels for sm_100a.
//
//   K1 partition_kernel       cross-diagonal binary search in HBM
//                             (core.hpp:99-146) at tile or p-way spacing
//   K2 merge_tiles_kernel     one CTA = one Segmented-Parallel-Merge window
//                             (parallel.hpp:90-145): bulk-copy (TMA engine)
//                             the tile's A/B windows into smem, split the
//                             window among threads by a second diagonal
//                             search in smem, serial stable merge of VT
//                             items per thread (core.hpp:151-180), stage the
//                             output in smem and write it back coalesced
//                             (bulk store when aligned).
//   K3 block_sort_kernel      stable sort of NT*VT-key runs in registers +
//                             smem (replaces sort.hpp:59-67's 32-runs)
//   K4 round_partition_kernel tile boundaries for every run pair of one
//                             bottom-up round (sort.hpp:71-101), left run = A
#pragma once

#include <type_traits>

#include "mp_common.cuh"

namespace mpb {

// ---------------------------------------------------------------------------
// K1: diagonal search in global memory.
// ---------------------------------------------------------------------------
template <class KT>
__device__ __forceinline__ uint64_t diag_search_global(
    const typename KT::T *__restrict__ a, uint64_t na,
    const typename KT::T *__restrict__ b, uint64_t nb, uint64_t d,
    uint32_t *probes = nullptr) {
  uint64_t lo = d > nb ? d - nb : 0;
  uint64_t hi = d < na ? d : na;
  uint32_t c = 0;
  while (lo < hi) {
    ++c;
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (take_b<KT>(b[d - 1 - mid], a[mid]))
      hi = mid;
    else
      lo = mid + 1;
  }
  if (probes)
    *probes = c;
  return lo;
}

// The same split found by one warp with 32-ary steps: lane l probes
// lo + l*step (step = ceil(span/32)); the predicate take_b(B[d-1-m], A[m])
// is false..true along m (core.hpp:110), so the first lane that sees true
// brackets the split between its probe and the previous lane's.  About
// log32(span) + 1 dependent rounds of loads instead of log2(span): for a CTA
// that searches its own tile boundary (SearchMap) the latency is what
// counts.  All lanes return the same (exact) split.
template <class KT>
__device__ __forceinline__ uint64_t diag_search_warp(
    const typename KT::T *__restrict__ a, uint64_t na,
    const typename KT::T *__restrict__ b, uint64_t nb, uint64_t d, int lane) {
  uint64_t lo = d > nb ? d - nb : 0;
  uint64_t hi = d < na ? d : na;  // split in [lo, hi]
  while (lo < hi) {
    const uint64_t step = (hi - lo + 31) >> 5;
    const uint64_t m = lo + static_cast<uint64_t>(lane) * step;
    const bool t = m >= hi || take_b<KT>(b[d - 1 - m], a[m]);
    const unsigned ball = __ballot_sync(0xffffffffu, t);
    if (ball == 0) {  // every probe false: split above the last probe
      lo = lo + 31 * step + 1;
    } else {
      const int k = __ffs(ball) - 1;  // first probe that is true
      const uint64_t mk = lo + static_cast<uint64_t>(k) * step;
      hi = mk < hi ? mk : hi;
      lo = k ? lo + static_cast<uint64_t>(k - 1) * step + 1 : lo;
    }
  }
  return lo;
}

// The same search with the top levels snapped to a shared grid (every
// GRID-th element of A and B).  A probe at a grid position mid is decided
// from the two grid neighbours of B[d-1-mid] when they bracket A[mid]
// conclusively (Bhi < A[mid] => move right; Blo >= A[mid] => move down) and
// by the exact element otherwise, so it is still an exact binary search for
// the same split.  Grid lines are shared by every thread's search and stay
// in L2; only the last ~log2(2*GRID) probes are private DRAM sectors.
// (Measured on B200: the plain search's 139 812 tile searches read 615 MB
// of DRAM at a 6 % L2 hit rate.)
template <class KT, uint64_t GRID = 1024>
__device__ __forceinline__ uint64_t diag_search_grid(
    const typename KT::T *__restrict__ a, uint64_t na,
    const typename KT::T *__restrict__ b, uint64_t nb, uint64_t d) {
  using T = typename KT::T;
  uint64_t lo = d > nb ? d - nb : 0;
  uint64_t hi = d < na ? d : na;
  while (hi - lo > 2 * GRID) {
    uint64_t mid = (lo + ((hi - lo) >> 1)) & ~(GRID - 1);
    if (mid <= lo)
      mid = lo + GRID;  // stays < hi since hi - lo > 2*GRID
    const uint64_t j = d - 1 - mid;  // B index, in [0, nb)
    const uint64_t jl = j & ~(GRID - 1);
    const uint64_t jh = jl + GRID < nb ? jl + GRID : nb - 1;
    const T x = a[mid];
    bool right;
    if (take_b<KT>(b[jh], x))  // B[j] <= B[jh] < A[mid]
      right = true;
    else if (!take_b<KT>(b[jl], x))  // B[j] >= B[jl] >= A[mid]
      right = false;
    else
      right = take_b<KT>(b[j], x);
    if (right)
      hi = mid;
    else
      lo = mid + 1;
  }
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (take_b<KT>(b[d - 1 - mid], a[mid]))
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

#ifndef MP_K1_GRID
#define MP_K1_GRID 16384  // B200 config 2 K1: 1024 34.0 us, 4096 27.2,
#endif                    // 16384 24.8, 65536 23.7 (step 0.662 -> 0.650 ms)
// Point t sits on diagonal min(t*spacing, N) (tile mode, p == 0) or on
// floor(t*N/p) (p-way mode, core.hpp:90-92).  Writes a_off for t < count.
template <class KT>
__global__ void partition_kernel(const typename KT::T *__restrict__ a,
                                 uint64_t na,
                                 const typename KT::T *__restrict__ b,
                                 uint64_t nb, uint64_t spacing, uint64_t p,
                                 uint64_t count, uint64_t *__restrict__ a_offs,
                                 unsigned long long *__restrict__ cmp = nullptr,
                                 uint64_t t0 = 0) {
  const uint64_t t = t0 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= count)
    return;
  const uint64_t n = na + nb;
  uint64_t d;
  if (p) {
    d = static_cast<uint64_t>((static_cast<unsigned __int128>(t) * n) / p);
  } else {
    const unsigned __int128 x = static_cast<unsigned __int128>(t) * spacing;
    d = x < n ? static_cast<uint64_t>(x) : n;
  }
  if (cmp) {  // replay the reference's exact probe sequence to count it
    uint32_t c = 0;
    a_offs[t] = diag_search_global<KT>(a, na, b, nb, d, &c);
    if (c)  // comparison count of the reference's search (core.hpp:128)
      atomicAdd(cmp, static_cast<unsigned long long>(c));
  } else {
    a_offs[t] = diag_search_grid<KT, MP_K1_GRID>(a, na, b, nb, d);
  }
}

// Refine a split plan made at tile NV*R to tile NV: boundary f lies between
// the planned points of its wider tile, so the search is bounded by them.
template <class KT>
__global__ void refine_partition_kernel(const typename KT::T *__restrict__ a,
                                        uint64_t na,
                                        const typename KT::T *__restrict__ b,
                                        uint64_t nb,
                                        const uint64_t *__restrict__ Pc,
                                        uint32_t nv, uint32_t R, uint64_t count,
                                        uint64_t *__restrict__ Pf) {
  const uint64_t f = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (f >= count)
    return;
  const uint64_t c = f / R, r = f % R;
  if (r == 0) {
    Pf[f] = Pc[c];
    return;
  }
  const uint64_t n = na + nb;
  const uint64_t d = f * nv < n ? f * nv : n;
  uint64_t lo = d > nb ? d - nb : 0;
  uint64_t hi = d < na ? d : na;
  lo = lo > Pc[c] ? lo : Pc[c];
  hi = hi < Pc[c + 1] ? hi : Pc[c + 1];
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (take_b<KT>(b[d - 1 - mid], a[mid]))
      hi = mid;
    else
      lo = mid + 1;
  }
  Pf[f] = lo;
}

// Arbitrary diagonals (used by the drop-in API for single searches and for
// the segmented-merge plan).
template <class KT>
__global__ void diagonals_kernel(const typename KT::T *__restrict__ a,
                                 uint64_t na,
                                 const typename KT::T *__restrict__ b,
                                 uint64_t nb, const uint64_t *__restrict__ diags,
                                 uint64_t count, uint64_t *__restrict__ a_offs,
                                 unsigned long long *__restrict__ cmp) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= count)
    return;
  const uint64_t n = na + nb;
  const uint64_t d = diags[t] < n ? diags[t] : n;
  uint32_t c = 0;
  a_offs[t] = diag_search_global<KT>(a, na, b, nb, d, &c);
  if (cmp && c)
    atomicAdd(cmp, static_cast<unsigned long long>(c));
}

// ---------------------------------------------------------------------------
// Tile -> window maps for K2.
// ---------------------------------------------------------------------------
struct TileWin {
  uint64_t a0;  // first A element (index into the `a` base pointer)
  uint64_t b0;  // first B element (index into the `b` base pointer)
  uint64_t o0;  // first output position
  int na;       // A elements in the window
  int nb;       // B elements in the window
};

// Plain merge of A and B: tile t owns outputs [t*NV, min((t+1)*NV, N)).
struct PlainMap {
  const uint64_t *P;  // a_off at diagonal t*NV, t = 0..tiles
  uint64_t n;
  uint32_t nv;
  __device__ __forceinline__ TileWin window(uint64_t t) const {
    const uint64_t d0 = t * nv;
    const uint64_t d1 = d0 + nv < n ? d0 + nv : n;
    const uint64_t a0 = P[t], a1 = P[t + 1];
    TileWin w;
    w.a0 = a0;
    w.b0 = d0 - a0;
    w.o0 = d0;
    w.na = static_cast<int>(a1 - a0);
    w.nb = static_cast<int>((d1 - a1) - (d0 - a0));
    return w;
  }
};

// Plain merge whose tile split points are searched by the tile's own CTA
// (no K1 launch): for merges that fit in one wave of CTAs, where K1's launch
// and dependent-probe latency is a large share of the call (config 1:
// K1 ~15 us cold + K2 ~10 us).  Warp 0 searches diagonal t*NV and warp 1
// diagonal (t+1)*NV (diag_search_warp: core.hpp:99-132 semantics, exact
// split points), then window() takes them like PlainMap takes P[t], P[t+1].
struct SearchMap {
  uint64_t na, n;
  uint32_t nv;
  static constexpr bool kSearch = true;
  // split point of boundary `end` (0: tile start, 1: tile end) of tile t
  template <class KT>
  __device__ __forceinline__ uint64_t split(const typename KT::T *a, const typename KT::T *b,
                                            uint64_t t, int end, int lane) const {
    const uint64_t d = (t + end) * nv < n ? (t + end) * nv : n;
    return diag_search_warp<KT>(a, na, b, n - na, d, lane);
  }
  __device__ __forceinline__ TileWin window(uint64_t t, uint64_t a0, uint64_t a1) const {
    const uint64_t d0 = t * nv;
    const uint64_t d1 = d0 + nv < n ? d0 + nv : n;
    TileWin w;
    w.a0 = a0;
    w.b0 = d0 - a0;
    w.o0 = d0;
    w.na = static_cast<int>(a1 - a0);
    w.nb = static_cast<int>((d1 - a1) - (d0 - a0));
    return w;
  }
};
template <class Map, class = void> struct map_searches : std::false_type {};
template <class Map>
struct map_searches<Map, std::void_t<decltype(Map::kSearch)>> : std::true_type {};

// One bottom-up round over runs of `width` (sort.hpp:71-101): pair k merges
// A = src[2kw, 2kw+w) with B = src[2kw+w, 2kw+2w) (clipped to n); an
// unpaired tail run has an empty B and is copied.  The tile NV divides the
// pair width 2w = NV << tshift, so a tile never straddles two pairs and the
// pair of tile t is t >> tshift (widths need not be powers of two: the bare
// 32-bit block sort makes 4352-key runs).  P[t] = pair-local a_off at the
// tile start.
__device__ __forceinline__ uint64_t round_pair_start(uint64_t t, uint32_t nv,
                                                     uint32_t tshift) {
  return (t >> tshift) * (uint64_t(nv) << tshift);
}

struct RoundMap {
  const uint64_t *P;
  uint64_t n;
  uint64_t width;
  uint32_t nv;
  uint32_t tshift;
  __device__ __forceinline__ TileWin window(uint64_t t) const {
    const uint64_t d0 = t * nv;
    const uint64_t s = round_pair_start(t, nv, tshift);
    const uint64_t la = (n - s) < width ? (n - s) : width;
    const uint64_t rest = n - s - la;
    const uint64_t lb = rest < width ? rest : width;
    const uint64_t dl0 = d0 - s;
    const uint64_t dl1 = dl0 + nv < la + lb ? dl0 + nv : la + lb;
    const uint64_t a0 = P[t];
    const uint64_t a1 = (dl1 == la + lb) ? la : P[t + 1];
    TileWin w;
    w.a0 = s + a0;
    w.b0 = s + la + (dl0 - a0);
    w.o0 = d0;
    w.na = static_cast<int>(a1 - a0);
    w.nb = static_cast<int>((dl1 - a1) - (dl0 - a0));
    return w;
  }
};

// RoundMap whose split points the tile's CTA searches itself (SearchMap's
// scheme for rounds of small sorts: one launch per round instead of K4 + K2).
struct RoundSearchMap {
  uint64_t n;
  uint64_t width;
  uint32_t nv;
  uint32_t tshift;
  static constexpr bool kSearch = true;
  template <class KT>
  __device__ __forceinline__ uint64_t split(const typename KT::T *src, const typename KT::T *,
                                            uint64_t t, int end, int lane) const {
    const uint64_t d0 = t * nv;
    const uint64_t s = round_pair_start(t, nv, tshift);
    const uint64_t la = (n - s) < width ? (n - s) : width;
    const uint64_t rest = n - s - la;
    const uint64_t lb = rest < width ? rest : width;
    const uint64_t dl0 = d0 - s;
    const uint64_t dl = end ? (dl0 + nv < la + lb ? dl0 + nv : la + lb) : dl0;
    return diag_search_warp<KT>(src + s, la, src + s + la, lb, dl, lane);
  }
  __device__ __forceinline__ TileWin window(uint64_t t, uint64_t a0, uint64_t a1) const {
    const uint64_t d0 = t * nv;
    const uint64_t s = round_pair_start(t, nv, tshift);
    const uint64_t la = (n - s) < width ? (n - s) : width;
    const uint64_t rest = n - s - la;
    const uint64_t lb = rest < width ? rest : width;
    const uint64_t dl0 = d0 - s;
    const uint64_t dl1 = dl0 + nv < la + lb ? dl0 + nv : la + lb;
    TileWin w;
    w.a0 = s + a0;
    w.b0 = s + la + (dl0 - a0);
    w.o0 = d0;
    w.na = static_cast<int>(a1 - a0);
    w.nb = static_cast<int>((dl1 - a1) - (dl0 - a0));
    return w;
  }
};

// K4: pair-local a_off at the start of every tile of one round.
template <class KT>
__global__ void round_partition_kernel(const typename KT::T *__restrict__ src,
                                       uint64_t n, uint64_t width,
                                       uint32_t tshift, uint32_t nv,
                                       uint64_t tiles,
                                       uint64_t *__restrict__ P,
                                       uint64_t t0 = 0) {
  const uint64_t t = t0 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= tiles)
    return;
  const uint64_t d0 = t * nv;
  const uint64_t s = round_pair_start(t, nv, tshift);
  const uint64_t la = (n - s) < width ? (n - s) : width;
  const uint64_t rest = n - s - la;
  const uint64_t lb = rest < width ? rest : width;
#ifndef MP_K4_GRID
#define MP_K4_GRID 4096  // B200, 2^30 u32 sort, 18 rounds of K4: 0 (plain
#endif                   // search) 2.70 ms, 256 2.94, 1024 2.08, 4096 1.76, 16384 1.83
  if constexpr (MP_K4_GRID == 0)
    P[t] = diag_search_global<KT>(src + s, la, src + s + la, lb, d0 - s);
  else
    P[t] = diag_search_grid<KT, MP_K4_GRID>(src + s, la, src + s + la, lb, d0 - s);
}

// K4 with one warp per tile boundary (diag_search_warp: ~log32 dependent
// rounds of 32 parallel probes instead of ~log2 single probes): for rounds
// whose K4 is latency-bound rather than bound by its DRAM sectors (a warp
// reads ~32x the sectors of a single-thread search).
template <class KT>
__global__ void round_partition_warp_kernel(const typename KT::T *__restrict__ src,
                                            uint64_t n, uint64_t width, uint32_t tshift,
                                            uint32_t nv, uint64_t tiles,
                                            uint64_t *__restrict__ P) {
  const uint64_t t = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= tiles)
    return;
  const uint64_t d0 = t * nv;
  const uint64_t s = round_pair_start(t, nv, tshift);
  const uint64_t la = (n - s) < width ? (n - s) : width;
  const uint64_t rest = n - s - la;
  const uint64_t lb = rest < width ? rest : width;
  const uint64_t a = diag_search_warp<KT>(src + s, la, src + s + la, lb, d0 - s, lane);
  if (lane == 0)
    P[t] = a;
}

// ---------------------------------------------------------------------------
// K2: tile merge.
// ---------------------------------------------------------------------------
// Staging index: odd VT keeps the per-thread strided stores conflict-free;
// even VT gets one pad element per 32 (breaks the power-of-two stride).
template <int VT>
__device__ __forceinline__ int stage_idx(int p) {
  if constexpr (VT & 1)
    return p;
  else
    return p + (p >> 5);
}

template <int NT, int VT>
__host__ __device__ constexpr int stage_elems() {
  return (VT & 1) ? NT * VT : NT * VT + (NT * VT) / 32;
}

// Bare keys (no values, not the AoS element) run K2 with sentinels: VT
// copies of the largest key after A's window and one after B's, so every
// thread takes the bounds-free serial merge (serial_merge, SENT = true).
template <class KT, bool VALS>
__host__ __device__ constexpr bool merge_sentinels() {
  return !VALS && KT::kind != kElement;
}

template <class KT, bool VALS, int NT, int VT>
__host__ __device__ constexpr uint32_t merge_smem_bytes() {
  using T = typename KT::T;
  constexpr uint32_t NV = NT * VT;
  constexpr uint32_t in_bytes =
      // windows + alignment gaps + one element of read slack per window
      NV * sizeof(T) + 96 + (VALS ? NV * 4 + 64 : 0) +
      (merge_sentinels<KT, VALS>() ? (VT + 1) * sizeof(T) + 16 : 0);
  constexpr uint32_t st_bytes =
      stage_elems<NT, VT>() * sizeof(T) + 16 +
      (VALS ? stage_elems<NT, VT>() * 4 + 16 : 0);
  return 16 + (in_bytes > st_bytes ? in_bytes : st_bytes);
}

// smem byte offset of the 16 B-aligned slot that mirrors global address g:
// offset congruent to g (mod 16) so the bulk-copy interior is aligned.
__device__ __forceinline__ uint32_t mirror_off(uint32_t at, const void *g) {
  return ((at + 15u) & ~15u) + static_cast<uint32_t>(reinterpret_cast<uintptr_t>(g) & 15u);
}

// Stage `bytes` of global memory at g into smem[off, off+bytes): the aligned
// interior through the bulk-copy engine (issued by thread 0, completes on
// bar), the unaligned head and tail (< 16 B each) with ordinary loads.
// Called by one warp (lane = 0..31): the head [0, lo) and tail [hi, bytes)
// outside the 16 B-aligned interior are < 32 B in total.
template <int ES>
__device__ __forceinline__ void stage_edges(char *smem, uint32_t off,
                                            const char *g, uint32_t bytes,
                                            int lane) {
  using W = typename std::conditional<
      ES == 4, uint32_t,
      typename std::conditional<ES == 8, unsigned long long, int4>::type>::type;
  const uintptr_t s = reinterpret_cast<uintptr_t>(g);
  const uintptr_t is = (s + 15) & ~uintptr_t(15);
  const uintptr_t ie = (s + bytes) & ~uintptr_t(15);
  const uint32_t lo = ie > is ? static_cast<uint32_t>(is - s) : bytes;
  const uint32_t hi = ie > is ? static_cast<uint32_t>(ie - s) : bytes;
  const uint32_t nh = lo / ES, nt = (bytes - hi) / ES;
  const uint32_t l = static_cast<uint32_t>(lane);
  if (l < nh + nt) {
    const uint32_t o = l < nh ? l * ES : hi + (l - nh) * ES;
    *reinterpret_cast<W *>(smem + off + o) = __ldg(reinterpret_cast<const W *>(g + o));
  }
}

__device__ __forceinline__ char *align16p(char *p) {
  return reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(p) + 15) &
                                  ~uintptr_t(15));
}

__device__ __forceinline__ uint32_t interior_bytes(const char *g, uint32_t bytes,
                                                   uint32_t *lo_out) {
  const uintptr_t s = reinterpret_cast<uintptr_t>(g);
  const uintptr_t is = (s + 15) & ~uintptr_t(15);
  const uintptr_t ie = (s + bytes) & ~uintptr_t(15);
  *lo_out = static_cast<uint32_t>(is - s);
  return ie > is ? static_cast<uint32_t>(ie - is) : 0u;
}

// Checksum sink support (core.hpp:200-245): key_of is static_cast<uint64_t>
// for integer keys; f32 keys are bit-cast (documented in DESIGN.md).
__device__ __forceinline__ uint64_t mix64_dev(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t key_of(uint32_t x) { return x; }
__device__ __forceinline__ uint64_t key_of(int32_t x) {
  return static_cast<uint64_t>(static_cast<long long>(x));
}
__device__ __forceinline__ uint64_t key_of(unsigned long long x) { return x; }
__device__ __forceinline__ uint64_t key_of(long long x) {
  return static_cast<uint64_t>(x);
}
__device__ __forceinline__ uint64_t key_of(const Element &x) {
  return static_cast<uint64_t>(x.key);
}

template <class T>
__device__ __forceinline__ T lds(const char *smem, uint32_t off) {
  return *reinterpret_cast<const T *>(smem + off);
}

// Serial stable merge of VT outputs from split (i, j) of the smem windows
// A = [oA, oA + na*KS), B = [oB, oB + nb*KS) (core.hpp:166-176; ties to A).
// Branch-free: one predicated choice and ONE smem load (the consumed side's
// next element) per output.  Fast path: when neither window can run out
// within VT steps (i + VT <= na and j + VT <= nb -- all but the threads at a
// window's end) the bounds tests vanish and the cursors are byte offsets
// (~8 instructions per output).  Loads may touch one element past a window
// (into the next window or the slack) and are then never used.
// SENT (bare keys, sentinels behind both windows -- see merge_sentinels):
// every thread takes the fast path.  Once A is exhausted its cursor walks
// A's VT sentinels (the largest key), which lose to every smaller B key and
// tie with a B key equal to them -- emitting the same value -- and B's
// cursor never passes its own sentinel (never strictly below an A key), so
// the VT output values are exact; outputs past the window are not stored.
template <class KT, int VT, bool VALS, bool SENT = false>
__device__ __forceinline__ void serial_merge(const char *smem, uint32_t oA,
                                             int na, uint32_t oB, int nb,
                                             uint32_t oAv, uint32_t oBv, int i,
                                             int j, typename KT::T (&keys)[VT],
                                             uint32_t (&vals)[VT]) {
  using T = typename KT::T;
  constexpr uint32_t KS = sizeof(T);
  uint32_t pa = oA + i * KS, pb = oB + j * KS;
  uint32_t pva = oAv + i * 4u, pvb = oBv + j * 4u;
  static_assert(!(SENT && VALS), "sentinels are for bare keys");
  if (SENT || (i + VT <= na && j + VT <= nb)) {
    T ka = lds<T>(smem, pa), kb = lds<T>(smem, pb);
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      const bool tb = take_b<KT>(kb, ka);
      keys[k] = tb ? kb : ka;
      if constexpr (VALS) {
        vals[k] = lds<uint32_t>(smem, tb ? pvb : pva);
        pva += tb ? 0u : 4u;
        pvb += tb ? 4u : 0u;
      }
      pa += tb ? 0u : KS;
      pb += tb ? KS : 0u;
      const T nxt = lds<T>(smem, tb ? pb : pa);
      kb = tb ? nxt : kb;
      ka = tb ? ka : nxt;
    }
    return;
  }
  const uint32_t ea = oA + na * KS, eb = oB + nb * KS;
  const uint32_t eva = oAv + na * 4u, evb = oBv + nb * 4u;
  T ka = lds<T>(smem, min(pa, ea)), kb = lds<T>(smem, min(pb, eb));
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    const bool tb = (pb < eb) && ((pa >= ea) || take_b<KT>(kb, ka));
    keys[k] = tb ? kb : ka;
    if constexpr (VALS) {
      vals[k] = lds<uint32_t>(smem, tb ? min(pvb, evb) : min(pva, eva));
      pva += tb ? 0u : 4u;
      pvb += tb ? 4u : 0u;
    }
    pa += tb ? 0u : KS;
    pb += tb ? KS : 0u;
    const T nxt = lds<T>(smem, tb ? min(pb, eb) : min(pa, ea));
    kb = tb ? nxt : kb;
    ka = tb ? ka : nxt;
  }
}

// SINK = the register-sink mode (parallel.hpp:181-198): nothing is stored;
// each thread folds (pos+1)*mix64(key) over its outputs and the CTA adds its
// partial sum into *sum.
// Residency target: a full SM (2048 threads, <= 32 registers) for bare
// keys up to 8 B; 3/4 of it when values or 16-byte elements ride along.
template <class KT, bool VALS, int NT, bool SINK = false>
constexpr int merge_min_blocks() {
  return (VALS && sizeof(typename KT::T) == 4)      ? 1024 / NT
         : (VALS || SINK)                           ? 1280 / NT
         : sizeof(typename KT::T) == 4               ? 2048 / NT  // f32 too: B200 config 5 K2 5.77 -> 5.38 ms
         : sizeof(typename KT::T) <= 8               ? 1536 / NT
                                                     : 1280 / NT;
}
template <class KT, bool VALS, int NT>
constexpr int block_sort_min_blocks() {
  return sizeof(typename KT::T) > 8   ? 512 / NT
         : VALS                        ? 1024 / NT
         : sizeof(typename KT::T) == 4 ? 2048 / NT
                                       : 1024 / NT;
}

// Interior copy by the LSU: 16-byte vector loads, all threads (the peer-
// memory loader: NVLink reads of mapped peer pointers are plain LDG.128).
// Four loads are issued before their stores so each thread keeps four
// NVLink reads in flight (peer LDG latency is ~1 us; B300_MICROARCH.md).
template <int NT>
__device__ __forceinline__ void lsu_copy16(char *smem, const char *g, uint32_t bytes,
                                           int tid) {
  const uint4 *src = reinterpret_cast<const uint4 *>(g);
  uint4 *dst = reinterpret_cast<uint4 *>(smem);
  const uint32_t n = bytes / 16;
  uint32_t q = tid;
  for (; q + 3 * NT < n; q += 4 * NT) {
    const uint4 v0 = src[q], v1 = src[q + NT], v2 = src[q + 2 * NT], v3 = src[q + 3 * NT];
    dst[q] = v0;
    dst[q + NT] = v1;
    dst[q + 2 * NT] = v2;
    dst[q + 3 * NT] = v3;
  }
  for (; q < n; q += NT)
    dst[q] = src[q];
}

// The half of K2 after the tile's windows are staged in smem (A at oA, B at
// oB, values at oAv/oBv; sentinels behind both windows when SENT): split the
// window among the threads by a diagonal search in smem, merge VT outputs per
// thread, then fold them into the checksum (SINK) or stage them in smem and
// write out[win.o0, win.o0 + na + nb) back (one bulk store when aligned).
// Shared by merge_tiles_kernel and the piece-list merge (mp_pieces.cuh).
template <class KT, bool VALS, int NT, int VT, bool SINK, bool SENT>
__device__ __forceinline__ void merge_staged_window(
    char *smem, const TileWin &win, uint32_t oA, uint32_t oB, uint32_t oAv, uint32_t oBv,
    typename KT::T *__restrict__ out, uint32_t *__restrict__ outv,
    unsigned long long *__restrict__ sum) {
  using T = typename KT::T;
  constexpr uint32_t KS = sizeof(T);
  const int tid = threadIdx.x;
  const int na_t = win.na, nb_t = win.nb, total = na_t + nb_t;
  // --- split the window among threads: diagonal search in smem ---
  const int diag = min(tid * VT, total);
  int lo = diag > nb_t ? diag - nb_t : 0;
  int hi = diag < na_t ? diag : na_t;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (take_b<KT>(lds<T>(smem, oB + (diag - 1 - mid) * KS),
                   lds<T>(smem, oA + mid * KS)))
      hi = mid;
    else
      lo = mid + 1;
  }
  int i = lo, j = diag - lo;

  // --- serial stable merge of VT outputs (core.hpp:166-176), branchless:
  //     one predicated choice and ONE smem load (the consumed side's next
  //     element) per output.  Reads may run one element past a window
  //     (into the next window or the slack) but are never used. ---
  T keys[VT];
  uint32_t vals[VT];
  serial_merge<KT, VT, VALS, SENT>(smem, oA, na_t, oB, nb_t, oAv, oBv, i, j, keys,
                                   vals);
  if constexpr (SINK) {
    unsigned long long acc = 0;
#pragma unroll
    for (int k = 0; k < VT; ++k)
      if (diag + k < total)
        acc += (win.o0 + diag + k + 1) * mix64_dev(key_of(keys[k]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
      acc += __shfl_xor_sync(0xffffffffu, acc, off);
    __shared__ unsigned long long warp_sums[NT / 32];
    if ((tid & 31) == 0)
      warp_sums[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      unsigned long long s = 0;
#pragma unroll
      for (int w = 0; w < NT / 32; ++w)
        s += warp_sums[w];
      atomicAdd(sum, s);
    }
    return;
  }
  __syncthreads();  // all windows consumed; reuse smem for output staging

  constexpr uint32_t oS = 16;
  constexpr uint32_t oSv = (oS + stage_elems<NT, VT>() * KS + 15u) & ~15u;
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    *reinterpret_cast<T *>(smem + oS + stage_idx<VT>(tid * VT + k) * KS) = keys[k];
    if constexpr (VALS)
      *reinterpret_cast<uint32_t *>(smem + oSv + stage_idx<VT>(tid * VT + k) * 4) = vals[k];
  }

  T *dst = out + win.o0;
  uint32_t *dstv = VALS ? outv + win.o0 : nullptr;
  const bool bulk_ok =
      (VT & 1) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) &&
      ((static_cast<uint32_t>(total) * KS) % 16 == 0) &&
      (!VALS || (((reinterpret_cast<uintptr_t>(dstv) & 15) == 0) &&
                 (static_cast<uint32_t>(total) * 4) % 16 == 0));
  if (bulk_ok) {
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      bulk_s2g(dst, smem + oS, static_cast<uint32_t>(total) * KS);
      if constexpr (VALS)
        bulk_s2g(dstv, smem + oSv, static_cast<uint32_t>(total) * 4);
      bulk_commit();
      bulk_wait_read0();
    }
  } else {
    __syncthreads();
    for (int q = tid; q < total; q += NT) {
      dst[q] = lds<T>(smem, oS + stage_idx<VT>(q) * KS);
      if constexpr (VALS)
        dstv[q] = lds<uint32_t>(smem, oSv + stage_idx<VT>(q) * 4);
    }
  }
}

// K2: one CTA per tile.  The window interiors arrive through the bulk-copy
// engine (TMA, cp.async.bulk) on an mbarrier; windows in another GPU's
// memory are the piece-list merge's job (mp_pieces.cuh).
template <class KT, bool VALS, int NT, int VT, class Map, bool SINK = false>
__global__ void __launch_bounds__(NT, (merge_min_blocks<KT, VALS, NT, SINK>()))
    merge_tiles_kernel(Map map, const typename KT::T *__restrict__ a,
                       const uint32_t *__restrict__ av,
                       const typename KT::T *__restrict__ b,
                       const uint32_t *__restrict__ bv,
                       typename KT::T *__restrict__ out,
                       uint32_t *__restrict__ outv,
                       unsigned long long *__restrict__ sum = nullptr,
                       uint64_t tile0 = 0) {
  using T = typename KT::T;
  constexpr uint32_t KS = sizeof(T);
  extern __shared__ __align__(128) char smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  const int tid = threadIdx.x;

  TileWin win;
  if constexpr (map_searches<Map>::value) {
    __shared__ unsigned long long split[2];
    if (tid < 64) {  // warp 0: the tile's start diagonal, warp 1: its end
      const int w = tid >> 5;
      const uint64_t sp = map.template split<KT>(a, b, tile0 + blockIdx.x, w, tid & 31);
      if ((tid & 31) == 0)
        split[w] = sp;
    }
    __syncthreads();
    win = map.window(tile0 + blockIdx.x, split[0], split[1]);
  } else {
    win = map.window(tile0 + blockIdx.x);
  }
  const int na_t = win.na, nb_t = win.nb;

  // --- smem layout (byte offsets): each window congruent mod 16 to its
  //     global source, so its 16 B-aligned interior is one bulk copy ---
  const char *gA = reinterpret_cast<const char *>(a + win.a0);
  const char *gB = reinterpret_cast<const char *>(b + win.b0);
  const uint32_t bA = na_t * KS, bB = nb_t * KS;
  constexpr bool SENT = merge_sentinels<KT, VALS>();
  const uint32_t oA = mirror_off(16, gA);
  const uint32_t oB = mirror_off(oA + bA + (SENT ? VT * KS : 0), gB);
  const char *gAv = nullptr, *gBv = nullptr;
  uint32_t oAv = 0, oBv = 0;
  if constexpr (VALS) {
    gAv = reinterpret_cast<const char *>(av + win.a0);
    gBv = reinterpret_cast<const char *>(bv + win.b0);
    oAv = mirror_off(oB + bB, gAv);
    oBv = mirror_off(oAv + na_t * 4, gBv);
  }

  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    uint32_t loA, loB, loAv = 0, loBv = 0;
    const uint32_t iA = interior_bytes(gA, bA, &loA);
    const uint32_t iB = interior_bytes(gB, bB, &loB);
    uint32_t iAv = 0, iBv = 0;
    if constexpr (VALS) {
      iAv = interior_bytes(gAv, na_t * 4, &loAv);
      iBv = interior_bytes(gBv, nb_t * 4, &loBv);
    }
    mbar_arrive_expect_tx(bar, iA + iB + iAv + iBv);
    if (iA)
      bulk_g2s(smem + oA + loA, gA + loA, iA, bar);
    if (iB)
      bulk_g2s(smem + oB + loB, gB + loB, iB, bar);
    if constexpr (VALS) {
      if (iAv)
        bulk_g2s(smem + oAv + loAv, gAv + loAv, iAv, bar);
      if (iBv)
        bulk_g2s(smem + oBv + loBv, gBv + loBv, iBv, bar);
    }
  }
  // unaligned heads/tails: warp 0 takes A, warp 1 takes B (values: 2, 3)
  {
    const int w = tid >> 5, l = tid & 31;
    static_assert(NT >= 128, "edge staging uses warps 0..3");
    if (w == 0)
      stage_edges<KS>(smem, oA, gA, bA, l);
    else if (w == 1)
      stage_edges<KS>(smem, oB, gB, bB, l);
    if constexpr (VALS) {
      if (w == 2)
        stage_edges<4>(smem, oAv, gAv, na_t * 4, l);
      else if (w == 3)
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

  merge_staged_window<KT, VALS, NT, VT, SINK, SENT>(smem, win, oA, oB, oAv, oBv, out, outv,
                                                    sum);
}

// ---------------------------------------------------------------------------
// K3: stable block sort of NV = NT*VT keys per CTA.
// 1) each thread sorts its VT keys in registers: an odd-even transposition
//    network with strict swaps (stable; needed when values or the element
//    tag are visible), or a Batcher odd-even merge network of min/max for
//    bare keys (equal bare keys are indistinguishable, so the bytes are the
//    same as a stable sort's);
// 2) log2(NT) Merge Path passes in smem: each thread finds its split on its
//    pair's cross diagonal and merges VT outputs branch-free.
// smem index p is padded to p + p/32, which spreads the stride-VT and
// stride-VT/2 access patterns over all 32 banks.  A short last block is
// padded with the maximum key; padding sits at the highest positions, so
// stability keeps it behind every real key.
// ---------------------------------------------------------------------------
template <class KT, bool VALS, int NT, int VT>
__host__ __device__ constexpr uint32_t block_sort_smem_bytes() {
  using T = typename KT::T;
  constexpr uint32_t E = NT * VT + (NT * VT) / 32;
  // + one element of read slack past each array (fast merge path)
  return ((E * sizeof(T) + 15) & ~15u) + (VALS ? E * 4 : 0) + 64;
}

template <class KT>
__device__ __forceinline__ void ce_minmax(typename KT::T &x, typename KT::T &y) {
  const bool sw = KT::less(y, x);
  const typename KT::T lo = sw ? y : x;
  y = sw ? x : y;
  x = lo;
}

// Batcher odd-even merge sort network on a register array (n = power of 2).
template <class KT, int N>
__device__ __forceinline__ void batcher_sort(typename KT::T (&x)[N]) {
#pragma unroll
  for (int p = 1; p < N; p <<= 1) {
#pragma unroll
    for (int k = p; k >= 1; k >>= 1) {
#pragma unroll
      for (int j = k % p; j + k < N; j += 2 * k) {
#pragma unroll
        for (int i = 0; i < k; ++i) {
          if (i + j + k < N && (i + j) / (2 * p) == (i + j + k) / (2 * p))
            ce_minmax<KT>(x[i + j], x[i + j + k]);
        }
      }
    }
  }
}

template <class KT, bool VALS, int NT, int VT>
__global__ void __launch_bounds__(NT, (block_sort_min_blocks<KT, VALS, NT>()))
    block_sort_kernel(const typename KT::T *__restrict__ in,
                      const uint32_t *__restrict__ inv,
                      typename KT::T *__restrict__ out,
                      uint32_t *__restrict__ outv, uint64_t n) {
  using T = typename KT::T;
  constexpr int NV = NT * VT;
  constexpr uint32_t KS = sizeof(T);
  constexpr int E = NV + NV / 32;
  constexpr uint32_t oV = (E * KS + 15) & ~15u;  // values after keys
  constexpr bool kStable = VALS || KT::kind == kElement;
  extern __shared__ __align__(128) char smem[];
  const int tid = threadIdx.x;
  const uint64_t base = uint64_t(blockIdx.x) * NV;
  const int cnt = static_cast<int>((n - base) < NV ? (n - base) : NV);
  auto sk = [&](int p) -> T & {
    return *reinterpret_cast<T *>(smem + (p + (p >> 5)) * KS);
  };
  auto sv = [&](int p) -> uint32_t & {
    return *reinterpret_cast<uint32_t *>(smem + oV + (p + (p >> 5)) * 4);
  };

  for (int q = tid; q < NV; q += NT) {
    sk(q) = q < cnt ? in[base + q] : KT::max_key();
    if constexpr (VALS)
      sv(q) = q < cnt ? inv[base + q] : 0u;
  }
  __syncthreads();

  T x[VT];
  uint32_t v[VT];
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    x[k] = sk(tid * VT + k);
    if constexpr (VALS)
      v[k] = sv(tid * VT + k);
  }
  if constexpr (kStable) {
#pragma unroll
    for (int pass = 0; pass < VT; ++pass) {
#pragma unroll
      for (int k = pass & 1; k + 1 < VT; k += 2) {
        const bool sw = KT::less(x[k + 1], x[k]);
        const T lo = sw ? x[k + 1] : x[k];
        x[k + 1] = sw ? x[k] : x[k + 1];
        x[k] = lo;
        if constexpr (VALS) {
          const uint32_t lv = sw ? v[k + 1] : v[k];
          v[k + 1] = sw ? v[k] : v[k + 1];
          v[k] = lv;
        }
      }
    }
  } else {
    batcher_sort<KT, VT>(x);
  }

#pragma unroll 1
  for (int width = VT; width < NV; width *= 2) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      sk(tid * VT + k) = x[k];
      if constexpr (VALS)
        sv(tid * VT + k) = v[k];
    }
    __syncthreads();
    const int gs = (tid * VT) & ~(2 * width - 1);
    const int diag = tid * VT - gs;
    const int A0 = gs, B0 = gs + width;
    int lo = diag > width ? diag - width : 0;
    int hi = diag < width ? diag : width;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (take_b<KT>(sk(B0 + diag - 1 - mid), sk(A0 + mid)))
        hi = mid;
      else
        lo = mid + 1;
    }
    int i = lo, j = diag - lo;
    // (a bounds-free fast path like serial_merge's was measured slower here,
    //  both with an unrolled and with a rolled slow path: 8.3 -> 11.0 ms)
    {
      T ka = sk(A0 + min(i, width - 1));
      T kb = sk(B0 + min(j, width - 1));
#pragma unroll
      for (int k = 0; k < VT; ++k) {
        const bool tb = (j < width) && ((i >= width) || take_b<KT>(kb, ka));
        x[k] = tb ? kb : ka;
        if constexpr (VALS)
          v[k] = sv(tb ? B0 + j : A0 + i);
        i += tb ? 0 : 1;
        j += tb ? 1 : 0;
        const T nxt = sk(tb ? B0 + min(j, width - 1) : A0 + min(i, width - 1));
        kb = tb ? nxt : kb;
        ka = tb ? ka : nxt;
      }
    }
  }

  __syncthreads();
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    sk(tid * VT + k) = x[k];
    if constexpr (VALS)
      sv(tid * VT + k) = v[k];
  }
  __syncthreads();
  for (int q = tid; q < cnt; q += NT) {
    out[base + q] = sk(q);
    if constexpr (VALS)
      outv[base + q] = sv(q);
  }
}

}  // namespace mpb

namespace mpb {

// ---------------------------------------------------------------------------
// Statistics of the Segmented Parallel Merge schedule (parallel.hpp:90-145,
// :262-292), computed on the device so drop-in callers get the reference's
// exact counters.  Window k starts on global diagonal k*L (the reference
// proves this equivalence, test_parallel.cpp:120-137), with its start split
// in starts_a[k].  Thread (k, r): r < p_eff replays worker r's window-local
// search; r == p_eff replays plan_segments' end-of-window search.
// ---------------------------------------------------------------------------
template <class KT>
__global__ void segment_stats_kernel(const typename KT::T *__restrict__ a,
                                     uint64_t na,
                                     const typename KT::T *__restrict__ b,
                                     uint64_t nb, uint64_t L, uint64_t p_eff,
                                     uint64_t iters,
                                     const uint64_t *__restrict__ starts_a,
                                     unsigned long long *__restrict__ plan_cmp,
                                     unsigned long long *__restrict__ merge_cmp) {
  const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  const uint64_t k = idx / (p_eff + 1), r = idx % (p_eff + 1);
  if (k >= iters)
    return;
  const uint64_t n = na + nb;
  const uint64_t d0 = k * L;
  const uint64_t ca = starts_a[k], cb = d0 - ca;
  const uint64_t rest = n - d0;
  const uint64_t Lw = L < rest ? L : rest;
  const uint64_t sna = Lw < na - ca ? Lw : na - ca;
  const uint64_t snb = Lw < nb - cb ? Lw : nb - cb;
  uint32_t c = 0;
  if (r == p_eff) {
    if (k + 1 == iters)
      return;
    diag_search_global<KT>(a + ca, sna, b + cb, snb, Lw, &c);
    if (c)
      atomicAdd(plan_cmp, static_cast<unsigned long long>(c));
  } else {
    const uint64_t pw = p_eff < Lw ? p_eff : Lw;
    if (r >= pw)
      return;
    const uint64_t dl = (r * Lw) / pw;
    diag_search_global<KT>(a + ca, sna, b + cb, snb, dl, &c);
    if (c)
      atomicAdd(merge_cmp, static_cast<unsigned long long>(c));
  }
}

}  // namespace mpb
