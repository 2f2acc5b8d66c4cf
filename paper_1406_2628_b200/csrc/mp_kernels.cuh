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

// Point t sits on diagonal min(t*spacing, N) (tile mode, p == 0) or on
// floor(t*N/p) (p-way mode, core.hpp:90-92).  Writes a_off for t < count.
template <class KT>
__global__ void partition_kernel(const typename KT::T *__restrict__ a,
                                 uint64_t na,
                                 const typename KT::T *__restrict__ b,
                                 uint64_t nb, uint64_t spacing, uint64_t p,
                                 uint64_t count, uint64_t *__restrict__ a_offs,
                                 unsigned long long *__restrict__ cmp = nullptr) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
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
  uint32_t c = 0;
  a_offs[t] = diag_search_global<KT>(a, na, b, nb, d, &c);
  if (cmp && c)  // comparison count of the reference's search (core.hpp:128)
    atomicAdd(cmp, static_cast<unsigned long long>(c));
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

// One bottom-up round over runs of `width` (sort.hpp:71-101): pair k merges
// A = src[2kw, 2kw+w) with B = src[2kw+w, 2kw+2w) (clipped to n); an
// unpaired tail run has an empty B and is copied.  NV divides 2w, so a tile
// never straddles two pairs.  P[t] = a_off (pair-local) at the tile start.
struct RoundMap {
  const uint64_t *P;
  uint64_t n;
  uint64_t width;
  uint32_t nv;
  __device__ __forceinline__ TileWin window(uint64_t t) const {
    const uint64_t d0 = t * nv;
    const uint64_t s = (d0 / (2 * width)) * (2 * width);
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

// K4: pair-local a_off at the start of every tile of one round.
template <class KT>
__global__ void round_partition_kernel(const typename KT::T *__restrict__ src,
                                       uint64_t n, uint64_t width,
                                       uint32_t nv, uint64_t tiles,
                                       uint64_t *__restrict__ P) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= tiles)
    return;
  const uint64_t d0 = t * nv;
  const uint64_t s = (d0 / (2 * width)) * (2 * width);
  const uint64_t la = (n - s) < width ? (n - s) : width;
  const uint64_t rest = n - s - la;
  const uint64_t lb = rest < width ? rest : width;
  P[t] = diag_search_global<KT>(src + s, la, src + s + la, lb, d0 - s);
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

template <class KT, bool VALS, int NT, int VT>
__host__ __device__ constexpr uint32_t merge_smem_bytes() {
  using T = typename KT::T;
  constexpr uint32_t NV = NT * VT;
  constexpr uint32_t in_bytes =
      NV * sizeof(T) + 48 + (VALS ? NV * 4 + 48 : 0);
  constexpr uint32_t st_bytes =
      stage_elems<NT, VT>() * sizeof(T) + 16 +
      (VALS ? stage_elems<NT, VT>() * 4 + 16 : 0);
  return 16 + (in_bytes > st_bytes ? in_bytes : st_bytes);
}

__device__ __forceinline__ char *align16p(char *p) {
  return reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(p) + 15) &
                                  ~uintptr_t(15));
}

// Copy the unaligned head [0, lo) and tail [hi, bytes) of a staged range
// with ordinary loads, ES bytes at a time (ES divides 16 and the range).
template <int ES, int NT>
__device__ __forceinline__ void copy_edges(const ByteRange &r, uint32_t lo,
                                           uint32_t hi) {
  using W = typename std::conditional<
      ES == 4, uint32_t,
      typename std::conditional<ES == 8, unsigned long long, int4>::type>::type;
  for (uint32_t o = threadIdx.x * ES; o < lo; o += NT * ES)
    *reinterpret_cast<W *>(r.dst + o) =
        __ldg(reinterpret_cast<const W *>(r.src + o));
  for (uint32_t o = hi + threadIdx.x * ES; o < r.bytes; o += NT * ES)
    *reinterpret_cast<W *>(r.dst + o) =
        __ldg(reinterpret_cast<const W *>(r.src + o));
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

// SINK = the register-sink mode (parallel.hpp:181-198): nothing is stored;
// each thread folds (pos+1)*mix64(key) over its outputs and the CTA adds its
// partial sum into *sum.
template <class KT, bool VALS, int NT, int VT, class Map, bool SINK = false>
__global__ void __launch_bounds__(NT)
    merge_tiles_kernel(Map map, const typename KT::T *__restrict__ a,
                       const uint32_t *__restrict__ av,
                       const typename KT::T *__restrict__ b,
                       const uint32_t *__restrict__ bv,
                       typename KT::T *__restrict__ out,
                       uint32_t *__restrict__ outv,
                       unsigned long long *__restrict__ sum = nullptr) {
  using T = typename KT::T;
  constexpr int KS = sizeof(T);
  extern __shared__ __align__(128) char smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  char *base = smem + 16;
  const int tid = threadIdx.x;

  const TileWin win = map.window(blockIdx.x);
  const int na_t = win.na, nb_t = win.nb, total = na_t + nb_t;

  // --- smem layout: each window congruent (mod 16) to its global source ---
  ByteRange rg[4];
  int nr = 2;
  rg[0].src = reinterpret_cast<const char *>(a + win.a0);
  rg[0].bytes = static_cast<uint32_t>(na_t) * KS;
  rg[0].dst = base + (reinterpret_cast<uintptr_t>(rg[0].src) & 15);
  rg[1].src = reinterpret_cast<const char *>(b + win.b0);
  rg[1].bytes = static_cast<uint32_t>(nb_t) * KS;
  rg[1].dst = align16p(rg[0].dst + rg[0].bytes) +
              (reinterpret_cast<uintptr_t>(rg[1].src) & 15);
  if constexpr (VALS) {
    nr = 4;
    rg[2].src = reinterpret_cast<const char *>(av + win.a0);
    rg[2].bytes = static_cast<uint32_t>(na_t) * 4;
    rg[2].dst = align16p(rg[1].dst + rg[1].bytes) +
                (reinterpret_cast<uintptr_t>(rg[2].src) & 15);
    rg[3].src = reinterpret_cast<const char *>(bv + win.b0);
    rg[3].bytes = static_cast<uint32_t>(nb_t) * 4;
    rg[3].dst = align16p(rg[2].dst + rg[2].bytes) +
                (reinterpret_cast<uintptr_t>(rg[3].src) & 15);
  }

  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    uint32_t tx = 0, lo, hi;
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (r < nr)
        tx += bulk_interior(rg[r], &lo, &hi);
    mbar_arrive_expect_tx(bar, tx);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (r < nr && bulk_interior(rg[r], &lo, &hi))
        bulk_g2s(rg[r].dst + lo, rg[r].src + lo, hi - lo, bar);
    }
  }
  {
    uint32_t lo, hi;
    bulk_interior(rg[0], &lo, &hi);
    copy_edges<KS, NT>(rg[0], lo, hi);
    bulk_interior(rg[1], &lo, &hi);
    copy_edges<KS, NT>(rg[1], lo, hi);
    if constexpr (VALS) {
      bulk_interior(rg[2], &lo, &hi);
      copy_edges<4, NT>(rg[2], lo, hi);
      bulk_interior(rg[3], &lo, &hi);
      copy_edges<4, NT>(rg[3], lo, hi);
    }
  }
  __syncthreads();
  mbar_wait(bar, 0);

  const T *sA = reinterpret_cast<const T *>(rg[0].dst);
  const T *sB = reinterpret_cast<const T *>(rg[1].dst);

  // --- split the window among threads: diagonal search in smem ---
  const int diag = min(tid * VT, total);
  int lo = diag > nb_t ? diag - nb_t : 0;
  int hi = diag < na_t ? diag : na_t;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (take_b<KT>(sB[diag - 1 - mid], sA[mid]))
      hi = mid;
    else
      lo = mid + 1;
  }
  int i = lo, j = diag - lo;

  // --- serial stable merge of VT outputs (core.hpp:166-176) ---
  T keys[VT];
  uint32_t vals[VT];
  T ka = i < na_t ? sA[i] : T{};
  T kb = j < nb_t ? sB[j] : T{};
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    const bool tb = (j < nb_t) && ((i >= na_t) || take_b<KT>(kb, ka));
    keys[k] = tb ? kb : ka;
    if constexpr (VALS) {
      const uint32_t *sAv = reinterpret_cast<const uint32_t *>(rg[2].dst);
      const uint32_t *sBv = reinterpret_cast<const uint32_t *>(rg[3].dst);
      if (diag + k < total)
        vals[k] = tb ? sBv[j] : sAv[i];
    }
    if (tb) {
      ++j;
      if (j < nb_t)
        kb = sB[j];
    } else {
      ++i;
      if (i < na_t)
        ka = sA[i];
    }
  }
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

  T *stage = reinterpret_cast<T *>(base);
  uint32_t *stagev = reinterpret_cast<uint32_t *>(
      align16p(base + stage_elems<NT, VT>() * KS));
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    stage[stage_idx<VT>(tid * VT + k)] = keys[k];
    if constexpr (VALS)
      stagev[stage_idx<VT>(tid * VT + k)] = vals[k];
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
      bulk_s2g(dst, stage, static_cast<uint32_t>(total) * KS);
      if constexpr (VALS)
        bulk_s2g(dstv, stagev, static_cast<uint32_t>(total) * 4);
      bulk_commit();
      bulk_wait_read0();
    }
  } else {
    __syncthreads();
    for (int q = tid; q < total; q += NT) {
      dst[q] = stage[stage_idx<VT>(q)];
      if constexpr (VALS)
        dstv[q] = stagev[stage_idx<VT>(q)];
    }
  }
}

// ---------------------------------------------------------------------------
// K3: stable block sort of NV = NT*VT keys per CTA.
// Odd-even transposition inside each thread (strict swaps => stable), then
// log2(NT) Merge Path passes in smem.  Short last block is padded with the
// maximum key; padding sits at the highest positions so stability keeps it
// behind every real key.
// ---------------------------------------------------------------------------
template <class KT, bool VALS, int NT, int VT>
__host__ __device__ constexpr uint32_t block_sort_smem_bytes() {
  using T = typename KT::T;
  constexpr uint32_t E = NT * VT + (NT * VT) / 32;
  return E * sizeof(T) + 16 + (VALS ? E * 4 : 0);
}

template <class KT, bool VALS, int NT, int VT>
__global__ void __launch_bounds__(NT)
    block_sort_kernel(const typename KT::T *__restrict__ in,
                      const uint32_t *__restrict__ inv,
                      typename KT::T *__restrict__ out,
                      uint32_t *__restrict__ outv, uint64_t n) {
  using T = typename KT::T;
  constexpr int NV = NT * VT;
  constexpr int E = NV + NV / 32;
  extern __shared__ __align__(128) char smem[];
  T *sk = reinterpret_cast<T *>(smem);
  uint32_t *sv = reinterpret_cast<uint32_t *>(align16p(smem + E * sizeof(T)));
  const int tid = threadIdx.x;
  const uint64_t base = uint64_t(blockIdx.x) * NV;
  const int cnt = static_cast<int>((n - base) < NV ? (n - base) : NV);
  auto sidx = [](int p) { return p + (p >> 5); };

  for (int q = tid; q < NV; q += NT) {
    sk[sidx(q)] = q < cnt ? in[base + q] : KT::max_key();
    if constexpr (VALS)
      sv[sidx(q)] = q < cnt ? inv[base + q] : 0u;
  }
  __syncthreads();

  T x[VT];
  uint32_t v[VT];
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    x[k] = sk[sidx(tid * VT + k)];
    if constexpr (VALS)
      v[k] = sv[sidx(tid * VT + k)];
  }
#pragma unroll
  for (int pass = 0; pass < VT; ++pass) {
#pragma unroll
    for (int k = pass & 1; k + 1 < VT; k += 2) {
      if (KT::less(x[k + 1], x[k])) {
        const T t = x[k];
        x[k] = x[k + 1];
        x[k + 1] = t;
        if constexpr (VALS) {
          const uint32_t tv = v[k];
          v[k] = v[k + 1];
          v[k + 1] = tv;
        }
      }
    }
  }

#pragma unroll 1
  for (int width = VT; width < NV; width *= 2) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      sk[sidx(tid * VT + k)] = x[k];
      if constexpr (VALS)
        sv[sidx(tid * VT + k)] = v[k];
    }
    __syncthreads();
    const int gs = ((tid * VT) / (2 * width)) * (2 * width);
    const int diag = tid * VT - gs;
    const int A0 = gs, B0 = gs + width;
    int lo = diag > width ? diag - width : 0;
    int hi = diag < width ? diag : width;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (take_b<KT>(sk[sidx(B0 + diag - 1 - mid)], sk[sidx(A0 + mid)]))
        hi = mid;
      else
        lo = mid + 1;
    }
    int i = lo, j = diag - lo;
    T ka = sk[sidx(A0 + (i < width ? i : width - 1))];
    T kb = sk[sidx(B0 + (j < width ? j : width - 1))];
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      const bool tb = (j < width) && ((i >= width) || take_b<KT>(kb, ka));
      x[k] = tb ? kb : ka;
      if constexpr (VALS)
        v[k] = tb ? sv[sidx(B0 + j)] : sv[sidx(A0 + i)];
      if (tb) {
        ++j;
        if (j < width)
          kb = sk[sidx(B0 + j)];
      } else {
        ++i;
        if (i < width)
          ka = sk[sidx(A0 + i)];
      }
    }
  }

  __syncthreads();
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    sk[sidx(tid * VT + k)] = x[k];
    if constexpr (VALS)
      sv[sidx(tid * VT + k)] = v[k];
  }
  __syncthreads();
  for (int q = tid; q < cnt; q += NT) {
    out[base + q] = sk[sidx(q)];
    if constexpr (VALS)
      outv[base + q] = sv[sidx(q)];
  }
}

}  // namespace mpb
