// mp_quad.cuh -- two bottom-up merge rounds in one pass over HBM.
//
// Rounds r and r+1 of sort.hpp:71-128 merge, for every group of four runs
// R0..R3 of width w (group start S = 4gw, runs clipped to n):
//     X = merge(R0, R1), Y = merge(R2, R3)        (round r, ties to the left)
//     out = merge(X, Y)                            (round r+1, ties to X)
// with an unpaired tail run carried, exactly as two separate rounds would.
// The fused pass produces the same bytes without materialising X and Y:
//
// K4q (quad_partition_kernel): the merge path of (X, Y) is cut where it
//   crosses the grid lines x = kG and y = jG (G divides 2w).  A crossing at
//   x = kG is the element v = X[kG] (a diagonal search on R0/R1 gives its
//   split (a, kG - a)); the Y elements before it are those < v, i.e.
//   (lower_bound(R2, v), lower_bound(R3, v)).  A crossing at y = jG is
//   u = Y[jG] (diagonal search on R2/R3); the X elements before it are those
//   <= u (ties go to X): (upper_bound(R0, u), upper_bound(R1, u)).  Each
//   crossing is thus a 4-way split (i0, i1, i2, i3) of the group.  The
//   crossing at x = kG is preceded by ceil(y/G) y-crossings and vice versa,
//   which gives every crossing its slot in path order directly.
//   No grid line lies strictly inside a segment between consecutive
//   crossings, so a segment holds at most G elements of X and G of Y.
// K4r (quad_refine_kernel): the exact 4-way split at every tile boundary
//   t*T: find the segment holding it, then a nested Merge Path search inside
//   the segment (outer on X/Y, inner on R0/R1 and R2/R3 for X[x], Y[y]).
// K5e (quad_tile_kernel): one CTA per tile of exactly T outputs bulk-copies
//   its four run slices into smem, merges R0/R1 and R2/R3 (threads dealt to
//   X and Y by size), writes X and Y back over the windows, merges X with Y
//   and bulk-stores the tile.
// Both inner merges and the outer one use take_b (ties to the left
// operand), so the result is the two-round result byte for byte.
#pragma once

#include "mp_kernels.cuh"

namespace mpb {

struct QuadPt {
  unsigned long long i[4];  // consumed prefix of R0..R3 at the crossing
};

struct QuadGroup {
  uint64_t S;     // first element of the group
  uint64_t l[4];  // run lengths (0 past n)
};

__device__ __forceinline__ QuadGroup quad_group(uint64_t g, uint64_t n,
                                                uint64_t w) {
  QuadGroup q;
  q.S = g * 4 * w;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint64_t s = q.S + r * w;
    q.l[r] = s < n ? (n - s < w ? n - s : w) : 0;
  }
  return q;
}

// number of elements < v
template <class KT>
__device__ __forceinline__ uint64_t lower_bound_dev(const typename KT::T *a,
                                                    uint64_t n,
                                                    typename KT::T v) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (KT::less(a[mid], v))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// number of elements <= v
template <class KT>
__device__ __forceinline__ uint64_t upper_bound_dev(const typename KT::T *a,
                                                    uint64_t n,
                                                    typename KT::T v) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (KT::less(v, a[mid]))
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ uint64_t cdiv_dev(uint64_t a, uint64_t b) {
  return (a + b - 1) / b;
}

// K4q: one thread per grid line of a group; 4w/G = 1 << lshift lines per
// full group.  P[(g << lshift) + slot] = the crossing in path order.
template <class KT, uint32_t G>
__global__ void quad_partition_kernel(const typename KT::T *__restrict__ src,
                                      uint64_t n, uint64_t w, uint32_t lshift,
                                      uint64_t lines, QuadPt *__restrict__ P) {
  using T = typename KT::T;
  const uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (p >= lines)
    return;
  const uint64_t g = p >> lshift;
  const uint64_t u = p & ((uint64_t(1) << lshift) - 1);
  const QuadGroup q = quad_group(g, n, w);
  const T *R0 = src + q.S, *R1 = R0 + w, *R2 = R1 + w, *R3 = R2 + w;
  const uint64_t cx = cdiv_dev(q.l[0] + q.l[1], G);
  const uint64_t cy = cdiv_dev(q.l[2] + q.l[3], G);
  QuadPt pt;
  uint64_t slot;
  if (u < cx) {
    const uint64_t d = u * G;
    const uint64_t a = diag_search_grid<KT>(R0, q.l[0], R1, q.l[1], d);
    const uint64_t b = d - a;
    const bool from_b = b < q.l[1] && (a >= q.l[0] || take_b<KT>(R1[b], R0[a]));
    const T v = from_b ? R1[b] : R0[a];
    const uint64_t i2 = lower_bound_dev<KT>(R2, q.l[2], v);
    const uint64_t i3 = lower_bound_dev<KT>(R3, q.l[3], v);
    pt.i[0] = a;
    pt.i[1] = b;
    pt.i[2] = i2;
    pt.i[3] = i3;
    slot = u + cdiv_dev(i2 + i3, G);
  } else if (u - cx < cy) {
    const uint64_t j = u - cx, d = j * G;
    const uint64_t c = diag_search_grid<KT>(R2, q.l[2], R3, q.l[3], d);
    const uint64_t e = d - c;
    const bool from_b = e < q.l[3] && (c >= q.l[2] || take_b<KT>(R3[e], R2[c]));
    const T v = from_b ? R3[e] : R2[c];
    const uint64_t i0 = upper_bound_dev<KT>(R0, q.l[0], v);
    const uint64_t i1 = upper_bound_dev<KT>(R1, q.l[1], v);
    pt.i[0] = i0;
    pt.i[1] = i1;
    pt.i[2] = c;
    pt.i[3] = e;
    slot = j + cdiv_dev(i0 + i1, G);
  } else {
    return;  // the short last group has fewer lines
  }
  ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(P + (g << lshift) + slot);
  dst[0] = make_ulonglong2(pt.i[0], pt.i[1]);
  dst[1] = make_ulonglong2(pt.i[2], pt.i[3]);
}

// ---------------------------------------------------------------------------
// (Round 2: K4q's two bounds and K4r's two inner splits searched in lockstep
// -- independent loads of one step issued together -- K4q 70.5 -> 66 us,
// K4r 117 -> 130 us per pass: not kept.)
// K4r guess window (B200, 8 K4r launches of a 2^30 sort, ncu: 64 1061 us,
// 128 986, 256 906, 512 1047, 1024 1186; sort 27.37 ms at 128, 27.29 at 256)
#ifndef MP_K4R_GUESS_R
#define MP_K4R_GUESS_R 256
#endif
// K4r / K5e (see the header).  An earlier variant ran one CTA per segment
// (0..2G outputs, bimodal around G): half of every CTA idle, 3.48 ms per
// fused pass.
// ---------------------------------------------------------------------------

// element x of merge(R0[0..l0), R1[0..l1)) (ties to R0) and its split
template <class KT>
__device__ __forceinline__ typename KT::T merged_at(const typename KT::T *R0, uint64_t l0,
                                                    const typename KT::T *R1, uint64_t l1,
                                                    uint64_t x) {
  uint64_t lo = x > l1 ? x - l1 : 0, hi = x < l0 ? x : l0;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (take_b<KT>(R1[x - 1 - mid], R0[mid]))
      hi = mid;
    else
      lo = mid + 1;
  }
  const uint64_t b = x - lo;
  const bool from_b = b < l1 && (lo >= l0 || take_b<KT>(R1[b], R0[lo]));
  return from_b ? R1[b] : R0[lo];
}

// split of merge(R0, R1) at diagonal x, searched within [lo0, hi0]
template <class KT>
__device__ __forceinline__ uint64_t split_in(const typename KT::T *R0, uint64_t l0,
                                             const typename KT::T *R1, uint64_t l1,
                                             uint64_t x, uint64_t lo0, uint64_t hi0) {
  uint64_t lo = x > l1 ? x - l1 : 0, hi = x < l0 ? x : l0;
  lo = lo > lo0 ? lo : lo0;
  hi = hi < hi0 ? hi : hi0;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (take_b<KT>(R1[x - 1 - mid], R0[mid]))
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

template <class KT>
__device__ __forceinline__ typename KT::T elem_at_split(const typename KT::T *R0, uint64_t l0,
                                                        const typename KT::T *R1, uint64_t l1,
                                                        uint64_t x, uint64_t a) {
  const uint64_t b = x - a;
  const bool from_b = b < l1 && (a >= l0 || take_b<KT>(R1[b], R0[a]));
  return from_b ? R1[b] : R0[a];
}

template <class KT>
__device__ __forceinline__ uint64_t split_at(const typename KT::T *R0, uint64_t l0,
                                             const typename KT::T *R1, uint64_t l1,
                                             uint64_t x) {
  uint64_t lo = x > l1 ? x - l1 : 0, hi = x < l0 ? x : l0;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (take_b<KT>(R1[x - 1 - mid], R0[mid]))
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

// K4r: Q[t] = the 4-way split at output position t*T of the fused pass (T
// divides the group size 4w, so tiles never straddle groups).
template <class KT, uint32_t G>
__global__ void quad_refine_kernel(const typename KT::T *__restrict__ src, uint64_t n,
                                   uint64_t w, uint32_t lshift, uint32_t T,
                                   uint64_t tiles, const QuadPt *__restrict__ P,
                                   QuadPt *__restrict__ Q) {
  using T_ = typename KT::T;
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= tiles)
    return;
  const uint64_t pos = t * T;
  const uint64_t g = pos / (4 * w);
  const uint64_t dl = pos - g * 4 * w;  // group-local output position
  QuadPt out;
  if (dl == 0) {
    out.i[0] = out.i[1] = out.i[2] = out.i[3] = 0;
  } else {
    const QuadGroup q = quad_group(g, n, w);
    const T_ *R0 = src + q.S, *R1 = R0 + w, *R2 = R1 + w, *R3 = R2 + w;
    const uint64_t pts = q.S + 4 * w <= n
                             ? (uint64_t(1) << lshift)
                             : cdiv_dev(q.l[0] + q.l[1], G) + cdiv_dev(q.l[2] + q.l[3], G);
    const QuadPt *Pg = P + (g << lshift);
    auto diag = [&](uint64_t k) {
      const QuadPt &p = Pg[k];
      return p.i[0] + p.i[1] + p.i[2] + p.i[3];
    };
    // last crossing at or before dl (crossing 0 is at diagonal 0)
    uint64_t lo = 0, hi = pts - 1;
    while (lo < hi) {
      const uint64_t mid = (lo + hi + 1) >> 1;
      if (diag(mid) <= dl)
        lo = mid;
      else
        hi = mid - 1;
    }
    const QuadPt p0 = Pg[lo];
    QuadPt p1;
    if (lo + 1 < pts) {
      p1 = Pg[lo + 1];
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r)
        p1.i[r] = q.l[r];
    }
    // segment: X-part = merge(R0[p0.i0..p1.i0), R1[..)), Y-part likewise
    const T_ *A0 = R0 + p0.i[0], *A1 = R1 + p0.i[1], *B0 = R2 + p0.i[2], *B1 = R3 + p0.i[3];
    const uint64_t la0 = p1.i[0] - p0.i[0], la1 = p1.i[1] - p0.i[1];
    const uint64_t lb0 = p1.i[2] - p0.i[2], lb1 = p1.i[3] - p0.i[3];
    const uint64_t nx = la0 + la1, ny = lb0 + lb1;
    const uint64_t d = dl - (p0.i[0] + p0.i[1] + p0.i[2] + p0.i[3]);
    // outer Merge Path search on (X-part, Y-part) at diagonal d, ties to X.
    // The inner splits are monotone (a(x) non-decreasing in x, c(y) in y),
    // so every probe narrows the range the next inner searches scan.
    uint64_t xl = d > ny ? d - ny : 0, xh = d < nx ? d : nx;
    uint64_t aL = 0, aH = la0, cL = 0, cH = lb0;  // a(x) for x in [xl,xh]; c(y)
    // The first two probes go to the proportional guess +- R instead of
    // the midpoint (any probe in [xl, xh) keeps the bisection exact); for
    // random-order runs they leave a 257-wide range, ~6 probes fewer than
    // bisecting the whole segment.  B200: see DESIGN.md.
    const uint64_t guess =
        nx + ny ? static_cast<uint64_t>(static_cast<float>(d) * static_cast<float>(nx) /
                                        static_cast<float>(nx + ny))
                : 0;
    int it = 0;
    while (xl < xh) {
      uint64_t x = xl + ((xh - xl) >> 1);
      if (it < 2 && xh - xl > 4 * MP_K4R_GUESS_R) {
        const uint64_t t = it == 0 ? (guess > MP_K4R_GUESS_R ? guess - MP_K4R_GUESS_R : 0)
                                   : guess + MP_K4R_GUESS_R;
        if (t >= xl && t < xh)
          x = t;
      }
      ++it;
      const uint64_t y = d - 1 - x;
      const uint64_t ax = split_in<KT>(A0, la0, A1, la1, x, aL, aH);
      const uint64_t cy = split_in<KT>(B0, lb0, B1, lb1, y, cL, cH);
      const T_ xv = elem_at_split<KT>(A0, la0, A1, la1, x, ax);
      const T_ yv = elem_at_split<KT>(B0, lb0, B1, lb1, y, cy);
      if (take_b<KT>(yv, xv)) {
        xh = x;  // answer <= x: a(answer) <= a(x), y grows: c >= c(y)
        aH = ax;
        cL = cy;
      } else {
        xl = x + 1;  // answer > x: a >= a(x), y(answer) <= d-2-x < y: c <= c(y)
        aL = ax;
        cH = cy + 1 < lb0 ? cy + 1 : lb0;
      }
    }
    const uint64_t x = xl, y = d - xl;
    const uint64_t a = split_in<KT>(A0, la0, A1, la1, x, aL, aH);
    const uint64_t c = split_in<KT>(B0, lb0, B1, lb1, y, cL, cH);
    out.i[0] = p0.i[0] + a;
    out.i[1] = p0.i[1] + (x - a);
    out.i[2] = p0.i[2] + c;
    out.i[3] = p0.i[3] + (y - c);
  }
  ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(Q + t);
  dst[0] = make_ulonglong2(out.i[0], out.i[1]);
  dst[1] = make_ulonglong2(out.i[2], out.i[3]);
}

// K5e: one CTA per tile of T outputs (NT*VT >= T + 2*VT).  Phase 1 deals
// ceil(nx/VT) threads to X = merge(R0w, R1w) and the rest to Y; both are
// written over their input windows; phase 2 merges X with Y.
// Every merge runs bounds-free on sentinels (serial_merge SENT, as K2):
// VT copies of the largest key behind each A-side window (R0w, R2w, then
// X) and one behind each B-side window (R1w, R3w, then Y).  The group of a
// tile is pos >> lg4w (4w is a power of two).  B200 source counters before
// (tools/ncu_src_capture.sh): 57.2 instructions per element, of which 6.8
// in warp 0's 64-bit window setup and 5.6 in bounds-checked tail merges.
template <class KT, int VT>
__host__ __device__ constexpr uint32_t quad_gap_bytes() {
  return (VT + 1) * sizeof(typename KT::T) + 16;
}
template <class KT, int NT, int VT>
__host__ __device__ constexpr uint32_t quad_smem_bytes() {
  return 64 + NT * VT * sizeof(typename KT::T) + 4 * quad_gap_bytes<KT, VT>() + 64;
}

// K5e's split searches start from the
// proportional guess d * na / (na + nb) with a +-2^W window.  Two probes
// (at the window's edges, issued together) check that the split lies
// inside it -- a* >= lo0 iff lo0 is the range start or pred(lo0 - 1) is
// false, a* <= hi0 iff hi0 is the range end or pred(hi0) is true -- and a
// binary search of ~W+1 steps finishes it; otherwise the full search runs.
// Random-order merges deviate from the guess by O(sqrt(n)), so the window
// usually holds; skewed inputs just take the fallback.  B200 (whole 2^30
// sort): off 28.16 ms, window 2^5 28.59, 2^6 27.90-28.0, 2^7 28.06.
// Round 2 (tools/ab_k5e_spec.sh, 2^30 sort 25.79 ms): neither fewer nor more
// shared-memory loads per search helped -- bisecting inside the window first
// and probing an edge only when the answer lands on it (4 of ~18 loads less,
// the same in K3w's passes) 27.34 ms (K5e 2.09 -> 2.25 ms, K3w 7.63 -> 7.86);
// probing the first one / two bisection levels together with the edges (one /
// two dependent round trips less) 26.00 / 26.62 ms.  The same lazy edge
// probes with the window recomputed after the loop (no extra live
// registers): 25.74 ms, within noise of 25.79.  The window search as 7
// unrolled binary-lifting steps with predicated probes (no loop counter or
// branch, ~55 instructions less per search): 27.39 ms.
#ifndef MP_QUAD_PRED_LOGW
#define MP_QUAD_PRED_LOGW 6
#endif
template <class KT, int LOGW>
__device__ __forceinline__ int split_predicted(const char *smem, uint32_t oA, int na,
                                               uint32_t oB, int nb, int d, float ratio) {
  using T = typename KT::T;
  constexpr uint32_t KS = sizeof(T);
  const int lo = d > nb ? d - nb : 0;
  const int hi = d < na ? d : na;
  auto pred = [&](int m) {  // take B at A index m on diagonal d
    return take_b<KT>(lds<T>(smem, oB + (d - 1 - m) * KS), lds<T>(smem, oA + m * KS));
  };
  int l = lo, h = hi;
  if (hi - lo > (2 << LOGW)) {
    const int guess = min(max(__float2int_rn(static_cast<float>(d) * ratio), lo), hi);
    const int lo0 = max(lo, guess - (1 << LOGW)), hi0 = min(hi, guess + (1 << LOGW));
    const bool ok_lo = lo0 == lo || !pred(lo0 - 1);
    const bool ok_hi = hi0 == hi || pred(hi0);
    if (ok_lo && ok_hi) {
      l = lo0;
      h = hi0;
    }
  }
  while (l < h) {
    const int mid = (l + h) >> 1;
    if (pred(mid))
      h = mid;
    else
      l = mid + 1;
  }
  return l;
}

// A fused-pass tile's four run windows into smem at kWin0 (K5e's
// prologue).  The windows travel as whole 16-byte granules: one bulk copy
// per window covers its unaligned head and tail too (the extra bytes land
// in the gap before the window and in its sentinel area, which is written
// after the copy), so thread 0's setup is one dependent load (the split
// points) and the copy issue -- no edge loads.  Only where a granule would
// leave the array (its first / last window) are those < 16 bytes read by
// plain loads.  The other threads wait on the mbarrier for the copies and
// the header; one barrier at the end orders the sentinel stores.  Returns
// the windows' offsets and lengths and the tile's first output position.
struct QuadTileHdr {
  uint32_t oW[4];
  int cnt[4];
  unsigned long long o0;
};

template <class KT, int VT>
__device__ __forceinline__ void quad_load_tile(char *smem, const typename KT::T *__restrict__ src,
                                               uint64_t n, uint64_t w, uint32_t lg4w, uint32_t T,
                                               const QuadPt *__restrict__ Q, uint32_t (&oW)[4],
                                               int (&cnt)[4], uint64_t &o0) {
  using T_ = typename KT::T;
  constexpr uint32_t KS = sizeof(T_);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  QuadTileHdr *hdr = reinterpret_cast<QuadTileHdr *>(smem + 16);
  constexpr uint32_t kWin0 = 64;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uintptr_t arr_lo = reinterpret_cast<uintptr_t>(src);
  const uintptr_t arr_hi = reinterpret_cast<uintptr_t>(src + n);
  if (tid == 0) {
    const uint64_t t = blockIdx.x;
    const uint64_t pos = t * T;
    // 4w is a power of two after K3w's runs (lg4w < 64); otherwise divide
    const uint64_t g = lg4w < 64 ? (pos >> lg4w) : pos / (4 * w);
    const QuadGroup q = quad_group(g, n, w);
    const QuadPt p0 = Q[t];
    QuadPt p1;
    const uint64_t gend = q.S + q.l[0] + q.l[1] + q.l[2] + q.l[3];
    if (pos + T < gend) {
      p1 = Q[t + 1];
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r)
        p1.i[r] = q.l[r];
    }
    uint32_t at = kWin0, tx = 0;
    uintptr_t wa[4], wb[4];
    uint32_t oW[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int c = static_cast<int>(p1.i[r] - p0.i[r]);
      const uintptr_t s0 = reinterpret_cast<uintptr_t>(src + q.S + r * w + p0.i[r]);
      const uintptr_t e0 = s0 + c * KS;
      oW[r] = mirror_off(at, reinterpret_cast<const void *>(s0));
      at = oW[r] + c * KS + quad_gap_bytes<KT, VT>();
      uintptr_t a = s0 & ~uintptr_t(15), b = (e0 + 15) & ~uintptr_t(15);
      if (a < arr_lo)
        a = (s0 + 15) & ~uintptr_t(15);
      if (b > arr_hi)
        b = e0 & ~uintptr_t(15);
      if (!c || b <= a)
        a = b = 0;
      wa[r] = a;
      wb[r] = b;
      tx += static_cast<uint32_t>(b - a);
      hdr->oW[r] = oW[r];
      hdr->cnt[r] = c;
    }
    hdr->o0 = pos;
    mbar_arrive_expect_tx(bar, tx);
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (wb[r] > wa[r]) {
        const uintptr_t s0 = reinterpret_cast<uintptr_t>(src + q.S + r * w + p0.i[r]);
        bulk_g2s(smem + oW[r] - static_cast<uint32_t>(s0 - wa[r]),
                 reinterpret_cast<const void *>(wa[r]), static_cast<uint32_t>(wb[r] - wa[r]), bar);
      }
  }
  mbar_wait(bar, 0);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    oW[r] = hdr->oW[r];
    cnt[r] = hdr->cnt[r];
  }
  o0 = hdr->o0;
  {
    const int w_ = tid >> 5, l = tid & 31;
    if (w_ == 0) {  // sentinels behind the windows (after the copies landed)
      for (int k = l; k <= VT; k += 32) {
        if (k < VT) {
          *reinterpret_cast<T_ *>(smem + oW[0] + (cnt[0] + k) * KS) = KT::max_key();
          *reinterpret_cast<T_ *>(smem + oW[2] + (cnt[2] + k) * KS) = KT::max_key();
        } else {
          *reinterpret_cast<T_ *>(smem + oW[1] + cnt[1] * KS) = KT::max_key();
          *reinterpret_cast<T_ *>(smem + oW[3] + cnt[3] * KS) = KT::max_key();
        }
      }
    } else if (w_ == 1) {  // window edges a granule would have read outside the array
      const int r = l >> 3, e = l & 7;
      const uint32_t oWr = r == 0 ? oW[0] : r == 1 ? oW[1] : r == 2 ? oW[2] : oW[3];
      const int cr = r == 0 ? cnt[0] : r == 1 ? cnt[1] : r == 2 ? cnt[2] : cnt[3];
      const uint64_t pos = o0;
      const uint64_t g = lg4w < 64 ? (pos >> lg4w) : pos / (4 * w);
      // window r's first element: the tile's split point, recomputed from Q
      const QuadPt p0 = Q[blockIdx.x];
      const uintptr_t s0 = reinterpret_cast<uintptr_t>(src + g * 4 * w + r * w + p0.i[r]);
      const uintptr_t e0 = s0 + cr * KS;
      if (cr && (((s0 & ~uintptr_t(15)) < arr_lo) || (((e0 + 15) & ~uintptr_t(15)) > arr_hi))) {
        uintptr_t a = s0 & ~uintptr_t(15), b = (e0 + 15) & ~uintptr_t(15);
        if (a < arr_lo)
          a = (s0 + 15) & ~uintptr_t(15);
        if (b > arr_hi)
          b = e0 & ~uintptr_t(15);
        if (b <= a)
          a = b = e0;  // nothing came by bulk copy: plain loads for all
        const uint32_t nh = static_cast<uint32_t>((a > s0 ? a - s0 : 0) / KS);
        const uint32_t nt = static_cast<uint32_t>((e0 > b ? e0 - b : 0) / KS);
        // head [s0, a) and tail [b, e0): at most 3 + 3 elements (or the
        // whole window of <= 7 elements when no granule fits)
        for (uint32_t k = e; k < nh + nt; k += 8) {
          const uintptr_t gaddr = k < nh ? s0 + k * KS : b + (k - nh) * KS;
          *reinterpret_cast<T_ *>(smem + oWr + (gaddr - s0)) =
              *reinterpret_cast<const T_ *>(gaddr);
        }
      }
    }
  }
  __syncthreads();

}

// K5e's two merge phases over the loaded windows
template <class KT, int NT, int VT>
__device__ __forceinline__ void quad_tile_merge(char *smem, typename KT::T *__restrict__ dst,
                                                const uint32_t (&oW)[4], const int (&cnt)[4],
                                                uint64_t o0) {
  using T_ = typename KT::T;
  constexpr uint32_t KS = sizeof(T_);
  const int tid = threadIdx.x;
  const int nx = cnt[0] + cnt[1], ny = cnt[2] + cnt[3], total = nx + ny;

  // ---- phase 1: dynamic split of the threads between X and Y ----
  T_ keys[VT];
  uint32_t vals[VT];
  const int tx = (nx + VT - 1) / VT;
  const int side = tid >= tx ? 1 : 0;
  const int t1 = tid - side * tx;
  const uint32_t oA = side ? oW[2] : oW[0], oB = side ? oW[3] : oW[1];
  const int na = side ? cnt[2] : cnt[0], nb = side ? cnt[3] : cnt[1];
  const int d1 = t1 * VT;
  const bool act1 = d1 < na + nb;
  if (act1) {
    const int lo = split_predicted<KT, MP_QUAD_PRED_LOGW>(smem, oA, na, oB, nb, d1,
                                          static_cast<float>(na) / static_cast<float>(na + nb));
    serial_merge<KT, VT, false, true>(smem, oA, na, oB, nb, 0, 0, lo, d1 - lo, keys, vals);
  }
  __syncthreads();  // every window consumed
  // X over [oW0, oW0 + nx), Y over [oW2, oW2 + ny): each fits in the span
  // of the two windows (and gaps) it was merged from, sentinels included
  const uint32_t oX = oW[0], oY = oW[2];
  if (act1) {
    const uint32_t op = side ? oY : oX;
    const int lim = side ? ny : nx;
    if (d1 + VT <= lim) {
#pragma unroll
      for (int k = 0; k < VT; ++k)
        *reinterpret_cast<T_ *>(smem + op + (d1 + k) * KS) = keys[k];
    } else {
#pragma unroll
      for (int k = 0; k < VT; ++k)
        if (d1 + k < lim)
          *reinterpret_cast<T_ *>(smem + op + (d1 + k) * KS) = keys[k];
    }
  }
  if (tid >= NT - 32) {  // the last warp: X's VT sentinels and Y's one
    for (int l = tid - (NT - 32); l <= VT; l += 32) {
      if (l < VT)
        *reinterpret_cast<T_ *>(smem + oX + (nx + l) * KS) = KT::max_key();
      else
        *reinterpret_cast<T_ *>(smem + oY + ny * KS) = KT::max_key();
    }
  }
  __syncthreads();

  // ---- phase 2: out = merge(X, Y), ties to X ----
  const int d2 = tid * VT;
  if (d2 < total) {
    const int lo = split_predicted<KT, MP_QUAD_PRED_LOGW>(smem, oX, nx, oY, ny, d2,
                                          static_cast<float>(nx) / static_cast<float>(total));
    serial_merge<KT, VT, false, true>(smem, oX, nx, oY, ny, 0, 0, lo, d2 - lo, keys, vals);
  }
  __syncthreads();  // X and Y consumed

  T_ *out = dst + o0;
  const uint32_t oS = mirror_off(16, out);
  if (d2 + VT <= total) {
#pragma unroll
    for (int k = 0; k < VT; ++k)
      *reinterpret_cast<T_ *>(smem + oS + (d2 + k) * KS) = keys[k];
  } else if (d2 < total) {
#pragma unroll
    for (int k = 0; k < VT; ++k)
      if (d2 + k < total)
        *reinterpret_cast<T_ *>(smem + oS + (d2 + k) * KS) = keys[k];
  }
  fence_proxy_async_smem();
  __syncthreads();
  uint32_t lo;
  const uint32_t ib = interior_bytes(reinterpret_cast<const char *>(out),
                                     static_cast<uint32_t>(total) * KS, &lo);
  if (tid == 0 && ib) {
    bulk_s2g(reinterpret_cast<char *>(out) + lo, smem + oS + lo, ib);
    bulk_commit();
  }
  if (tid >= 32 && tid < 64) {
    const uint32_t bytes = static_cast<uint32_t>(total) * KS;
    const uint32_t hi = ib ? lo + ib : bytes;
    const uint32_t hlo = ib ? lo : bytes;
    const uint32_t nh = hlo / KS, nt = (bytes - hi) / KS;
    const uint32_t l = tid - 32;
    if (l < nh + nt) {
      const uint32_t e = l < nh ? l : (hi / KS) + (l - nh);
      out[e] = lds<T_>(smem, oS + e * KS);
    }
  }
  if (tid == 0 && ib)
    bulk_wait_read0();
}

template <class KT, int NT, int VT>
__global__ void __launch_bounds__(NT, 1536 / NT)
    quad_tile_kernel(const typename KT::T *__restrict__ src,
                     typename KT::T *__restrict__ dst, uint64_t n, uint64_t w,
                     uint32_t lg4w, uint32_t T, const QuadPt *__restrict__ Q) {
  extern __shared__ __align__(128) char smem[];
  uint32_t oW[4];
  int cnt[4];
  uint64_t o0;
  quad_load_tile<KT, VT>(smem, src, n, w, lg4w, T, Q, oW, cnt, o0);
  quad_tile_merge<KT, NT, VT>(smem, dst, oW, cnt, o0);
}

}  // namespace mpb
