// mp_pieces.cuh -- merging sequences that are concatenations of pieces
// (shards that may live on other GPUs, mapped over NVLink / NVSwitch).
//
// A = A_0 ++ A_1 ++ ... and B = B_0 ++ B_1 ++ ... (virtual index spaces).
// The merge path of (A, B) crosses every piece boundary exactly once:
//   row a = s (first element of an A piece) at the point (s, lb_B(A[s])),
//     lb_B(x) = #{B[j] < x}            (B keys equal to A[s] follow it),
//   column b = t (first element of a B piece) at (ub_A(B[t]), t),
//     ub_A(y) = #{A[i] <= y}           (A keys equal to B[t] precede it).
// Cutting the requested output range at those crossings leaves segments
// whose A-range lies in ONE A piece and B-range in ONE B piece; each is a
// plain merge of two contiguous ranges (Merge Path locality),
// run by the ordinary K1 + K2 kernels straight from the (peer) pointers:
// the NVLink pull is fused into the tile loads, no staging exchange.
#pragma once

#include "mp_kernels.cuh"

namespace mpb {

constexpr int kMaxPieces = 16;

struct VPieces {
  const void *ptr[kMaxPieces];
  uint64_t start[kMaxPieces + 1];  // start[n] = total length
  int n;
};

template <class KT>
__device__ __forceinline__ typename KT::T vget(const VPieces &v, uint64_t i) {
  int k = 0;
#pragma unroll 1
  while (k + 1 < v.n && i >= v.start[k + 1])
    ++k;
  return static_cast<const typename KT::T *>(v.ptr[k])[i - v.start[k]];
}

// #{B[j] < x}
template <class KT>
__device__ uint64_t v_lower_bound(const VPieces &B, const typename KT::T &x) {
  uint64_t lo = 0, hi = B.start[B.n];
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (KT::less(vget<KT>(B, mid), x))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// #{A[i] <= y}
template <class KT>
__device__ uint64_t v_upper_bound(const VPieces &A, const typename KT::T &y) {
  uint64_t lo = 0, hi = A.start[A.n];
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (KT::less(y, vget<KT>(A, mid)))
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
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

// One thread per probe:
//   out[0], out[1]           a_off at the range ends d0, d1
//   out[2 + k], k < nA - 1   diagonal where row A.start[k+1] is crossed
//   out[1 + nA + k], k < nB-1 diagonal where column B.start[k+1] is crossed
// (as (a, b) pairs packed in two uint64 each: out[2*idx], out[2*idx+1])
template <class KT>
__global__ void pieces_probe_kernel(VPieces A, VPieces B, uint64_t d0,
                                    uint64_t d1, uint64_t *__restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int nA = A.n, nB = B.n;
  const uint64_t na = A.start[nA], nb = B.start[nB];
  if (t == 0 || t == 1) {
    const uint64_t d = t == 0 ? d0 : d1;
    const uint64_t a = v_diag_search<KT>(A, B, d);
    out[2 * t] = a;
    out[2 * t + 1] = d - a;
  } else if (t < 2 + (nA - 1)) {
    const uint64_t s = A.start[t - 1];  // starts of pieces 1..nA-1
    uint64_t b = nb;
    if (s < na)
      b = v_lower_bound<KT>(B, vget<KT>(A, s));
    out[2 * t] = s;
    out[2 * t + 1] = b;
  } else if (t < 2 + (nA - 1) + (nB - 1)) {
    const uint64_t s = B.start[t - 1 - (nA - 1)];
    uint64_t a = na;
    if (s < nb)
      a = v_upper_bound<KT>(A, vget<KT>(B, s));
    out[2 * t] = a;
    out[2 * t + 1] = s;
  }
}

}  // namespace mpb
