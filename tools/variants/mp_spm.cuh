// mp_spm.cuh -- K2s: the persistent streaming Segmented Parallel Merge.
//
// Taken out of the product build in round 2 (MP_MERGE_ENGINE=spm): bit-exact
// but 2.3x slower than K1 + K2 on the B200 (one CTA's rings keep ~17 KB per
// stream in flight vs ~120 KB for 8 tile CTAs per SM).  Not compiled.
//
// The paper's cache-efficient SPM (parallel.hpp:90-145)
// mapped onto one B200 SM: a persistent CTA owns a contiguous output range
// [D_c, D_{c+1}) (D_c = floor(c*N/G)), i.e. the reference's worker segment.
// Only the two ends of that range are found by cross-diagonal search in HBM
// (one warp-cooperative 16-ary search per end, in the prologue).  Inside the
// range the CTA walks the merge path window by window (window = NV outputs,
// the SPM's L): A and B are STREAMED sequentially through two shared-memory
// rings fed by a producer warp with 1-D bulk copies (TMA engine) ahead of
// consumption, and each window's split is found in smem (the SPM hand-over:
// "the last worker's end point starts the next window").  There is no global
// split pass (K1) and every input byte is read from HBM exactly once.
//
//   warp NT/32 (producer): lane 0 issues cp.async.bulk for ring chunks as
//       slots free up (empty mbarriers), completion on full mbarriers.
//   warps 0..NT/32-1 (consumers): per window: wait full chunks, per-thread
//       diagonal search + VT-output branch-free merge from the rings, stage,
//       one bulk store per window (double-buffered staging), release chunks.
#pragma once

#include "mp_kernels.cuh"

namespace mpb {

// Warp-cooperative K-ary diagonal search (K = 16 lanes per search): each
// step probes 16 positions of the remaining range in parallel, so a 2^31
// range needs ceil(31/4) = 8 dependent DRAM round trips instead of 31.
// `lane16` in [0, 16), `mask` = the 16 participating lanes.
template <class KT>
__device__ uint64_t halfwarp_diag_search(const typename KT::T *__restrict__ a,
                                         uint64_t na,
                                         const typename KT::T *__restrict__ b,
                                         uint64_t nb, uint64_t d, int lane16,
                                         unsigned mask, int base_lane) {
  uint64_t lo = d > nb ? d - nb : 0;
  uint64_t hi = d < na ? d : na;
  while (lo < hi) {
    const uint64_t span = hi - lo;
    uint64_t m;
    bool valid;
    if (span <= 16) {
      m = lo + lane16;
      valid = static_cast<uint64_t>(lane16) < span;
    } else {
      m = lo + (span * static_cast<uint64_t>(lane16 + 1)) / 17;
      valid = true;
    }
    const bool pred = valid && take_b<KT>(b[d - 1 - m], a[m]);
    const unsigned bal = (__ballot_sync(mask, pred) >> base_lane) & 0xFFFFu;
    // positions are increasing in lane order; pred is monotone
    const int first = bal ? __ffs(bal) - 1 : 16;
    uint64_t m_first = __shfl_sync(mask, m, base_lane + (first < 16 ? first : 0));
    uint64_t m_prev = first > 0 ? __shfl_sync(mask, m, base_lane + first - 1)
                                : __shfl_sync(mask, m, base_lane);
    const int nvalid = span <= 16 ? static_cast<int>(span) : 16;
    uint64_t m_last = __shfl_sync(mask, m, base_lane + nvalid - 1);
    if (first < 16) {
      hi = m_first;
      lo = first > 0 ? m_prev + 1 : lo;
    } else {
      lo = m_last + 1;
    }
  }
  return lo;
}

template <class KT, int NT, int VT, int CH, int SLOTS>
struct SpmCfg {
  using T = typename KT::T;
  static constexpr int KS = sizeof(T);
  static constexpr int NV = NT * VT;
  static constexpr int RING = CH * SLOTS;  // elements per ring (power of 2)
  static_assert((RING & (RING - 1)) == 0, "ring must be a power of two");
  static_assert((SLOTS - 1) * CH >= NV, "ring too small for one window");
  static_assert((CH * KS) % 16 == 0, "chunk must be whole 16 B units");
  static constexpr uint32_t oRingA = 0;
  static constexpr uint32_t oRingB = oRingA + RING * KS;
  static constexpr uint32_t oStage = oRingB + RING * KS;  // 2 x NV keys
  static constexpr uint32_t oBar = (oStage + 2 * NV * KS + 127) & ~127u;
  // barriers: fullA[S], emptyA[S], fullB[S], emptyB[S]
  static constexpr uint32_t oMisc = oBar + 4 * SLOTS * 8;
  static constexpr uint32_t bytes = oMisc + 64;
};

template <class KT, int NT, int VT, int CH, int SLOTS>
__global__ void __launch_bounds__(NT + 32, 1)
    spm_merge_kernel(const typename KT::T *__restrict__ a, uint64_t na,
                     const typename KT::T *__restrict__ b, uint64_t nb,
                     typename KT::T *__restrict__ out) {
  using C = SpmCfg<KT, NT, VT, CH, SLOTS>;
  using T = typename KT::T;
  constexpr int KS = C::KS, NV = C::NV, RING = C::RING;
  extern __shared__ __align__(128) char smem[];
  uint64_t *fullA = reinterpret_cast<uint64_t *>(smem + C::oBar);
  uint64_t *emptyA = fullA + SLOTS;
  uint64_t *fullB = emptyA + SLOTS;
  uint64_t *emptyB = fullB + SLOTS;
  uint64_t *misc = reinterpret_cast<uint64_t *>(smem + C::oMisc);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint64_t n = na + nb;
  const uint64_t G = gridDim.x;
  // CTA output ranges start on 16 B boundaries of `out` (the caller
  // guarantees `out` is 16 B aligned), so every window store is a bulk copy
  constexpr uint64_t AL = 16 / KS;
  auto range_start = [&](uint64_t c) -> uint64_t {
    if (c >= G)
      return n;
    const uint64_t d = static_cast<uint64_t>(
        (static_cast<unsigned __int128>(c) * n) / G);
    return d & ~(AL - 1);
  };
  const uint64_t D0 = range_start(blockIdx.x);
  const uint64_t D1 = range_start(blockIdx.x + 1);

  // ---- prologue: this CTA's two end splits (producer warp, 2 x 16 lanes) --
  if (warp == NT / 32) {
    const int half = lane >> 4, l16 = lane & 15;
    const uint64_t d = half ? D1 : D0;
    const uint64_t s = halfwarp_diag_search<KT>(
        a, na, b, nb, d, l16, 0xFFFFu << (half * 16), half * 16);
    if (l16 == 0)
      misc[half] = s;  // misc[0] = a at D0, misc[1] = a at D1
    if (lane == 0) {
      for (int i = 0; i < SLOTS; ++i) {
        mbar_init(&fullA[i], 1);
        mbar_init(&emptyA[i], 1);
        mbar_init(&fullB[i], 1);
        mbar_init(&emptyB[i], 1);
      }
      fence_mbar_init();
    }
  }
  __syncthreads();
  const uint64_t a_s = misc[0], a_e = misc[1];
  const uint64_t b_s = D0 - a_s, b_e = D1 - a_e;
  // chunk grids start at 16 B-aligned element indices
  const uint64_t baseA = a_s & ~(AL - 1), baseB = b_s & ~(AL - 1);

  if (warp == NT / 32) {
    // ---------------- producer ----------------
    if (lane != 0)
      return;
    const uint64_t endA = a_e, endB = b_e;
    const uint64_t nchA = endA > baseA ? (endA - baseA + CH - 1) / CH : 0;
    const uint64_t nchB = endB > baseB ? (endB - baseB + CH - 1) / CH : 0;
    uint64_t kA = 0, kB = 0;
    auto issue = [&](const T *src, uint64_t base, uint64_t end, uint64_t k,
                     uint32_t oRing, uint64_t *full) {
      const int slot = static_cast<int>(k % SLOTS);
      const uint64_t e0 = base + k * CH;
      const uint64_t e1 = e0 + CH < end ? e0 + CH : end;
      // bulk part: whole 16 B units; the tail (< 16 B) by ordinary loads
      const uint64_t e1a = e0 + ((e1 - e0) & ~(AL - 1));
      char *dst = smem + oRing + static_cast<uint32_t>(slot) * CH * KS;
      for (uint64_t e = e1a; e < e1; ++e)
        reinterpret_cast<T *>(dst)[e - e0] = src[e];
      const uint32_t bytes = static_cast<uint32_t>((e1a - e0) * KS);
      mbar_arrive_expect_tx(&full[slot], bytes);
      if (bytes)
        bulk_g2s(dst, src + e0, bytes, &full[slot]);
    };
    while (kA < nchA || kB < nchB) {
      bool progressed = false;
      if (kA < nchA) {
        const int slot = static_cast<int>(kA % SLOTS);
        const uint32_t par = static_cast<uint32_t>((kA / SLOTS) & 1) ^ 1u;
        if (kA < SLOTS || mbar_test_wait(&emptyA[slot], par)) {
          issue(a, baseA, endA, kA, C::oRingA, fullA);
          ++kA;
          progressed = true;
        }
      }
      if (kB < nchB) {
        const int slot = static_cast<int>(kB % SLOTS);
        const uint32_t par = static_cast<uint32_t>((kB / SLOTS) & 1) ^ 1u;
        if (kB < SLOTS || mbar_test_wait(&emptyB[slot], par)) {
          issue(b, baseB, endB, kB, C::oRingB, fullB);
          ++kB;
          progressed = true;
        }
      }
      (void)progressed;
    }
    return;
  }

  // ---------------- consumers (NT threads) ----------------
  auto bar_c = [] { asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory"); };
  auto ldA = [&](uint64_t e) -> T {  // global A element index -> ring
    return *reinterpret_cast<const T *>(
        smem + C::oRingA + static_cast<uint32_t>((e - baseA) & (RING - 1)) * KS);
  };
  auto ldB = [&](uint64_t e) -> T {
    return *reinterpret_cast<const T *>(
        smem + C::oRingB + static_cast<uint32_t>((e - baseB) & (RING - 1)) * KS);
  };
  uint64_t ca = a_s, cb = b_s, o = D0;
  uint64_t relA = 0, relB = 0;  // next chunk to release
  uint64_t waitedA = 0, waitedB = 0;  // chunks known full
  int sb = 0;
  while (o < D1) {
    const int total = static_cast<int>(D1 - o < NV ? D1 - o : NV);
    const int wa = static_cast<int>(a_e - ca < static_cast<uint64_t>(total) ? a_e - ca : total);
    const int wb = static_cast<int>(b_e - cb < static_cast<uint64_t>(total) ? b_e - cb : total);
    // wait for every chunk the window touches
    const uint64_t needA = wa ? (ca + wa - 1 - baseA) / CH + 1 : 0;
    const uint64_t needB = wb ? (cb + wb - 1 - baseB) / CH + 1 : 0;
    for (; waitedA < needA; ++waitedA)
      mbar_wait(&fullA[waitedA % SLOTS], static_cast<uint32_t>((waitedA / SLOTS) & 1));
    for (; waitedB < needB; ++waitedB)
      mbar_wait(&fullB[waitedB % SLOTS], static_cast<uint32_t>((waitedB / SLOTS) & 1));

    // per-thread split on its diagonal within the window
    const int diag = min(tid * VT, total);
    int lo = diag > wb ? diag - wb : 0;
    int hi = diag < wa ? diag : wa;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (take_b<KT>(ldB(cb + (diag - 1 - mid)), ldA(ca + mid)))
        hi = mid;
      else
        lo = mid + 1;
    }
    int i = lo, j = diag - lo;
    T keys[VT];
    T ka = ldA(ca + min(i, wa));
    T kb = ldB(cb + min(j, wb));
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      const bool tb = (j < wb) && ((i >= wa) || take_b<KT>(kb, ka));
      keys[k] = tb ? kb : ka;
      i += tb ? 0 : 1;
      j += tb ? 1 : 0;
      const T nxt = tb ? ldB(cb + min(j, wb)) : ldA(ca + min(i, wa));
      kb = tb ? nxt : kb;
      ka = tb ? ka : nxt;
    }
    // the window's end split: the thread that owns output total-1 knows it
    if (diag < total && diag + VT >= total) {
      // replay to exactly `total - diag` outputs
      int ii = lo, jj = diag - lo;
      for (int k = 0; k < total - diag; ++k) {
        const bool tb = (jj < wb) && ((ii >= wa) ||
                                      take_b<KT>(ldB(cb + jj), ldA(ca + ii)));
        ii += tb ? 0 : 1;
        jj += tb ? 1 : 0;
      }
      misc[2] = static_cast<uint64_t>(ii);
    }
    if (tid == 0)
      bulk_wait_read<1>();  // staging buffer sb (used two windows ago) free
    bar_c();
    const uint64_t ua = misc[2];
    const uint64_t ub = static_cast<uint64_t>(total) - ua;
    ca += ua;
    cb += ub;
    // release ring chunks entirely below the new heads
    if (tid == 0) {
      for (; relA < waitedA && baseA + (relA + 1) * CH <= ca; ++relA)
        mbar_arrive(&emptyA[relA % SLOTS]);
      for (; relB < waitedB && baseB + (relB + 1) * CH <= cb; ++relB)
        mbar_arrive(&emptyB[relB % SLOTS]);
    }
    const uint32_t oS = C::oStage + static_cast<uint32_t>(sb) * NV * KS;
#pragma unroll
    for (int k = 0; k < VT; ++k)
      *reinterpret_cast<T *>(smem + oS + (tid * VT + k) * KS) = keys[k];
    fence_proxy_async_smem();
    bar_c();
    if (tid == 0) {
      const int tot_al = total & ~static_cast<int>(AL - 1);
      if (tot_al)
        bulk_s2g(out + o, smem + oS, static_cast<uint32_t>(tot_al) * KS);
      for (int q = tot_al; q < total; ++q)  // < 16 B tail, last window only
        out[o + q] = *reinterpret_cast<const T *>(smem + oS + q * KS);
      bulk_commit();
    }
    o += static_cast<uint64_t>(total);
    sb ^= 1;
  }
  if (tid == 0)
    bulk_wait_read<0>();
}

}  // namespace mpb
