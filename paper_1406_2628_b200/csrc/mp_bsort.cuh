// mp_bsort.cuh -- K3b: block sort for bare 32-bit keys (u32, i32, f32
// totalOrder), the first pass of mp_sort when no values ride along
// (replaces sort.hpp:59-67's insertion-sorted base runs).
//
// Bare keys carry no payload, so equal keys are indistinguishable: any
// correct sort of a block yields the bytes of the stable one, and the keys
// may be dealt to threads in any order.  The kernel is issue-bound, so the
// design minimises instructions per key:
//   * keys enter as their order-preserving u32 image (i32: sign flip, f32:
//     totalOrder image) -- one unsigned compare per merge step for all three
//     types -- and leave through the inverse image;
//   * keys come in as 16-byte vectors (any dealing to threads is fine) and
//     leave through one bulk store (cp.async.bulk) of the staged block;
//   * a Batcher network sorts each thread's VT keys in registers;
//   * log2(NT) Merge Path passes (core.hpp:99-180) in shared memory.  Each run
//     of the pass is followed by one word holding the sentinel 0xFFFFFFFF,
//     and A's cursor saturates at its sentinel, so the per-output step needs
//     no bounds tests: once A is exhausted its sentinel loses to every B key
//     below the maximum and ties with a B key equal to it -- which emits the
//     same value, so the output bytes are exact.  (B's cursor cannot pass
//     its sentinel: the sentinel is never strictly below an A key.)
//     VT is odd, so the stride-VT stores hit 32 distinct banks and the
//     merge cursors of neighbouring threads (~VT/2 apart) spread over banks.
#pragma once

#include "mp_common.cuh"

namespace mpb {

template <class KT> __device__ __forceinline__ uint32_t order_u32(typename KT::T x);
template <> __device__ __forceinline__ uint32_t order_u32<KeyU32>(uint32_t x) { return x; }
template <> __device__ __forceinline__ uint32_t order_u32<KeyI32>(int32_t x) {
  return static_cast<uint32_t>(x) ^ 0x80000000u;
}
template <> __device__ __forceinline__ uint32_t order_u32<KeyF32>(uint32_t x) {
  return f32_order(x);
}
template <class KT> __device__ __forceinline__ typename KT::T from_order_u32(uint32_t u);
template <> __device__ __forceinline__ uint32_t from_order_u32<KeyU32>(uint32_t u) { return u; }
template <> __device__ __forceinline__ int32_t from_order_u32<KeyI32>(uint32_t u) {
  return static_cast<int32_t>(u ^ 0x80000000u);
}
template <> __device__ __forceinline__ uint32_t from_order_u32<KeyF32>(uint32_t u) {
  return (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;  // inverse of f32_order
}

// smem: the finest level (NT runs of VT) has the most sentinel words
template <int NT, int VT>
__host__ __device__ constexpr uint32_t bare_sort_smem_bytes() {
  return static_cast<uint32_t>(NT) * (VT + 1) * 4 + 64;
}

__device__ __forceinline__ void ce_u32(uint32_t &x, uint32_t &y) {
  const uint32_t lo = min(x, y);
  y = max(x, y);
  x = lo;
}

// Batcher's odd-even merge sort network for the next power of two above N,
// truncated to N inputs (the missing inputs act as +inf, so comparators that
// touch them never fire and are dropped).
template <int N>
__device__ __forceinline__ void batcher_u32(uint32_t (&x)[N]) {
  constexpr int P2 = N <= 1 ? 1 : 1 << (32 - __builtin_clz(N - 1));
#pragma unroll
  for (int p = 1; p < P2; p <<= 1) {
#pragma unroll
    for (int k = p; k >= 1; k >>= 1) {
#pragma unroll
      for (int j = k % p; j + k < P2; j += 2 * k) {
#pragma unroll
        for (int i = 0; i < k; ++i) {
          if (i + j + k < N && (i + j) / (2 * p) == (i + j + k) / (2 * p))
            ce_u32(x[i + j], x[i + j + k]);
        }
      }
    }
  }
}

// One CTA sorts NV = NT * VT keys (VT odd).  Pass k merges runs of
// w = VT << k held by 2^k threads each; the pair of thread t is t >> (k+1).
// Level-k layout: run r at word r * (w + 1), its sentinel at r * (w + 1) + w.
template <class KT, int NT, int VT, bool ALIGNED>
__global__ void __launch_bounds__(NT, 2048 / NT)
    block_sort_bare_kernel(const typename KT::T *__restrict__ in,
                           typename KT::T *__restrict__ out, uint64_t n,
                           uint64_t block0) {
  static_assert(sizeof(typename KT::T) == 4 && (VT & 1) && (NT & (NT - 1)) == 0,
                "bare 32-bit keys, odd VT, NT a power of two");
  constexpr int NV = NT * VT;
  constexpr int LNT = __builtin_ctz(NT);
  static_assert((NV * 4) % 16 == 0, "bulk store granularity");
  extern __shared__ __align__(128) uint32_t s[];
  const int tid = threadIdx.x;
  const uint64_t base = (block0 + blockIdx.x) * NV;
  // ALIGNED launches cover whole 16 B-aligned blocks only (the host sends a
  // short last block or unaligned buffers to the generic instantiation)
  const int cnt = ALIGNED ? NV : static_cast<int>((n - base) < NV ? (n - base) : NV);
  constexpr bool full = ALIGNED;

  // ---- load: any dealing of the block's keys to threads will do ----
  uint32_t x[VT];
  if constexpr (full) {
    constexpr int V4 = NV / 4 / NT;  // 16-byte vectors per thread
    const uint4 *src = reinterpret_cast<const uint4 *>(in + base);
#pragma unroll
    for (int m = 0; m < V4; ++m) {
      const uint4 v = __ldg(src + tid + m * NT);
      x[4 * m + 0] = order_u32<KT>(static_cast<typename KT::T>(v.x));
      x[4 * m + 1] = order_u32<KT>(static_cast<typename KT::T>(v.y));
      x[4 * m + 2] = order_u32<KT>(static_cast<typename KT::T>(v.z));
      x[4 * m + 3] = order_u32<KT>(static_cast<typename KT::T>(v.w));
    }
#pragma unroll
    for (int k = 4 * V4; k < VT; ++k)
      x[k] = order_u32<KT>(in[base + (k - 4 * V4) * NT + 4 * V4 * NT + tid]);
  } else {
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      const int q = tid + k * NT;
      x[k] = q < cnt ? order_u32<KT>(in[base + q]) : 0xFFFFFFFFu;
    }
  }
  batcher_u32<VT>(x);

#pragma unroll 1
  for (int k = 0; k < LNT; ++k) {
    const int w = VT << k;
    // ---- store the thread's sorted VT keys (stride VT, odd: no conflicts) ----
    {
      const int r = tid >> k, off = (tid & ((1 << k) - 1)) * VT;
      const int o = r * (w + 1) + off;
#pragma unroll
      for (int q = 0; q < VT; ++q)
        s[o + q] = x[q];
      if (off + VT == w)
        s[o + VT] = 0xFFFFFFFFu;
    }
    __syncthreads();
    // ---- split: diagonal search within the pair (ties to A) ----
    const int diag = (tid & ((2 << k) - 1)) * VT;
    const int aO = ((tid >> (k + 1)) << 1) * (w + 1);
    const int bO = aO + w + 1;
    int lo = diag > w ? diag - w : 0;
    int hi = diag < w ? diag : w;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s[bO + diag - 1 - mid] < s[aO + mid])
        hi = mid;
      else
        lo = mid + 1;
    }
    // ---- serial merge of VT outputs, no bounds tests (see header) ----
    int pa = aO + lo, pb = bO + (diag - lo);
    const int ea = aO + w;  // A's sentinel
    uint32_t ka = s[pa], kb = s[pb];
#pragma unroll
    for (int q = 0; q < VT; ++q) {
      const bool tb = kb < ka;
      x[q] = tb ? kb : ka;
      pa = tb ? pa : min(pa + 1, ea);
      pb = tb ? pb + 1 : pb;
      const uint32_t nx = s[tb ? pb : pa];
      kb = tb ? nx : kb;
      ka = tb ? ka : nx;
    }
    __syncthreads();
  }

  // ---- x = sorted positions [tid*VT, tid*VT + VT); stage, write back ----
#pragma unroll
  for (int q = 0; q < VT; ++q)
    s[tid * VT + q] = static_cast<uint32_t>(from_order_u32<KT>(x[q]));
  if constexpr (full) {
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      bulk_s2g(out + base, s, NV * 4);
      bulk_commit();
      bulk_wait_read0();
    }
  } else {
    __syncthreads();
    for (int q = tid; q < cnt; q += NT)
      out[base + q] = static_cast<typename KT::T>(s[q]);
  }
}

}  // namespace mpb

namespace mpb {

// ---------------------------------------------------------------------------
// K3w: block sort of 4096 bare 32-bit keys per CTA (256 threads x 16) that
// keeps the first five merge levels in registers:
//   * Batcher network on each thread's 16 keys (u32 order image);
//   * warp levels m = 1..5 (groups of 2^m lanes, runs of 16 * 2^(m-1)
//     merged): a bitonic merge of the two halves' ascending runs -- the
//     "flip" stage compares element e with element 16*2^m - 1 - e (partner
//     lane ^ (2^m - 1), register 15 - q), then half-cleaners at lane strides
//     2^(m-2) .. 1 (shfl.xor) and register strides 8 .. 1 -- so a warp ends
//     with one sorted run of 512 in lane-major order and no smem traffic;
//   * three Merge Path passes in smem (runs of 512 -> 4096) with one
//     sentinel word after every run and a p + p/32 padded layout (the
//     stride-16 stores and loads stay conflict-free), A's cursor saturating
//     at its sentinel as in K3b;
//   * each thread's 16 sorted keys leave with four 16-byte stores.
// Bare keys only (no stability question: equal keys are equal bytes).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ce_dir(uint32_t &x, uint32_t y, bool upper) {
  x = upper ? max(x, y) : min(x, y);
}

__host__ __device__ __forceinline__ constexpr int pad32(int p) { return p + (p >> 5); }

// Pass layout: run r of width W at word r * (W + 32) (32-aligned, so
// pad32(run + k) = pad32(run) + pad32(k) and a thread's 16 keys -- at a
// multiple of 16 -- land at pad32(o) + q), followed by 16 copies of the
// sentinel 0xFFFFFFFF: A's cursor may walk 16 of them, so it needs no
// saturation (see the K3b header for why the output bytes stay exact).
template <int NT>
__host__ __device__ constexpr uint32_t warp_sort_smem_bytes() {
  return static_cast<uint32_t>(pad32(NT * 16 + NT * 16 / 512 * 32 + 32)) * 4 + 64;
}

// Merge Path passes over runs of W, 2W, .. < NV (compile-time widths: the
// run/pair/diagonal arithmetic is shifts and masks, the stores take
// immediate offsets).  B200 ncu, 2^30 keys, before: 321 + ~150 (search)
// warp instructions per pass and warp with runtime widths (an integer
// division per pass), a saturating A cursor and per-key padded addresses.
template <int W, int NV>
__device__ __forceinline__ void warp_sort_passes(uint32_t (&x)[16], uint32_t *s, int p0) {
  if constexpr (W < NV) {
    constexpr int VT = 16, S = W + 32;
    {
      const int r = p0 / W, off = p0 % W;
      uint32_t *p = s + pad32(r * S + off);
#pragma unroll
      for (int q = 0; q < VT; ++q)
        p[q] = x[q];
      if (off + VT == W) {
        uint32_t *ps = s + pad32(r * S + W);
#pragma unroll
        for (int q = 0; q < 16; ++q)
          ps[q] = 0xFFFFFFFFu;
      }
    }
    __syncthreads();
    const int diag = p0 % (2 * W);
    const int aO = (p0 / (2 * W)) * 2 * S;
    const int bO = aO + S;
    int lo = diag > W ? diag - W : 0;
    int hi = diag < W ? diag : W;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s[pad32(bO + diag - 1 - mid)] < s[pad32(aO + mid)])
        hi = mid;
      else
        lo = mid + 1;
    }
    int pa = aO + lo, pb = bO + (diag - lo);
    uint32_t ka = s[pad32(pa)], kb = s[pad32(pb)];
#pragma unroll
    for (int q = 0; q < VT; ++q) {
      const bool tb = kb < ka;
      x[q] = min(ka, kb);
      pa += tb ? 0 : 1;
      pb += tb ? 1 : 0;
      const uint32_t nx = s[pad32(tb ? pb : pa)];
      kb = tb ? nx : kb;
      ka = tb ? ka : nx;
    }
    __syncthreads();
    warp_sort_passes<2 * W, NV>(x, s, p0);
  }
}

template <class KT, int NT, bool ALIGNED>
__global__ void __launch_bounds__(NT, 2048 / NT)
    block_sort_warp_kernel(const typename KT::T *__restrict__ in,
                           typename KT::T *__restrict__ out, uint64_t n,
                           uint64_t block0) {
  static_assert(sizeof(typename KT::T) == 4 && NT % 32 == 0 && (NT & (NT - 1)) == 0,
                "bare 32-bit keys, NT a power of two");
  constexpr int VT = 16;
  constexpr int NV = NT * VT;
  extern __shared__ __align__(128) uint32_t s[];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint64_t base = (block0 + blockIdx.x) * NV;
  const int cnt = ALIGNED ? NV : static_cast<int>((n - base) < NV ? (n - base) : NV);

  uint32_t x[VT];
  if constexpr (ALIGNED) {
    const uint4 *src = reinterpret_cast<const uint4 *>(in + base);
#pragma unroll
    for (int m = 0; m < VT / 4; ++m) {
      const uint4 v = __ldg(src + tid + m * NT);
      x[4 * m + 0] = order_u32<KT>(static_cast<typename KT::T>(v.x));
      x[4 * m + 1] = order_u32<KT>(static_cast<typename KT::T>(v.y));
      x[4 * m + 2] = order_u32<KT>(static_cast<typename KT::T>(v.z));
      x[4 * m + 3] = order_u32<KT>(static_cast<typename KT::T>(v.w));
    }
  } else {
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      const int q = tid + k * NT;
      x[k] = q < cnt ? order_u32<KT>(in[base + q]) : 0xFFFFFFFFu;
    }
  }
  batcher_u32<VT>(x);

  // ---- warp levels: runs of 16 -> 512 in registers ----
#pragma unroll
  for (int m = 1; m <= 5; ++m) {
    const int g = 1 << m;
    {  // flip: element e <-> 16g - 1 - e
      const bool upper = (lane & (g - 1)) >= (g >> 1);
#pragma unroll
      for (int q = 0; q < VT / 2; ++q) {
        const uint32_t a = __shfl_xor_sync(0xffffffffu, x[VT - 1 - q], g - 1);
        const uint32_t b = __shfl_xor_sync(0xffffffffu, x[q], g - 1);
        ce_dir(x[q], a, upper);
        ce_dir(x[VT - 1 - q], b, upper);
      }
    }
#pragma unroll
    for (int st = g >> 2; st >= 1; st >>= 1) {  // half-cleaners across lanes
      const bool upper = (lane & st) != 0;
#pragma unroll
      for (int q = 0; q < VT; ++q)
        ce_dir(x[q], __shfl_xor_sync(0xffffffffu, x[q], st), upper);
    }
#pragma unroll
    for (int st = VT / 2; st >= 1; st >>= 1)  // half-cleaners in registers
#pragma unroll
      for (int q = 0; q < VT; ++q)
        if ((q & st) == 0)
          ce_u32(x[q], x[q + st]);
  }

  // ---- smem Merge Path passes: runs of 512 -> NV ----
  const int p0 = tid * VT;
  warp_sort_passes<512, NV>(x, s, p0);

  // ---- x = sorted positions [p0, p0 + 16) of the block ----
  if constexpr (ALIGNED) {
    uint4 *dst = reinterpret_cast<uint4 *>(out + base + p0);
#pragma unroll
    for (int m = 0; m < VT / 4; ++m) {
      uint4 v;
      v.x = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 0]));
      v.y = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 1]));
      v.z = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 2]));
      v.w = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 3]));
      dst[m] = v;
    }
  } else {
#pragma unroll
    for (int q = 0; q < VT; ++q)
      if (p0 + q < cnt)
        out[base + p0 + q] = from_order_u32<KT>(x[q]);
  }
}

}  // namespace mpb

namespace mpb {

// ---------------------------------------------------------------------------
// K3t: block sort of NV = 16 * NT bare 32-bit keys per CTA as a bitonic
// sorting network whose compare-exchanges all run inside registers.
//
// K3w's levels cost per key: 3 instructions for every compare-exchange
// across lanes (SHFL + a max and a predicated min: the direction depends on
// the lane), and ~29 per Merge Path pass (split search + serial merge with
// padded addressing; B200 ncu: 321 + ~150 warp instructions per pass and
// warp).  K3t instead moves the keys so that the partners of a stage sit in
// one thread:
//   * layout G (G = 0 or G >= 5): thread t holds the 16 elements whose index
//     bits [G, G+4) are the register number r and whose other bits are t's
//     bits in order.  Layout 0 ("C") is 16 consecutive elements per thread.
//     A transpose between layouts is 16 STS + 16 LDS through a p + p/32
//     padded buffer; for G = 0 and G >= 5 the 32 lanes of every access hit
//     32 distinct banks and all offsets are compile-time immediates.
//   * merge level L (runs 2^(L-1) -> 2^L): the upper run is reversed on its
//     way into the first layout of the level (the registers in reverse order
//     and thread bits [0, L-5) flipped -- element e -> e ^ (2^(L-1) - 1)),
//     which makes every 2^L-group bitonic, so every stage is an ascending
//     half-cleaner: min to the lower index, max to the upper (ce_u32, one
//     instruction per key).  Bits L-1 .. 5 are processed four at a time in
//     layouts G >= 5, bit 4 (lane bit 0 of layout C) with one shfl.xor
//     stage, bits 3..0 in layout C.
//   * levels L <= 8 (runs up to 256, inside a warp) keep K3w's flip + shfl
//     formulation (no smem); the CTA ends in layout C and stores 16 keys per
//     thread with 16-byte vectors.
// Per key: Batcher 8, levels 5-8 46, level L >= 9 about L stages + 3 per
// lane stage + 2 per transpose + 1 for the reversal: 166 instructions per
// key in all against K3w's 207 -- but 104 of them are VIMNMX on the
// half-rate ALU pipe, and B200 runs K3t at 8.44 ms vs K3w's 8.26 ms (ALU
// pipe 80 % busy, LSU 59 %, barrier and MIO stalls), so K3t is opt-in
// (MP_K3W=tr).
// ---------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ int tr_base(int t) {
  const int e = G == 0 ? t * 16 : ((t & ((1 << G) - 1)) | ((t >> G) << (G + 4)));
  return pad32(e);
}
template <int G>
__host__ __device__ constexpr int tr_step() {
  return G == 0 ? 1 : (1 << G) + (1 << (G - 5));
}
template <int G>
__device__ __forceinline__ void tr_store(const uint32_t (&x)[16], uint32_t *s, int t) {
  uint32_t *p = s + tr_base<G>(t);
#pragma unroll
  for (int r = 0; r < 16; ++r)
    p[r * tr_step<G>()] = x[r];
}
template <int G>
__device__ __forceinline__ void tr_load(uint32_t (&x)[16], const uint32_t *s, int t) {
  const uint32_t *p = s + tr_base<G>(t);
#pragma unroll
  for (int r = 0; r < 16; ++r)
    x[r] = p[r * tr_step<G>()];
}
// ascending half-cleaners on register strides SR, SR/2, .., SR >> (K-1)
template <int SR, int K>
__device__ __forceinline__ void reg_stages(uint32_t (&x)[16]) {
  if constexpr (K > 0) {
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if ((q & SR) == 0)
        ce_u32(x[q], x[q + SR]);
    reg_stages<SR / 2, K - 1>(x);
  }
}

// Groups of element bits hb .. 5 of one level, four at a time (layout G =
// hb - 3), then the 2-3 leftover bits in layout 5, a single leftover bit as
// a lane stage later.  Returns through the layout-0 transpose.
// Level 9's groups (512 elements) are one warp's keys in every layout used,
// so its transposes only need warp-level barriers.
template <bool WARP>
__device__ __forceinline__ void tr_sync() {
  if constexpr (WARP)
    __syncwarp();
  else
    __syncthreads();
}

template <int HB, bool WARP>
__device__ __forceinline__ void tr_groups(uint32_t (&x)[16], uint32_t *s, int tid) {
  if constexpr (HB >= 8) {
    tr_load<HB - 3>(x, s, tid);
    reg_stages<8, 4>(x);
    tr_sync<WARP>();
    tr_store<HB - 3>(x, s, tid);
    tr_sync<WARP>();
    tr_groups<HB - 4, WARP>(x, s, tid);
  } else if constexpr (HB >= 6) {  // bits HB..5: layout 5, register strides
    tr_load<5>(x, s, tid);
    reg_stages<(1 << (HB - 5)), HB - 4>(x);
    tr_sync<WARP>();
    tr_store<5>(x, s, tid);
    tr_sync<WARP>();
    tr_load<0>(x, s, tid);
  } else {
    tr_load<0>(x, s, tid);
  }
}

template <int L, int LOGNV, int NT>
__device__ __forceinline__ void tr_levels(uint32_t (&x)[16], uint32_t *s, int tid) {
  if constexpr (L <= LOGNV) {
    const int lane = tid & 31;
    // reversal of the upper run: e -> e ^ (2^(L-1) - 1)
    const bool rev = (tid >> (L - 5)) & 1;
    const int tw = rev ? (tid ^ ((1 << (L - 5)) - 1)) : tid;
    uint32_t y[16];
#pragma unroll
    for (int r = 0; r < 16; ++r)
      y[r] = rev ? x[15 - r] : x[r];
    tr_store<0>(y, s, tw);
    tr_sync<L == 9>();
    tr_groups<L - 1, L == 9>(x, s, tid);  // ends with layout 0 loaded
    constexpr int HB = L - 1 - 4 * ((L - 1 - 4) / 4);  // bits left above 4
    if constexpr (HB == 5) {  // one leftover bit (5): lane stride 2
      const bool upper = (lane & 2) != 0;
#pragma unroll
      for (int q = 0; q < 16; ++q)
        ce_dir(x[q], __shfl_xor_sync(0xffffffffu, x[q], 2), upper);
    }
    {  // bit 4: lane stride 1
      const bool upper = (lane & 1) != 0;
#pragma unroll
      for (int q = 0; q < 16; ++q)
        ce_dir(x[q], __shfl_xor_sync(0xffffffffu, x[q], 1), upper);
    }
    reg_stages<8, 4>(x);
    tr_sync<L == 9>();  // layout-0 reads done before the next level's stores
    tr_levels<L + 1, LOGNV, NT>(x, s, tid);
  }
}

template <int NT>
__host__ __device__ constexpr uint32_t tr_sort_smem_bytes() {
  return static_cast<uint32_t>(pad32(NT * 16)) * 4 + 64;
}

template <class KT, int NT, bool ALIGNED>
__global__ void __launch_bounds__(NT, 2048 / NT)
    block_sort_tr_kernel(const typename KT::T *__restrict__ in,
                         typename KT::T *__restrict__ out, uint64_t n,
                         uint64_t block0) {
  static_assert(sizeof(typename KT::T) == 4 && NT >= 64 && (NT & (NT - 1)) == 0,
                "bare 32-bit keys, NT a power of two");
  constexpr int VT = 16;
  constexpr int NV = NT * VT;
  constexpr int LOGNV = __builtin_ctz(NV);
  extern __shared__ __align__(128) uint32_t s[];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint64_t base = (block0 + blockIdx.x) * NV;
  const int cnt = ALIGNED ? NV : static_cast<int>((n - base) < NV ? (n - base) : NV);

  uint32_t x[VT];
  if constexpr (ALIGNED) {
    const uint4 *src = reinterpret_cast<const uint4 *>(in + base);
#pragma unroll
    for (int m = 0; m < VT / 4; ++m) {
      const uint4 v = __ldg(src + tid + m * NT);
      x[4 * m + 0] = order_u32<KT>(static_cast<typename KT::T>(v.x));
      x[4 * m + 1] = order_u32<KT>(static_cast<typename KT::T>(v.y));
      x[4 * m + 2] = order_u32<KT>(static_cast<typename KT::T>(v.z));
      x[4 * m + 3] = order_u32<KT>(static_cast<typename KT::T>(v.w));
    }
  } else {
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      const int q = tid + k * NT;
      x[k] = q < cnt ? order_u32<KT>(in[base + q]) : 0xFFFFFFFFu;
    }
  }
  batcher_u32<VT>(x);

  // ---- levels 5..8 (runs 16 -> 256) inside the warp: flip + shfl ----
#pragma unroll
  for (int m = 1; m <= 4; ++m) {
    const int g = 1 << m;
    {
      const bool upper = (lane & (g - 1)) >= (g >> 1);
#pragma unroll
      for (int q = 0; q < VT / 2; ++q) {
        const uint32_t a = __shfl_xor_sync(0xffffffffu, x[VT - 1 - q], g - 1);
        const uint32_t b = __shfl_xor_sync(0xffffffffu, x[q], g - 1);
        ce_dir(x[q], a, upper);
        ce_dir(x[VT - 1 - q], b, upper);
      }
    }
#pragma unroll
    for (int st = g >> 2; st >= 1; st >>= 1) {
      const bool upper = (lane & st) != 0;
#pragma unroll
      for (int q = 0; q < VT; ++q)
        ce_dir(x[q], __shfl_xor_sync(0xffffffffu, x[q], st), upper);
    }
    reg_stages<8, 4>(x);
  }
  // ---- levels 9..LOGNV through register layouts ----
  tr_levels<9, LOGNV, NT>(x, s, tid);

  const int p0 = tid * VT;
  if constexpr (ALIGNED) {
    uint4 *dst = reinterpret_cast<uint4 *>(out + base + p0);
#pragma unroll
    for (int m = 0; m < VT / 4; ++m) {
      uint4 v;
      v.x = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 0]));
      v.y = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 1]));
      v.z = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 2]));
      v.w = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 3]));
      dst[m] = v;
    }
  } else {
#pragma unroll
    for (int q = 0; q < VT; ++q)
      if (p0 + q < cnt)
        out[base + p0 + q] = from_order_u32<KT>(x[q]);
  }
}

}  // namespace mpb
