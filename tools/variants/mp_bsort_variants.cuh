// mp_bsort_variants.cuh -- measured-slower variants taken out of the product build
// (round 2).  Kept for reference and for A/B experiments: NOT compiled into
// libmergepath_b200.so.  Each block is headed by what it was and the B200
// measurement that retired it; it needs the product headers
// (paper_1406_2628_b200/csrc/) to compile.
#pragma once

// ===== K3b block_sort_bare_kernel (MP_BLOCK_SORT=bare): 4352-key runs; B200 2^30 u32 block pass 9.0 ms vs K3w 7.1 ms =====
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



// ===== K3b smem size =====
// smem: the finest level (NT runs of VT) has the most sentinel words
template <int NT, int VT>
__host__ __device__ constexpr uint32_t bare_sort_smem_bytes() {
  return static_cast<uint32_t>(NT) * (VT + 1) * 4 + 64;
}



// ===== K3t block_sort_tr_kernel (MP_K3W=tr): bitonic network in registers with smem transposes; B200 8.44 ms vs K3w 8.26 ms =====
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



// ===== K3w double-load merge step (MP_K3W_DOUBLE_LOAD=1): ALU pipe 85 -> 69 % but 7.80 -> 8.20 ms =====
// MP_K3W_DOUBLE_LOAD=1 (compile-time A/B): the merge step reloads both heads
// with FMA-pipe addressing and no selects.  B200: ALU pipe 85 % -> 69 %, but
// the longer dependent chain per output (IMAD.HI -> IMAD -> IMAD -> LDS)
// makes K3w latency-bound: 7.80 -> 8.20 ms.  Off.
#ifndef MP_K3W_DOUBLE_LOAD
#define MP_K3W_DOUBLE_LOAD 0
#endif
// smem word k of a 32-aligned padded run at shared address `base`:
// base + 4 * (k + (k >> 5)), as IMAD.HI / IMAD (FMA pipe) instead of the
// LEA.HI / LEA pair ptxas picks for pad32 (ALU pipe, K3w's bottleneck).
__device__ __forceinline__ uint32_t lds_padded(uint32_t base, uint32_t k) {
  uint32_t h, a, v;
  asm("mul.hi.u32 %0, %1, 134217728;" : "=r"(h) : "r"(k));
  asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a) : "r"(k), "r"(base));
  asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a) : "r"(h), "r"(a));
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}



// ===== K3w double-load merge loop =====
#if MP_K3W_DOUBLE_LOAD
    // A cursor i only; B's is diag + q - i.  Both heads are reloaded every
    // step (one more LDS, no selects), addresses via IMAD.HI / IMAD on the
    // FMA pipe: aO, bO are multiples of 32, so pad32(run + k) =
    // pad32(run) + k + (k >> 5).
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(s + pad32(aO)));
    const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(s + pad32(bO)));
    uint32_t i = static_cast<uint32_t>(lo);
    uint32_t ua = lds_padded(sa, i), vb = lds_padded(sb, static_cast<uint32_t>(diag) - i);
#pragma unroll
    for (int q = 0; q < VT; ++q) {
      x[q] = min(ua, vb);
      i += ua <= vb ? 1u : 0u;  // ties take A
      ua = lds_padded(sa, i);
      vb = lds_padded(sb, static_cast<uint32_t>(diag + q + 1) - i);
    }
#else
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
#endif

// ===== K3w passes with FMA-pipe smem addressing (MP_K3W_FMA_ADDR, round 2):
// every padded LDS address of the split searches and merge loops formed by
// mul.hi / mad.lo (IMAD.HI / IMAD) instead of LEA.HI / LEA.  B200
// (tools/ab_k3w_fma.sh, 512 x 32): ALU pipe 80 -> 74 %, FMA 14 %, but K3w
// 8.05 -> 8.19 ms and the sort 26.27 -> 26.42 ms (a three-deep IMAD chain
// on every load).  Not kept.
//   uint32_t h, a;  // k -> shared address of padded word k
//   asm("mul.hi.u32 %0, %1, 134217728;" : "=r"(h) : "r"(k));
//   asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a) : "r"(k), "r"(base));
//   asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a) : "r"(h), "r"(a));
