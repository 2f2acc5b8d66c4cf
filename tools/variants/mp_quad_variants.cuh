// mp_quad_variants.cuh -- measured-slower variants taken out of the product build
// (round 2).  Kept for reference and for A/B experiments: NOT compiled into
// libmergepath_b200.so.  Each block is headed by what it was and the B200
// measurement that retired it; it needs the product headers
// (paper_1406_2628_b200/csrc/) to compile.
#pragma once

// ===== K5e fixed-step split search (MP_QUAD_FIXED_SEARCH=1): 1.35 vs 1.40 G instructions but 2.30 vs 2.07 ms =====
// MP_QUAD_FIXED_SEARCH=1 (compile-time A/B): K5e's splits by fixed-step
// binary lifting instead of the while loop.  B200: 1.35 vs 1.40 G
// instructions but K5e 2.30 vs 2.07 ms (sort 30.8 vs 29.0 ms) -- every
// warp now pays the longest chain of 13 dependent probe pairs.  Off.
#ifndef MP_QUAD_FIXED_SEARCH
#define MP_QUAD_FIXED_SEARCH 0
#endif
// Split of the smem windows A[0, na), B[0, nb) on diagonal d (core.hpp:110
// predicate, ties to A) by binary lifting with a fixed number of steps K
// (2^K > min(na, nb)): no loop branch, no divergence between lanes.  Probe
// indices are clamped into the windows' neighbourhood; a clamped probe never
// moves the answer.
template <class KT, int K>
__device__ __forceinline__ int split_fixed(const char *smem, uint32_t oA, int na,
                                           uint32_t oB, int nb, int d) {
  using T = typename KT::T;
  constexpr uint32_t KS = sizeof(T);
  int i = d > nb ? d - nb : 0;
  const int hi = d < na ? d : na;
#pragma unroll
  for (int step = 1 << (K - 1); step > 0; step >>= 1) {
    const int j = i + step;  // does the split lie at or beyond j?
    const int jj = j < hi ? j : hi;
    const bool stay = take_b<KT>(lds<T>(smem, oB + (d - jj) * KS), lds<T>(smem, oA + (jj - 1) * KS));
    i = (j <= hi && !stay) ? j : i;
  }
  return i;
}



// ===== K5e alternative split searches =====
#elif MP_QUAD_FIXED_SEARCH
    // min(na, nb) <= T / 2 <= 2^13 - 1 for tiles up to 16382 outputs
    const int lo = split_fixed<KT, 13>(smem, oA, na, oB, nb, d1);
#else
    int lo = d1 > nb ? d1 - nb : 0;
    int hi = d1 < na ? d1 : na;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (take_b<KT>(lds<T_>(smem, oB + (d1 - 1 - mid) * KS), lds<T_>(smem, oA + mid * KS)))
        hi = mid;
      else
        lo = mid + 1;
    }
#endif


// ===== K5e alternative split searches =====
#elif MP_QUAD_FIXED_SEARCH
    const int lo = split_fixed<KT, 13>(smem, oX, nx, oY, ny, d2);
#else
    int lo = d2 > ny ? d2 - ny : 0;
    int hi = d2 < nx ? d2 : nx;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (take_b<KT>(lds<T_>(smem, oY + (d2 - 1 - mid) * KS), lds<T_>(smem, oX + mid * KS)))
        hi = mid;
      else
        lo = mid + 1;
    }
#endif


// ===== K5e2 quad_tile2_kernel (MP_QUAD_ILP2=1): two merge slots per thread; 2.50 vs 2.07 ms per pass =====
// K5e2: K5e with two merge slots per thread.  K5e is latency-bound (B200:
// 59 % issue, barrier and short-scoreboard stalls on top, and a fixed-step
// search that lengthens the chains made it slower), so each thread carries
// two independent chains: in both phases it owns slots 2t and 2t+1 (two
// diagonals VT apart), searches them in one interleaved loop and merges them
// back to back (the unrolled serial merges are independent, so their steps
// interleave).  Same smem layout, sentinels and bytes as K5e.
template <class KT, int VT>
__device__ __forceinline__ void split2(const char *smem, uint32_t oA0, int na0, uint32_t oB0,
                                       int nb0, int d0, bool on0, uint32_t oA1, int na1,
                                       uint32_t oB1, int nb1, int d1, bool on1, int &r0,
                                       int &r1) {
  using T = typename KT::T;
  constexpr uint32_t KS = sizeof(T);
  int lo0 = d0 > nb0 ? d0 - nb0 : 0, hi0 = on0 ? (d0 < na0 ? d0 : na0) : lo0;
  int lo1 = d1 > nb1 ? d1 - nb1 : 0, hi1 = on1 ? (d1 < na1 ? d1 : na1) : lo1;
  while (lo0 < hi0 || lo1 < hi1) {
    if (lo0 < hi0) {
      const int mid = (lo0 + hi0) >> 1;
      if (take_b<KT>(lds<T>(smem, oB0 + (d0 - 1 - mid) * KS), lds<T>(smem, oA0 + mid * KS)))
        hi0 = mid;
      else
        lo0 = mid + 1;
    }
    if (lo1 < hi1) {
      const int mid = (lo1 + hi1) >> 1;
      if (take_b<KT>(lds<T>(smem, oB1 + (d1 - 1 - mid) * KS), lds<T>(smem, oA1 + mid * KS)))
        hi1 = mid;
      else
        lo1 = mid + 1;
    }
  }
  r0 = lo0;
  r1 = lo1;
}

template <class KT, int NT, int VT>
__host__ __device__ constexpr uint32_t quad2_smem_bytes() {
  return 64 + 2 * NT * VT * sizeof(typename KT::T) + 4 * quad_gap_bytes<KT, VT>() + 64;
}

template <class KT, int NT, int VT>
__global__ void __launch_bounds__(NT, 800 / NT)
    quad_tile2_kernel(const typename KT::T *__restrict__ src,
                      typename KT::T *__restrict__ dst, uint64_t n, uint64_t w,
                      uint32_t lg4w, uint32_t T, const QuadPt *__restrict__ Q) {
  using T_ = typename KT::T;
  constexpr uint32_t KS = sizeof(T_);
  extern __shared__ __align__(128) char smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  const int tid = threadIdx.x;
  struct Hdr {
    uint32_t oW[4];
    int cnt[4];
    unsigned long long o0;
  };
  Hdr *hdr = reinterpret_cast<Hdr *>(smem + 16);
  constexpr uint32_t kWin0 = 64;
  if (tid < 32) {
    const uint64_t t = blockIdx.x;
    const uint64_t pos = t * T;
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
    int cnt[4];
    const char *gW[4];
    uint32_t oW[4];
    uint32_t at = kWin0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      cnt[r] = static_cast<int>(p1.i[r] - p0.i[r]);
      gW[r] = reinterpret_cast<const char *>(src + q.S + r * w + p0.i[r]);
      oW[r] = mirror_off(at, gW[r]);
      at = oW[r] + cnt[r] * KS + quad_gap_bytes<KT, VT>();
    }
    const int l = tid;
    if (l == 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        hdr->oW[r] = oW[r];
        hdr->cnt[r] = cnt[r];
      }
      hdr->o0 = pos;
      mbar_init(bar, 1);
      fence_mbar_init();
      uint32_t lo[4], ib[4], tx = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        ib[r] = interior_bytes(gW[r], cnt[r] * KS, &lo[r]);
        tx += ib[r];
      }
      mbar_arrive_expect_tx(bar, tx);
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (ib[r])
          bulk_g2s(smem + oW[r] + lo[r], gW[r] + lo[r], ib[r], bar);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if ((l >> 3) == r)
        stage_edges<KS>(smem, oW[r], gW[r], cnt[r] * KS, l & 7);
    if (l < VT) {
      *reinterpret_cast<T_ *>(smem + oW[0] + (cnt[0] + l) * KS) = KT::max_key();
      *reinterpret_cast<T_ *>(smem + oW[2] + (cnt[2] + l) * KS) = KT::max_key();
    } else if (l == VT) {
      *reinterpret_cast<T_ *>(smem + oW[1] + cnt[1] * KS) = KT::max_key();
      *reinterpret_cast<T_ *>(smem + oW[3] + cnt[3] * KS) = KT::max_key();
    }
  }
  __syncthreads();
  uint32_t oW[4];
  int cnt[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    oW[r] = hdr->oW[r];
    cnt[r] = hdr->cnt[r];
  }
  const uint64_t o0 = hdr->o0;
  const int nx = cnt[0] + cnt[1], ny = cnt[2] + cnt[3], total = nx + ny;
  mbar_wait(bar, 0);

  // ---- phase 1: slots 2t, 2t+1 of the X slots then the Y slots ----
  T_ k0[VT], k1[VT];
  uint32_t vals[VT];
  const int tx = (nx + VT - 1) / VT, ty = (ny + VT - 1) / VT;
  const int s0 = 2 * tid, s1 = 2 * tid + 1;
  const int side0 = s0 >= tx, side1 = s1 >= tx;
  const int u0 = s0 - side0 * tx, u1 = s1 - side1 * tx;
  const bool on0 = side0 ? u0 < ty : true, on1 = side1 ? u1 < ty : true;
  const uint32_t oA0 = side0 ? oW[2] : oW[0], oB0 = side0 ? oW[3] : oW[1];
  const uint32_t oA1 = side1 ? oW[2] : oW[0], oB1 = side1 ? oW[3] : oW[1];
  const int na0 = side0 ? cnt[2] : cnt[0], nb0 = side0 ? cnt[3] : cnt[1];
  const int na1 = side1 ? cnt[2] : cnt[0], nb1 = side1 ? cnt[3] : cnt[1];
  const int e0 = u0 * VT, e1 = u1 * VT;
  {
    int r0, r1;
    split2<KT, VT>(smem, oA0, na0, oB0, nb0, e0, on0, oA1, na1, oB1, nb1, e1, on1, r0, r1);
    if (on0)
      serial_merge<KT, VT, false, true>(smem, oA0, na0, oB0, nb0, 0, 0, r0, e0 - r0, k0, vals);
    if (on1)
      serial_merge<KT, VT, false, true>(smem, oA1, na1, oB1, nb1, 0, 0, r1, e1 - r1, k1, vals);
  }
  __syncthreads();  // every window consumed
  const uint32_t oX = oW[0], oY = oW[2];
  auto put = [&](const T_(&k)[VT], bool on, int side, int e) {
    if (!on)
      return;
    const uint32_t op = side ? oY : oX;
    const int lim = side ? ny : nx;
    if (e + VT <= lim) {
#pragma unroll
      for (int q = 0; q < VT; ++q)
        *reinterpret_cast<T_ *>(smem + op + (e + q) * KS) = k[q];
    } else {
#pragma unroll
      for (int q = 0; q < VT; ++q)
        if (e + q < lim)
          *reinterpret_cast<T_ *>(smem + op + (e + q) * KS) = k[q];
    }
  };
  put(k0, on0, side0, e0);
  put(k1, on1, side1, e1);
  if (tid >= NT - 32) {
    const int l = tid - (NT - 32);
    if (l < VT)
      *reinterpret_cast<T_ *>(smem + oX + (nx + l) * KS) = KT::max_key();
    else if (l == VT)
      *reinterpret_cast<T_ *>(smem + oY + ny * KS) = KT::max_key();
  }
  __syncthreads();

  // ---- phase 2: out = merge(X, Y), diagonals 2t*VT and (2t+1)*VT ----
  const int f0 = s0 * VT, f1 = s1 * VT;
  const bool p0 = f0 < total, p1 = f1 < total;
  {
    int r0, r1;
    split2<KT, VT>(smem, oX, nx, oY, ny, f0, p0, oX, nx, oY, ny, f1, p1, r0, r1);
    if (p0)
      serial_merge<KT, VT, false, true>(smem, oX, nx, oY, ny, 0, 0, r0, f0 - r0, k0, vals);
    if (p1)
      serial_merge<KT, VT, false, true>(smem, oX, nx, oY, ny, 0, 0, r1, f1 - r1, k1, vals);
  }
  __syncthreads();  // X and Y consumed

  T_ *out = dst + o0;
  const uint32_t oS = mirror_off(16, out);
  auto stage = [&](const T_(&k)[VT], int f) {
    if (f + VT <= total) {
#pragma unroll
      for (int q = 0; q < VT; ++q)
        *reinterpret_cast<T_ *>(smem + oS + (f + q) * KS) = k[q];
    } else if (f < total) {
#pragma unroll
      for (int q = 0; q < VT; ++q)
        if (f + q < total)
          *reinterpret_cast<T_ *>(smem + oS + (f + q) * KS) = k[q];
    }
  };
  stage(k0, f0);
  stage(k1, f1);
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



// ===== K5p quad_persist_kernel (MP_QUAD_PERSIST, round 2): K5e as a
// persistent, warp-specialised kernel (producer warp: split points, window
// layout and edges one tile ahead, bulk loads/stores; NTC consumer threads:
// K5e's two merge phases with named barriers).  B200, 2^30 u32 sort,
// 30 steps each, 1965 MHz: K5e 27.31-27.37 ms; K5p 640x27 double-buffered
// (1 CTA/SM, 20 consumer warps) 34.39 ms; 992x17 x2 buffers 32.98; 640x27
// x3 buffers 33.16; 896x19 x2 32.97; 640x27 single buffer, 2 CTAs/SM
// 33.14 (K5p 2.85 ms per pass vs K5e 2.15, issue 46.7 %).  ncu stall
// sampling (profiles/r02/k5_stalls.md): K5e loses 55 % of its warp samples
// at the barrier behind warp 0's per-tile setup, but the persistent form
// cannot keep 40 consumer warps per SM with two 64 KB tile buffers each, and
// with 20 the dependent LDS chains of the merges are exposed.  Not kept.
// ---------------------------------------------------------------------------
// K5p: K5e as a persistent, warp-specialised kernel.  One CTA per SM walks
// the tiles t = blockIdx.x, + gridDim.x, ...; NBUF smem buffers hold
// consecutive tiles.  A producer warp (the last warp) prepares tile k + NBUF
// while NTC consumer threads merge tile k:
//   producer: reads the tile's 4-way split points (Q[t], Q[t+1]) from HBM,
//     lays out the four run windows in the free buffer, issues their bulk
//     copies (TMA engine) on the buffer's `full` mbarrier, stages the
//     unaligned window edges and the sentinels with ordinary stores; then,
//     once the consumers have staged a tile's output (`staged` mbarrier),
//     issues its bulk store and waits for the store to have read the
//     buffer before refilling it;
//   consumers: wait `full`, run K5e's two merge phases (same code, same
//     bytes) on that buffer with named barriers among themselves only,
//     stage the output, arrive on `staged`.
// So the split-point loads, the window copies and the output stores of
// neighbouring tiles overlap the merges: K5e paid a global-load latency and
// a bulk-copy wait per tile with every thread of the CTA idle.
// ---------------------------------------------------------------------------
template <class KT, int NTC, int VT, int NBUF, uint32_t TT>
struct QuadPersistCfg {
  static constexpr uint32_t KS = sizeof(typename KT::T);
  // one tile's four windows (TT elements) + gaps/sentinels + alignment slack
  static constexpr uint32_t BUF = ((TT * KS + 4 * quad_gap_bytes<KT, VT>() + 256) + 127) & ~127u;
  static constexpr uint32_t HDR = 512;  // mbarriers + per-buffer headers
  static constexpr uint32_t bytes = HDR + NBUF * BUF;
  static_assert(NTC * VT >= int(TT) + 2 * VT && (VT & 1) && NTC % 32 == 0, "K5p shape");
  static_assert(NBUF * (16 + 48) + 64 <= HDR, "K5p header");
};

struct QuadHdr {
  uint32_t oW[4];
  int cnt[4];
  unsigned long long o0;
  unsigned long long pad;
};

__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <class KT, int NTC, int VT, int NBUF, uint32_t TT>
__global__ void __launch_bounds__(NTC + 32, NBUF == 1 ? 2 : 1)
    quad_persist_kernel(const typename KT::T *__restrict__ src,
                        typename KT::T *__restrict__ dst, uint64_t n, uint64_t w,
                        uint32_t lg4w, const QuadPt *__restrict__ Q, uint64_t tiles) {
  using T_ = typename KT::T;
  using Cfg = QuadPersistCfg<KT, NTC, VT, NBUF, TT>;
  constexpr uint32_t KS = sizeof(T_);
  extern __shared__ __align__(128) char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem);
  uint64_t *staged = full + NBUF;
  QuadHdr *hdr = reinterpret_cast<QuadHdr *>(smem + 64);
  auto buf = [&](int b) { return smem + Cfg::HDR + b * Cfg::BUF; };
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(full + b, 1);
      mbar_init(staged + b, 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  constexpr uint32_t kWin0 = 64;

  if (tid >= NTC) {  // ---------------- producer warp ----------------
    const int l = tid - NTC;
    // Everything about tile t that needs HBM round trips -- its split
    // points, window layout and the unaligned window edges (lane l holds
    // edge element l & 7 of window l >> 3) -- is read one tile ahead, while
    // the consumers merge; filling a buffer then only waits for the buffer.
    struct Prep {
      uint64_t pos;
      const char *gW[4];
      uint32_t oW[4];
      int cnt[4];
      T_ edge;
      uint32_t edge_off;  // byte offset in the buffer (~0u: none)
    };
    auto prepare = [&](uint64_t t) {
      Prep p;
      p.pos = t * TT;
      const uint64_t g = p.pos >> lg4w;
      const QuadGroup q = quad_group(g, n, w);
      const QuadPt p0 = Q[t];
      QuadPt p1;
      const uint64_t gend = q.S + q.l[0] + q.l[1] + q.l[2] + q.l[3];
      if (p.pos + TT < gend) {
        p1 = Q[t + 1];
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r)
          p1.i[r] = q.l[r];
      }
      uint32_t at = kWin0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        p.cnt[r] = static_cast<int>(p1.i[r] - p0.i[r]);
        p.gW[r] = reinterpret_cast<const char *>(src + q.S + r * w + p0.i[r]);
        p.oW[r] = mirror_off(at, p.gW[r]);
        at = p.oW[r] + p.cnt[r] * KS + quad_gap_bytes<KT, VT>();
      }
      // this lane's edge element (stage_edges' split, as a load now and a
      // store at fill time): heads [0, lo) and tails [hi, bytes) < 32 B
      const int r = l >> 3, e = l & 7;
      const uintptr_t s0 = reinterpret_cast<uintptr_t>(p.gW[r]);
      const uint32_t bytes = p.cnt[r] * KS;
      const uintptr_t is = (s0 + 15) & ~uintptr_t(15);
      const uintptr_t ie = (s0 + bytes) & ~uintptr_t(15);
      const uint32_t lo = ie > is ? static_cast<uint32_t>(is - s0) : bytes;
      const uint32_t hi = ie > is ? static_cast<uint32_t>(ie - s0) : bytes;
      const uint32_t nh = lo / KS, nt = (bytes - hi) / KS;
      p.edge_off = ~0u;
      if (static_cast<uint32_t>(e) < nh + nt) {
        const uint32_t o = static_cast<uint32_t>(e) < nh ? e * KS : hi + (e - nh) * KS;
        p.edge = *reinterpret_cast<const T_ *>(p.gW[r] + o);
        p.edge_off = p.oW[r] + o;
      }
      return p;
    };
    auto fill = [&](const Prep &p, int b) {
      char *base = buf(b);
      if (p.edge_off != ~0u)
        *reinterpret_cast<T_ *>(base + p.edge_off) = p.edge;
      if (l < VT) {  // sentinels behind the windows (outside the bulk copies)
        *reinterpret_cast<T_ *>(base + p.oW[0] + (p.cnt[0] + l) * KS) = KT::max_key();
        *reinterpret_cast<T_ *>(base + p.oW[2] + (p.cnt[2] + l) * KS) = KT::max_key();
      } else if (l == VT) {
        *reinterpret_cast<T_ *>(base + p.oW[1] + p.cnt[1] * KS) = KT::max_key();
        *reinterpret_cast<T_ *>(base + p.oW[3] + p.cnt[3] * KS) = KT::max_key();
      }
      if (l == 0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          hdr[b].oW[r] = p.oW[r];
          hdr[b].cnt[r] = p.cnt[r];
        }
        hdr[b].o0 = p.pos;
      }
      __syncwarp();
      if (l == 0) {
        uint32_t lo[4], ib[4], tx = 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          ib[r] = interior_bytes(p.gW[r], p.cnt[r] * KS, &lo[r]);
          tx += ib[r];
        }
        mbar_arrive_expect_tx(full + b, tx);
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (ib[r])
            bulk_g2s(base + p.oW[r] + lo[r], p.gW[r] + lo[r], ib[r], full + b);
      }
    };
    // issue the bulk store of the tile staged in buffer b (lane 0), then
    // wait until the store has read the buffer
    auto store_out = [&](int b) {
      char *base = buf(b);
      const QuadHdr &h = hdr[b];
      const int total = h.cnt[0] + h.cnt[1] + h.cnt[2] + h.cnt[3];
      T_ *out = dst + h.o0;
      const uint32_t oS = mirror_off(16, out);
      uint32_t lo;
      const uint32_t ib = interior_bytes(reinterpret_cast<const char *>(out),
                                         static_cast<uint32_t>(total) * KS, &lo);
      if (l == 0 && ib) {
        bulk_s2g(reinterpret_cast<char *>(out) + lo, base + oS + lo, ib);
        bulk_commit();
        bulk_wait_read0();
      }
      __syncwarp();
    };
    uint64_t k = 0;
    uint64_t t = blockIdx.x;
    if (t < tiles) {
      Prep next = prepare(t);
      for (; t < tiles; t += gridDim.x, ++k) {
        const Prep cur = next;
        const int b = static_cast<int>(k % NBUF);
        const uint32_t use = static_cast<uint32_t>(k / NBUF);
        if (t + gridDim.x < tiles)  // tile k + 1's HBM round trips, now
          next = prepare(t + gridDim.x);
        if (k >= NBUF) {  // buffer b still holds tile k - NBUF: store it first
          mbar_wait(staged + b, (use - 1) & 1);
          store_out(b);
        }
        fill(cur, b);
      }
    }
    // drain: the last min(k, NBUF) tiles' outputs
    for (uint64_t j = k > NBUF ? k - NBUF : 0; j < k; ++j) {
      const int b = static_cast<int>(j % NBUF);
      mbar_wait(staged + b, static_cast<uint32_t>(j / NBUF) & 1);
      store_out(b);
    }
    if (l == 0)
      bulk_wait0();  // the stores' global writes complete before the CTA exits
    return;
  }

  // ---------------- consumers ----------------
  uint64_t k = 0;
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
    const int b = static_cast<int>(k % NBUF);
    mbar_wait(full + b, static_cast<uint32_t>(k / NBUF) & 1);
    const char *base = buf(b);
    char *wbase = buf(b);
    uint32_t oW[4];
    int cnt[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      oW[r] = hdr[b].oW[r];
      cnt[r] = hdr[b].cnt[r];
    }
    const uint64_t o0 = hdr[b].o0;
    const int nx = cnt[0] + cnt[1], ny = cnt[2] + cnt[3], total = nx + ny;

    // phase 1: X = merge(R0w, R1w), Y = merge(R2w, R3w) (threads dealt by size)
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
      const int lo = split_predicted<KT, MP_QUAD_PRED_LOGW>(
          base, oA, na, oB, nb, d1, static_cast<float>(na) / static_cast<float>(na + nb));
      serial_merge<KT, VT, false, true>(base, oA, na, oB, nb, 0, 0, lo, d1 - lo, keys, vals);
    }
    consumer_sync(NTC);  // every window consumed
    const uint32_t oX = oW[0], oY = oW[2];
    if (act1) {
      const uint32_t op = side ? oY : oX;
      const int lim = side ? ny : nx;
      if (d1 + VT <= lim) {
#pragma unroll
        for (int e = 0; e < VT; ++e)
          *reinterpret_cast<T_ *>(wbase + op + (d1 + e) * KS) = keys[e];
      } else {
#pragma unroll
        for (int e = 0; e < VT; ++e)
          if (d1 + e < lim)
            *reinterpret_cast<T_ *>(wbase + op + (d1 + e) * KS) = keys[e];
      }
    }
    if (tid >= NTC - 32) {  // the last consumer warp: X's VT sentinels and Y's one
      const int l = tid - (NTC - 32);
      if (l < VT)
        *reinterpret_cast<T_ *>(wbase + oX + (nx + l) * KS) = KT::max_key();
      else if (l == VT)
        *reinterpret_cast<T_ *>(wbase + oY + ny * KS) = KT::max_key();
    }
    consumer_sync(NTC);

    // phase 2: out = merge(X, Y), ties to X
    const int d2 = tid * VT;
    if (d2 < total) {
      const int lo = split_predicted<KT, MP_QUAD_PRED_LOGW>(
          base, oX, nx, oY, ny, d2, static_cast<float>(nx) / static_cast<float>(total));
      serial_merge<KT, VT, false, true>(base, oX, nx, oY, ny, 0, 0, lo, d2 - lo, keys, vals);
    }
    consumer_sync(NTC);  // X and Y consumed

    T_ *out = dst + o0;
    const uint32_t oS = mirror_off(16, out);
    // the 16 B-aligned interior goes out through the producer's bulk store;
    // the < 16 B head [0, h_end) and tail [t_beg, total) straight from the
    // registers of the threads that own them (nothing reads the buffer
    // after `staged`)
    uint32_t olo;
    const uint32_t oib = interior_bytes(reinterpret_cast<const char *>(out),
                                        static_cast<uint32_t>(total) * KS, &olo);
    const int h_end = oib ? static_cast<int>(olo / KS) : total;
    const int t_beg = oib ? static_cast<int>((olo + oib) / KS) : total;
    if (d2 >= h_end && d2 + VT <= t_beg) {
#pragma unroll
      for (int e = 0; e < VT; ++e)
        *reinterpret_cast<T_ *>(wbase + oS + (d2 + e) * KS) = keys[e];
    } else if (d2 < total) {
#pragma unroll
      for (int e = 0; e < VT; ++e) {
        const int x = d2 + e;
        if (x < h_end || (x >= t_beg && x < total))
          out[x] = keys[e];
        else if (x < total)
          *reinterpret_cast<T_ *>(wbase + oS + x * KS) = keys[e];
      }
    }
    fence_proxy_async_smem();
    consumer_sync(NTC);
    if (tid == 0)
      mbar_arrive(staged + b);
  }
}



// ===== K5e with two merge chains per thread (MP_K5E_CHAINS=2, round 2):
// each thread's VT outputs as two halves from two splits (the second by a
// short search bounded by the first), stepped alternately for ILP.  B200
// (tools/ab_k5e_chains.sh): K5e 2.09 -> 2.26 ms per pass, sort 26.3 ->
// 27.6-27.7 ms (48 registers either way; the extra search costs more than
// the shorter chains save).  Not kept.
// Two independent merge chains per thread (bare keys on sentinels, as
// serial_merge SENT): outputs [0, H) from split (i0, j0) and [H, VT) from
// split (i1, j1), stepped alternately so each dependent LDS -> compare ->
// select chain has the other one's instructions to hide behind.
template <class KT, int VT, int H>
__device__ __forceinline__ void serial_merge2(const char *smem, uint32_t oA, uint32_t oB,
                                              int i0, int j0, int i1, int j1,
                                              typename KT::T (&keys)[VT]) {
  using T = typename KT::T;
  constexpr uint32_t KS = sizeof(T);
  uint32_t pa0 = oA + i0 * KS, pb0 = oB + j0 * KS;
  uint32_t pa1 = oA + i1 * KS, pb1 = oB + j1 * KS;
  T ka0 = lds<T>(smem, pa0), kb0 = lds<T>(smem, pb0);
  T ka1 = lds<T>(smem, pa1), kb1 = lds<T>(smem, pb1);
#pragma unroll
  for (int k = 0; k < H; ++k) {
    {
      const bool tb = take_b<KT>(kb0, ka0);
      keys[k] = tb ? kb0 : ka0;
      pa0 += tb ? 0u : KS;
      pb0 += tb ? KS : 0u;
      const T nxt = lds<T>(smem, tb ? pb0 : pa0);
      kb0 = tb ? nxt : kb0;
      ka0 = tb ? ka0 : nxt;
    }
    if (H + k < VT) {
      const bool tb = take_b<KT>(kb1, ka1);
      keys[H + k] = tb ? kb1 : ka1;
      pa1 += tb ? 0u : KS;
      pb1 += tb ? KS : 0u;
      const T nxt = lds<T>(smem, tb ? pb1 : pa1);
      kb1 = tb ? nxt : kb1;
      ka1 = tb ? ka1 : nxt;
    }
  }
}

// Split on diagonal d knowing the split on diagonal d0 < d is a0: it lies
// in [a0, a0 + (d - d0)] (and the usual range) -- a short search.
template <class KT>
__device__ __forceinline__ int split_after(const char *smem, uint32_t oA, int na, uint32_t oB,
                                           int nb, int d, int d0, int a0) {
  using T = typename KT::T;
  constexpr uint32_t KS = sizeof(T);
  int lo = max(d > nb ? d - nb : 0, a0);
  int hi = min(d < na ? d : na, a0 + (d - d0));
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (take_b<KT>(lds<T>(smem, oB + (d - 1 - mid) * KS), lds<T>(smem, oA + mid * KS)))
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

#ifndef MP_K5E_CHAINS
#define MP_K5E_CHAINS 2
#endif



// ===== K5f quad_tile_split_kernel (MP_K5F, round 2): X and Y in their own
// smem region so both merge phases store each output as produced (no VT
// output registers, 3 barriers instead of 5), at twice the smem per tile.
// B200 (tools/ab_k5f.sh, 2^30 sort, 50 steps): K5e 26.28-26.31 ms; K5f at
// 8192-output tiles 640 x 13, 3 CTAs/SM: 33.13 ms (K5f 2.79 ms per pass at
// 65 % issue, K4q + K4r 0.36 ms at the 8192 spacing); 448 x 19: 29.66-29.70
// (2.35 ms); 16384 tiles 1024 x 17, 1 CTA/SM: 39.93.  Not kept.
// ---------------------------------------------------------------------------
// K5f: the fused pass with X and Y in their own smem region.  K5e writes X
// and Y over the input windows and the output over X and Y, so every merge
// first collects its VT outputs in registers and waits at a barrier before
// storing them (VT registers per thread, two CTAs of 20 warps per SM).
// Here the merges store each output as it is produced: phase 1 into the
// X/Y region, phase 2 into the (dead) input region as the output staging.
// No output registers, three barriers instead of five -- at the price of
// twice the smem per tile, so the tile is TILE outputs (8192: three CTAs
// per SM) and K4q/K4r run at that spacing.
// ---------------------------------------------------------------------------
template <class KT, int VT, int TILE>
__host__ __device__ constexpr uint32_t quad_split_in_bytes() {
  return ((64 + TILE * sizeof(typename KT::T) + 4 * quad_gap_bytes<KT, VT>() + 64) + 127) & ~127u;
}
template <class KT, int VT, int TILE>
__host__ __device__ constexpr uint32_t quad_split_smem_bytes() {
  return quad_split_in_bytes<KT, VT, TILE>() + TILE * sizeof(typename KT::T) +
         (VT + 1) * sizeof(typename KT::T) + 64;
}

// Serial stable merge of up to VT outputs (bare keys on sentinels) from split
// (i, j) of the smem windows at oA / oB, each output stored at once to smem
// offset oOut + k * KS (k < cnt).
template <class KT, int VT>
__device__ __forceinline__ void merge_store_smem(char *smem, uint32_t oA, uint32_t oB, int i,
                                                 int j, uint32_t oOut, int cnt) {
  using T = typename KT::T;
  constexpr uint32_t KS = sizeof(T);
  uint32_t pa = oA + i * KS, pb = oB + j * KS;
  T ka = lds<T>(smem, pa), kb = lds<T>(smem, pb);
  if (cnt >= VT) {
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      const bool tb = take_b<KT>(kb, ka);
      *reinterpret_cast<T *>(smem + oOut + k * KS) = tb ? kb : ka;
      pa += tb ? 0u : KS;
      pb += tb ? KS : 0u;
      const T nxt = lds<T>(smem, tb ? pb : pa);
      kb = tb ? nxt : kb;
      ka = tb ? ka : nxt;
    }
  } else {
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      if (k >= cnt)
        break;
      const bool tb = take_b<KT>(kb, ka);
      *reinterpret_cast<T *>(smem + oOut + k * KS) = tb ? kb : ka;
      pa += tb ? 0u : KS;
      pb += tb ? KS : 0u;
      const T nxt = lds<T>(smem, tb ? pb : pa);
      kb = tb ? nxt : kb;
      ka = tb ? ka : nxt;
    }
  }
}

template <class KT, int NT, int VT, int TILE, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    quad_tile_split_kernel(const typename KT::T *__restrict__ src,
                           typename KT::T *__restrict__ dst, uint64_t n, uint64_t w,
                           uint32_t lg4w, const QuadPt *__restrict__ Q) {
  using T_ = typename KT::T;
  constexpr uint32_t KS = sizeof(T_);
  static_assert(NT * VT >= TILE + 2 * VT && (VT & 1), "K5f shape");
  extern __shared__ __align__(128) char smem[];
  const int tid = threadIdx.x;
  uint32_t oW[4];
  int cnt[4];
  uint64_t o0;
  quad_load_tile<KT, VT>(smem, src, n, w, lg4w, TILE, Q, oW, cnt, o0);
  const int nx = cnt[0] + cnt[1], ny = cnt[2] + cnt[3], total = nx + ny;
  // X and Y (plus their sentinels) in their own region
  constexpr uint32_t XY0 = quad_split_in_bytes<KT, VT, TILE>();
  const uint32_t oX = XY0;
  const uint32_t oY = (oX + (nx + VT) * KS + 15u) & ~15u;

  // ---- phase 1: X = merge(R0w, R1w), Y = merge(R2w, R3w), stored at once ----
  {
    const int tx = (nx + VT - 1) / VT;
    const int side = tid >= tx ? 1 : 0;
    const int t1 = tid - side * tx;
    const uint32_t oA = side ? oW[2] : oW[0], oB = side ? oW[3] : oW[1];
    const int na = side ? cnt[2] : cnt[0], nb = side ? cnt[3] : cnt[1];
    const int d1 = t1 * VT;
    if (d1 < na + nb) {
      const int lo = split_predicted<KT, MP_QUAD_PRED_LOGW>(
          smem, oA, na, oB, nb, d1, static_cast<float>(na) / static_cast<float>(na + nb));
      merge_store_smem<KT, VT>(smem, oA, oB, lo, d1 - lo, (side ? oY : oX) + d1 * KS,
                               na + nb - d1);
    }
    if (tid >= NT - 32) {  // the last warp: X's VT sentinels and Y's one
      const int l = tid - (NT - 32);
      if (l < VT)
        *reinterpret_cast<T_ *>(smem + oX + (nx + l) * KS) = KT::max_key();
      else if (l == VT)
        *reinterpret_cast<T_ *>(smem + oY + ny * KS) = KT::max_key();
    }
  }
  __syncthreads();  // X and Y complete; the input windows are dead

  // ---- phase 2: out = merge(X, Y), ties to X, staged over the input region ----
  T_ *out = dst + o0;
  const uint32_t oS = mirror_off(16, out);
  uint32_t olo;
  const uint32_t oib = interior_bytes(reinterpret_cast<const char *>(out),
                                      static_cast<uint32_t>(total) * KS, &olo);
  const int d2 = tid * VT;
  if (d2 < total) {
    const int lo = split_predicted<KT, MP_QUAD_PRED_LOGW>(
        smem, oX, nx, oY, ny, d2, static_cast<float>(nx) / static_cast<float>(total));
    merge_store_smem<KT, VT>(smem, oX, oY, lo, d2 - lo, oS + d2 * KS, total - d2);
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (tid == 0 && oib) {
    bulk_s2g(reinterpret_cast<char *>(out) + olo, smem + oS + olo, oib);
    bulk_commit();
  }
  if (tid >= 32 && tid < 64) {  // unaligned head / tail (< 16 B each)
    const uint32_t bytes = static_cast<uint32_t>(total) * KS;
    const uint32_t hi = oib ? olo + oib : bytes;
    const uint32_t hlo = oib ? olo : bytes;
    const uint32_t nh = hlo / KS, nt = (bytes - hi) / KS;
    const uint32_t l = tid - 32;
    if (l < nh + nt) {
      const uint32_t e = l < nh ? l : (hi / KS) + (l - nh);
      out[e] = lds<T_>(smem, oS + e * KS);
    }
  }
  if (tid == 0 && oib)
    bulk_wait_read0();
}



// ===== K5g: conflict-free gathered outer merge (MP_QUAD_GATHER=1): correct, 3.04 vs 2.09 ms per pass =====
// Round 2, session 5.  The fused pass with its outer merge (X with Y) done by
// a bank-conflict-free gather into registers and a bitonic merge network
// instead of a serial merge from shared memory.  Byte-exact (37 GPU sort
// parity tests) but slower on B200: 2^30 u32 sort 33.9 vs 26.3 ms.  ncu
// (profiles/r02/k5g/): the gather itself is conflict-free as designed (32
// loads, 1 wavefront each, vs 3.5 for a serial merge's load) and all shared
// loads drop 399 -> 343 M wavefronts per pass, but
//   * 32 outputs per thread put neighbouring lanes' diagonals 32 apart, so
//     the phase-2 split search probes X[16 l + c]: 16-way bank conflicts (6-7.5
//     wavefronts per probe, 124 M wavefronts per pass -- more than the gather
//     saved); probes would have to be re-aligned per lane;
//   * the 32 sorted keys of a thread leave as eight 16-byte stores at a
//     128-byte lane stride: 32 sectors per request, lg_throttle + drain
//     stalls (staging them through shared memory needs a conflict-free
//     blocked -> linear transpose, i.e. direction flags in the network);
//   * 64 registers x 512 threads leave 2 CTAs = 1024 threads per SM (K5e:
//     1280): the inner merges and the tile prologue, unchanged work, take
//     0.5 ms longer per pass.
// The ALU pipe (one warp instruction per 2 cycles per sub-partition) would
// bound a fully gathered pass at ~13 ALU instructions per key and level --
// no better than K5e's ~11 -- so the idea was retired rather than tuned.
// Needs mp_bsort.cuh (order_u32, ce_u32) and the launch code below.
//
//   constexpr int kGatherNT = int(kQuadTile) / 32, kGatherVT = 33;
//   constexpr uint32_t qsmem = quad_gather_smem_bytes<KT, kGatherNT, kGatherVT>();
//   quad_tile_gather_kernel<KT, kGatherNT, kGatherVT><<<qtiles, kGatherNT, qsmem, s>>>(src, dst, n, w, lg4w, QT, QQ);
// ---------------------------------------------------------------------------
// K5g: K5e whose outer merge (X with Y) reads shared memory without bank
// conflicts and has no dependent load chain.
//
// ncu on K5e (profiles/r02/k5e_full_raw.csv): the LSU data pipe runs at 81 %
// of its wavefront peak and 277 M of the 399 M load wavefronts per pass are
// bank conflicts -- every thread of a serial merge walks its own cursor, so a
// warp's 32 loads fall on random banks (3.3 wavefronts per load).  K5g keeps
// K5e's prologue and inner merges (VT = 33 outputs per thread, NT = 512) and
// replaces the outer merge for full tiles (T = 32 * NT outputs):
//   * phase 1 writes X forward from a 128-byte boundary (X[k] in bank k % 32)
//     and Y REVERSED, ending in bank 31 (Y[k] in bank (31 - k) % 32), both as
//     order-preserving u32 images;
//   * thread i takes outputs [32 i, 32 i + 32): a Merge Path search gives its
//     split a_s (its neighbour's is a_e), so it owns X[a_s, a_e) and
//     Y[32 i - a_s, 32 (i + 1) - a_e) -- 32 elements whose banks are the 32
//     consecutive residues (a_e - 32 .. a_e - 1) % 32: Y's descending part
//     sits right below X's ascending part in bank space because the two
//     cursors of a diagonal sum to a multiple of 32;
//   * in load round j lane l fetches its element of bank (l + j) % 32 into
//     register j: 32 loads, one wavefront each, all independent;
//   * the registers then hold a rotation of (Y part descending, X part
//     ascending) -- a bitonic sequence, which the five half-cleaner stages of
//     a bitonic merge network sort whatever the rotation;
//   * the 32 sorted outputs leave as eight 16-byte stores (no staging copy).
// Bare keys only: equal keys are equal bytes, so the network's unstable order
// is the stable merge's bytes.  Partial tiles and unaligned outputs take
// K5e's path (quad_tile_merge).
// ---------------------------------------------------------------------------
template <class KT, int NT, int VT>
__host__ __device__ constexpr uint32_t quad_gather_split_off() {
  return (quad_smem_bytes<KT, NT, VT>() + 15u) & ~15u;
}
template <class KT, int NT, int VT>
__host__ __device__ constexpr uint32_t quad_gather_smem_bytes() {
  return quad_gather_split_off<KT, NT, VT>() + NT * 4u + 16u;
}

template <class KT, int NT, int VT>
__global__ void __launch_bounds__(NT, 1024 / NT)
    quad_tile_gather_kernel(const typename KT::T *__restrict__ src,
                            typename KT::T *__restrict__ dst, uint64_t n, uint64_t w,
                            uint32_t lg4w, uint32_t T, const QuadPt *__restrict__ Q) {
  using T_ = typename KT::T;
  static_assert(sizeof(T_) == 4, "bare 32-bit keys");
  constexpr uint32_t KS = 4;
  extern __shared__ __align__(128) char smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  uint32_t oW[4];
  int cnt[4];
  uint64_t o0;
  quad_load_tile<KT, VT>(smem, src, n, w, lg4w, T, Q, oW, cnt, o0);
  const int nx = cnt[0] + cnt[1], ny = cnt[2] + cnt[3], total = nx + ny;
  if (total != 32 * NT || (reinterpret_cast<uintptr_t>(dst) & 15) != 0) {  // CTA-uniform
    quad_tile_merge<KT, NT, VT>(smem, dst, oW, cnt, o0);
    return;
  }

  // ---- phase 1: X = merge(R0w, R1w), Y = merge(R2w, R3w) as K5e ----
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
  // X[k] at bX + 4k (bank k % 32); Y[k] at bY - 4k with bY in bank 31.  Each
  // lies inside the span of the windows (and gaps) it was merged from: the
  // alignment slack is < 128 bytes, two gaps are 2 * (4 VT + 20) bytes.
  const uint32_t bX = (oW[0] + 127u) & ~127u;
  const uint32_t bY = ((oW[2] + 4u * static_cast<uint32_t>(ny) + 127u - 128u) & ~127u) + 124u;
  if (act1) {
    const int lim = side ? ny : nx;
    if (side == 0) {
#pragma unroll
      for (int k = 0; k < VT; ++k)
        if (d1 + k < lim)
          *reinterpret_cast<uint32_t *>(smem + bX + (d1 + k) * KS) = order_u32<KT>(keys[k]);
    } else {
#pragma unroll
      for (int k = 0; k < VT; ++k)
        if (d1 + k < lim)
          *reinterpret_cast<uint32_t *>(smem + bY - (d1 + k) * KS) = order_u32<KT>(keys[k]);
    }
  }
  __syncthreads();

  // ---- phase 2: thread tid owns outputs [32 tid, 32 tid + 32) ----
  int *sp = reinterpret_cast<int *>(smem + quad_gather_split_off<KT, NT, VT>());
  const int d2 = tid * 32;
  int a_s;
  {
    const int lo = d2 > ny ? d2 - ny : 0;
    const int hi = d2 < nx ? d2 : nx;
    auto pred = [&](int m) {  // take Y at X index m on diagonal d2 (u32 order images)
      return lds<uint32_t>(smem, bY - (d2 - 1 - m) * KS) < lds<uint32_t>(smem, bX + m * KS);
    };
    int l = lo, h = hi;
    constexpr int LOGW = MP_QUAD_PRED_LOGW;
    if (hi - lo > (2 << LOGW)) {
      const float ratio = static_cast<float>(nx) / static_cast<float>(total);
      const int guess = min(max(__float2int_rn(static_cast<float>(d2) * ratio), lo), hi);
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
    a_s = l;
  }
  sp[tid] = a_s;
  __syncthreads();
  const int a_e = tid + 1 < NT ? sp[tid + 1] : nx;
  uint32_t x[32];
  {
    const int b_i = 32 - (a_e - a_s);  // Y elements of this block
    const int base = a_e - 32;         // virtual index of the block's first element
    const uint32_t c = static_cast<uint32_t>(lane - base) & 31u;
    const uint32_t KA = bX + 4u * static_cast<uint32_t>(base);
    const uint32_t KB = bY + 4u - 128u * static_cast<uint32_t>(tid) + 4u * static_cast<uint32_t>(base);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t tj = (c + j) & 31u;
      const uint32_t off = static_cast<int>(tj) >= b_i ? KA : KB;
      x[j] = lds<uint32_t>(smem, off + 4u * tj);
    }
  }
#pragma unroll
  for (int st = 16; st >= 1; st >>= 1)
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if ((q & st) == 0)
        ce_u32(x[q], x[q + st]);
  uint4 *out = reinterpret_cast<uint4 *>(dst + o0 + d2);
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    uint4 v;
    v.x = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 0]));
    v.y = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 1]));
    v.z = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 2]));
    v.w = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 3]));
    out[m] = v;
  }
}

