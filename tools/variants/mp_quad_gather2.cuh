// mp_quad_gather2.cuh -- K5g v2 (experiment, not in the product build): the
// gathered outer merge of K5g (mp_quad_variants.cuh) with the two problems its
// ncu capture showed repaired -- split-search probes aligned to the lane's
// bank, and the sorted keys staged through a swizzled 16-byte layout so the
// global stores are coalesced.  Byte-exact (37 GPU sort parity tests); B200,
// 2^30 u32 sort: 29.17 ms (2.54 ms per pass) vs K5g 33.9 (3.04) and K5e 25.57
// (2.09).  ncu (profiles/r02/k5g2/): LSU data pipe 58 % (K5e 82 %), 381 M
// shared-memory wavefronts (479 M), but 1.50 G instructions (1.31 G), issue
// 52 %, warps active 48 %: with 32 keys live per thread the kernel needs 64
// registers, so an SM holds 2 x 512 threads (K5e: 2 x 640) and nothing hides
// the tile prologue (19 % of the samples) and the store tail (11 %).
// At 8192-output tiles (256 threads, 48 registers, 5 CTAs = 1280 threads per
// SM, crossings still on the 16384 grid): 2.40 ms per pass, and K4r's twice as
// many tile boundaries cost 0.28 instead of 0.12 ms: 29.3 ms per sort.
// To build it: include this header after mp_quad.cuh in mp_capi.cu (-I
// tools/variants) and launch, where K5e is launched for QT == kQuadTile,
//   constexpr int GNT = int(kQuadTile) / 32, GVT = 33;
//   quad_tile_gather_kernel<KT, GNT, GVT><<<qtiles, GNT,
//       quad_gather_smem_bytes<KT, GNT, GVT>(), s>>>(src, dst, n, w, lg4w, QT, QQ);
#pragma once
#include "mp_quad.cuh"
#include "mp_bsort.cuh"
namespace mpb {
template <class KT, int NT, int VT>
__host__ __device__ constexpr uint32_t quad_gather_split_off() {
  return (quad_smem_bytes<KT, NT, VT>() + 15u) & ~15u;
}
template <class KT, int NT, int VT>
__host__ __device__ constexpr uint32_t quad_gather_smem_bytes() {
  return quad_gather_split_off<KT, NT, VT>() + NT * 4u + 16u;
}

template <class KT, int NT, int VT>
__global__ void __launch_bounds__(NT, NT <= 256 ? 1280 / NT : 1024 / NT)
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
    // probes are moved to indices = lane (mod 32): X[m] sits in bank m % 32 and
    // the Y probe of diagonal d2 (a multiple of 32) in bank m % 32 too, so the
    // warp's probes fall in 32 different banks instead of two (neighbouring
    // diagonals are 32 apart and their splits ~16)
    if (hi - lo > (2 << LOGW)) {
      const float ratio = static_cast<float>(nx) / static_cast<float>(total);
      const int guess = min(max(__float2int_rn(static_cast<float>(d2) * ratio), lo), hi);
      int lo0 = guess - (1 << LOGW), hi0 = guess + (1 << LOGW);
      lo0 -= (lo0 - 1 - lane) & 31;  // lo0 - 1 = lane (mod 32)
      hi0 += (lane - hi0) & 31;      // hi0 = lane (mod 32)
      lo0 = max(lo, lo0);
      hi0 = min(hi, hi0);
      const bool ok_lo = lo0 == lo || !pred(lo0 - 1);
      const bool ok_hi = hi0 == hi || pred(hi0);
      if (ok_lo && ok_hi) {
        l = lo0;
        h = hi0;
      }
    }
    while (l < h) {
      int mid = (l + h) >> 1;
      if (h - l >= 64) {
        int m2 = mid - ((mid - lane) & 31);
        if (m2 < l)
          m2 += 32;
        mid = m2 < h ? m2 : mid;
      }
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
  // The thread's 32 sorted keys go to shared memory as eight 16-byte stores,
  // quad g of row tid at quad slot g ^ (tid & 7) (8 consecutive lanes hit 8
  // different bank groups), and leave as 16-byte loads + coalesced 16-byte
  // global stores: linear quad Qi = row * 8 + g lives at slot g ^ (row & 7).
  __syncthreads();  // X and Y consumed (the staging area overlays them)
  uint4 *stg = reinterpret_cast<uint4 *>(smem + 128);
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    uint4 v;
    v.x = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 0]));
    v.y = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 1]));
    v.z = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 2]));
    v.w = static_cast<uint32_t>(from_order_u32<KT>(x[4 * m + 3]));
    stg[tid * 8 + (m ^ (tid & 7))] = v;
  }
  __syncthreads();
  uint4 *out = reinterpret_cast<uint4 *>(dst + o0);
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int qi = tid + m * NT;
    const int row = qi >> 3, g = qi & 7;
    out[qi] = stg[row * 8 + (g ^ (row & 7))];
  }
}

}  // namespace mpb
