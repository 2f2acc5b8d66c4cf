/*
 * mp_oracle.c -- CPU restatement of the reference Merge Path algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker the parity tests,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg compare the CUDA
 * path against.  Nothing in the product (paper_1406_2628_b200/, include/)
 * links, loads or calls it.
 *
 * It restates, in plain C, the reference library at
 *   /root/reference/proj/include/mergepath/core.hpp      (diagonal search,
 *                                                        partition, merge)
 *   /root/reference/proj/include/mergepath/parallel.hpp  (parallel / SPM)
 *   /root/reference/proj/include/mergepath/sort.hpp      (merge sorts)
 * Each function cites the file:line it follows.  It is single-threaded: the
 * reference's worker decomposition is replayed sequentially (outputs and
 * statistics do not depend on the interleaving).
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * the reference's own known-answer tests (tests/golden/kats.json) and
 * against outputs of the reference itself compiled from /root/reference
 * (oracle/_ref, fixtures in tests/golden/ref_*.json).
 *
 * Key kinds (suffix):  u32, i32, f32 (IEEE totalOrder on the raw bits),
 * u64, i64, el (the reference's 16-byte `element`, core.hpp:39-51).
 * Optional uint32 payloads ("values") travel with u32/i32/f32/u64/i64 keys
 * (struct-of-arrays form of a {key, value} record ordered by key only).
 *
 * Status codes match the C ABI: 0 ok, 1 invalid argument.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t key;
  uint32_t tag;
  uint32_t pad;
} orc_element; /* core.hpp:39-51: 16 B, ordered by key only */

/* ---- comparators: all strict "less" (core.hpp:81-87 uses comp(b, a)) ---- */
static inline uint32_t orc_f32_order(uint32_t u) {
  /* IEEE 754 totalOrder as an unsigned key: flip all bits of negatives,
   * set the sign bit of non-negatives.  -0.0 < +0.0, NaNs at the ends. */
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
#define LESS_u32(x, y) ((x) < (y))
#define LESS_i32(x, y) ((x) < (y))
#define LESS_f32(x, y) (orc_f32_order(x) < orc_f32_order(y))
#define LESS_u64(x, y) ((x) < (y))
#define LESS_i64(x, y) ((x) < (y))
#define LESS_el(x, y) ((x).key < (y).key)

/* key_of for the checksum sink (core.hpp:209-214: static_cast<uint64_t>).
 * f32 keys are bit-cast (documented divergence: the reference's value
 * conversion of negative floats is undefined behaviour). */
#define KEYOF_u32(x) ((uint64_t)(x))
#define KEYOF_i32(x) ((uint64_t)(int64_t)(x))
#define KEYOF_f32(x) ((uint64_t)(x))
#define KEYOF_u64(x) ((uint64_t)(x))
#define KEYOF_i64(x) ((uint64_t)(x))
#define KEYOF_el(x) ((uint64_t)(x).key)

/* core.hpp:200-205 */
uint64_t orc_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* core.hpp:90-92, in 128-bit so i*n never overflows */
uint64_t orc_diagonal_of(uint64_t n, uint64_t p, uint64_t i) {
  return (uint64_t)(((unsigned __int128)i * n) / p);
}

#define MP_MIN(x, y) ((x) < (y) ? (x) : (y))

#define DEFINE_ORACLE(S, T)                                                    \
  /* core.hpp:99-132: smallest a_off on diagonal d with comp(B[d-1-m],A[m]) */ \
  uint64_t orc_diagonal_search_##S(const T *a, uint64_t na, const T *b,        \
                                   uint64_t nb, uint64_t d, uint64_t *cmp) {   \
    uint64_t lo = d > nb ? d - nb : 0;                                         \
    uint64_t hi = d < na ? d : na;                                             \
    while (lo < hi) {                                                          \
      const uint64_t mid = lo + (hi - lo) / 2;                                 \
      if (cmp)                                                                 \
        ++*cmp;                                                                \
      if (LESS_##S(b[d - 1 - mid], a[mid]))                                    \
        hi = mid;                                                              \
      else                                                                     \
        lo = mid + 1;                                                          \
    }                                                                          \
    return lo;                                                                 \
  }                                                                            \
                                                                               \
  /* core.hpp:136-146: p+1 points on diagonals i*N/p (a_off only) */          \
  int orc_partition_##S(const T *a, uint64_t na, const T *b, uint64_t nb,      \
                        uint64_t p, uint64_t *a_offs, uint64_t *cmp) {         \
    if (p == 0)                                                                \
      return 1;                                                                \
    const uint64_t n = na + nb;                                                \
    for (uint64_t i = 0; i <= p; ++i)                                          \
      a_offs[i] = orc_diagonal_search_##S(a, na, b, nb,                        \
                                          orc_diagonal_of(n, p, i), cmp);      \
    return 0;                                                                  \
  }                                                                            \
                                                                               \
  /* core.hpp:151-180: stable merge of `len` outputs from (sa, sb); ties to A  \
   * (core.hpp:167-170).  Values (optional) travel with their keys. */        \
  int orc_sequential_merge_##S(const T *a, const uint32_t *av, uint64_t na,    \
                               const T *b, const uint32_t *bv, uint64_t nb,    \
                               uint64_t sa, uint64_t sb, uint64_t len, T *out, \
                               uint32_t *outv, uint64_t *end_a,                \
                               uint64_t *end_b, uint64_t *steps) {             \
    if (sa > na || sb > nb)                                                    \
      return 1; /* core.hpp:159-160 aborts; report it instead */              \
    if (len > na + nb - (sa + sb))                                             \
      return 1; /* core.hpp:161-162 */                                        \
    uint64_t i = sa, j = sb, r = len, o = 0;                                   \
    while (r > 0 && i < na && j < nb) {                                        \
      if (LESS_##S(b[j], a[i])) {                                              \
        if (outv)                                                              \
          outv[o] = bv[j];                                                     \
        out[o++] = b[j++];                                                     \
      } else {                                                                 \
        if (outv)                                                              \
          outv[o] = av[i];                                                     \
        out[o++] = a[i++];                                                     \
      }                                                                        \
      --r;                                                                     \
    }                                                                          \
    for (; r > 0 && i < na; --r) {                                             \
      if (outv)                                                                \
        outv[o] = av[i];                                                       \
      out[o++] = a[i++];                                                       \
    }                                                                          \
    for (; r > 0 && j < nb; --r) {                                             \
      if (outv)                                                                \
        outv[o] = bv[j];                                                       \
      out[o++] = b[j++];                                                       \
    }                                                                          \
    if (steps)                                                                 \
      *steps += len;                                                           \
    if (end_a)                                                                 \
      *end_a = i;                                                              \
    if (end_b)                                                                 \
      *end_b = j;                                                              \
    return 0;                                                                  \
  }                                                                            \
                                                                               \
  /* parallel.hpp:67-88 + :151-179: worker w searches diagonal w*N/p and     \
   * merges up to (w+1)*N/p; workers replayed in order. */                    \
  int orc_parallel_merge_##S(const T *a, const uint32_t *av, uint64_t na,      \
                             const T *b, const uint32_t *bv, uint64_t nb,      \
                             T *out, uint32_t *outv, uint64_t p,               \
                             uint64_t *cmp, uint64_t *steps) {                 \
    if (p == 0)                                                                \
      return 1; /* parallel.hpp:54-57 */                                      \
    const uint64_t n = na + nb;                                                \
    for (uint64_t w = 0; w < p; ++w) {                                         \
      const uint64_t d_lo = orc_diagonal_of(n, p, w);                          \
      const uint64_t d_hi = orc_diagonal_of(n, p, w + 1);                      \
      if (d_lo == d_hi)                                                        \
        continue;                                                              \
      const uint64_t s = orc_diagonal_search_##S(a, na, b, nb, d_lo, cmp);     \
      orc_sequential_merge_##S(a, av, na, b, bv, nb, s, d_lo - s,              \
                               d_hi - d_lo, out + d_lo,                        \
                               outv ? outv + d_lo : NULL, NULL, NULL, steps);  \
    }                                                                          \
    return 0;                                                                  \
  }                                                                            \
                                                                               \
  /* parallel.hpp:90-145 + :202-236: Segmented Parallel Merge.  Windows of   \
   * L = C/3 outputs; window-local searches on L-capped sub-arrays; the last  \
   * active worker's end point starts the next window.  win_a/win_b (may be   \
   * NULL) receive each window's consumption; *iterations = ceil(N/L). */     \
  int orc_segmented_merge_##S(                                                 \
      const T *a, const uint32_t *av, uint64_t na, const T *b,                 \
      const uint32_t *bv, uint64_t nb, T *out, uint32_t *outv, uint64_t p,     \
      uint64_t C, uint64_t *cmp, uint64_t *steps, uint64_t *win_a,             \
      uint64_t *win_b, uint64_t *iterations) {                                 \
    if (p == 0 || C < 3)                                                       \
      return 1; /* parallel.hpp:54-63 */                                      \
    const uint64_t L = C / 3;                                                  \
    const uint64_t n = na + nb;                                                \
    const uint64_t iters = (n + L - 1) / L;                                    \
    const uint64_t p_eff = MP_MIN(p, L);                                       \
    uint64_t ca = 0, cb = 0;                                                   \
    for (uint64_t k = 0; k < iters; ++k) {                                     \
      const uint64_t d0 = ca + cb;                                             \
      const uint64_t rest = n - d0;                                            \
      const uint64_t Lw = MP_MIN(L, rest);                                     \
      const uint64_t pw = MP_MIN(p_eff, Lw);                                   \
      const uint64_t sub_na = MP_MIN(Lw, na - ca);                             \
      const uint64_t sub_nb = MP_MIN(Lw, nb - cb);                             \
      uint64_t na_next = ca, nb_next = cb;                                     \
      for (uint64_t w = 0; w < pw; ++w) {                                      \
        const uint64_t dl = orc_diagonal_of(Lw, pw, w);                        \
        const uint64_t dh = orc_diagonal_of(Lw, pw, w + 1);                    \
        const uint64_t la = orc_diagonal_search_##S(a + ca, sub_na, b + cb,    \
                                                    sub_nb, dl, cmp);          \
        uint64_t ea, eb;                                                       \
        orc_sequential_merge_##S(a, av, na, b, bv, nb, ca + la, cb + dl - la,  \
                                 dh - dl, out + d0 + dl,                       \
                                 outv ? outv + d0 + dl : NULL, &ea, &eb,       \
                                 steps);                                       \
        if (w + 1 == pw) {                                                     \
          na_next = ea;                                                        \
          nb_next = eb;                                                        \
        }                                                                      \
      }                                                                        \
      if (win_a)                                                               \
        win_a[k] = na_next - ca;                                               \
      if (win_b)                                                               \
        win_b[k] = nb_next - cb;                                               \
      ca = na_next;                                                            \
      cb = nb_next;                                                            \
    }                                                                          \
    if (iterations)                                                            \
      *iterations = iters;                                                     \
    return 0;                                                                  \
  }                                                                            \
                                                                               \
  /* parallel.hpp:262-292: window starting points of the SPM schedule.       \
   * start_a/start_b need ceil(N/L) entries (0 when N == 0). */               \
  int orc_plan_segments_##S(const T *a, uint64_t na, const T *b, uint64_t nb,  \
                            uint64_t p, uint64_t C, uint64_t *start_a,         \
                            uint64_t *start_b, uint64_t *window_len,           \
                            uint64_t *p_eff, uint64_t *iterations,             \
                            uint64_t *cmp) {                                   \
    if (p == 0 || C < 3)                                                       \
      return 1;                                                                \
    const uint64_t L = C / 3;                                                  \
    const uint64_t n = na + nb;                                                \
    const uint64_t iters = (n + L - 1) / L;                                    \
    *window_len = L;                                                           \
    *p_eff = MP_MIN(p, L);                                                     \
    *iterations = iters;                                                       \
    uint64_t ca = 0, cb = 0;                                                   \
    for (uint64_t k = 0; k < iters; ++k) {                                     \
      start_a[k] = ca;                                                         \
      start_b[k] = cb;                                                         \
      if (k + 1 == iters)                                                      \
        break;                                                                 \
      const uint64_t rest = n - (ca + cb);                                     \
      const uint64_t Lw = MP_MIN(L, rest);                                     \
      const uint64_t sub_na = MP_MIN(Lw, na - ca);                             \
      const uint64_t sub_nb = MP_MIN(Lw, nb - cb);                             \
      const uint64_t la =                                                      \
          orc_diagonal_search_##S(a + ca, sub_na, b + cb, sub_nb, Lw, cmp);    \
      ca += la;                                                                \
      cb += Lw - la;                                                           \
    }                                                                          \
    return 0;                                                                  \
  }                                                                            \
                                                                               \
  /* sort.hpp:59-67: stable binary-insertion sort (upper_bound) */            \
  static void orc_insertion_sort_##S(T *r, uint32_t *rv, uint64_t len) {       \
    for (uint64_t k = 1; k < len; ++k) {                                       \
      const T v = r[k];                                                        \
      const uint32_t vv = rv ? rv[k] : 0;                                      \
      uint64_t lo = 0, hi = k; /* upper_bound: first x with v < x */          \
      while (lo < hi) {                                                        \
        const uint64_t mid = lo + (hi - lo) / 2;                               \
        if (LESS_##S(v, r[mid]))                                               \
          hi = mid;                                                            \
        else                                                                   \
          lo = mid + 1;                                                        \
      }                                                                        \
      memmove(r + lo + 1, r + lo, (k - lo) * sizeof(T));                       \
      r[lo] = v;                                                               \
      if (rv) {                                                                \
        memmove(rv + lo + 1, rv + lo, (k - lo) * sizeof(uint32_t));           \
        rv[lo] = vv;                                                           \
      }                                                                        \
    }                                                                          \
  }                                                                            \
                                                                               \
  /* sort.hpp:71-101: one round, left run is A; unpaired tail copied */       \
  static void orc_merge_round_##S(const T *src, const uint32_t *srcv, T *dst,  \
                                  uint32_t *dstv, uint64_t len,                \
                                  uint64_t width) {                            \
    const uint64_t stride = 2 * width;                                         \
    const uint64_t pairs = len > width ? (len + width - 1) / stride : 0;       \
    for (uint64_t pr = 0; pr < pairs; ++pr) {                                  \
      const uint64_t i = pr * stride;                                          \
      const uint64_t bl = MP_MIN(width, len - i - width);                      \
      orc_sequential_merge_##S(src + i, srcv ? srcv + i : NULL, width,         \
                               src + i + width,                                \
                               srcv ? srcv + i + width : NULL, bl, 0, 0,       \
                               width + bl, dst + i, dstv ? dstv + i : NULL,    \
                               NULL, NULL, NULL);                              \
    }                                                                          \
    const uint64_t tail = pairs * stride;                                      \
    if (tail < len) {                                                          \
      memcpy(dst + tail, src + tail, (len - tail) * sizeof(T));                \
      if (dstv)                                                                \
        memcpy(dstv + tail, srcv + tail, (len - tail) * sizeof(uint32_t));     \
    }                                                                          \
  }                                                                            \
                                                                               \
  /* sort.hpp:105-128: 32-runs by insertion sort, then ping-pong rounds;      \
   * result lands in data.  Returns the round count. */                       \
  static uint64_t orc_sort_rounds_##S(T *data, uint32_t *datav, T *aux,        \
                                      uint32_t *auxv, uint64_t len) {          \
    if (len <= 1)                                                              \
      return 0;                                                                \
    for (uint64_t i = 0; i < len; i += 32)                                     \
      orc_insertion_sort_##S(data + i, datav ? datav + i : NULL,               \
                             MP_MIN(32, len - i));                             \
    T *src = data, *dst = aux;                                                 \
    uint32_t *srcv = datav, *dstv = auxv;                                      \
    uint64_t rounds = 0;                                                       \
    for (uint64_t width = 32; width < len; width *= 2) {                       \
      orc_merge_round_##S(src, srcv, dst, dstv, len, width);                   \
      T *t = src;                                                              \
      src = dst;                                                               \
      dst = t;                                                                 \
      uint32_t *tv = srcv;                                                     \
      srcv = dstv;                                                             \
      dstv = tv;                                                               \
      ++rounds;                                                                \
    }                                                                          \
    if (src != data) {                                                         \
      memcpy(data, src, len * sizeof(T));                                      \
      if (datav)                                                               \
        memcpy(datav, srcv, len * sizeof(uint32_t));                           \
    }                                                                          \
    return rounds;                                                             \
  }                                                                            \
                                                                               \
  /* sort.hpp:132-148: parallel_merge_sort (out may alias data) */            \
  int orc_merge_sort_##S(const T *data, const uint32_t *vals, uint64_t n,      \
                         uint64_t p, T *out, uint32_t *outv,                   \
                         uint64_t *rounds) {                                   \
    if (p == 0)                                                                \
      return 1;                                                                \
    if (out != data)                                                           \
      memmove(out, data, n * sizeof(T));                                       \
    if (outv && outv != vals)                                                  \
      memmove(outv, vals, n * sizeof(uint32_t));                               \
    if (n <= 1)                                                                \
      return 0;                                                                \
    T *aux = (T *)malloc(n * sizeof(T));                                       \
    uint32_t *auxv = outv ? (uint32_t *)malloc(n * sizeof(uint32_t)) : NULL;   \
    const uint64_t r = orc_sort_rounds_##S(out, outv, aux, auxv, n);           \
    free(aux);                                                                 \
    free(auxv);                                                                \
    if (rounds)                                                                \
      *rounds += r;                                                            \
    return 0;                                                                  \
  }                                                                            \
                                                                               \
  /* sort.hpp:150-195: cache_efficient_parallel_sort.  Phase 1 sorts blocks  \
   * of C/3, phase 2 merges block pairs level by level (odd block carried).   \
   * Segmented and plain merges produce identical bytes, so    \
   * phase 2 uses the sequential merge of the whole pair. */                  \
  int orc_ce_sort_##S(const T *data, const uint32_t *vals, uint64_t n,         \
                      uint64_t p, uint64_t C, T *out, uint32_t *outv,          \
                      uint64_t *levels_out) {                                  \
    if (p == 0 || C < 3)                                                       \
      return 1;                                                                \
    const uint64_t block = C / 3;                                              \
    if (out != data)                                                           \
      memmove(out, data, n * sizeof(T));                                       \
    if (outv && outv != vals)                                                  \
      memmove(outv, vals, n * sizeof(uint32_t));                               \
    if (n <= 1)                                                                \
      return 0;                                                                \
    T *aux = (T *)malloc(n * sizeof(T));                                       \
    uint32_t *auxv = outv ? (uint32_t *)malloc(n * sizeof(uint32_t)) : NULL;   \
    for (uint64_t i = 0; i < n; i += block) {                                  \
      const uint64_t bl = MP_MIN(block, n - i);                                \
      orc_sort_rounds_##S(out + i, outv ? outv + i : NULL, aux + i,            \
                          auxv ? auxv + i : NULL, bl);                         \
    }                                                                          \
    T *src = out, *dst = aux;                                                  \
    uint32_t *srcv = outv, *dstv = auxv;                                       \
    uint64_t levels = 0;                                                       \
    for (uint64_t width = block; width < n; width *= 2) {                      \
      orc_merge_round_##S(src, srcv, dst, dstv, n, width);                     \
      T *t = src;                                                              \
      src = dst;                                                               \
      dst = t;                                                                 \
      uint32_t *tv = srcv;                                                     \
      srcv = dstv;                                                             \
      dstv = tv;                                                               \
      ++levels;                                                                \
    }                                                                          \
    if (src != out) {                                                          \
      memcpy(out, src, n * sizeof(T));                                         \
      if (outv)                                                                \
        memcpy(outv, srcv, n * sizeof(uint32_t));                              \
    }                                                                          \
    free(aux);                                                                 \
    free(auxv);                                                                \
    if (levels_out)                                                            \
      *levels_out += levels;                                                   \
    return 0;                                                                  \
  }                                                                            \
                                                                               \
  /* core.hpp:240-245: position-weighted checksum of an output array */       \
  uint64_t orc_checksum_##S(const T *out, uint64_t n) {                        \
    uint64_t sum = 0;                                                          \
    for (uint64_t i = 0; i < n; ++i)                                           \
      sum += (i + 1) * orc_mix64(KEYOF_##S(out[i]));                           \
    return sum;                                                                \
  }

DEFINE_ORACLE(u32, uint32_t)
DEFINE_ORACLE(i32, int32_t)
DEFINE_ORACLE(f32, uint32_t)
DEFINE_ORACLE(u64, uint64_t)
DEFINE_ORACLE(i64, int64_t)
DEFINE_ORACLE(el, orc_element)

/* ------------------------------------------------------------------------
 * Config input generators.  x_i(seed) = mix64(seed + i*G),
 * the (i+1)-th SplitMix64 output from state `seed`.  `first` is the global
 * index of out[0] so shards can be generated independently.
 * kind: 0 u32 = x>>32; 1 i32 in [0,1024) = x>>54; 2 u64 = x;
 *       3 u64 below 2^40 = x>>24; 4 u64 in [2^40,2^64) = 2^40+mulhi(x,2^64-2^40)
 *       5 f32 Normal(0,1) (Box-Muller, cosine branch); 6 f32 Exp(1).
 * ------------------------------------------------------------------------ */
#define ORC_GOLDEN 0x9E3779B97F4A7C15ULL
static inline uint64_t orc_x(uint64_t seed, uint64_t i) {
  return orc_mix64(seed + i * ORC_GOLDEN);
}

int orc_generate(int kind, uint64_t seed, uint64_t first, uint64_t n,
                 void *out) {
  const double two53 = 1.0 / 9007199254740992.0;
  for (uint64_t k = 0; k < n; ++k) {
    const uint64_t i = first + k;
    switch (kind) {
    case 0:
      ((uint32_t *)out)[k] = (uint32_t)(orc_x(seed, i) >> 32);
      break;
    case 1:
      ((int32_t *)out)[k] = (int32_t)(orc_x(seed, i) >> 54);
      break;
    case 2:
      ((uint64_t *)out)[k] = orc_x(seed, i);
      break;
    case 3:
      ((uint64_t *)out)[k] = orc_x(seed, i) >> 24;
      break;
    case 4: {
      const unsigned __int128 m =
          (unsigned __int128)orc_x(seed, i) * (~0ULL - (1ULL << 40) + 1ULL);
      ((uint64_t *)out)[k] = (1ULL << 40) + (uint64_t)(m >> 64);
      break;
    }
    case 5: {
      const double u1 = ((double)((orc_x(seed, 2 * i) >> 11) + 1)) * two53;
      const double u2 = ((double)(orc_x(seed, 2 * i + 1) >> 11)) * two53;
      const double v = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
      const float f = (float)v;
      memcpy((uint32_t *)out + k, &f, 4);
      break;
    }
    case 6: {
      const double u = ((double)((orc_x(seed, i) >> 11) + 1)) * two53;
      const float f = (float)(-log(u));
      memcpy((uint32_t *)out + k, &f, 4);
      break;
    }
    default:
      return 1;
    }
  }
  return 0;
}

/* Test helper: the ascending sort of generated inputs (not a reference
 * algorithm, just the "sorted ascending" of BASELINE.json's configs).
 * LSD radix sort on the order-preserving unsigned image of each key type;
 * stable, so values (optional) keep input order among equal keys. */
static inline uint64_t orc_radix_key(int kt, const void *keys, uint64_t i) {
  switch (kt) {
  case 0:
    return ((const uint32_t *)keys)[i];
  case 1:
    return (uint32_t)(((const int32_t *)keys)[i]) ^ 0x80000000u;
  case 2:
    return orc_f32_order(((const uint32_t *)keys)[i]);
  case 3:
    return ((const uint64_t *)keys)[i];
  default:
    return ((const uint64_t *)keys)[i] ^ 0x8000000000000000ULL;
  }
}

int orc_radix_sort(int kt, void *keys, uint32_t *vals, uint64_t n) {
  if (kt < 0 || kt > 4)
    return 1;
  const size_t ks = kt <= 2 ? 4 : 8;
  const int passes = kt <= 2 ? 2 : 4; /* 16-bit digits */
  uint8_t *tmpk = (uint8_t *)malloc(n * ks + 1);
  uint32_t *tmpv = vals ? (uint32_t *)malloc(n * 4 + 4) : NULL;
  uint64_t *count = (uint64_t *)malloc(65536 * sizeof(uint64_t));
  uint8_t *src = (uint8_t *)keys, *dst = tmpk;
  uint32_t *srcv = vals, *dstv = tmpv;
  for (int pass = 0; pass < passes; ++pass) {
    const int shift = 16 * pass;
    memset(count, 0, 65536 * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i)
      ++count[(orc_radix_key(kt, src, i) >> shift) & 0xFFFF];
    uint64_t sum = 0;
    for (int d = 0; d < 65536; ++d) {
      const uint64_t c = count[d];
      count[d] = sum;
      sum += c;
    }
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t pos = count[(orc_radix_key(kt, src, i) >> shift) & 0xFFFF]++;
      memcpy(dst + pos * ks, src + i * ks, ks);
      if (vals)
        dstv[pos] = srcv[i];
    }
    uint8_t *t = src;
    src = dst;
    dst = t;
    uint32_t *tv = srcv;
    srcv = dstv;
    dstv = tv;
  }
  /* even pass count: result is back in keys/vals */
  free(tmpk);
  free(tmpv);
  free(count);
  return 0;
}
