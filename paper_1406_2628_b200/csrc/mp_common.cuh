// mp_common.cuh -- key traits, comparators and sm_100a PTX helpers shared by
// every Merge Path kernel.
//
// The whole library is built around ONE predicate, the merge-matrix entry of
// the reference (core.hpp:79-87): M[i,j] = comp(B[j], A[i]), i.e. "take B"
// only when B is strictly less.  Equal keys go to A first, which makes every
// merge here stable with A as the left operand.  `take_b()`
// below is that predicate; the partition kernel, the in-CTA thread split and
// the serial merge all use it, so the tie rule is identical at all levels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mpb {

// ---------------------------------------------------------------------------
// Key kinds (match include/mergepath_b200.h's mp_key_type).
// ---------------------------------------------------------------------------
enum KeyKind : int {
  kU32 = 0,
  kI32 = 1,
  kF32 = 2,  // IEEE totalOrder on the raw bits
  kU64 = 3,
  kI64 = 4,
  kElement = 5,  // reference `element` {int64 key; uint32 tag}, 16 B AoS
};

// The reference's test element (core.hpp:39-51): 16 bytes, ordered by key.
struct alignas(16) Element {
  long long key;
  unsigned int tag;
  unsigned int pad;
};

__host__ __device__ __forceinline__ uint32_t f32_order(uint32_t u) {
  // totalOrder image: negatives bit-flipped, non-negatives get the sign bit.
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

struct KeyU32 {
  using T = uint32_t;
  static constexpr int kind = kU32;
  __host__ __device__ __forceinline__ static bool less(T x, T y) { return x < y; }
  __host__ __device__ __forceinline__ static T max_key() { return 0xFFFFFFFFu; }
};
struct KeyI32 {
  using T = int32_t;
  static constexpr int kind = kI32;
  __host__ __device__ __forceinline__ static bool less(T x, T y) { return x < y; }
  __host__ __device__ __forceinline__ static T max_key() { return 0x7FFFFFFF; }
};
struct KeyF32 {  // keys stored as their raw uint32 bit patterns
  using T = uint32_t;
  static constexpr int kind = kF32;
  __host__ __device__ __forceinline__ static bool less(T x, T y) {
    return f32_order(x) < f32_order(y);
  }
  // f32_order(0x7FFFFFFF) == 0xFFFFFFFF: the largest key in totalOrder.
  __host__ __device__ __forceinline__ static T max_key() { return 0x7FFFFFFFu; }
};
struct KeyU64 {
  using T = unsigned long long;
  static constexpr int kind = kU64;
  __host__ __device__ __forceinline__ static bool less(T x, T y) { return x < y; }
  __host__ __device__ __forceinline__ static T max_key() { return ~0ULL; }
};
struct KeyI64 {
  using T = long long;
  static constexpr int kind = kI64;
  __host__ __device__ __forceinline__ static bool less(T x, T y) { return x < y; }
  __host__ __device__ __forceinline__ static T max_key() { return 0x7FFFFFFFFFFFFFFFLL; }
};
struct KeyElement {
  using T = Element;
  static constexpr int kind = kElement;
  __host__ __device__ __forceinline__ static bool less(const T &x, const T &y) {
    return x.key < y.key;
  }
  __host__ __device__ __forceinline__ static T max_key() {
    T e;
    e.key = 0x7FFFFFFFFFFFFFFFLL;
    e.tag = 0xFFFFFFFFu;
    e.pad = 0;
    return e;
  }
};

// The merge-matrix predicate (core.hpp:86): true = the path moves right
// (consume B).  Strict, so ties go to A.
template <class KT>
__device__ __forceinline__ bool take_b(const typename KT::T &b,
                                       const typename KT::T &a) {
  return KT::less(b, a);
}

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + 1-D bulk async copies (TMA engine, UBLKCP in SASS).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar,
                                                      uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Non-blocking probe (test_wait never suspends the thread, unlike try_wait):
// for a producer that polls several barriers in turn.
__device__ __forceinline__ bool mbar_test_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// global -> shared bulk copy completing on an mbarrier (16 B aligned, size %16)
__device__ __forceinline__ void bulk_g2s(void *smem_dst, const void *gmem_src,
                                         uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// shared -> global bulk copy (bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void *gmem_dst, const void *smem_src,
                                         uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                   gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// at most N bulk groups may still be reading shared memory
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

// plain (non-transaction) arrive, release semantics at CTA scope
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Stage a byte range [src, src+bytes) of global memory into smem so that
// smem_base[k] mirrors src[k].  smem_base must be congruent to src mod 16.
// The 16 B-aligned interior goes through the bulk-copy engine (issued by the
// caller's elected thread, counted into *tx); the unaligned head and tail
// (< 16 B each) are copied by the CTA's threads with ordinary loads.
struct ByteRange {
  const char *src;
  char *dst;
  uint32_t bytes;
};

__device__ __forceinline__ uint32_t bulk_interior(const ByteRange &r,
                                                  uint32_t *lo,
                                                  uint32_t *hi) {
  const uintptr_t s = reinterpret_cast<uintptr_t>(r.src);
  const uintptr_t e = s + r.bytes;
  const uintptr_t is = (s + 15) & ~uintptr_t(15);
  const uintptr_t ie = e & ~uintptr_t(15);
  if (ie <= is) {
    *lo = r.bytes;
    *hi = r.bytes;
    return 0;
  }
  *lo = static_cast<uint32_t>(is - s);
  *hi = static_cast<uint32_t>(ie - s);
  return *hi - *lo;
}

}  // namespace mpb
