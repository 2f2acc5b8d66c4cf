#pragma once

// Glue between the drop-in mergepath templates and the C ABI of
// libmergepath_b200.so (include/mergepath_b200.h).
//
//  * key_traits<T, Comp> maps every supported (T, Comp) pair to an
//    mp_key_type at compile time.  Unsupported pairs are a compile error
//    (static_assert) -- there is no CPU fallback.
//  * check() turns an mp_status into the reference's error behaviour:
//    MP_ERR_INVALID -> std::invalid_argument, anything else ->
//    std::runtime_error (a CUDA failure has no reference counterpart).
//  * device(): the GPU that host-span calls stage through (default 0,
//    overridable with set_device() or the MERGEPATH_DEVICE variable).

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <new>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "../mergepath_b200.h"

namespace mergepath {

struct element;  // core.hpp

// IEEE 754 totalOrder on float: the comparator the configs use for f32
// keys (-0.0 < +0.0; NaNs ordered by payload at the ends).  The reference
// has no float carrier; its Comp parameter takes this comparator.
struct total_order_less {
  static std::uint32_t image(float f) {
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  }
  bool operator()(float l, float r) const { return image(l) < image(r); }
};

namespace b200 {

template <typename T, typename Comp> struct key_traits {
  static constexpr int value = -1;
};
template <> struct key_traits<std::uint32_t, std::less<std::uint32_t>> {
  static constexpr int value = MP_KEY_U32;
};
template <> struct key_traits<std::int32_t, std::less<std::int32_t>> {
  static constexpr int value = MP_KEY_I32;
};
template <> struct key_traits<float, total_order_less> {
  static constexpr int value = MP_KEY_F32;
};
template <> struct key_traits<unsigned long, std::less<unsigned long>> {
  static constexpr int value = sizeof(unsigned long) == 8 ? MP_KEY_U64 : MP_KEY_U32;
};
template <> struct key_traits<unsigned long long, std::less<unsigned long long>> {
  static constexpr int value = MP_KEY_U64;
};
template <> struct key_traits<long, std::less<long>> {
  static constexpr int value = sizeof(long) == 8 ? MP_KEY_I64 : MP_KEY_I32;
};
template <> struct key_traits<long long, std::less<long long>> {
  static constexpr int value = MP_KEY_I64;
};
// transparent comparator
template <typename T> struct key_traits<T, std::less<void>>
    : key_traits<T, std::less<T>> {};

template <typename T, typename Comp> constexpr int key_type() {
  constexpr int kt = key_traits<std::remove_cv_t<T>, Comp>::value;
  static_assert(kt >= 0,
                "mergepath (B200 backend): this (element type, comparator) "
                "pair has no device kernel; supported: uint32/int32/"
                "uint64/int64 with std::less, float with total_order_less, "
                "mergepath::element with key_less");
  return kt;
}

inline int &device_slot() {
  static int dev = [] {
    const char *e = std::getenv("MERGEPATH_DEVICE");
    return e ? std::atoi(e) : 0;
  }();
  return dev;
}
inline int device() { return device_slot(); }
inline void set_device(int d) { device_slot() = d; }

inline void check(int status) {
  if (status == MP_OK)
    return;
  const std::string msg = mp_last_error();
  if (status == MP_ERR_INVALID)
    throw std::invalid_argument(msg);
  throw std::runtime_error("mergepath (B200 backend): " + msg);
}

// Page-locked host memory for callers that own their buffers: host-span
// calls DMA it directly (config-2 merge 47 ms) instead of staging pageable
// memory through pinned slots (100 ms; the host's DRAM bandwidth bounds the
// extra copies).  std::vector<T, mergepath::b200::pinned_allocator<T>> is a
// drop-in container for the reference API's spans.
template <typename T> struct pinned_allocator {
  using value_type = T;
  pinned_allocator() = default;
  template <typename U> pinned_allocator(const pinned_allocator<U> &) noexcept {}
  T *allocate(std::size_t n) {
    void *p = mp_host_alloc(n * sizeof(T));
    if (!p && n)
      throw std::bad_alloc();
    return static_cast<T *>(p);
  }
  void deallocate(T *p, std::size_t) noexcept { mp_host_free(p); }
  template <typename U> bool operator==(const pinned_allocator<U> &) const noexcept {
    return true;
  }
  template <typename U> bool operator!=(const pinned_allocator<U> &) const noexcept {
    return false;
  }
};

}  // namespace b200
}  // namespace mergepath
