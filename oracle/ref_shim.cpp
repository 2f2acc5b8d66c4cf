// ref_shim.cpp -- extern "C" wrapper around the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile against the reference
// headers where they lie (-I /root/reference/proj/include) plus the
// reference's own thread_team.cpp, into oracle/_ref/libmergepath_ref.so.
// Nothing from the reference is copied into this repository; this file only
// instantiates the reference's public templates for the key types the
// configs use and exposes them over a C ABI so that
//   * tests/golden/make_golden.py can record reference outputs as fixtures,
//   * tests can cross-check the C restatement (oracle/mp_oracle.c), and
//   * bench.py --impl reference / cpu_baseline can time the reference's own
//     CPU path (parallel.hpp:151-162, sort.hpp:132-148) on the GPU box.
//
// Comparators follow BASELINE.md §3: std::less for integer keys, a key-only
// comparator for {u64 key, u32 value} records, IEEE totalOrder for floats.

#include <cstdint>
#include <cstring>
#include <span>
#include <vector>

#include "mergepath/core.hpp"
#include "mergepath/parallel.hpp"
#include "mergepath/sort.hpp"
#include "mergepath/thread_team.hpp"

namespace {

using namespace mergepath;

struct kv {  // config 3 record: u64 key, u32 value (16 B with padding)
  std::uint64_t key;
  std::uint32_t val;
  std::uint32_t pad;
};
struct kv_less {
  bool operator()(const kv &l, const kv &r) const { return l.key < r.key; }
};

inline std::uint32_t total_order_bits(float f) {
  std::uint32_t u;
  std::memcpy(&u, &f, 4);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
struct total_order_less {
  bool operator()(float l, float r) const {
    return total_order_bits(l) < total_order_bits(r);
  }
};

template <typename T> merge_input<T> view(const void *a, std::uint64_t na,
                                          const void *b, std::uint64_t nb) {
  return {std::span<const T>(static_cast<const T *>(a), na),
          std::span<const T>(static_cast<const T *>(b), nb)};
}

}  // namespace

extern "C" {

void *ref_team_new(std::uint64_t p) { return new thread_team(p); }
void ref_team_free(void *t) { delete static_cast<thread_team *>(t); }
std::uint64_t ref_team_lanes(void *t) {
  return static_cast<thread_team *>(t)->lanes();
}

#define REF_DEFINE(S, T, COMP)                                                 \
  std::uint64_t ref_diagonal_search_##S(const void *a, std::uint64_t na,       \
                                        const void *b, std::uint64_t nb,       \
                                        std::uint64_t d, std::uint64_t *cmp) { \
    return diagonal_search(view<T>(a, na, b, nb), d, COMP{}, cmp).a_off;       \
  }                                                                            \
  int ref_partition_##S(const void *a, std::uint64_t na, const void *b,        \
                        std::uint64_t nb, std::uint64_t p,                     \
                        std::uint64_t *a_offs, std::uint64_t *b_offs,          \
                        std::uint64_t *cmp) {                                  \
    try {                                                                      \
      const auto pts = partition(view<T>(a, na, b, nb), p, COMP{}, cmp);      \
      for (std::size_t i = 0; i < pts.size(); ++i) {                           \
        a_offs[i] = pts[i].a_off;                                              \
        b_offs[i] = pts[i].b_off;                                              \
      }                                                                        \
      return 0;                                                                \
    } catch (const std::invalid_argument &) {                                  \
      return 1;                                                                \
    }                                                                          \
  }                                                                            \
  int ref_parallel_merge_##S(void *team, const void *a, std::uint64_t na,      \
                             const void *b, std::uint64_t nb, void *out,       \
                             std::uint64_t *cmp, std::uint64_t *steps) {       \
    merge_stats st;                                                            \
    parallel_merge_into(view<T>(a, na, b, nb),                                 \
                        std::span<T>(static_cast<T *>(out), na + nb),          \
                        *static_cast<thread_team *>(team), COMP{}, &st);       \
    if (cmp)                                                                   \
      *cmp += st.partition_comparisons;                                        \
    if (steps)                                                                 \
      *steps += st.merge_steps;                                                \
    return 0;                                                                  \
  }                                                                            \
  int ref_parallel_merge_p_##S(std::uint64_t p, const void *a,                 \
                               std::uint64_t na, const void *b,                \
                               std::uint64_t nb, void *out,                    \
                               std::uint64_t *cmp, std::uint64_t *steps) {     \
    try {                                                                      \
      merge_stats st;                                                          \
      parallel_merge_into(view<T>(a, na, b, nb),                               \
                          std::span<T>(static_cast<T *>(out), na + nb), p,     \
                          COMP{}, &st);                                        \
      if (cmp)                                                                 \
        *cmp += st.partition_comparisons;                                      \
      if (steps)                                                               \
        *steps += st.merge_steps;                                              \
      return 0;                                                                \
    } catch (const std::invalid_argument &) {                                  \
      return 1;                                                                \
    }                                                                          \
  }                                                                            \
  int ref_segmented_merge_##S(std::uint64_t p, std::uint64_t C, const void *a, \
                              std::uint64_t na, const void *b,                 \
                              std::uint64_t nb, void *out, std::uint64_t *cmp, \
                              std::uint64_t *steps, std::uint64_t *win_a,      \
                              std::uint64_t *win_b, std::uint64_t *nwin) {     \
    try {                                                                      \
      merge_stats st;                                                          \
      segmented_parallel_merge_into(                                           \
          view<T>(a, na, b, nb), std::span<T>(static_cast<T *>(out), na + nb), \
          p, C, COMP{}, &st);                                                  \
      if (cmp)                                                                 \
        *cmp += st.partition_comparisons;                                      \
      if (steps)                                                               \
        *steps += st.merge_steps;                                              \
      for (std::size_t k = 0; k < st.windows.size(); ++k) {                    \
        if (win_a)                                                             \
          win_a[k] = st.windows[k].a_consumed;                                 \
        if (win_b)                                                             \
          win_b[k] = st.windows[k].b_consumed;                                 \
      }                                                                        \
      if (nwin)                                                                \
        *nwin = st.windows.size();                                             \
      return 0;                                                                \
    } catch (const std::invalid_argument &) {                                  \
      return 1;                                                                \
    }                                                                          \
  }                                                                            \
  int ref_plan_segments_##S(const void *a, std::uint64_t na, const void *b,    \
                            std::uint64_t nb, std::uint64_t p,                 \
                            std::uint64_t C, std::uint64_t *start_a,           \
                            std::uint64_t *start_b, std::uint64_t *window_len, \
                            std::uint64_t *p_eff, std::uint64_t *iterations,   \
                            std::uint64_t *cmp) {                              \
    try {                                                                      \
      const auto plan =                                                        \
          plan_segments(view<T>(a, na, b, nb), p, C, COMP{}, cmp);             \
      *window_len = plan.window_len;                                           \
      *p_eff = plan.p_eff;                                                     \
      *iterations = plan.iterations;                                           \
      for (std::size_t k = 0; k < plan.starting_points.size(); ++k) {          \
        start_a[k] = plan.starting_points[k].a_off;                            \
        start_b[k] = plan.starting_points[k].b_off;                            \
      }                                                                        \
      return 0;                                                                \
    } catch (const std::invalid_argument &) {                                  \
      return 1;                                                                \
    }                                                                          \
  }                                                                            \
  int ref_merge_sort_##S(const void *data, std::uint64_t n, std::uint64_t p,   \
                         void *out, std::uint64_t *rounds) {                   \
    try {                                                                      \
      sort_stats st;                                                           \
      const auto v = parallel_merge_sort(                                      \
          std::span<const T>(static_cast<const T *>(data), n), p, COMP{},      \
          &st);                                                                \
      std::memcpy(out, v.data(), n * sizeof(T));                               \
      if (rounds)                                                              \
        *rounds += st.merge_rounds;                                            \
      return 0;                                                                \
    } catch (const std::invalid_argument &) {                                  \
      return 1;                                                                \
    }                                                                          \
  }                                                                            \
  int ref_ce_sort_##S(const void *data, std::uint64_t n, std::uint64_t p,      \
                      std::uint64_t C, void *out, std::uint64_t *levels) {     \
    try {                                                                      \
      sort_stats st;                                                           \
      const auto v = cache_efficient_parallel_sort(                            \
          std::span<const T>(static_cast<const T *>(data), n), p, C, COMP{},   \
          &st);                                                                \
      std::memcpy(out, v.data(), n * sizeof(T));                               \
      if (levels)                                                              \
        *levels += st.merge_rounds;                                            \
      return 0;                                                                \
    } catch (const std::invalid_argument &) {                                  \
      return 1;                                                                \
    }                                                                          \
  }

REF_DEFINE(u32, std::uint32_t, std::less<std::uint32_t>)
REF_DEFINE(i32, std::int32_t, std::less<std::int32_t>)
REF_DEFINE(f32, float, total_order_less)
REF_DEFINE(u64, std::uint64_t, std::less<std::uint64_t>)
REF_DEFINE(i64, std::int64_t, std::less<std::int64_t>)
REF_DEFINE(el, element, key_less)
REF_DEFINE(kv, kv, kv_less)

// Register-sink merge (parallel.hpp:183-198) on the test element type and
// on int64 (checksum is defined for integer keys, core.hpp:209-214).
std::uint64_t ref_merge_checksum_i64(std::uint64_t p, const void *a,
                                     std::uint64_t na, const void *b,
                                     std::uint64_t nb) {
  return parallel_merge_checksum(view<std::int64_t>(a, na, b, nb), p);
}
std::uint64_t ref_merge_checksum_el(std::uint64_t p, const void *a,
                                    std::uint64_t na, const void *b,
                                    std::uint64_t nb) {
  return parallel_merge_checksum(view<element>(a, na, b, nb), p, key_less{});
}
std::uint64_t ref_segmented_checksum_el(std::uint64_t p, std::uint64_t C,
                                        const void *a, std::uint64_t na,
                                        const void *b, std::uint64_t nb) {
  return segmented_parallel_merge_checksum(view<element>(a, na, b, nb), p, C,
                                           key_less{});
}
std::uint64_t ref_checksum_of_el(const void *out, std::uint64_t n) {
  return checksum_of(
      std::span<const element>(static_cast<const element *>(out), n));
}

}  // extern "C"
