#pragma once

// Drop-in replacement for the reference's mergepath/sort.hpp
// (/root/reference/proj/include/mergepath/sort.hpp) backed by the B200
// library.  Both sorts are one call to mp_sort_host, which runs mp_sort's
// schedule on the device: a block sort into sorted runs -- K3w (16384-key
// runs, bare 32-bit keys: u32 / i32 / f32) or the stable K3 (2048-key runs:
// values, 64-bit keys, element) -- then ceil(log2(N / run)) Merge Path
// rounds, run as fused round pairs (one HBM pass per two rounds, mp_quad.cuh)
// for large bare 32-bit sorts and as K4 split points + K2 tile merges
// otherwise; left run = A in every pair, so the result is stable with
// respect to input index -- the same bytes as the reference's plain and
// cache-efficient sorts (test_sort.cpp:128-135).
//
// make_sort_plan() still describes the REFERENCE CPU plan (32-element base
// runs or C/3 blocks) so sort_stats::merge_rounds keeps its meaning for
// drop-in callers (test_sort.cpp:27-67 pins it).

#include <bit>
#include <cstdint>
#include <span>
#include <vector>

#include "mergepath/core.hpp"
#include "mergepath/parallel.hpp"
#include "mergepath/thread_team.hpp"

namespace mergepath {

inline constexpr std::size_t sort_base_run = 32;

enum class sort_variant { plain, cache_efficient };

struct sort_plan {
  sort_variant variant = sort_variant::plain;
  std::size_t block_size = 0;
  std::size_t blocks = 0;
  std::size_t tree_levels = 0;
};

struct sort_stats {
  std::size_t merge_rounds = 0;
};

inline sort_plan make_sort_plan(sort_variant variant, std::size_t n,
                                std::size_t cache_elems) {
  sort_plan plan;
  plan.variant = variant;
  plan.block_size = variant == sort_variant::plain
                        ? sort_base_run
                        : detail::window_of(cache_elems);
  plan.blocks = n == 0 ? 0 : (n + plan.block_size - 1) / plan.block_size;
  plan.tree_levels =
      plan.blocks <= 1 ? 0 : static_cast<std::size_t>(std::bit_width(plan.blocks - 1));
  return plan;
}

namespace detail {
template <typename T, typename Comp>
std::vector<T> device_sort(std::span<const T> data) {
  std::vector<T> out(data.size());
  if (!data.empty())
    b200::check(mp_sort_host(b200::key_type<T, Comp>(), data.data(), nullptr,
                             data.size(), out.data(), nullptr,
                             b200::device()));
  return out;
}
}  // namespace detail

template <typename T, typename Comp = std::less<T>>
std::vector<T> parallel_merge_sort(std::span<const T> data, std::size_t p,
                                   Comp comp = {},
                                   sort_stats *stats = nullptr) {
  (void)comp;
  detail::check_merge_args(p);
  std::vector<T> out = detail::device_sort<T, Comp>(data);
  if (stats)
    stats->merge_rounds +=
        make_sort_plan(sort_variant::plain, data.size(), 0).tree_levels;
  return out;
}

template <typename T, typename Comp = std::less<T>>
std::vector<T> cache_efficient_parallel_sort(std::span<const T> data,
                                             std::size_t p,
                                             std::size_t cache_elems,
                                             Comp comp = {},
                                             sort_stats *stats = nullptr) {
  (void)comp;
  detail::check_merge_args(p);
  detail::window_of(cache_elems);
  std::vector<T> out = detail::device_sort<T, Comp>(data);
  if (stats)
    stats->merge_rounds +=
        make_sort_plan(sort_variant::cache_efficient, data.size(), cache_elems)
            .tree_levels;
  return out;
}

}  // namespace mergepath
