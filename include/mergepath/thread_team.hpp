#pragma once

// Drop-in for the reference's mergepath/thread_team.hpp
// (/root/reference/proj/include/mergepath/thread_team.hpp:19-57).
//
// In the reference the team IS the runtime: p logical workers on OS threads,
// fork/join dispatch and a barrier per phase.  In the B200 build that role
// belongs to the CUDA grid: a merge's "workers" are CTAs and threads, a phase
// barrier is a kernel boundary or __syncthreads.  The class is kept so every
// `(..., thread_team &team, ...)` overload compiles unchanged; the merges
// read only size() (the caller's p, which shapes statistics, never bytes).
//
// run()/run_phased() keep their contract (fn(w) exactly once per worker per
// phase, completion(phase) once after all workers of that phase) and execute
// on the calling thread; no OS threads are spawned.

#include <cstddef>
#include <cstdint>
#include <functional>
#include <stdexcept>

namespace mergepath {

class thread_team {
public:
  explicit thread_team(std::size_t workers) : thread_team(workers, 1) {}
  thread_team(std::size_t workers, std::size_t max_os_threads)
      : workers_(workers) {
    (void)max_os_threads;
    if (workers == 0)  // thread_team.cpp:22-23
      throw std::invalid_argument("thread_team: worker count must be positive");
  }
  ~thread_team() = default;

  thread_team(const thread_team &) = delete;
  thread_team &operator=(const thread_team &) = delete;

  std::size_t size() const { return workers_; }
  std::size_t lanes() const { return 1; }

  void run(const std::function<void(std::size_t)> &fn) {
    for (std::size_t w = 0; w < workers_; ++w)
      fn(w);
  }

  void run_phased(std::size_t phases,
                  const std::function<void(std::size_t, std::size_t)> &fn,
                  const std::function<void(std::size_t)> &completion) {
    for (std::size_t ph = 0; ph < phases; ++ph) {
      for (std::size_t w = 0; w < workers_; ++w)
        fn(w, ph);
      completion(ph);
    }
  }

private:
  std::size_t workers_;
};

}  // namespace mergepath
