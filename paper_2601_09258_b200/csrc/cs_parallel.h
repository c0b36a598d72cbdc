// cs_parallel.h — the host services' fork-join helper: f(begin, end, thread)
// on n_threads contiguous slices of [0, n) (at most one thread per item).
#pragma once
#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <thread>
#include <vector>

namespace cs_host {

template <typename F>
void parallel_for(size_t n, uint32_t n_threads, F f) {
  const uint32_t nt = std::max<uint32_t>(1, static_cast<uint32_t>(std::min<size_t>(n_threads, n ? n : 1)));
  std::vector<std::thread> th;
  for (uint32_t t = 0; t < nt; ++t) th.emplace_back([&, t] { f(n * t / nt, n * (t + 1) / nt, t); });
  for (auto& x : th) x.join();
}

}  // namespace cs_host
