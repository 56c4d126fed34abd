// ORACLE — TEST INFRASTRUCTURE ONLY (see sko.hpp).
// Restates parallel.hpp:17-40: static contiguous chunking with a fresh
// std::thread pool per call, capped by max_threads(); tasks write disjoint
// outputs so results do not depend on scheduling.
#pragma once

#include <algorithm>
#include <thread>
#include <vector>

namespace sko {

template <typename Fn>
void parallel_for(Index begin, Index end, Fn&& fn) {
  const Index n = end - begin;
  if (n <= 0) return;
  const int nt = int(std::max<Index>(1, std::min<Index>(max_threads(), n)));
  if (nt == 1) {
    for (Index i = begin; i < end; ++i) fn(i);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(std::size_t(nt - 1));
  const Index chunk = (n + nt - 1) / nt;
  for (int t = 1; t < nt; ++t) {
    const Index lo = begin + t * chunk;
    const Index hi = std::min(end, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([lo, hi, &fn] {
      for (Index i = lo; i < hi; ++i) fn(i);
    });
  }
  const Index hi0 = std::min(end, begin + chunk);
  for (Index i = begin; i < hi0; ++i) fn(i);
  for (auto& th : pool) th.join();
}

}  // namespace sko
