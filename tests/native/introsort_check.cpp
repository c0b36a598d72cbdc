// Checks cs_introsort.h against the host's std::sort: sorting (key, payload)
// pairs with a key-only comparator must give the same permutation as
// cs_sort::sort on positions and as the device fit's range-step scheme.  Many ties, sorted / reversed / organ-pipe
// inputs, and median-of-three-adversarial inputs that reach the heap-sort
// fallback.  Prints "ok <cases>" or the first mismatch.
#include <algorithm>
#include <cstdio>
#include <random>
#include <utility>
#include <vector>

#include "../../paper_2601_09258_b200/csrc/cs_introsort.h"

struct KP {
  double key;
  uint32_t pos, pad;
};
struct KPLess {
  bool operator()(const KP& a, const KP& b) const { return a.key < b.key; }
};

// the device fit's scheme: (key, position) pairs, partition ranges taken in
// an arbitrary (here LIFO-from-the-left) order, final ranges insertion-sorted
// independently afterwards
static std::vector<uint32_t> range_steps(const std::vector<double>& key, uint64_t seed) {
  const uint32_t n = static_cast<uint32_t>(key.size());
  std::vector<KP> a(n);
  for (uint32_t i = 0; i < n; ++i) a[i] = {key[i], i, 0};
  std::vector<cs_sort::Range> work, fin;
  if (n > cs_sort::kThreshold) work.push_back(cs_sort::start(0, n));
  else fin.push_back({0, n, 0});
  std::mt19937_64 rng(seed);
  while (!work.empty()) {
    const size_t k = rng() % work.size();  // any order
    const cs_sort::Range r = work[k];
    work.erase(work.begin() + static_cast<long>(k));
    cs_sort::Range out[2];
    unsigned fm = 0;
    const int c = cs_sort::step(a.data(), r, KPLess{}, out, &fm);
    for (int i = 0; i < c; ++i) ((fm >> i) & 1 ? fin : work).push_back(out[i]);
  }
  for (const auto& r : fin) cs_sort::insertion_sort(a.data(), r.first, r.last, KPLess{});
  std::vector<uint32_t> p(n);
  for (uint32_t i = 0; i < n; ++i) p[i] = a[i].pos;
  return p;
}

static bool check(const std::vector<double>& key, const char* what) {
  std::vector<std::pair<double, uint32_t>> p(key.size());
  for (size_t i = 0; i < key.size(); ++i) p[i] = {key[i], static_cast<uint32_t>(i)};
  std::sort(p.begin(), p.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  std::vector<uint32_t> a(key.size());
  for (size_t i = 0; i < key.size(); ++i) a[i] = static_cast<uint32_t>(i);
  cs_sort::sort(a.data(), static_cast<int64_t>(a.size()), key.data());
  const std::vector<uint32_t> b = range_steps(key, key.size());
  for (size_t i = 0; i < key.size(); ++i)
    if (a[i] != p[i].second || b[i] != p[i].second) {
      std::printf("mismatch %s n=%zu at %zu (%s)\n", what, key.size(), i,
                  a[i] != p[i].second ? "index sort" : "range steps");
      return false;
    }
  return true;
}

// the "median-of-3 killer" permutation (Musser) for n even
static std::vector<double> m3_killer(size_t n) {
  std::vector<double> v(n);
  const size_t k = n / 2;
  for (size_t i = 1; i <= k; ++i) {
    if (i % 2) {
      v[i - 1] = static_cast<double>(i);
      v[i] = static_cast<double>(k + i);
    }
    v[k + i - 1] = static_cast<double>(2 * i);
  }
  return v;
}

int main() {
  std::mt19937_64 rng(7);
  size_t cases = 0;
  for (int rep = 0; rep < 3000; ++rep) {
    const size_t n = rep < 200 ? rep : 1 + rng() % 5000;
    const int distinct = 1 + static_cast<int>(rng() % (rep % 3 == 0 ? 4 : rep % 3 == 1 ? 64 : 100000));
    std::vector<double> k(n);
    for (auto& x : k) x = static_cast<double>(rng() % distinct);
    if (!check(k, "random")) return 1;
    std::vector<double> s = k;
    std::sort(s.begin(), s.end());
    if (!check(s, "sorted")) return 1;
    std::reverse(s.begin(), s.end());
    if (!check(s, "reversed")) return 1;
    std::vector<double> organ(n);
    for (size_t i = 0; i < n; ++i) organ[i] = static_cast<double>(std::min(i, n - i) % (distinct + 1));
    if (!check(organ, "organ")) return 1;
    cases += 4;
  }
  for (size_t n = 2; n < 6000; n += 98) {
    if (!check(m3_killer(n), "m3killer")) return 1;
    ++cases;
  }
  // signed zeros compare equal; NaN-free inputs only (the fit's features are finite)
  std::vector<double> z = {0.0, -0.0, 1.0, -0.0, 0.0, 2.0, -1.0, 0.0};
  for (int i = 0; i < 5; ++i) z.insert(z.end(), z.begin(), z.end());
  if (!check(z, "zeros")) return 1;
  std::printf("ok %zu\n", cases + 1);
  return 0;
}
