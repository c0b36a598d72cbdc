// cs_introsort.h — libstdc++'s std::sort (bits/stl_algo.h, bits/stl_heap.h:
// __introsort_loop with the median-of-three unguarded partition, heap-sort
// fallback at depth 2*lg(n), final insertion sort with threshold 16) restated
// on an index array, usable on the host and the device.
//
// The GBDT fit (gbdt.cpp:60-63) sorts (feature value, residual) pairs with a
// comparator on the feature value only, so the order of equal keys — and with
// it the order in which residuals are summed — is whatever this algorithm
// produces from the input order.  Sorting positions with key[pos] reproduces
// the pairs' permutation exactly: the comparisons and moves are the same.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define CS_HD __host__ __device__ __forceinline__
#else
#define CS_HD inline
#endif

namespace cs_sort {

// Element-generic restatement: E is the moved element, lt(E, E) the
// comparator.  Index sorts use E = uint32_t with Less (key[a] < key[b]);
// the device fit sorts (key, row) pairs directly.
struct Less {
  const double* key;
  CS_HD bool operator()(uint32_t a, uint32_t b) const { return key[a] < key[b]; }
};

CS_HD int lg(int64_t n) {  // std::__lg
  int k = 0;
  while (n > 1) {
    n >>= 1;
    ++k;
  }
  return k;
}

template <typename E>
CS_HD void swap(E* a, int64_t i, int64_t j) {
  const E t = a[i];
  a[i] = a[j];
  a[j] = t;
}

// ---- heap (stl_heap.h)
template <typename E, typename Lt>
CS_HD void push_heap(E* a, int64_t hole, int64_t top, E value, const Lt& lt) {
  int64_t parent = (hole - 1) / 2;
  while (hole > top && lt(a[parent], value)) {
    a[hole] = a[parent];
    hole = parent;
    parent = (hole - 1) / 2;
  }
  a[hole] = value;
}

template <typename E, typename Lt>
CS_HD void adjust_heap(E* a, int64_t hole, int64_t len, E value, const Lt& lt) {
  const int64_t top = hole;
  int64_t child = hole;
  while (child < (len - 1) / 2) {
    child = 2 * (child + 1);
    if (lt(a[child], a[child - 1])) --child;
    a[hole] = a[child];
    hole = child;
  }
  if ((len & 1) == 0 && child == (len - 2) / 2) {
    child = 2 * (child + 1);
    a[hole] = a[child - 1];
    hole = child - 1;
  }
  push_heap(a, hole, top, value, lt);
}

template <typename E, typename Lt>
CS_HD void make_heap(E* a, int64_t len, const Lt& lt) {
  if (len < 2) return;
  int64_t parent = (len - 2) / 2;
  while (true) {
    adjust_heap(a, parent, len, a[parent], lt);
    if (parent == 0) return;
    --parent;
  }
}

// __partial_sort(first, last, last): __heap_select (make_heap only) + __sort_heap
template <typename E, typename Lt>
CS_HD void heap_sort(E* a, int64_t len, const Lt& lt) {
  make_heap(a, len, lt);
  while (len > 1) {
    --len;
    const E value = a[len];
    a[len] = a[0];
    adjust_heap(a, 0, len, value, lt);
  }
}

// ---- partition
template <typename E, typename Lt>
CS_HD void move_median_to_first(E* a, int64_t result, int64_t x, int64_t y, int64_t z, const Lt& lt) {
  if (lt(a[x], a[y])) {
    if (lt(a[y], a[z])) swap(a, result, y);
    else if (lt(a[x], a[z])) swap(a, result, z);
    else swap(a, result, x);
  } else if (lt(a[x], a[z])) {
    swap(a, result, x);
  } else if (lt(a[y], a[z])) {
    swap(a, result, z);
  } else {
    swap(a, result, y);
  }
}

// the pivot sits outside [first, last) and is never moved by the scan, so
// its value is held in a register
template <typename E, typename Lt>
CS_HD int64_t unguarded_partition(E* a, int64_t first, int64_t last, int64_t pivot, const Lt& lt) {
  const E pv = a[pivot];
  while (true) {
    while (lt(a[first], pv)) ++first;
    --last;
    while (lt(pv, a[last])) --last;
    if (!(first < last)) return first;
    swap(a, first, last);
    ++first;
  }
}

template <typename E, typename Lt>
CS_HD int64_t partition_pivot(E* a, int64_t first, int64_t last, const Lt& lt) {
  const int64_t mid = first + (last - first) / 2;
  move_median_to_first(a, first, first + 1, mid, last - 1, lt);
  return unguarded_partition(a, first + 1, last, first, lt);
}

// ---- insertion sorts
template <typename E, typename Lt>
CS_HD void unguarded_linear_insert(E* a, int64_t last, const Lt& lt) {
  const E val = a[last];
  int64_t next = last - 1;
  while (lt(val, a[next])) {
    a[last] = a[next];
    last = next;
    --next;
  }
  a[last] = val;
}

template <typename E, typename Lt>
CS_HD void insertion_sort(E* a, int64_t first, int64_t last, const Lt& lt) {
  if (first == last) return;
  for (int64_t i = first + 1; i != last; ++i) {
    if (lt(a[i], a[first])) {
      const E val = a[i];
      for (int64_t k = i; k > first; --k) a[k] = a[k - 1];
      a[first] = val;
    } else {
      unguarded_linear_insert(a, i, lt);
    }
  }
}

constexpr int64_t kThreshold = 16;

// __introsort_loop, with the recursion on the right part made explicit (a
// stack of pending [first, last, depth) ranges).  The ranges are disjoint,
// so the order in which they are processed does not change the result.
template <typename E, typename Lt>
CS_HD void introsort_loop(E* a, int64_t first0, int64_t last0, int depth0, const Lt& lt) {
  struct Range {
    int64_t first, last;
    int depth;
  };
  Range stack[66];  // pending continuations <= the depth limit 2*lg(n) <= 64
  int sp = 0;
  stack[sp++] = {first0, last0, depth0};
  while (sp) {
    Range r = stack[--sp];
    while (r.last - r.first > kThreshold) {
      if (r.depth == 0) {
        heap_sort(a + r.first, r.last - r.first, lt);
        break;
      }
      --r.depth;
      const int64_t cut = partition_pivot(a, r.first, r.last, lt);
      stack[sp++] = {r.first, cut, r.depth};  // continuation of this call
      r = Range{cut, r.last, r.depth};          // the nested call, run now
    }
  }
}

// __final_insertion_sort.  After the partitions no element is smaller than
// anything in an earlier partition range (left part <= pivot <= right part),
// so this is also an independent insertion sort of each final range.
template <typename E, typename Lt>
CS_HD void final_insertion_sort(E* a, int64_t n, const Lt& lt) {
  if (n > kThreshold) {
    insertion_sort(a, 0, kThreshold, lt);
    for (int64_t i = kThreshold; i < n; ++i) unguarded_linear_insert(a, i, lt);
  } else {
    insertion_sort(a, 0, n, lt);
  }
}

// ---- the same sort as independent range steps (the device fit runs the
// partition tree level by level, then the final ranges in parallel):
// start(n) -> one work range or one final range; step(range) -> heap sort
// (depth exhausted: sorted, nothing left to do) or a partition into two
// children, each a work range (> kThreshold) or a final range; finally
// insertion_sort(a, first, last) of every final range.
struct Range {
  uint32_t first, last, depth;
};
// returns the number of children written to out[0..1]; *final_mask bit i
// set when out[i] is a final range
template <typename E, typename Lt>
CS_HD int step(E* a, const Range& r, const Lt& lt, Range out[2], unsigned* final_mask) {
  *final_mask = 0;
  if (r.depth == 0) {
    heap_sort(a + r.first, r.last - r.first, lt);
    return 0;
  }
  const uint32_t cut = (uint32_t)partition_pivot(a, r.first, r.last, lt);
  out[0] = Range{r.first, cut, r.depth - 1};
  out[1] = Range{cut, r.last, r.depth - 1};
  if (cut - r.first <= (uint32_t)kThreshold) *final_mask |= 1u;
  if (r.last - cut <= (uint32_t)kThreshold) *final_mask |= 2u;
  return 2;
}
CS_HD Range start(uint32_t first, uint32_t n) { return Range{first, first + n, (uint32_t)(2 * lg(n))}; }

// std::sort(a, a + n, lt)
template <typename E, typename Lt>
CS_HD void sort_with(E* a, int64_t n, const Lt& lt) {
  if (n <= 1) return;
  introsort_loop(a, 0, n, 2 * lg(n), lt);
  final_insertion_sort(a, n, lt);
}

// std::sort of positions by key[position]
CS_HD void sort(uint32_t* a, int64_t n, const double* key) { sort_with(a, n, Less{key}); }

}  // namespace cs_sort
