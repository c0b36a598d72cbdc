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

CS_HD void swap(uint32_t* a, int64_t i, int64_t j) {
  const uint32_t t = a[i];
  a[i] = a[j];
  a[j] = t;
}

// ---- heap (stl_heap.h)
CS_HD void push_heap(uint32_t* a, int64_t hole, int64_t top, uint32_t value, const Less& lt) {
  int64_t parent = (hole - 1) / 2;
  while (hole > top && lt(a[parent], value)) {
    a[hole] = a[parent];
    hole = parent;
    parent = (hole - 1) / 2;
  }
  a[hole] = value;
}

CS_HD void adjust_heap(uint32_t* a, int64_t hole, int64_t len, uint32_t value, const Less& lt) {
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

CS_HD void make_heap(uint32_t* a, int64_t len, const Less& lt) {
  if (len < 2) return;
  int64_t parent = (len - 2) / 2;
  while (true) {
    adjust_heap(a, parent, len, a[parent], lt);
    if (parent == 0) return;
    --parent;
  }
}

// __partial_sort(first, last, last): __heap_select (make_heap only) + __sort_heap
CS_HD void heap_sort(uint32_t* a, int64_t len, const Less& lt) {
  make_heap(a, len, lt);
  while (len > 1) {
    --len;
    const uint32_t value = a[len];
    a[len] = a[0];
    adjust_heap(a, 0, len, value, lt);
  }
}

// ---- partition
CS_HD void move_median_to_first(uint32_t* a, int64_t result, int64_t x, int64_t y, int64_t z,
                                const Less& lt) {
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

CS_HD int64_t unguarded_partition(uint32_t* a, int64_t first, int64_t last, int64_t pivot, const Less& lt) {
  while (true) {
    while (lt(a[first], a[pivot])) ++first;
    --last;
    while (lt(a[pivot], a[last])) --last;
    if (!(first < last)) return first;
    swap(a, first, last);
    ++first;
  }
}

CS_HD int64_t partition_pivot(uint32_t* a, int64_t first, int64_t last, const Less& lt) {
  const int64_t mid = first + (last - first) / 2;
  move_median_to_first(a, first, first + 1, mid, last - 1, lt);
  return unguarded_partition(a, first + 1, last, first, lt);
}

// ---- insertion sorts
CS_HD void unguarded_linear_insert(uint32_t* a, int64_t last, const Less& lt) {
  const uint32_t val = a[last];
  int64_t next = last - 1;
  while (lt(val, a[next])) {
    a[last] = a[next];
    last = next;
    --next;
  }
  a[last] = val;
}

CS_HD void insertion_sort(uint32_t* a, int64_t first, int64_t last, const Less& lt) {
  if (first == last) return;
  for (int64_t i = first + 1; i != last; ++i) {
    if (lt(a[i], a[first])) {
      const uint32_t val = a[i];
      for (int64_t k = i; k > first; --k) a[k] = a[k - 1];
      a[first] = val;
    } else {
      unguarded_linear_insert(a, i, lt);
    }
  }
}

constexpr int64_t kThreshold = 16;

// __introsort_loop, with the recursion on the right part made explicit (a
// stack of pending [first, last, depth) ranges processed in the same order)
CS_HD void introsort_loop(uint32_t* a, int64_t first0, int64_t last0, int depth0, const Less& lt) {
  struct Range {
    int64_t first, last;
    int depth;
  };
  Range stack[66];  // pending continuations <= the depth limit 2*lg(n) <= 64
  int sp = 0;
  stack[sp++] = {first0, last0, depth0};
  while (sp) {
    Range r = stack[--sp];
    // a call: loop on [first, last); each cut's right part is a nested call
    // that completes before this call continues with the left part, so the
    // left part is pushed first and the right part on top of it
    while (r.last - r.first > kThreshold) {
      if (r.depth == 0) {
        heap_sort(a + r.first, r.last - r.first, lt);
        r.last = r.first;  // this call returns
        break;
      }
      --r.depth;
      const int64_t cut = partition_pivot(a, r.first, r.last, lt);
      stack[sp++] = {r.first, cut, r.depth};  // continuation of this call
      r = Range{cut, r.last, r.depth};          // the nested call, run now
    }
  }
}

// std::sort(a, a + n, key-less-than)
CS_HD void sort(uint32_t* a, int64_t n, const double* key) {
  const Less lt{key};
  if (n <= 1) return;
  introsort_loop(a, 0, n, 2 * lg(n), lt);
  if (n > kThreshold) {
    insertion_sort(a, 0, kThreshold, lt);
    for (int64_t i = kThreshold; i < n; ++i) unguarded_linear_insert(a, i, lt);
  } else {
    insertion_sort(a, 0, n, lt);
  }
}

}  // namespace cs_sort
