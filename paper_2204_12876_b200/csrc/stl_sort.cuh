// std::sort(first, last) on doubles with operator<, step for step as the
// reference's toolchain runs it (libstdc++ introsort: depth limit 2*floor(log2 n),
// median-of-three pivot moved to the front, unguarded Hoare partition, heap sort
// when the depth limit runs out, then a final insertion sort over 16-element
// runs). The reference's median filter sorts each window with it
// (postprocess.cpp:134-162) and takes the middle element(s); which of two
// equal-comparing values (+0 / -0) or where a NaN ends up there depends on
// these exact moves, so the device repeats them instead of using any sort.
// __host__ __device__: tests/native/stl_sort_check.cpp runs it against
// std::sort on the host (random, tied, signed-zero and NaN windows).
#pragma once

#if defined(__CUDACC__)
#define RB_HD __host__ __device__ __forceinline__
#else
#define RB_HD inline
#endif

namespace rb200 {
namespace stl {

constexpr int kThreshold = 16;  // libstdc++ _S_threshold

RB_HD void swapAt(double* a, int i, int j) {
  const double t = a[i];
  a[i] = a[j];
  a[j] = t;
}

RB_HD void moveMedianToFirst(double* a, int result, int x, int y, int z) {
  if (a[x] < a[y]) {
    if (a[y] < a[z]) swapAt(a, result, y);
    else if (a[x] < a[z]) swapAt(a, result, z);
    else swapAt(a, result, x);
  } else if (a[x] < a[z]) {
    swapAt(a, result, x);
  } else if (a[y] < a[z]) {
    swapAt(a, result, z);
  } else {
    swapAt(a, result, y);
  }
}

// __unguarded_partition(first, last, pivot): the scans stop at the array ends
// too (the library relies on sentinels there, which hold for any input in
// which it does not run off the array).
RB_HD int unguardedPartition(double* a, int first, int last, int pivot, int lo, int hi) {
  while (true) {
    while (first < hi && a[first] < a[pivot]) ++first;
    --last;
    while (last > lo && a[pivot] < a[last]) --last;
    if (!(first < last)) return first;
    swapAt(a, first, last);
    ++first;
  }
}

RB_HD void pushHeap(double* a, int first, int hole, int top, double value) {
  int parent = (hole - 1) / 2;
  while (hole > top && a[first + parent] < value) {
    a[first + hole] = a[first + parent];
    hole = parent;
    parent = (hole - 1) / 2;
  }
  a[first + hole] = value;
}

RB_HD void adjustHeap(double* a, int first, int hole, int len, double value) {
  const int top = hole;
  int child = hole;
  while (child < (len - 1) / 2) {
    child = 2 * (child + 1);
    if (a[first + child] < a[first + child - 1]) --child;
    a[first + hole] = a[first + child];
    hole = child;
  }
  if ((len & 1) == 0 && child == (len - 2) / 2) {
    child = 2 * (child + 1);
    a[first + hole] = a[first + child - 1];
    hole = child - 1;
  }
  pushHeap(a, first, hole, top, value);
}

// __partial_sort(first, last, last) = make_heap + sort_heap
RB_HD void heapSort(double* a, int first, int last) {
  const int len = last - first;
  if (len >= 2) {
    for (int parent = (len - 2) / 2;; --parent) {
      adjustHeap(a, first, parent, len, a[first + parent]);
      if (parent == 0) break;
    }
  }
  while (last - first > 1) {
    --last;
    const double value = a[last];
    a[last] = a[first];
    adjustHeap(a, first, 0, last - first, value);
  }
}

RB_HD void unguardedLinearInsert(double* a, int i, int lo) {
  const double val = a[i];
  int next = i - 1;
  while (next >= lo && val < a[next]) {
    a[i] = a[next];
    i = next;
    --next;
  }
  a[i] = val;
}

RB_HD void insertionSort(double* a, int first, int last) {
  if (first == last) return;
  for (int i = first + 1; i < last; ++i) {
    if (a[i] < a[first]) {
      const double val = a[i];
      for (int k = i; k > first; --k) a[k] = a[k - 1];
      a[first] = val;
    } else {
      unguardedLinearInsert(a, i, first);
    }
  }
}

// n <= 128. __introsort_loop partitions [first, last), recurses into the
// right part and loops on the left one; the two parts are disjoint and each
// one's moves depend only on its own contents and depth, so they are taken
// here from an explicit stack (at most one entry per depth level).
RB_HD void sort(double* a, int n) {
  if (n <= 1) return;
  int lg = 0;
  while ((2 << lg) <= n) ++lg;  // floor(log2 n)
  int st_first[16], st_last[16], st_depth[16];
  int sp = 0;
  st_first[sp] = 0;
  st_last[sp] = n;
  st_depth[sp] = 2 * lg;
  ++sp;
  while (sp > 0) {
    --sp;
    const int first = st_first[sp];
    int last = st_last[sp];
    int depth = st_depth[sp];
    while (last - first > kThreshold) {
      if (depth == 0) {
        heapSort(a, first, last);
        break;
      }
      --depth;
      const int mid = first + (last - first) / 2;
      moveMedianToFirst(a, first, first + 1, mid, last - 1);
      const int cut = unguardedPartition(a, first + 1, last, first, 0, n);
      st_first[sp] = cut;
      st_last[sp] = last;
      st_depth[sp] = depth;
      ++sp;
      last = cut;
    }
  }
  // __final_insertion_sort
  if (n > kThreshold) {
    insertionSort(a, 0, kThreshold);
    for (int i = kThreshold; i < n; ++i) unguardedLinearInsert(a, i, 0);
  } else {
    insertionSort(a, 0, n);
  }
}

}  // namespace stl
}  // namespace rb200
