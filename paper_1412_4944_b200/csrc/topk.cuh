// Register-resident selection networks for the hard-threshold step (onb.py:58-76)
// in the tensor-core epilogues.  All indices are compile-time constants, so the
// arrays stay in registers; every comparator is one FMNMX pair.
#pragma once

namespace sbo {
namespace topk {

// element max / min: FMNMX for float32 values, IMNMX for integer keys
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ float vmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ int vmax(int a, int b) { return max(a, b); }
__device__ __forceinline__ int vmin(int a, int b) { return min(a, b); }

// compare-exchange so that v[i] >= v[j]
template <typename T>
__device__ __forceinline__ void cx(T& a, T& b) {
  const T hi = vmax(a, b), lo = vmin(a, b);
  a = hi;
  b = lo;
}

// a bitonic sequence of N -> sorted descending
template <int N, typename T>
__device__ __forceinline__ void merge_desc(T* v) {
#pragma unroll
  for (int half = N / 2; half >= 1; half >>= 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if ((i & half) == 0) cx(v[i], v[i + half]);
    }
  }
}

// 8 values -> sorted descending with the optimal 19-comparator network (depth 6)
template <typename T>
__device__ __forceinline__ void sort8_desc(T* v) {
  cx(v[0], v[2]); cx(v[1], v[3]); cx(v[4], v[6]); cx(v[5], v[7]);
  cx(v[0], v[4]); cx(v[1], v[5]); cx(v[2], v[6]); cx(v[3], v[7]);
  cx(v[0], v[1]); cx(v[2], v[3]); cx(v[4], v[5]); cx(v[6], v[7]);
  cx(v[2], v[4]); cx(v[3], v[5]);
  cx(v[1], v[4]); cx(v[3], v[6]);
  cx(v[1], v[2]); cx(v[3], v[4]); cx(v[5], v[6]);
}

// any N (power of two) -> sorted descending (bitonic sort; 8 uses sort8_desc)
template <int N, typename T>
__device__ __forceinline__ void sort_desc(T* v) {
  if constexpr (N == 8) {
    sort8_desc(v);
    return;
  }
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int half = size / 2; half >= 1; half >>= 1) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int j = i ^ half;
        if (j > i) {
          // descending inside even `size`-blocks, ascending inside odd ones,
          // except the final pass which is all descending
          const bool desc = (size == N) || ((i & size) == 0);
          if (desc) cx(v[i], v[j]);
          else cx(v[j], v[i]);
        }
      }
    }
  }
}

// top-G (sorted descending) of the union of two sorted-descending lists a, b;
// result in a.  c_i = max(a_i, b_{G-1-i}) is bitonic and holds the top G.
template <int G, typename T>
__device__ __forceinline__ void merge_top(T* a, const T* b) {
#pragma unroll
  for (int i = 0; i < G; ++i) a[i] = vmax(a[i], b[G - 1 - i]);
  merge_desc<G>(a);
}

// top-G of 64 values, sorted descending, into v[0..G) (v is destroyed)
template <int G>
__device__ __forceinline__ void top_of_64(float* v) {
  static_assert(G >= 1 && G <= 64 && (G & (G - 1)) == 0, "G must be a power of two <= 64");
#pragma unroll
  for (int g = 0; g < 64; g += G) sort_desc<G>(v + g);
#pragma unroll
  for (int step = G; step < 64; step <<= 1) {
#pragma unroll
    for (int g = 0; g + step < 64; g += 2 * step) merge_top<G>(v + g, v + g + step);
  }
}

// As top_of_64, also summing every value the network discards (each merge
// keeps max(a_i, b_{G-1-i}) and drops the min): sum(v) = sum(top) + dropped,
// with dropped accumulated from the small values themselves (no cancellation).
// SORTED = false: the final merge leaves v[0..G) as the top-G SET (bitonic, not
// sorted) — enough when every one of them is kept (k == G).
template <int G, bool SORTED = true>
__device__ __forceinline__ float top_of_64_dropped(float* v) {
  float dropped = 0.0f;
#pragma unroll
  for (int g = 0; g < 64; g += G) sort_desc<G>(v + g);
#pragma unroll
  for (int step = G; step < 64; step <<= 1) {
#pragma unroll
    for (int g = 0; g + step < 64; g += 2 * step) {
      float* a = v + g;
      const float* b = v + g + step;
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const float x = a[i], y = b[G - 1 - i];
        a[i] = fmaxf(x, y);
        dropped += fminf(x, y);
      }
      if (SORTED || 2 * step < 64) merge_desc<G>(a);
    }
  }
  return dropped;
}

}  // namespace topk
}  // namespace sbo
