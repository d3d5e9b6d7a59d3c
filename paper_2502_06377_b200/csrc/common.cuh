// Shared device helpers for the IBMI B200 library (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>

namespace ibmi {

// Logical index -> physical index with at most one gap.  A contiguous set
// [lo, hi) of a p-index problem has complement [0, lo) u [hi, p): logical
// complement index i maps to i (< lo) or i + (hi - lo) (>= lo).  This is how
// every kernel addresses Σ[c, c] without gathering it (the reference gathers
// with np.ix_, linalg.py:186-191).
// A general (non-contiguous) index set uses an explicit device index list
// instead (`idx`, sorted ascending), e.g. the sets of a custom overlapping
// partition (reference partition.py:124-141).
struct RowMap {
  int split;      // i < split -> off0 + i ; else off1 + (i - split)
  int64_t off0;
  int64_t off1;
  const int64_t* idx;   // non-null: i -> idx[i]
};

__host__ __device__ __forceinline__ int64_t map_idx(const RowMap& m, int i) {
  if (m.idx) return m.idx[i];
  return i < m.split ? m.off0 + i : m.off1 + (int64_t)(i - m.split);
}

inline RowMap contig_map(int64_t off) { return RowMap{INT_MAX, off, 0, nullptr}; }
inline RowMap list_map(const int64_t* idx) { return RowMap{INT_MAX, 0, 0, idx}; }
// complement of [lo, hi): logical [0, lo) -> [0, lo), [lo, ..) -> [hi, ..)
inline RowMap complement_map(int64_t lo, int64_t hi) {
  return RowMap{(int)lo, 0, hi, nullptr};
}

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// 16-byte async copy global->shared, zero-filling the tail beyond src_bytes.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes));
}
// 8-byte async copy (unaligned problems), zero-fill when src_bytes == 0.
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace ibmi
