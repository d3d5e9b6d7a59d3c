// Fused sweep for small problems (p <= 1024; BASELINE c1 is p = 512, two sets).
//
// One sweep of the reference's solve loop (solver.py:257-265) — the K block
// updates of _BlockOp.apply (solver.py:122-129) and the matrix of the error
// estimate (solver.py:154) with its Gram form — as ONE cooperative kernel.
//
// Why: at p = 512 every GEMM of a block step is ~33 MFLOP, about 1 µs of FP64
// tensor work, but each launch of the big-tile TMA GEMM costs 15-35 µs of
// latency (pipeline fill, 128×128 tiles on 4 of 148 SMs, split-K reduction
// launches).  The 14 launches of a c1 sweep took 0.235 ms for 0.2 GFLOP.  Here
// the phases are separated by grid barriers (1.3-1.7 µs each) instead of launches,
// tiles are 16×32 so 128 CTAs share a 256×256 product (a 32×32 tile with K = 256
// is 2.1 µs of DMMA on one SM: the first version's 64 CTAs left 84 SMs idle and
// spent 5.7 µs per phase, this one 4.0), and operands stream from L2 straight
// into DMMA fragments (Σ, A and W are 2 MB each at c1: L2-resident; staging them
// through shared memory with cp.async was measured slower, 7.1 µs per phase).
//
// Phases (set k: I = [lo, hi), b rows, complement c through a one-gap map):
//   A_k  Σ[I, c] = −W_k·Σ[c, c],  Σ[c, I] = its transpose          (b × c tiles, K = c)
//   B_k  Σ[I, I] = A_II⁻¹ − Σ[I, c]·W_kᵀ, lower tiles mirrored     (b × b lower tiles, K = c)
//   C    B = Σ[I_K, :]·A[:, c_K]                                   (b × c tiles, K = p)
//   D    G = B·Bᵀ (lower tiles mirrored), y₁ = B·(1/√c)            (feeds the power iteration)
// Each CTA computes 16×32 output tiles; its 8 warps split K, each holding a
// 16×32 accumulator in DMMA fragments, summed through shared memory in a fixed
// pairwise order (deterministic).  Σ and B are read with ld.global.cg: other CTAs wrote
// them earlier in this kernel, so L1 must be bypassed.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace ibmi {
namespace cg = cooperative_groups;

constexpr int SS_MAX_SETS = 16;
constexpr int SS_TILE = 32;       // tile columns (N)
constexpr int SS_TM = 16;         // tile rows (M): 16 × 32 tiles put 128+ CTAs on a 256 × 256 product (c1)
constexpr int SS_THREADS = 256;
constexpr int SS_SMEM = 8 * SS_TM * (SS_TILE + 1) * (int)sizeof(double);   // 8 warps × 16 × 33 doubles

struct SmallSet {
  int lo, hi;
  const double* W;      // b × ld, global column coordinates, zero on I
  const double* ainv;   // b × ldb
  int64_t ldb;
};

struct SmallSweepParams {
  double* S;
  const double* A;
  int64_t ld;
  int p, K;
  SmallSet set[SS_MAX_SETS];
  int estimate;         // 1: phases C and D on the last set
  double* B; int64_t ldB;
  double* G; int64_t ldG;
  double* y1;
  unsigned long long* trace;   // optional (IBMI_SS_TRACE=1): %globaltimer of block 0 after each phase
};

struct SsOperand {
  const double* base;
  int64_t ld;
  int split;            // logical row i -> i < split ? off0 + i : off1 + (i - split)
  int off0, off1;
  int rows;
  bool cg;              // read through L2 only (written earlier in this kernel)
};

__device__ __forceinline__ int ss_row(const SsOperand& o, int i) { return i < o.split ? o.off0 + i : o.off1 + (i - o.split); }

// acc(32×32 at tile tm, tn) = Σ_seg Σ_k X[xrow(m)][k0 + k]·Y[yrow(n)][k0 + k]; element (r, c) of the
// tile is handed to epi(m, n, value) by exactly one thread.
template <class Epi>
__device__ __forceinline__ void ss_tile(const SsOperand& X, const SsOperand& Y, int nseg, const int* seg_k0,
                                        const int* seg_len, int tm, int tn, double* red, Epi epi) {
  constexpr int MI = SS_TM / 8, NJ = SS_TILE / 8;      // 2 × 4 DMMA tiles of 8 × 8 per warp
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const double* xr[MI];
  const double* yr[NJ];
  bool xv[MI], yv[NJ];
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int m = tm * SS_TM + 8 * i + g;
    xv[i] = m < X.rows;
    xr[i] = X.base + (int64_t)(xv[i] ? ss_row(X, m) : 0) * X.ld;
  }
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int n = tn * SS_TILE + 8 * j + g;
    yv[j] = n < Y.rows;
    yr[j] = Y.base + (int64_t)(yv[j] ? ss_row(Y, n) : 0) * Y.ld;
  }
  for (int s = 0; s < nseg; ++s) {
    const int k0 = seg_k0[s], len = seg_len[s];
    const int steps = (len + 3) >> 2;
    const int per = (steps + 7) >> 3;                  // k-steps per warp, contiguous slice
    const int s0 = wid * per, s1 = min(steps, s0 + per);
#pragma unroll 4
    for (int ks = s0; ks < s1; ++ks) {
      const int k = 4 * ks + t;
      const bool kv = k < len;
      double a[MI], b[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = (kv && xv[i]) ? (X.cg ? __ldcg(xr[i] + k0 + k) : __ldg(xr[i] + k0 + k)) : 0.0;
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[j] = (kv && yv[j]) ? (Y.cg ? __ldcg(yr[j] + k0 + k) : __ldg(yr[j] + k0 + k)) : 0.0;
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  double* mine = red + wid * SS_TM * (SS_TILE + 1);
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      mine[(8 * i + g) * (SS_TILE + 1) + 8 * j + 2 * t] = acc[i][j][0];
      mine[(8 * i + g) * (SS_TILE + 1) + 8 * j + 2 * t + 1] = acc[i][j][1];
    }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < SS_TM * SS_TILE / SS_THREADS; ++q) {
    const int e = tid + SS_THREADS * q;
    const int r = e >> 5, c = e & 31;
    double v[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) v[w] = red[w * SS_TM * (SS_TILE + 1) + r * (SS_TILE + 1) + c];
    epi(tm * SS_TM + r, tn * SS_TILE + c, ((v[0] + v[4]) + (v[2] + v[6])) + ((v[1] + v[5]) + (v[3] + v[7])));
  }
  __syncthreads();
}

// Lower-triangle tile walk of a b × b symmetric product with SS_TM × SS_TILE tiles: tile (tm, tn) is kept when
// its first column is not above its last row; elements above the diagonal are masked by the epilogue.
__device__ __forceinline__ bool ss_lower_tile(int tile, int b, int& tm, int& tn) {
  const int ntn = (b + SS_TILE - 1) / SS_TILE;
  tm = tile / ntn;
  tn = tile % ntn;
  return tn * SS_TILE <= tm * SS_TM + SS_TM - 1;
}

__device__ __forceinline__ void ss_stamp(const SmallSweepParams& P, int& slot) {
  if (P.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.trace[slot] = t;
  }
  ++slot;
}

__global__ void __launch_bounds__(SS_THREADS, 1) small_sweep_kernel(SmallSweepParams P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double ss_red[];
  const int p = P.p;
  const int64_t ld = P.ld;
  int slot = 0;
  ss_stamp(P, slot);
  for (int k = 0; k < P.K; ++k) {
    const SmallSet st = P.set[k];
    const int lo = st.lo, hi = st.hi, b = hi - lo, c = p - b;
    const int seg_k0[2] = {0, hi};
    const int seg_len[2] = {lo, p - hi};
    // ---- A_k: Σ[I, c] = −W·Σ[c, c], mirrored
    {
      const SsOperand X{st.W, ld, INT_MAX, 0, 0, b, false};
      const SsOperand Y{P.S, ld, lo, 0, hi, c, true};
      const int ntm = (b + SS_TM - 1) / SS_TM, ntn = (c + SS_TILE - 1) / SS_TILE;
      for (int tile = blockIdx.x; tile < ntm * ntn; tile += gridDim.x) {
        ss_tile(X, Y, 2, seg_k0, seg_len, tile / ntn, tile % ntn, ss_red, [&](int m, int n, double v) {
          if (m < b && n < c) {
            const int cn = n < lo ? n : n + b;
            P.S[(int64_t)(lo + m) * ld + cn] = -v;
            P.S[(int64_t)cn * ld + lo + m] = -v;
          }
        });
      }
    }
    ss_stamp(P, slot);
    __threadfence();
    grid.sync();
    ss_stamp(P, slot);
    // ---- B_k: Σ[I, I] = A_II⁻¹ − Σ[I, c]·Wᵀ, lower tiles mirrored
    {
      const SsOperand X{P.S, ld, INT_MAX, lo, 0, b, true};
      const SsOperand Y{st.W, ld, INT_MAX, 0, 0, b, false};
      const int ntiles = ((b + SS_TM - 1) / SS_TM) * ((b + SS_TILE - 1) / SS_TILE);
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int tm, tn;
        if (!ss_lower_tile(tile, b, tm, tn)) continue;
        ss_tile(X, Y, 2, seg_k0, seg_len, tm, tn, ss_red, [&](int m, int n, double v) {
          if (m < b && n <= m) {
            const double r = st.ainv[(int64_t)m * st.ldb + n] - v;
            P.S[(int64_t)(lo + m) * ld + lo + n] = r;
            P.S[(int64_t)(lo + n) * ld + lo + m] = r;
          }
        });
      }
    }
    ss_stamp(P, slot);
    __threadfence();
    grid.sync();
    ss_stamp(P, slot);
  }
  if (!P.estimate) return;
  const SmallSet st = P.set[P.K - 1];
  const int lo = st.lo, hi = st.hi, b = hi - lo, c = p - b;
  // ---- C: B = Σ[I, :]·A[:, c]   (A symmetric: A[j][c_n] = A[c_n][j])
  {
    const int k0[1] = {0}, len[1] = {p};
    const SsOperand X{P.S, ld, INT_MAX, lo, 0, b, true};
    const SsOperand Y{P.A, ld, lo, 0, hi, c, false};
    const int ntm = (b + SS_TM - 1) / SS_TM, ntn = (c + SS_TILE - 1) / SS_TILE;
    for (int tile = blockIdx.x; tile < ntm * ntn; tile += gridDim.x) {
      ss_tile(X, Y, 1, k0, len, tile / ntn, tile % ntn, ss_red, [&](int m, int n, double v) {
        if (m < b && n < c) P.B[(int64_t)m * P.ldB + n] = v;
      });
    }
  }
  ss_stamp(P, slot);
  __threadfence();
  grid.sync();
  ss_stamp(P, slot);
  // ---- D: G = B·Bᵀ (lower tiles mirrored), y₁ = B·(1/√c)
  {
    const int k0[1] = {0}, len[1] = {c};
    const SsOperand X{P.B, P.ldB, INT_MAX, 0, 0, b, true};
    const int ntiles = ((b + SS_TM - 1) / SS_TM) * ((b + SS_TILE - 1) / SS_TILE);
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int tm, tn;
      if (!ss_lower_tile(tile, b, tm, tn)) continue;
      ss_tile(X, X, 1, k0, len, tm, tn, ss_red, [&](int m, int n, double v) {
        if (m < b && n <= m) {
          P.G[(int64_t)m * P.ldG + n] = v;
          P.G[(int64_t)n * P.ldG + m] = v;
        }
      });
    }
    const double scale = 1.0 / sqrt((double)c);
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (SS_THREADS / 32) + (threadIdx.x >> 5), tw = gridDim.x * (SS_THREADS / 32);
    for (int r = gw; r < b; r += tw) {
      const double* row = P.B + (int64_t)r * P.ldB;
      double s = 0.0;
      for (int j = lane; j < c; j += 32) s = fma(__ldcg(row + j), scale, s);
      s = warp_sum(s);
      if (lane == 0) P.y1[r] = s;
    }
  }
  ss_stamp(P, slot);
}

}  // namespace ibmi
