// FP64 tensor-core (DMMA) "NT" GEMM for sm_100a:
//
//     C[cm(m)][cn(n)] = alpha * sum_k X(m, k) * Y(n, k)  + beta * D[dm(m)][dn(n)]
//
// Blackwell has no FP64 tcgen05/UMMA kind (ptxas rejects .kind::f64), so the
// FP64 tensor path is the warp-synchronous DMMA.8x8x4 issued by
// mma.sync.m8n8k4.f64 (37.1 TFLOP/s measured on B200 = 148 SM x 128 flop/clk x
// 1.965 GHz).  This kernel is built to keep that pipe saturated:
//   * 128x128 CTA tile, 8 warps of 64x32, 64 FP64 accumulators per thread;
//   * 4-stage cp.async shared-memory pipeline, BK = 16;
//   * k-slot permutation: lane (g, t) holds k = 2t and 2t+1 of every 8-k half,
//     so one LDS.128 feeds two DMMAs (XOR-swizzled rows -> conflict-free);
//   * operands are addressed through RowMaps (at most one gap) and up to two
//     K segments, so Σ[c, c] of a contiguous set is read in place, never
//     gathered;
//   * fused epilogues: scaled store (+beta*D), mirrored (transposed) store for
//     the Σ[c, I] = -Mᵀ half of the update, lower-triangle-only tiles for
//     symmetric products, and a (δ - acc)² reduction for ‖I − AΣ‖_F.
//
// Every GEMM of the sweep (solver.py:124-125, :154), of the setup
// (solver.py:119-120) and of the residual is of this NT form because A and Σ
// are symmetric: a column of Σ is the row with the same index.
#pragma once
#include "common.cuh"

namespace ibmi {

constexpr int GB_M = 128;
constexpr int GB_N = 128;
constexpr int GB_K = 16;
constexpr int G_STAGES = 4;
constexpr int G_THREADS = 256;
constexpr int T_LD = 130;                          // padded row of a transposed tile
constexpr int TILE_DBL = (GB_K * T_LD > GB_M * GB_K) ? GB_K * T_LD : GB_M * GB_K;  // 2080
constexpr size_t GEMM_SMEM = (size_t)G_STAGES * 2 * TILE_DBL * sizeof(double);   // 133120

struct KSeg {
  int64_t x0, y0;  // first physical K column (or row, for transposed operands) of X and Y
  int len;
};

enum { EPI_STORE = 0, EPI_FROB = 1 };

struct GemmParams {
  const double* X; int64_t ldx; RowMap xm;   // XT=false: X[xm(m)*ldx + x0 + k]; XT=true: X[(x0+k)*ldx + xm.off0 + m]
  const double* Y; int64_t ldy; RowMap yn;
  int M, N;
  int nseg; KSeg seg[2];
  int kt0, kt_total;                         // k-tiles in segment 0, in total
  double* C; int64_t ldc; RowMap cm, cn;
  double alpha, beta;
  const double* D; int64_t ldd; RowMap dm, dn;
  int mirror;                                // also store C[cn(n)][cm(m)]
  int lower;                                 // only tiles tm >= tn; in diagonal tiles only m >= n
  int tiles_m, tiles_n;
  double* partial;                           // EPI_FROB: one partial sum per CTA
};

__device__ __forceinline__ int swz(int r, int k) {   // non-transposed tile element (r, k)
  return r * GB_K + ((((k >> 1) ^ ((r & 1) << 2))) << 1) + (k & 1);
}

// Issue the cp.async loads of k-tile `kt` of one operand into `dst`.
template <bool TR, bool V16>
__device__ __forceinline__ void load_operand(double* dst, const double* base, int64_t ld, const RowMap& map,
                                             int rows_total, int r0, const KSeg& sg, int ktl, int tid) {
  const int kbase = ktl * GB_K;
  if (!TR) {
    if (V16) {
      const int ch = tid & 7;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = (tid >> 3) + 32 * i;
        const int gr = r0 + r;
        const int kc = kbase + 2 * ch;
        int bytes = 0;
        const double* src = base;
        if (gr < rows_total) {
          const int rem = sg.len - kc;
          bytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
          if (bytes) src = base + map_idx(map, gr) * ld + sg.x0 + kc;
        }
        cp_async16(dst + r * GB_K + ((ch ^ ((r & 1) << 2)) << 1), src, bytes);
      }
    } else {
      const int e = tid & 15;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = (tid >> 4) + 16 * i;
        const int gr = r0 + r;
        const int kc = kbase + e;
        int bytes = 0;
        const double* src = base;
        if (gr < rows_total && kc < sg.len) {
          bytes = 8;
          src = base + map_idx(map, gr) * ld + sg.x0 + kc;
        }
        cp_async8(dst + swz(r, e), src, bytes);
      }
    }
  } else {
    // transposed operand: tile is [GB_K k-rows][128 columns], columns contiguous from map.off0
    if (V16) {
      const int ch = tid & 63;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int kr = (tid >> 6) + 4 * i;
        const int col = r0 + 2 * ch;
        int bytes = 0;
        const double* src = base;
        if (kbase + kr < sg.len) {
          const int rem = rows_total - col;
          bytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
          if (bytes) src = base + (sg.x0 + kbase + kr) * ld + map.off0 + col;
        }
        cp_async16(dst + kr * T_LD + 2 * ch, src, bytes);
      }
    } else {
      const int e = tid & 127;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int kr = (tid >> 7) + 2 * i;
        const int col = r0 + e;
        int bytes = 0;
        const double* src = base;
        if (kbase + kr < sg.len && col < rows_total) {
          bytes = 8;
          src = base + (sg.x0 + kbase + kr) * ld + map.off0 + col;
        }
        cp_async8(dst + kr * T_LD + e, src, bytes);
      }
    }
  }
}

template <bool XT, bool YT, bool V16, int EPI>
__global__ void __launch_bounds__(G_THREADS, 1) gemm_nt_kernel(const GemmParams P) {
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int g = lane >> 2;
  const int t = lane & 3;
  const int wm0 = (warp & 1) * 64;
  const int wn0 = (warp >> 1) * 32;

  int tm, tn;
  if (P.lower) {
    const int b = blockIdx.x;
    int r = (int)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= b) ++r;
    while (r * (r + 1) / 2 > b) --r;
    tm = r;
    tn = b - r * (r + 1) / 2;
  } else {
    tm = blockIdx.x % P.tiles_m;
    tn = blockIdx.x / P.tiles_m;
  }
  const int m0 = tm * GB_M;
  const int n0 = tn * GB_N;

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto stage_x = [&](int s) { return smem + (size_t)s * 2 * TILE_DBL; };
  auto stage_y = [&](int s) { return smem + (size_t)s * 2 * TILE_DBL + TILE_DBL; };

  auto issue = [&](int s, int kt) {
    const int sgi = kt < P.kt0 ? 0 : 1;
    const int ktl = sgi ? kt - P.kt0 : kt;
    KSeg sx = P.seg[sgi];
    KSeg sy = sx;
    sy.x0 = sx.y0;
    load_operand<XT, V16>(stage_x(s), P.X, P.ldx, P.xm, P.M, m0, sx, ktl, tid);
    load_operand<YT, V16>(stage_y(s), P.Y, P.ldy, P.yn, P.N, n0, sy, ktl, tid);
  };

  const int KT = P.kt_total;
#pragma unroll
  for (int s = 0; s < G_STAGES - 1; ++s) {
    if (s < KT) issue(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<G_STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + G_STAGES - 1;
      if (nk < KT) issue(nk % G_STAGES, nk);
      cp_async_commit();
    }
    const double* xs = stage_x(kt % G_STAGES);
    const double* ys = stage_y(kt % G_STAGES);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int kk = half * 8;
      double a[8][2], b[4][2];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = wm0 + 8 * i + g;
        if (!XT) {
          const double2 v = *reinterpret_cast<const double2*>(xs + r * GB_K + ((((kk >> 1) + t) ^ ((r & 1) << 2)) << 1));
          a[i][0] = v.x;
          a[i][1] = v.y;
        } else {
          a[i][0] = xs[(kk + 2 * t) * T_LD + r];
          a[i][1] = xs[(kk + 2 * t + 1) * T_LD + r];
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = wn0 + 8 * j + g;
        if (!YT) {
          const double2 v = *reinterpret_cast<const double2*>(ys + r * GB_K + ((((kk >> 1) + t) ^ ((r & 1) << 2)) << 1));
          b[j][0] = v.x;
          b[j][1] = v.y;
        } else {
          b[j][0] = ys[(kk + 2 * t) * T_LD + r];
          b[j][1] = ys[(kk + 2 * t + 1) * T_LD + r];
        }
      }
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i][s], b[j][s]);
    }
  }
  cp_async_wait<0>();

  // ------------------------------------------------------------- epilogue
  if (EPI == EPI_STORE) {
    const bool diag_tile = P.lower && tm == tn;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = m0 + wm0 + 8 * i + g;
      if (m >= P.M) continue;
      const int64_t rowc = map_idx(P.cm, m);
      const int64_t rowd = P.beta != 0.0 ? map_idx(P.dm, m) : 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + wn0 + 8 * j + 2 * t + e;
          if (n >= P.N) continue;
          if (diag_tile && m < n) continue;
          double v = P.alpha * acc[i][j][e];
          if (P.beta != 0.0) v += P.beta * P.D[rowd * P.ldd + map_idx(P.dn, n)];
          const int64_t colc = map_idx(P.cn, n);
          P.C[rowc * P.ldc + colc] = v;
          if (P.mirror) P.C[colc * P.ldc + rowc] = v;
        }
      }
    }
  } else {
    // ‖I − XYᵀ‖_F² partial: (δ(cm(m), cn(n)) − acc)²
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = m0 + wm0 + 8 * i + g;
      if (m >= P.M) continue;
      const int64_t rowc = map_idx(P.cm, m);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + wn0 + 8 * j + 2 * t + e;
          if (n >= P.N) continue;
          const double d = (rowc == map_idx(P.cn, n) ? 1.0 : 0.0) - acc[i][j][e];
          s = fma(d, d, s);
        }
    }
    s = warp_sum(s);
    __syncthreads();
    double* red = smem;
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < G_THREADS / 32; ++w) tot += red[w];
      P.partial[blockIdx.x] = tot;
    }
  }
}

}  // namespace ibmi
