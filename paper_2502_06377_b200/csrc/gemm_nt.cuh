// FP64 tensor-core (DMMA) "NT" GEMM for sm_100a:
//
//     C[cm(m)][cn(n)] = alpha * sum_k X(m, k) * Y(n, k)  + beta * D[dm(m)][dn(n)]
//
// Blackwell has no FP64 tcgen05/UMMA kind (ptxas rejects .kind::f64), so the
// FP64 tensor path is the warp-synchronous DMMA.8x8x4 issued by
// mma.sync.m8n8k4.f64 (37.1 TFLOP/s measured on B200 = 148 SM x 128 flop/clk x
// 1.965 GHz).  This kernel is built to keep that pipe saturated:
//   * 128x128 CTA tile, WM x WN warp tiles (64x32 / 32x32), FP64 accumulators
//     in registers;
//   * multi-stage cp.async shared-memory pipeline (BK = 16 or 32);
//   * k-slot permutation: lane (g, t) holds k = 2t and 2t+1 of every 8-k group,
//     so one LDS.128 feeds two DMMAs (XOR-swizzled rows -> conflict-free);
//   * operands are addressed through RowMaps (at most one gap) and up to two
//     K segments, so Σ[c, c] of a contiguous set is read in place, never
//     gathered;
//   * fused epilogues: scaled store (+beta*D), mirrored (transposed) store for
//     the Σ[c, I] = -Mᵀ half of the update, lower-triangle-only tiles for
//     symmetric products, split-K partial tiles, and a (δ - acc)² reduction
//     for ‖I − AΣ‖_F.
//
// Every GEMM of the sweep (solver.py:124-125, :154), of the setup
// (solver.py:119-120) and of the residual is of this NT form because A and Σ
// are symmetric: a column of Σ is the row with the same index.
#pragma once
#include "common.cuh"

namespace ibmi {

constexpr int GB_M = 128;
constexpr int GB_N = 128;
constexpr int T_PAD = 2;                 // transposed tile row = 128 + 2 doubles

template <int BK_, int STAGES_, int WM_, int WN_>
struct GemmCfg {
  static constexpr int BK = BK_;
  static constexpr int STAGES = STAGES_;
  static constexpr int WM = WM_;
  static constexpr int WN = WN_;
  static constexpr int WARPS_M = GB_M / WM;
  static constexpr int WARPS_N = GB_N / WN;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int MI = WM / 8;      // 8x8 sub-tiles per warp in M
  static constexpr int NJ = WN / 8;
  static constexpr int T_LD = GB_M + T_PAD;
  static constexpr int TILE_DBL = (BK * T_LD > GB_M * BK) ? BK * T_LD : GB_M * BK;
  static constexpr size_t SMEM = (size_t)STAGES * 2 * TILE_DBL * sizeof(double);
  static constexpr int MIN_BLOCKS = 1;
};

using CfgA = GemmCfg<16, 4, 64, 32>;     // 256 threads, 2 warps / scheduler
using CfgB = GemmCfg<16, 4, 32, 32>;     // 512 threads, 4 warps / scheduler
using CfgC = GemmCfg<32, 3, 32, 32>;     // 512 threads, BK 32

struct KSeg {
  int64_t x0, y0;  // first physical K column (or row, for transposed operands) of X and Y
  int len;
};

enum { EPI_STORE = 0, EPI_FROB = 1, EPI_PARTIAL = 2 };

struct GemmParams {
  const double* X; int64_t ldx; RowMap xm;   // XT=false: X[xm(m)*ldx + x0 + k]; XT=true: X[(x0+k)*ldx + xm.off0 + m]
  const double* Y; int64_t ldy; RowMap yn;
  int M, N;
  int nseg; KSeg seg[2];
  int kt0, kt_total;                         // k-tiles in segment 0, in total
  int splits;                                // split-K factor (EPI_PARTIAL)
  double* C; int64_t ldc; RowMap cm, cn;
  double alpha, beta;
  const double* D; int64_t ldd; RowMap dm, dn;
  int mirror;                                // also store C2[c2n(n)][c2m(m)]
  double* C2; int64_t ldc2; RowMap c2m, c2n;   // mirror target (defaults to C, cm, cn)
  const int64_t* cidx;                       // optional: direct-store / δ row = cidx[m] instead of cm(m)
  int direct;                                // write the direct store C[cm(m)][cn(n)] (default 1)
  // peer mode (sharded sweep, fused exchange): the direct store goes to the
  // row-panel owner's Σ through NVLink peer pointers.  cm(m) is the global
  // row r, cn(n) this rank's local row l; block-cyclic panels of bc_panel rows.
  double* const* peers;
  int64_t bc_panel;
  int bc_world, bc_rank;
  int lower;                                 // only tiles tm >= tn; in diagonal tiles only m >= n
  int tiles_m, tiles_n;
  int group_m = 0;                           // raster: bands of group_m tile rows, tn-major inside (0: tm-major)
  double* partial;                           // EPI_FROB: one partial sum per CTA; EPI_PARTIAL: split tiles
  int* tile_count = nullptr;                 // EPI_PARTIAL on the TMA kernel: per-tile arrival counters (zeroed
                                             // before the launch); the split that arrives last reduces the tile
                                             // and runs the epilogue, so no separate reduction launch is needed
};

// Output tile of linear tile index `tile` (the GEMM kernels and the split-K
// reduction must agree).  lower: row-major over the lower triangle.  group_m:
// the M tiles are cut into bands of group_m rows and each band is walked
// column by column, so the CTAs resident at once share a few X row blocks and
// a few Y row blocks (L2 hits) instead of all of X.  Otherwise tm-major.
__device__ __forceinline__ void tile_coords(const GemmParams& P, int tile, int& tm, int& tn) {
  if (P.lower) {
    int r = (int)((sqrt(8.0 * (double)tile + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= tile) ++r;
    while (r * (r + 1) / 2 > tile) --r;
    tm = r;
    tn = tile - r * (r + 1) / 2;
  } else if (P.group_m > 0 && P.group_m < P.tiles_m) {
    const int per = P.group_m * P.tiles_n;
    const int band = tile / per;
    const int first = band * P.group_m;
    const int gm = min(P.group_m, P.tiles_m - first);
    const int r = tile - band * per;
    tm = first + r % gm;
    tn = r / gm;
  } else {
    tm = tile % P.tiles_m;
    tn = tile / P.tiles_m;
  }
}

// Direct-store address of element (m, n) (rowc = cidx/cm row already mapped).
__device__ __forceinline__ double* direct_addr(const GemmParams& P, int64_t rowc, int n) {
  return P.C + rowc * P.ldc + map_idx(P.cn, n);
}

// Peer store (fused exchange): element (m, n) of the panel GEMM is Σ[r][gc]
// with r = c2m(m) the global row and gc the global column of this rank's
// local row l = c2n(n); it goes to the owner of row r (block-cyclic panels).
__device__ __forceinline__ void peer_store(const GemmParams& P, int m, int n, double v) {
  const int64_t r = map_idx(P.c2m, m);
  const int64_t T = P.bc_panel, G = P.bc_world;
  const int h = (int)((r / T) % G);
  const int64_t lr = (r / (T * G)) * T + r % T;
  const int64_t l = map_idx(P.c2n, n);
  const int64_t gc = ((l / T) * G + P.bc_rank) * T + l % T;
  P.peers[h][lr * P.ldc2 + gc] = v;
}

template <int BK>
__device__ __forceinline__ int swz(int r, int k) {   // non-transposed tile element (r, k)
  return r * BK + ((((k >> 1) ^ ((r & 1) << 2))) << 1) + (k & 1);
}

// Issue the cp.async loads of k-tile `ktl` of one operand into `dst`.
template <class CF, bool TR, bool V16>
__device__ __forceinline__ void load_operand(double* dst, const double* base, int64_t ld, const RowMap& map,
                                             int rows_total, int r0, const KSeg& sg, int ktl, int tid) {
  constexpr int BK = CF::BK;
  constexpr int NT = CF::THREADS;
  const int kbase = ktl * BK;
  if (!TR) {
    if (V16) {
      constexpr int CPR = BK / 2;                    // 16-byte chunks per row
      constexpr int PER = GB_M * CPR / NT;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int q = tid + NT * i;
        const int r = q / CPR, ch = q % CPR;
        const int gr = r0 + r;
        const int kc = kbase + 2 * ch;
        int bytes = 0;
        const double* src = base;
        if (gr < rows_total) {
          const int rem = sg.len - kc;
          bytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
          if (bytes) src = base + map_idx(map, gr) * ld + sg.x0 + kc;
        }
        cp_async16(dst + r * BK + ((ch ^ ((r & 1) << 2)) << 1), src, bytes);
      }
    } else {
      constexpr int PER = GB_M * BK / NT;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int q = tid + NT * i;
        const int r = q / BK, e = q % BK;
        const int gr = r0 + r;
        const int kc = kbase + e;
        int bytes = 0;
        const double* src = base;
        if (gr < rows_total && kc < sg.len) {
          bytes = 8;
          src = base + map_idx(map, gr) * ld + sg.x0 + kc;
        }
        cp_async8(dst + swz<BK>(r, e), src, bytes);
      }
    }
  } else {
    // transposed operand: tile is [BK k-rows][128 columns], columns contiguous from map.off0
    constexpr int TL = CF::T_LD;
    if (V16) {
      constexpr int PER = BK * (GB_M / 2) / NT;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int q = tid + NT * i;
        const int kr = q / (GB_M / 2), ch = q % (GB_M / 2);
        const int col = r0 + 2 * ch;
        int bytes = 0;
        const double* src = base;
        if (kbase + kr < sg.len) {
          const int rem = rows_total - col;
          bytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
          if (bytes) src = base + (sg.x0 + kbase + kr) * ld + map.off0 + col;
        }
        cp_async16(dst + kr * TL + 2 * ch, src, bytes);
      }
    } else {
      constexpr int PER = BK * GB_M / NT;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int q = tid + NT * i;
        const int kr = q / GB_M, e = q % GB_M;
        const int col = r0 + e;
        int bytes = 0;
        const double* src = base;
        if (kbase + kr < sg.len && col < rows_total) {
          bytes = 8;
          src = base + (sg.x0 + kbase + kr) * ld + map.off0 + col;
        }
        cp_async8(dst + kr * TL + e, src, bytes);
      }
    }
  }
}

template <class CF, bool XT, bool YT, bool V16, int EPI>
__global__ void __launch_bounds__(CF::THREADS, 1) gemm_nt_kernel(const GemmParams P) {
  constexpr int BK = CF::BK, ST = CF::STAGES, MI = CF::MI, NJ = CF::NJ, TL = CF::T_LD;
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int g = lane >> 2;
  const int t = lane & 3;
  const int wm0 = (warp % CF::WARPS_M) * CF::WM;
  const int wn0 = (warp / CF::WARPS_M) * CF::WN;

  int tile = blockIdx.x;
  int split = 0;
  if (EPI == EPI_PARTIAL) {
    split = tile % P.splits;
    tile /= P.splits;
  }
  int tm, tn;
  tile_coords(P, tile, tm, tn);
  const int m0 = tm * GB_M;
  const int n0 = tn * GB_N;

  // k-tile range of this CTA (split-K: contiguous chunk of the global k-tile list)
  int kt_begin = 0, kt_end = P.kt_total;
  if (EPI == EPI_PARTIAL) {
    const int per = (P.kt_total + P.splits - 1) / P.splits;
    kt_begin = min(P.kt_total, split * per);
    kt_end = min(P.kt_total, kt_begin + per);
  }

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto stage_x = [&](int s) { return smem + (size_t)s * 2 * CF::TILE_DBL; };
  auto stage_y = [&](int s) { return smem + (size_t)s * 2 * CF::TILE_DBL + CF::TILE_DBL; };

  auto issue = [&](int s, int kt) {
    const int sgi = kt < P.kt0 ? 0 : 1;
    const int ktl = sgi ? kt - P.kt0 : kt;
    KSeg sx = P.seg[sgi];
    KSeg sy = sx;
    sy.x0 = sx.y0;
    load_operand<CF, XT, V16>(stage_x(s), P.X, P.ldx, P.xm, P.M, m0, sx, ktl, tid);
    load_operand<CF, YT, V16>(stage_y(s), P.Y, P.ldy, P.yn, P.N, n0, sy, ktl, tid);
  };

  const int KT = kt_end - kt_begin;
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < KT) issue(s, kt_begin + s);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<ST - 2>();
    __syncthreads();
    {
      const int nk = kt + ST - 1;
      if (nk < KT) issue(nk % ST, kt_begin + nk);
      cp_async_commit();
    }
    const double* xs = stage_x(kt % ST);
    const double* ys = stage_y(kt % ST);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 8) {
      double a[MI][2], b[NJ][2];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int r = wm0 + 8 * i + g;
        if (!XT) {
          const double2 v = *reinterpret_cast<const double2*>(xs + r * BK + ((((kk >> 1) + t) ^ ((r & 1) << 2)) << 1));
          a[i][0] = v.x;
          a[i][1] = v.y;
        } else {
          a[i][0] = xs[(kk + 2 * t) * TL + r];
          a[i][1] = xs[(kk + 2 * t + 1) * TL + r];
        }
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int r = wn0 + 8 * j + g;
        if (!YT) {
          const double2 v = *reinterpret_cast<const double2*>(ys + r * BK + ((((kk >> 1) + t) ^ ((r & 1) << 2)) << 1));
          b[j][0] = v.x;
          b[j][1] = v.y;
        } else {
          b[j][0] = ys[(kk + 2 * t) * TL + r];
          b[j][1] = ys[(kk + 2 * t + 1) * TL + r];
        }
      }
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i][s], b[j][s]);
    }
  }
  cp_async_wait<0>();

  // ------------------------------------------------------------- epilogue
  if (EPI == EPI_STORE) {
    const bool diag_tile = P.lower && tm == tn;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int m = m0 + wm0 + 8 * i + g;
      if (m >= P.M) continue;
      const int64_t rowc = P.cidx ? P.cidx[m] : map_idx(P.cm, m);
      const int64_t rowd = P.beta != 0.0 ? map_idx(P.dm, m) : 0;
      const int64_t mcol2 = map_idx(P.c2m, m);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + wn0 + 8 * j + 2 * t + e;
          if (n >= P.N) continue;
          if (diag_tile && m < n) continue;
          double v = P.alpha * acc[i][j][e];
          if (P.beta != 0.0) v += P.beta * P.D[rowd * P.ldd + map_idx(P.dn, n)];
          if (P.direct) *direct_addr(P, rowc, n) = v;
          if (P.mirror) P.C2[map_idx(P.c2n, n) * P.ldc2 + mcol2] = v;
          if (P.peers) peer_store(P, m, n, v);
        }
      }
    }
    if (P.peers) __threadfence_system();   // peer stores visible before the exchange barrier
  } else if (EPI == EPI_PARTIAL) {
    // raw partial tile [128][128] of (tile, split), reduced later in fixed split order
    double* dst = P.partial + ((size_t)blockIdx.x) * GB_M * GB_N;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int r = wm0 + 8 * i + g;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int c = wn0 + 8 * j + 2 * t;
        *reinterpret_cast<double2*>(dst + r * GB_N + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    }
  } else {
    // ‖I − XYᵀ‖_F² partial: (δ(cm(m), cn(n)) − acc)²
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int m = m0 + wm0 + 8 * i + g;
      if (m >= P.M) continue;
      const int64_t rowc = P.cidx ? P.cidx[m] : map_idx(P.cm, m);
#pragma unroll
      for (int j = 0; j < NJ; ++j)
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
      for (int w = 0; w < CF::THREADS / 32; ++w) tot += red[w];
      P.partial[blockIdx.x] = tot;
    }
  }
}

// Fixed-order reduction of split-K partial tiles + the STORE epilogue.
// grid: one CTA per output tile, 256 threads.  The tile is processed in
// 32-row chunks: partial sums and the direct store are coalesced along the
// row; the mirrored (transposed) store and the peer store go through a shared
// memory transpose so they are written as contiguous 32-element runs too.
// One CTA per (tile, 32-row chunk): grid = tiles * GB_M / 32.  Each thread
// keeps 16 row accumulators and streams the split partials with the split
// loop outside, so 16 independent loads are in flight per thread; every
// element is still summed in split order 0..s-1 (deterministic, unchanged bits).
// One 32-row chunk (rows rc..rc+31) of output tile `tile`: sum the split partials in split order and run the
// STORE epilogue.  All 256 threads of the CTA call it together; `tr` is 32 × 129 doubles of shared memory.
template <bool STREAM>
__device__ __forceinline__ void splitk_reduce_chunk(const GemmParams& P, int tile, int rc, double (*tr)[129]) {
  int tm, tn;
  tile_coords(P, tile, tm, tn);
  const bool diag_tile = P.lower && tm == tn;
  const double* src = P.partial + (size_t)tile * P.splits * GB_M * GB_N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = tid & 127;
  const int n = tn * GB_N + c;
  const bool ncol_ok = n < P.N;
  const int64_t colc = ncol_ok ? map_idx(P.cn, n) : 0;
  const int64_t cold = (ncol_ok && P.beta != 0.0) ? map_idx(P.dn, n) : 0;
  const int r0 = rc + (tid >> 7);
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  for (int sp = 0; sp < P.splits; ++sp) {
    const double* base = src + (size_t)sp * GB_M * GB_N + (size_t)r0 * GB_N + c;
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] += STREAM ? __ldcs(base + 2 * q * GB_N) : __ldcg(base + 2 * q * GB_N);
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int r = r0 + 2 * q;
    const int m = tm * GB_M + r;
    double v = P.alpha * acc[q];
    const bool ok = ncol_ok && m < P.M && !(diag_tile && m < n);
    if (ok) {
      if (P.beta != 0.0) v += P.beta * P.D[map_idx(P.dm, m) * P.ldd + cold];
      if (P.direct) P.C[(P.cidx ? P.cidx[m] : map_idx(P.cm, m)) * P.ldc + colc] = v;
    }
    tr[r - rc][c] = v;
  }
  if (P.mirror || P.peers) {
    __syncthreads();
    const int m = tm * GB_M + rc + lane;
    const bool mrow_ok = m < P.M;
    const int64_t mcol2 = mrow_ok ? map_idx(P.c2m, m) : 0;
    for (int cc = warp; cc < GB_N; cc += 8) {
      const int nn = tn * GB_N + cc;
      if (!mrow_ok || nn >= P.N || (diag_tile && m < nn)) continue;
      const double v = tr[lane][cc];
      if (P.mirror) P.C2[map_idx(P.c2n, nn) * P.ldc2 + mcol2] = v;
      if (P.peers) peer_store(P, m, nn, v);
    }
  }
}

__global__ void __launch_bounds__(256) splitk_reduce_kernel(const GemmParams P) {
  __shared__ double tr[32][129];
  splitk_reduce_chunk<true>(P, blockIdx.x / (GB_M / 32), (blockIdx.x % (GB_M / 32)) * 32, tr);
  if (P.peers) __threadfence_system();
}

}  // namespace ibmi
