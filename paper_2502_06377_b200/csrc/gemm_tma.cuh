// TMA + mbarrier variant of the FP64 DMMA NT GEMM (sm_100a), used for the hot
// sweep GEMMs when the operand geometry allows it.
//
// Differences from gemm_nt.cuh (cp.async + __syncthreads pipeline):
//   * operand tiles arrive by cp.async.bulk.tensor (TMA, SASS UTMALDG) with
//     the 128-byte hardware swizzle, issued by one elected thread;
//   * each stage has a "full" mbarrier (TMA transaction bytes) and an "empty"
//     mbarrier (one arrive per consumer warp); there is no CTA-wide barrier in
//     the main loop, so warps drift apart and the DMMA pipe always has a warp
//     with operands ready;
//   * a tile whose 128 rows cross the RowMap gap is fetched as sixteen 8-row
//     boxes, otherwise as one 128-row box.
// Fragment rows inside every 8-row group are permuted (g -> perm(g)) so that
// the two rows served in one LDS.128 phase differ in bit 2 of (row % 8) and
// the swizzled reads stay bank-conflict free.
#pragma once
#include <cuda.h>
#include "gemm_nt.cuh"

namespace ibmi {

constexpr int TMA_ST = 6;                      // stages
constexpr int TMA_D = TMA_ST - 2;              // prefetch distance (tiles in flight)
constexpr int TMA_BK = 16;                     // 16 doubles = 128 B rows (SWIZZLE_128B)
constexpr int TMA_TILE_BYTES = GB_M * TMA_BK * 8;          // 16 KB per operand
constexpr int TMA_STAGE_BYTES = 2 * TMA_TILE_BYTES;        // 32 KB
constexpr size_t TMA_SMEM = (size_t)TMA_ST * TMA_STAGE_BYTES + 1024 + 2 * TMA_ST * 8;

// One set of maps per K segment: the inner extent of each map ends where its
// segment ends, so a box that runs past the segment is zero-filled by TMA
// (exact semantics, no masking in the main loop).
struct TmaMaps {
  CUtensorMap xb[2], xs[2], yb[2], ys[2];      // big (128-row) and small (8-row) boxes per segment
};

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(mbar)
      : "memory");
}

__device__ __forceinline__ int perm8(int g) { return (g >> 1) | ((g & 1) << 2); }

// Load one operand tile (128 logical rows starting at r0, 16 K-columns at kx).
__device__ __forceinline__ void tma_operand(uint32_t dst, const CUtensorMap* big, const CUtensorMap* small,
                                            const RowMap& map, int r0, int kx, uint32_t mbar) {
  const bool contiguous = (r0 + GB_M <= map.split) || (r0 >= map.split);
  if (contiguous) {
    tma_load_2d(dst, big, kx, (int)map_idx(map, r0), mbar);
  } else {
#pragma unroll 1
    for (int i = 0; i < GB_M / 8; ++i) tma_load_2d(dst + i * 8 * 128, small, kx, (int)map_idx(map, r0 + 8 * i), mbar);
  }
}

// FIX (EPI_PARTIAL only): the split-K fix-up inside the kernel.  A template parameter, not a run-time
// branch: even never taken, the extra code cost the default split-K instance 0.3-1.4% (register allocation).
template <int EPI, bool FIX = false>
__global__ void __launch_bounds__(256, 1) gemm_tma_kernel(const GemmParams P, const __grid_constant__ TmaMaps maps) {
  constexpr int MI = 8, NJ = 4;
  extern __shared__ __align__(1024) unsigned char tsmem_raw[];
  __shared__ double red[8];
  // 1024-byte aligned stage ring (SWIZZLE_128B pattern repeats every 1024 B)
  const uint32_t raw = smem_u32(tsmem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* gbase = tsmem_raw + (base - raw);
  const uint32_t bar_full = base + TMA_ST * TMA_STAGE_BYTES;
  const uint32_t bar_empty = bar_full + TMA_ST * 8;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int g = lane >> 2;
  const int t = lane & 3;
  const int wm0 = (warp & 1) * 64;
  const int wn0 = (warp >> 1) * 32;
  const int pg = perm8(g);

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
  int kt_begin = 0, kt_end = P.kt_total;
  if (EPI == EPI_PARTIAL) {
    const int per = (P.kt_total + P.splits - 1) / P.splits;
    kt_begin = min(P.kt_total, split * per);
    kt_end = min(P.kt_total, kt_begin + per);
  }
  const int KT = kt_end - kt_begin;

  if (tid == 0) {
    for (int s = 0; s < TMA_ST; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.xb[0])) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.yb[0])) : "memory");
  }
  __syncthreads();

  auto issue = [&](int j) {   // tile j (relative) -> stage j % ST
    const int kt = kt_begin + j;
    const int sgi = kt < P.kt0 ? 0 : 1;
    const int ktl = sgi ? kt - P.kt0 : kt;
    const int s = j % TMA_ST;
    const uint32_t fb = bar_full + 8 * s;
    mbar_expect_tx(fb, TMA_STAGE_BYTES);
    const uint32_t dx = base + s * TMA_STAGE_BYTES;
    tma_operand(dx, &maps.xb[sgi], &maps.xs[sgi], P.xm, m0, (int)(P.seg[sgi].x0 + ktl * TMA_BK), fb);
    tma_operand(dx + TMA_TILE_BYTES, &maps.yb[sgi], &maps.ys[sgi], P.yn, n0, (int)(P.seg[sgi].y0 + ktl * TMA_BK), fb);
  };

  if (tid == 0) {
    for (int j = 0; j < TMA_D && j < KT; ++j) issue(j);
  }

  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // per-thread fragment offsets (doubles) inside a 16 KB tile, before the k swizzle
  int xrow[MI], yrow[NJ];
#pragma unroll
  for (int i = 0; i < MI; ++i) xrow[i] = wm0 + 8 * i + pg;
#pragma unroll
  for (int j = 0; j < NJ; ++j) yrow[j] = wn0 + 8 * j + pg;
  const int sw = pg;   // (row & 7) == pg for every fragment row

  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % TMA_ST;
    if (tid == 0 && kt + TMA_D < KT) {
      const int j = kt + TMA_D;
      const int round = j / TMA_ST;
      if (round > 0) mbar_wait(bar_empty + 8 * (j % TMA_ST), (round - 1) & 1);
      issue(j);
    }
    mbar_wait(bar_full + 8 * s, (kt / TMA_ST) & 1);
    const double* xs = reinterpret_cast<const double*>(gbase + s * TMA_STAGE_BYTES);
    const double* ys = xs + GB_M * TMA_BK;
#pragma unroll
    for (int kk = 0; kk < TMA_BK; kk += 8) {
      const int ch = ((kk >> 1) + t) ^ sw;
      double a[MI][2], b[NJ][2];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const double2 v = *reinterpret_cast<const double2*>(xs + xrow[i] * TMA_BK + (ch << 1));
        a[i][0] = v.x;
        a[i][1] = v.y;
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const double2 v = *reinterpret_cast<const double2*>(ys + yrow[j] * TMA_BK + (ch << 1));
        b[j][0] = v.x;
        b[j][1] = v.y;
      }
#pragma unroll
      for (int ss = 0; ss < 2; ++ss)
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i][ss], b[j][ss]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_empty + 8 * s);
  }

  // ------------------------------------------------------------- epilogue
  // accumulator (i, j, e) of this thread is C[m0 + xrow[i]][n0 + wn0 + 8j + perm8(2t + e)]
  if (EPI == EPI_STORE) {
    const bool diag_tile = P.lower && tm == tn;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int m = m0 + xrow[i];
      if (m >= P.M) continue;
      const int64_t rowc = P.cidx ? P.cidx[m] : map_idx(P.cm, m);
      const int64_t rowd = P.beta != 0.0 ? map_idx(P.dm, m) : 0;
      const int64_t mcol2 = map_idx(P.c2m, m);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + wn0 + 8 * j + perm8(2 * t + e);
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
    if (P.peers) __threadfence_system();
  } else if (EPI == EPI_PARTIAL) {
    double* dst = P.partial + ((size_t)blockIdx.x) * GB_M * GB_N;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) dst[xrow[i] * GB_N + wn0 + 8 * j + perm8(2 * t + e)] = acc[i][j][e];
    if (FIX) {
      // Fix-up inside the GEMM: the split that arrives last at this tile sums all partials in
      // split order (same bits as the separate reduction kernel) and runs the STORE epilogue.
      // The stage ring is free by now (every issued TMA load was consumed) and serves as the
      // 32 × 129 transpose buffer.
      __shared__ int last;
      __threadfence();
      __syncthreads();
      if (tid == 0) last = atomicAdd(P.tile_count + tile, 1) == P.splits - 1;
      __syncthreads();
      if (last) {
        __threadfence();
        double(*tr)[129] = reinterpret_cast<double(*)[129]>(gbase);
        for (int rc = 0; rc < GB_M; rc += 32) {
          splitk_reduce_chunk<false>(P, tile, rc, tr);
          __syncthreads();
        }
        if (P.peers) __threadfence_system();
      }
    }
  } else {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int m = m0 + xrow[i];
      if (m >= P.M) continue;
      const int64_t rowc = P.cidx ? P.cidx[m] : map_idx(P.cm, m);
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + wn0 + 8 * j + perm8(2 * t + e);
          if (n >= P.N) continue;
          const double d = (rowc == map_idx(P.cn, n) ? 1.0 : 0.0) - acc[i][j][e];
          s = fma(d, d, s);
        }
    }
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < 8; ++w) tot += red[w];
      P.partial[blockIdx.x] = tot;
    }
  }
}

}  // namespace ibmi
