// tcgen05 INT8 tensor-core GEMM (sm_100a) — the integer engine of the
// Ozaki-II FP64 emulation (ozaki.cuh).
//
//   R[m][n] = ( sum_k X[m][k] * Y[n][k] )  mod  modulus        (X, Y int8, K-major)
//
// Both operands are row-major with K contiguous ("NT"), the layout every IBMI
// GEMM already has (Σ is stored full-symmetric, so a column is the row with
// the same index).  One CTA per SM, persistent over 128 x 256 output tiles:
//   warp 0      TMA producer (one elected lane; 128-byte swizzled boxes of
//               128 K-bytes, one "full" mbarrier per stage with tx bytes)
//   warp 1      TMEM allocator + MMA issuer (one lane issues
//               tcgen05.mma.cta_group::1.kind::i8, M=128 N=256 K=32, and
//               tcgen05.commit's the smem stage back to the producer)
//   warps 2..5  epilogue: tcgen05.ld 32x32b from TMEM, reduce the exact int32
//               sums mod the modulus, store one uint8 residue per element
// Two TMEM accumulators (2 x 256 columns) let the epilogue of tile i overlap
// the MMAs of tile i+1.  A grid dimension runs over moduli (planes), so one
// launch computes every residue product of an Ozaki-II GEMM.
#pragma once
#include <cuda.h>
#include <stdint.h>
#include "common.cuh"

namespace ibmi {

constexpr int IG_BM = 128;            // tile rows  (UMMA M)
constexpr int IG_BN = 256;            // tile cols  (UMMA N)
constexpr int IG_BK = 128;            // K bytes per stage (= one 128B swizzle row)
constexpr int IG_UK = 32;             // K per tcgen05.mma kind::i8
constexpr int IG_ST = 4;              // smem stages
constexpr int IG_A_BYTES = IG_BM * IG_BK;
constexpr int IG_B_BYTES = IG_BN * IG_BK;
constexpr int IG_STAGE = IG_A_BYTES + IG_B_BYTES;   // 48 KB
constexpr int IG_THREADS = 192;
constexpr size_t IG_SMEM = (size_t)IG_ST * IG_STAGE + 1024 + 256;

// One plane of an int8 operand family: plane l of X lives at x + l * x_plane.
struct IgemmParams {
  int M, N, K;               // K in elements (bytes)
  int tiles_m, tiles_n, planes;
  uint8_t* R;                // residues, plane l at R + l * r_plane, row-major ld = ldr
  int64_t ldr, r_plane;
  int32_t* C32;              // optional raw int32 output (probe / tests), plane 0 only
  int64_t ldc32;
  int mod[32];               // modulus per plane (0: raw int32 to C32)
  int rows_per_plane_x;      // TMA row offset of plane l in the stacked X map
  int rows_per_plane_y;
  int lower;                 // only tiles whose columns start at or before the rows end (symmetric C)
  // Operand addressing inside a plane (all-zero = identity): X rows start at
  // x_row_off; logical Y row r sits at r < y_split ? r : r - y_split + y_off1
  // (the complement of a set, skipping its rows); logical K column k of X / Y
  // sits at k < *_ksplit ? k : k - *_ksplit + *_koff1 (the set's columns
  // skipped).  Splits are multiples of 128 so no TMA box straddles a gap.
  int x_row_off;
  int y_split, y_off1;
  int xk_split, xk_off1, yk_split, yk_off1;
};
__device__ __forceinline__ int ig_gap(int v, int split, int off1) { return v < split ? v : v - split + off1; }

__device__ __forceinline__ void ig_mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void ig_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void ig_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void ig_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "IGW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra IGW_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void ig_tma_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

// K-major operand tile with the 128-byte swizzle: 8-row atoms of 1024 bytes
// (SBO = 1024), LBO unused, descriptor version 1 (sm_100), layout 2 = SW128.
__device__ __forceinline__ uint64_t ig_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// kind::i8 instruction descriptor: s32 accumulate, signed A/B, K-major both.
__host__ __device__ constexpr uint32_t ig_idesc(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void ig_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void ig_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(mbar)
               : "memory");
}

#define IG_LD32(taddr, r)                                                                                          \
  asm volatile(                                                                                                    \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                                             \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),            \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),      \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),    \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])     \
      : "r"(taddr))

// tile t of plane l -> (tm, tn); tiles of one plane are column-major in tm so
// CTAs that run concurrently share the larger (256-row) Y tile through L2.
__device__ __forceinline__ bool ig_tile(const IgemmParams& P, int t, int& l, int& tm, int& tn) {
  const int per = P.tiles_m * P.tiles_n;
  l = t / per;
  const int r = t - l * per;
  tm = r % P.tiles_m;
  tn = r / P.tiles_m;
  if (P.lower && tn * IG_BN > tm * IG_BM + IG_BM - 1) return false;
  return true;
}

__global__ void __launch_bounds__(IG_THREADS, 1)
    igemm_tc_kernel(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap my,
                    const IgemmParams P) {
  extern __shared__ __align__(1024) unsigned char ig_smem_raw[];
  const uint32_t raw = smem_u32(ig_smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bar_full = base + IG_ST * IG_STAGE;
  const uint32_t bar_empty = bar_full + IG_ST * 8;
  const uint32_t bar_tfull = bar_empty + IG_ST * 8;
  const uint32_t bar_tempty = bar_tfull + 2 * 8;
  const uint32_t slot = bar_tempty + 2 * 8;
  uint32_t* slot_ptr = reinterpret_cast<uint32_t*>(ig_smem_raw + (slot - raw));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < IG_ST; ++s) {
      ig_mbar_init(bar_full + 8 * s, 1);
      ig_mbar_init(bar_empty + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      ig_mbar_init(bar_tfull + 8 * a, 1);
      ig_mbar_init(bar_tempty + 8 * a, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mx)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&my)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(slot));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot_ptr;

  const int KT = (P.K + IG_BK - 1) / IG_BK;
  const int total = P.tiles_m * P.tiles_n * P.planes;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int l, tm, tn;
        if (!ig_tile(P, t, l, tm, tn)) continue;
        const int xa = l * P.rows_per_plane_x + P.x_row_off + tm * IG_BM;
        const int ya0 = l * P.rows_per_plane_y + ig_gap(tn * IG_BN, P.y_split, P.y_off1);
        const int ya1 = l * P.rows_per_plane_y + ig_gap(tn * IG_BN + 128, P.y_split, P.y_off1);
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const uint32_t s = it % IG_ST;
          const uint32_t round = it / IG_ST;
          if (round > 0) ig_wait(bar_empty + 8 * s, (round - 1) & 1);
          const uint32_t fb = bar_full + 8 * s;
          ig_expect_tx(fb, IG_STAGE);
          const uint32_t dst = base + s * IG_STAGE;
          const int kl = kt * IG_BK;
          ig_tma_2d(dst, &mx, ig_gap(kl, P.xk_split, P.xk_off1), xa, fb);
          // the 256-row Y tile as two 128-row boxes (either may sit past the row gap)
          const int ky = ig_gap(kl, P.yk_split, P.yk_off1);
          ig_tma_2d(dst + IG_A_BYTES, &my, ky, ya0, fb);
          ig_tma_2d(dst + IG_A_BYTES + IG_B_BYTES / 2, &my, ky, ya1, fb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ig_idesc(IG_BM, IG_BN);
      uint32_t it = 0, tc = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int l, tm, tn;
        if (!ig_tile(P, t, l, tm, tn)) continue;
        const uint32_t a = tc & 1, use = tc >> 1;
        if (use > 0) ig_wait(bar_tempty + 8 * a, (use - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + a * IG_BN;
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const uint32_t s = it % IG_ST;
          ig_wait(bar_full + 8 * s, (it / IG_ST) & 1);
          tc_fence_after();
          const uint32_t sa = base + s * IG_STAGE;
          const uint64_t da = ig_desc(sa), db = ig_desc(sa + IG_A_BYTES);
#pragma unroll
          for (int j = 0; j < IG_BK / IG_UK; ++j)
            ig_mma(d, da + (uint64_t)(j * IG_UK / 16), db + (uint64_t)(j * IG_UK / 16), idesc, (kt | j) != 0);
          ig_commit(bar_empty + 8 * s);
        }
        ig_commit(bar_tfull + 8 * a);
        ++tc;
      }
    }
  } else {
    const int q = warp & 3;                  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    uint32_t tc = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int l, tm, tn;
      if (!ig_tile(P, t, l, tm, tn)) continue;
      const uint32_t a = tc & 1, use = tc >> 1;
      ig_wait(bar_tfull + 8 * a, use & 1);
      tc_fence_after();
      const int m = tm * IG_BM + row;
      const int md = P.mod[l];
      const bool mok = m < P.M;
#pragma unroll 1
      for (int c = 0; c < IG_BN / 32; ++c) {
        uint32_t r[32];
        IG_LD32(tmem + ((uint32_t)(q * 32) << 16) + a * IG_BN + c * 32, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        const int n0 = tn * IG_BN + c * 32;
        if (!mok) continue;
        if (md == 0) {
          int32_t* dst = P.C32 + (int64_t)m * P.ldc32 + n0;
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (n0 + e < P.N) dst[e] = (int32_t)r[e];
        } else {
          uint32_t w[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            uint32_t v = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              int x = (int32_t)r[4 * e + b] % md;
              x += x < 0 ? md : 0;
              v |= (uint32_t)x << (8 * b);
            }
            w[e] = v;
          }
          uint8_t* dst = P.R + (int64_t)l * P.r_plane + (int64_t)m * P.ldr + n0;
          if (n0 + 32 <= P.N) {
            reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
            reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
          } else {
            for (int e = 0; e < 32 && n0 + e < P.N; ++e) dst[e] = (uint8_t)(w[e >> 2] >> (8 * (e & 3)));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) ig_arrive(bar_tempty + 8 * a);
      ++tc;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}


// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05.mma.cta_group::2): a cluster of 2 CTAs on one TPC
// computes a 256 x 256 tile.  CTA r holds A rows [128r, 128r+128) and B rows
// (output columns) [128r, 128r+128) of the tile; the leader (rank 0) issues
// M=256 N=256 K=32 MMAs that read both CTAs' shared memory, and each CTA's
// TMEM receives its own 128 accumulator rows x 256 columns.  Per SM and MMA
// the operand traffic is 8 KB instead of 12 KB (the 1-CTA kernel is bounded
// by its shared-memory operand reads).  Both CTAs' TMA loads complete on the
// leader's "full" barrier; the leader's commits multicast to both CTAs'
// "empty" / "tmem full" barriers; both epilogues arrive on the leader's
// "tmem empty" barrier.
constexpr int IG2_BM = 256;           // pair tile rows
constexpr int IG2_BN = 256;           // pair tile cols
constexpr int IG2_ST = 6;             // stages (32 KB per CTA each)
constexpr int IG2_A_BYTES = 128 * IG_BK;
constexpr int IG2_B_BYTES = 128 * IG_BK;
constexpr int IG2_STAGE = IG2_A_BYTES + IG2_B_BYTES;
constexpr size_t IG2_SMEM = (size_t)IG2_ST * IG2_STAGE + 1024 + 256;

__device__ __forceinline__ uint32_t ig_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t ig_mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void ig_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void ig_tma_2d_pair(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(mbar_cluster)
      : "memory");
}
__device__ __forceinline__ void ig_mma2(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void ig_commit2(uint32_t mbar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(mbar),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void ig_arrive_cluster(uint32_t mbar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(mbar_cluster) : "memory");
}

__device__ __forceinline__ bool ig2_tile(const IgemmParams& P, int t, int& l, int& tm, int& tn) {
  const int tiles_m = (P.M + IG2_BM - 1) / IG2_BM, tiles_n = (P.N + IG2_BN - 1) / IG2_BN;
  const int per = tiles_m * tiles_n;
  l = t / per;
  const int r = t - l * per;
  tm = r % tiles_m;
  tn = r / tiles_m;
  if (P.lower && tn * IG2_BN > tm * IG2_BM + IG2_BM - 1) return false;
  return true;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(IG_THREADS, 1)
    igemm_tc2_kernel(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap my,
                     const IgemmParams P) {
  extern __shared__ __align__(1024) unsigned char ig_smem_raw[];
  const uint32_t raw = smem_u32(ig_smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bar_full = base + IG2_ST * IG2_STAGE;
  const uint32_t bar_empty = bar_full + IG2_ST * 8;
  const uint32_t bar_tfull = bar_empty + IG2_ST * 8;
  const uint32_t bar_tempty = bar_tfull + 2 * 8;
  const uint32_t slot = bar_tempty + 2 * 8;
  uint32_t* slot_ptr = reinterpret_cast<uint32_t*>(ig_smem_raw + (slot - raw));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ig_cluster_rank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < IG2_ST; ++s) {
      ig_mbar_init(bar_full + 8 * s, 1);      // leader: one expect_tx arrival; both CTAs' bytes
      ig_mbar_init(bar_empty + 8 * s, 1);     // one multicast commit from the leader
    }
    for (int a = 0; a < 2; ++a) {
      ig_mbar_init(bar_tfull + 8 * a, 1);
      ig_mbar_init(bar_tempty + 8 * a, 8);    // leader's: 4 epilogue warps x 2 CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mx)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&my)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(slot));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  ig_cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *slot_ptr;

  const int KT = (P.K + IG_BK - 1) / IG_BK;
  const int tiles_m = (P.M + IG2_BM - 1) / IG2_BM, tiles_n = (P.N + IG2_BN - 1) / IG2_BN;
  const int total = tiles_m * tiles_n * P.planes;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const uint32_t full_leader = ig_mapa(bar_full, 0);

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = cid; t < total; t += ncl) {
        int l, tm, tn;
        if (!ig2_tile(P, t, l, tm, tn)) continue;
        const int xa = l * P.rows_per_plane_x + P.x_row_off + tm * IG2_BM + (int)rank * 128;
        const int ya = l * P.rows_per_plane_y + ig_gap(tn * IG2_BN + (int)rank * 128, P.y_split, P.y_off1);
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const uint32_t s = it % IG2_ST;
          const uint32_t round = it / IG2_ST;
          if (round > 0) ig_wait(bar_empty + 8 * s, (round - 1) & 1);
          if (rank == 0) ig_expect_tx(bar_full + 8 * s, 2 * IG2_STAGE);
          const uint32_t dst = base + s * IG2_STAGE;
          const int kl = kt * IG_BK;
          ig_tma_2d_pair(dst, &mx, ig_gap(kl, P.xk_split, P.xk_off1), xa, full_leader + 8 * s);
          ig_tma_2d_pair(dst + IG2_A_BYTES, &my, ig_gap(kl, P.yk_split, P.yk_off1), ya, full_leader + 8 * s);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = ig_idesc(IG2_BM, IG2_BN);
      uint32_t it = 0, tc = 0;
      for (int t = cid; t < total; t += ncl) {
        int l, tm, tn;
        if (!ig2_tile(P, t, l, tm, tn)) continue;
        const uint32_t a = tc & 1, use = tc >> 1;
        if (use > 0) ig_wait(bar_tempty + 8 * a, (use - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + a * IG2_BN;
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const uint32_t s = it % IG2_ST;
          ig_wait(bar_full + 8 * s, (it / IG2_ST) & 1);
          tc_fence_after();
          const uint32_t sa = base + s * IG2_STAGE;
          const uint64_t da = ig_desc(sa), db = ig_desc(sa + IG2_A_BYTES);
#pragma unroll
          for (int j = 0; j < IG_BK / IG_UK; ++j)
            ig_mma2(d, da + (uint64_t)(j * IG_UK / 16), db + (uint64_t)(j * IG_UK / 16), idesc, (kt | j) != 0);
          ig_commit2(bar_empty + 8 * s);
        }
        ig_commit2(bar_tfull + 8 * a);
        ++tc;
      }
    }
  } else {
    const int q = warp & 3;
    const int row = (int)rank * 128 + q * 32 + lane;
    const uint32_t tempty_leader = ig_mapa(bar_tempty, 0);
    uint32_t tc = 0;
    for (int t = cid; t < total; t += ncl) {
      int l, tm, tn;
      if (!ig2_tile(P, t, l, tm, tn)) continue;
      const uint32_t a = tc & 1, use = tc >> 1;
      ig_wait(bar_tfull + 8 * a, use & 1);
      tc_fence_after();
      const int m = tm * IG2_BM + row;
      const int md = P.mod[l];
      const bool mok = m < P.M;
#pragma unroll 1
      for (int c = 0; c < IG2_BN / 32; ++c) {
        uint32_t r[32];
        IG_LD32(tmem + ((uint32_t)(q * 32) << 16) + a * IG2_BN + c * 32, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        const int n0 = tn * IG2_BN + c * 32;
        if (!mok || n0 >= P.N) continue;
        if (md == 0) {
          int32_t* dst = P.C32 + (int64_t)m * P.ldc32 + n0;
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (n0 + e < P.N) dst[e] = (int32_t)r[e];
        } else {
          uint32_t w[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            uint32_t v = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              int x = (int32_t)r[4 * e + b] % md;
              x += x < 0 ? md : 0;
              v |= (uint32_t)x << (8 * b);
            }
            w[e] = v;
          }
          uint8_t* dst = P.R + (int64_t)l * P.r_plane + (int64_t)m * P.ldr + n0;
          if (n0 + 32 <= P.N) {
            reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
            reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
          } else {
            for (int e = 0; e < 32 && n0 + e < P.N; ++e) dst[e] = (uint8_t)(w[e >> 2] >> (8 * (e & 3)));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) ig_arrive_cluster(tempty_leader + 8 * a);
      ++tc;
    }
  }
  tc_fence_before();
  ig_cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

}  // namespace ibmi
