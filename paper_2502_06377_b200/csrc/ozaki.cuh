// Ozaki-II FP64 GEMM emulation on the INT8 tensor cores (sm_100a).
//
//   C = X · Yᵀ  (FP64)   computed as
//   1. per-row power-of-two scaling: X'_ik = rint(X_ik · 2^ex_i), |X'| <= 2^t
//      (same for Y with ey_j), exact integers in int64;
//   2. residues of X', Y' modulo n pairwise-coprime moduli m_l <= 256, stored
//      as symmetric int8 planes (oz_split_kernel);
//   3. one exact INT8 GEMM per modulus on tcgen05 (igemm_tc.cuh), reduced
//      mod m_l in its epilogue to one uint8 residue per output element;
//   4. Chinese remaindering of the n residues to the exact integer
//      C'_ij = Σ_k X'_ik Y'_jk (|C'| <= K·2^2t <= P/4, P = Π m_l) in 192-bit
//      limb arithmetic, then C_ij = C'_ij · 2^-(ex_i + ey_j) rounded once to
//      FP64 (oz_crt_kernel), with the caller's GEMM epilogue fused (alpha,
//      beta·D, direct store, mirrored store, lower triangle).
// The only rounding is the truncation of step 1 (2^-t relative to each row's
// largest entry, t up to 62 bits > the 53 of FP64) and the final rounding.
// t follows from n and K: K · 2^(2t) <= P/4.
#pragma once
#include <stdint.h>
#include "common.cuh"
#include "gemm_nt.cuh"

namespace ibmi {

constexpr int OZ_MINN = 8;
constexpr int OZ_MAXN = 20;
constexpr int OZ_LIMBS = 6;    // 192-bit CRT arithmetic, 32-bit limbs

struct OzTable {
  int n;
  int m[OZ_MAXN];
  float invm[OZ_MAXN];
  uint32_t k21[OZ_MAXN];         // 2^21 mod m
  uint32_t k42[OZ_MAXN];         // 2^42 mod m
  uint32_t magic[OZ_MAXN];       // ceil(2^(32+sh)/m): floor(s/m) = umulhi(s, magic) >> sh for s < 2^31
  int sh[OZ_MAXN];
  int bias[OZ_MAXN];             // m·ceil(2^30/m): makes a signed limb sum non-negative, ≡ 0 mod m
  uint32_t w[OZ_MAXN][OZ_LIMBS]; // CRT weights (P/m_l)·((P/m_l)^-1 mod m_l) < P
  float f[OZ_MAXN];              // w_l / P (fp32 suffices: q = rint(Σ r_l f_l) needs |error| < 1/4)
  uint32_t P[OZ_LIMBS];
  double log2P;
};

__constant__ OzTable c_oz[OZ_MAXN - OZ_MINN + 1];

// ---- step 1: per-row exponent.  Row r of the operand is X[rm(r)][km(k)],
// k in [0, K).  ex[r] = t - 1 - floor(log2 max_k |X|)  (0 for a zero row).
__global__ void oz_rowexp_kernel(const double* __restrict__ X, int64_t ld, RowMap rm, RowMap km, int R, int K,
                                 int t, int* __restrict__ ex) {
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < R; w += nwarps) {
    const double* row = X + map_idx(rm, w) * ld;
    double mx = 0.0;
    if (km.idx == nullptr && km.split >= K) {
      const double* q = row + km.off0;
      for (int k = lane; k < K; k += 32) mx = fmax(mx, fabs(q[k]));
    } else {
      for (int k = lane; k < K; k += 32) mx = fmax(mx, fabs(row[map_idx(km, k)]));
    }
    mx = warp_max(mx);
    if (lane == 0) ex[w] = mx > 0.0 ? t - 1 - ilogb(mx) : 0;
  }
}

// |rint(x · 2^e)| as an unsigned integer (<= 2^62 by the choice of e), by
// integer operations on the IEEE fields (no ldexp / F2I.S64).  Subnormals and
// zero give 0.
__device__ __forceinline__ uint64_t oz_scaled_mag(double x, int e) {
  const uint64_t bits = (uint64_t)__double_as_longlong(x);
  const int E = (int)((bits >> 52) & 0x7ff);
  if (E == 0) return 0;
  const uint64_t mant = (bits & 0xfffffffffffffull) | 0x10000000000000ull;
  const int s = E - 1075 + e;                   // x = ±mant · 2^(E-1075)
  if (s >= 0) return mant << s;
  if (s < -54) return 0;
  return (mant + (1ull << (-s - 1))) >> (-s);
}

// symmetric residue (|r| <= m/2) of the signed a = c0 + c1·2^21 + c2·2^42
// (|c0|, |c1| < 2^21, |c2| < 2^20) modulo entry l: the limb sum plus a bias
// ≡ 0 (mod m) lies in [0, 2^31), where the multiply-high division is exact.
// Rounding the quotient of s + (m-1)/2 gives the symmetric remainder directly.
__device__ __forceinline__ int oz_sym_residue(const OzTable& T, int l, int c0, int c1, int c2) {
  const uint32_t m = (uint32_t)T.m[l];
  const uint32_t s = (uint32_t)(c2 * (int)T.k42[l] + T.bias[l] + c1 * (int)T.k21[l] + c0);
  const uint32_t q = __umulhi(s + ((m - 1) >> 1), T.magic[l]) >> 7;   // every modulus is in [129, 256]
  return (int)(s - q * m);
}

// ---- step 2: residue planes.  Thread = (row r, 8 consecutive logical k);
// plane l of row r lives at Q + l*qplane + r*ldq.  Columns k >= K are zero.
constexpr int OZ_SPLIT_V = 8;
template <int NM>
__global__ void __launch_bounds__(256, 4) oz_split_kernel(const double* __restrict__ X, int64_t ld, RowMap rm,
                                                          RowMap km, int R, int K, const int* __restrict__ ex,
                                                          int8_t* __restrict__ Q, int64_t ldq, int64_t qplane) {
  // persistent: a bounded grid walks (row, 2048-column slab) items, so the
  // conversion co-resides with a running INT8 GEMM (one CTA per SM) instead
  // of filling every SM slot before it
  constexpr int V = OZ_SPLIT_V;
  const OzTable& T = c_oz[NM - OZ_MINN];
  const int64_t slabs = (ldq + V * 256 - 1) / (V * 256);
  for (int64_t item = blockIdx.x; item < (int64_t)R * slabs; item += gridDim.x) {
    const int r = (int)(item / slabs);
    const int k0 = (int)((item - (int64_t)r * slabs) * (V * 256)) + threadIdx.x * V;
    if (k0 >= ldq) continue;
    const double* row = X + map_idx(rm, r) * ld;
    const int e = ex[r];
    double x[V];
    const bool fast = km.idx == nullptr && (km.split >= k0 + V || km.split <= k0) && k0 + V <= K;
    const double* q1 = row + map_idx(km, k0);
    if (fast && (reinterpret_cast<uintptr_t>(q1) & 15) == 0) {
      const double2* q = reinterpret_cast<const double2*>(q1);
#pragma unroll
      for (int i = 0; i < V / 2; ++i) {
        const double2 v = __ldcs(q + i);
        x[2 * i] = v.x;
        x[2 * i + 1] = v.y;
      }
    } else if (fast) {
#pragma unroll
      for (int i = 0; i < V; ++i) x[i] = q1[i];
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) x[i] = (k0 + i < K) ? row[map_idx(km, k0 + i)] : 0.0;
    }
    int c0[V], c1[V], c2[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const uint64_t a = oz_scaled_mag(x[i], e);
      const int sg = x[i] < 0.0 ? -1 : 1;
      c0[i] = sg * (int)((uint32_t)a & 0x1fffffu);
      c1[i] = sg * (int)((uint32_t)(a >> 21) & 0x1fffffu);
      c2[i] = sg * (int)(a >> 42);
    }
    int8_t* dst = Q + (int64_t)r * ldq + k0;
#pragma unroll
    for (int l = 0; l < NM; ++l) {
      {
        int v[V];
#pragma unroll
        for (int i = 0; i < V; ++i) v[i] = oz_sym_residue(T, l, c0[i], c1[i], c2[i]);
        const uint32_t w0 = __byte_perm(__byte_perm(v[0], v[1], 0x0040), __byte_perm(v[2], v[3], 0x0040), 0x5410);
        const uint32_t w1 = __byte_perm(__byte_perm(v[4], v[5], 0x0040), __byte_perm(v[6], v[7], 0x0040), 0x5410);
        *reinterpret_cast<uint2*>(dst + (int64_t)l * qplane) = make_uint2(w0, w1);
      }
    }
  }
}

// ---- step 4: CRT + fused GEMM epilogue.
struct OzCrt {
  const uint8_t* R; int64_t ldr, rplane;    // residues [l][i][j]
  const int* ex; const int* ey;
  RowMap exm, eym;  // row i / chunk column j -> exponent index (all-zero map = identity)
  int n;            // moduli
  int M, ncols;     // rows of the output, columns of this chunk
  int j_off;        // logical column of chunk column 0
};

// Exact C' from n residues; returns C' · 2^-shift as FP64.
// Limbs of the CRT arithmetic: |C'| <= P/4 < 2^(32·L - 1) suffices, the sum
// S = Σ r_l w_l being evaluated modulo 2^(32·L).  16 moduli (P < 2^126): 4.
template <int NM>
constexpr int oz_limbs() { return NM <= 16 ? 4 : 5; }

template <int NM>
__device__ __forceinline__ double oz_crt_value(const OzTable& T, const uint32_t* rs, int byte, int shift) {
  constexpr int LB = oz_limbs<NM>();
  int64_t acc[LB];
#pragma unroll
  for (int k = 0; k < LB; ++k) acc[k] = 0;
  float fq = 0.0f;
#pragma unroll
  for (int l = 0; l < NM; ++l) {
    {
      const uint32_t r = (rs[l] >> (8 * byte)) & 0xffu;
#pragma unroll
      for (int k = 0; k < LB; ++k) acc[k] += (int64_t)((uint64_t)r * T.w[l][k]);
      fq = fmaf((float)r, T.f[l], fq);
    }
  }
  const int64_t q = (int64_t)rintf(fq);
#pragma unroll
  for (int k = 0; k < LB; ++k) acc[k] -= q * (int64_t)T.P[k];
#pragma unroll
  for (int k = 0; k < LB - 1; ++k) {
    acc[k + 1] += acc[k] >> 32;            // arithmetic shift: signed carry
    acc[k] &= 0xffffffffll;
  }
  uint32_t L[LB];
#pragma unroll
  for (int k = 0; k < LB; ++k) L[k] = (uint32_t)acc[k];
  const bool neg = (int32_t)L[LB - 1] < 0;
  if (neg) {   // two's-complement negate the 192-bit value
    uint32_t carry = 1;
#pragma unroll
    for (int k = 0; k < LB; ++k) {
      const uint64_t s = (uint64_t)(~L[k]) + carry;
      L[k] = (uint32_t)s;
      carry = (uint32_t)(s >> 32);
    }
  }
  double d = 0.0;
#pragma unroll
  for (int k = LB - 1; k >= 0; --k) d = fma(d, 4294967296.0, (double)L[k]);
  d = neg ? -d : d;
  const int be = 1023 - shift;                 // 2^-shift as a normal double when in range
  if (be >= 1 && be <= 2046) return d * __longlong_as_double((int64_t)be << 52);
  return ldexp(d, -shift);
}

// Block: 256 threads = 8 warps; tile 16 rows x 128 columns; thread = 4
// consecutive columns of 2 rows.  Mirror stores go through a shared-memory
// transpose so both stores are coalesced.  Column 4·lane + b of a tile row sits
// at b·33 + lane: each warp store is 32 consecutive doubles (no bank conflicts;
// 4·lane + b would put lanes 8 banks apart, an 8-way conflict).
template <int NM>
__global__ void __launch_bounds__(256) oz_crt_kernel(const GemmParams P, const OzCrt E) {
  constexpr int TR = 16;          // tile rows (16.5 KB of shared memory: co-resides with the INT8 GEMM)
  __shared__ double tile[TR][4 * 33 + 1];
  const OzTable& T = c_oz[NM - OZ_MINN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tiles_j = (E.ncols + 127) / 128, tiles_i = (E.M + TR - 1) / TR;
  for (int tile_id = blockIdx.x; tile_id < tiles_i * tiles_j; tile_id += gridDim.x) {
  const int i0 = (tile_id / tiles_j) * TR, j0 = (tile_id % tiles_j) * 128;
  const int jl = j0 + 4 * lane;
  const bool diag_skip_all = P.lower && (E.j_off + j0) > (i0 + TR - 1);
  if (diag_skip_all) continue;
  __syncthreads();                // the previous tile's mirror reads are done
#pragma unroll 1
  for (int rr = 0; rr < TR / 8; ++rr) {
    const int il = warp + 8 * rr;
    const int i = i0 + il;
    double v4[4] = {0.0, 0.0, 0.0, 0.0};
    bool ok4[4] = {false, false, false, false};
    if (i < E.M && jl < E.ncols) {
      uint32_t rs[NM];
      const uint8_t* src = E.R + (int64_t)i * E.ldr + jl;
#pragma unroll
      for (int l = 0; l < NM; ++l) rs[l] = __ldcs(reinterpret_cast<const unsigned int*>(src + (int64_t)l * E.rplane));
      const int exi = E.ex[map_idx(E.exm, i)];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int j = jl + b;
        if (j >= E.ncols) break;
        const int n = E.j_off + j;
        if (P.lower && i < n) continue;
        double v = P.alpha * oz_crt_value<NM>(T, rs, b, exi + E.ey[map_idx(E.eym, j)]);
        if (P.beta != 0.0) v += P.beta * P.D[map_idx(P.dm, i) * P.ldd + map_idx(P.dn, n)];
        v4[b] = v;
        ok4[b] = true;
        if (P.direct) P.C[map_idx(P.cm, i) * P.ldc + map_idx(P.cn, n)] = v;
      }
    }
    if (P.mirror) {
#pragma unroll
      for (int b = 0; b < 4; ++b) tile[il][b * 33 + lane] = ok4[b] ? v4[b] : __longlong_as_double(-1ll);
    }
  }
  if (!P.mirror) continue;
  __syncthreads();
  // mirror: C2[c2n(n)][c2m(i)] for the 128 columns x TR rows of the tile
  // (half-warps: lanes 0..15 and 16..31 take two consecutive columns)
  const int il = lane & (TR - 1);
  const int i = i0 + il;
  if (i < E.M) {
    const int64_t mc = map_idx(P.c2m, i);
#pragma unroll 1
    for (int jj = 2 * warp + (lane >> 4); jj < 128; jj += 16) {
      const int j = j0 + jj;
      if (j >= E.ncols) break;
      const double v = tile[il][(jj & 3) * 33 + (jj >> 2)];
      if (__double_as_longlong(v) == -1ll) continue;   // not computed (lower mask)
      P.C2[map_idx(P.c2n, E.j_off + j) * P.ldc2 + mc] = v;
    }
  }
  }
}

// ---- incremental maintenance of the residue planes of Σ (full rows,
// exponent per row, plane stride qplane): after a block step only the set's
// columns changed in the other rows.  Rewrite their residues with the row's
// existing exponent; a value that no longer fits in t bits flags its row for
// a full re-conversion (oz_fix_rows_kernel).
template <int NM>
__global__ void __launch_bounds__(256) oz_update_cols_kernel(const double* __restrict__ S, int64_t ld, int rows,
                                                             int64_t lo, int b, const int* __restrict__ E, int t,
                                                             int8_t* __restrict__ Q, int64_t ldq, int64_t qplane,
                                                             int* __restrict__ flags) {
  constexpr int V = 8;
  const OzTable& T = c_oz[NM - OZ_MINN];
  const int per = (b + V - 1) / V;
  for (int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; item < (int64_t)rows * per;
       item += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(item / per);
    const int c0 = (int)(item - (int64_t)j * per) * V;
    const double* src = S + (int64_t)j * ld + lo + c0;
    const int e = E[j];
    int r0[V], r1[V], r2[V];
    bool over = false;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const double x = c0 + i < b ? src[i] : 0.0;
      // |x|·2^e must stay below 2^t; test the exponent (a shifted mantissa
      // would overflow 64 bits long before the test could see it)
      const int ex = (int)((__double_as_longlong(x) >> 52) & 0x7ff);
      const bool big = ex != 0 && ex - 1023 + e >= t;
      over |= big;
      const uint64_t a = big ? 0 : oz_scaled_mag(x, e);
      const int sg = x < 0.0 ? -1 : 1;
      r0[i] = sg * (int)((uint32_t)a & 0x1fffffu);
      r1[i] = sg * (int)((uint32_t)(a >> 21) & 0x1fffffu);
      r2[i] = sg * (int)(a >> 42);
    }
    if (over) flags[j] = 1;
    int8_t* dst = Q + (int64_t)j * ldq + lo + c0;
#pragma unroll
    for (int l = 0; l < NM; ++l) {
      int v[V];
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = oz_sym_residue(T, l, r0[i], r1[i], r2[i]);
      if (c0 + V <= b) {
        const uint32_t w0 = __byte_perm(__byte_perm(v[0], v[1], 0x0040), __byte_perm(v[2], v[3], 0x0040), 0x5410);
        const uint32_t w1 = __byte_perm(__byte_perm(v[4], v[5], 0x0040), __byte_perm(v[6], v[7], 0x0040), 0x5410);
        *reinterpret_cast<uint2*>(dst + (int64_t)l * qplane) = make_uint2(w0, w1);
      } else {
        for (int i = 0; c0 + i < b; ++i) dst[(int64_t)l * qplane + i] = (int8_t)v[i];
      }
    }
  }
}

// Re-convert every flagged row in full (fresh exponent), one block per row.
template <int NM>
__global__ void __launch_bounds__(256) oz_fix_rows_kernel(const double* __restrict__ S, int64_t ld, int rows, int K,
                                                          int* __restrict__ E, int t, int8_t* __restrict__ Q,
                                                          int64_t ldq, int64_t qplane, int* __restrict__ flags) {
  constexpr int V = 8;
  __shared__ double red[8];
  const OzTable& T = c_oz[NM - OZ_MINN];
  for (int j = blockIdx.x; j < rows; j += gridDim.x) {
    if (flags[j] == 0) continue;
    const double* row = S + (int64_t)j * ld;
    double mx = 0.0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) mx = fmax(mx, fabs(row[k]));
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
    const int e = mx > 0.0 ? t - 1 - ilogb(mx) : 0;
    for (int k0 = threadIdx.x * V; k0 < ldq; k0 += blockDim.x * V) {
      int r0[V], r1[V], r2[V];
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const double x = k0 + i < K ? row[k0 + i] : 0.0;
        const uint64_t a = oz_scaled_mag(x, e);
        const int sg = x < 0.0 ? -1 : 1;
        r0[i] = sg * (int)((uint32_t)a & 0x1fffffu);
        r1[i] = sg * (int)((uint32_t)(a >> 21) & 0x1fffffu);
        r2[i] = sg * (int)(a >> 42);
      }
      int8_t* dst = Q + (int64_t)j * ldq + k0;
#pragma unroll
      for (int l = 0; l < NM; ++l) {
        int v[V];
#pragma unroll
        for (int i = 0; i < V; ++i) v[i] = oz_sym_residue(T, l, r0[i], r1[i], r2[i]);
        const uint32_t w0 = __byte_perm(__byte_perm(v[0], v[1], 0x0040), __byte_perm(v[2], v[3], 0x0040), 0x5410);
        const uint32_t w1 = __byte_perm(__byte_perm(v[4], v[5], 0x0040), __byte_perm(v[6], v[7], 0x0040), 0x5410);
        *reinterpret_cast<uint2*>(dst + (int64_t)l * qplane) = make_uint2(w0, w1);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      E[j] = e;
      flags[j] = 0;
    }
  }
}

// n (moduli) -> template instance
#define OZ_DISPATCH(n, F, ...)                  \
  switch (n) {                                  \
    case 8: F<8>(__VA_ARGS__); break;           \
    case 9: F<9>(__VA_ARGS__); break;           \
    case 10: F<10>(__VA_ARGS__); break;         \
    case 11: F<11>(__VA_ARGS__); break;         \
    case 12: F<12>(__VA_ARGS__); break;         \
    case 13: F<13>(__VA_ARGS__); break;         \
    case 14: F<14>(__VA_ARGS__); break;         \
    case 15: F<15>(__VA_ARGS__); break;         \
    case 16: F<16>(__VA_ARGS__); break;         \
    case 17: F<17>(__VA_ARGS__); break;         \
    case 18: F<18>(__VA_ARGS__); break;         \
    case 19: F<19>(__VA_ARGS__); break;         \
    default: F<20>(__VA_ARGS__); break;         \
  }

// The conversion / CRT kernels keep the SM in its max-shared-memory
// configuration: a kernel that prefers L1 would have the SM re-carved, which
// needs it drained, and the INT8 GEMM (197 KB per CTA) could not co-reside.
template <class F>
void oz_carveout(F* f) {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    done = true;
  }
}
template <int NM>
void oz_split_launch(dim3 grid, cudaStream_t s, const double* X, int64_t ld, RowMap rm, RowMap km, int R, int K,
                     const int* ex, int8_t* Q, int64_t ldq, int64_t qplane) {
  oz_carveout(oz_split_kernel<NM>);
  oz_split_kernel<NM><<<grid, 256, 0, s>>>(X, ld, rm, km, R, K, ex, Q, ldq, qplane);
}
template <int NM>
void oz_update_cols_launch(dim3 grid, cudaStream_t s, const double* S, int64_t ld, int rows, int64_t lo, int b,
                           const int* E, int t, int8_t* Q, int64_t ldq, int64_t qplane, int* flags) {
  oz_update_cols_kernel<NM><<<grid, 256, 0, s>>>(S, ld, rows, lo, b, E, t, Q, ldq, qplane, flags);
}
template <int NM>
void oz_fix_rows_launch(dim3 grid, cudaStream_t s, const double* S, int64_t ld, int rows, int K, int* E, int t,
                        int8_t* Q, int64_t ldq, int64_t qplane, int* flags) {
  oz_fix_rows_kernel<NM><<<grid, 256, 0, s>>>(S, ld, rows, K, E, t, Q, ldq, qplane, flags);
}
template <int NM>
void oz_crt_launch(dim3 grid, cudaStream_t s, const GemmParams& P, const OzCrt& E) {
  oz_carveout(oz_crt_kernel<NM>);
  oz_crt_kernel<NM><<<grid, 256, 0, s>>>(P, E);
}

}  // namespace ibmi
