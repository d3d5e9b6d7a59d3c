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
  uint32_t cpow[OZ_MAXN][2];     // bytes i=0..3 / 4..7: 2^(8i) mod m, packed for dp4a
  int cneg[OZ_MAXN];             // (-2^64) mod m: two's-complement correction of a negative int64
  uint32_t w[OZ_MAXN][OZ_LIMBS]; // CRT weights (P/m_l)·((P/m_l)^-1 mod m_l) < P
  double f[OZ_MAXN];             // w_l / P
  uint32_t P[OZ_LIMBS];
  double log2P;
};

__constant__ OzTable c_oz[OZ_MAXN - OZ_MINN + 1];

// ---- step 1: per-row exponent.  Row r of the operand is X[rm(r)][km(k)],
// k in [0, K).  ex[r] = t - 1 - floor(log2 max_k |X|)  (0 for a zero row).
__global__ void oz_rowexp_kernel(const double* __restrict__ X, int64_t ld, RowMap rm, RowMap km, int R, int K,
                                 int t, int* __restrict__ ex) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= R) return;
  const double* row = X + map_idx(rm, warp) * ld;
  double mx = 0.0;
  if (km.idx == nullptr && km.split >= K) {
    const double* q = row + km.off0;
    for (int k = lane; k < K; k += 32) mx = fmax(mx, fabs(q[k]));
  } else {
    for (int k = lane; k < K; k += 32) mx = fmax(mx, fabs(row[map_idx(km, k)]));
  }
  mx = warp_max(mx);
  if (lane == 0) ex[warp] = mx > 0.0 ? t - 1 - ilogb(mx) : 0;
}

// residue of a two's-complement int64 v modulo table entry l, in [0, m)
__device__ __forceinline__ int oz_mod(const OzTable& T, int l, uint64_t v) {
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  int s = (int)__dp4a(lo, T.cpow[l][0], __dp4a(hi, T.cpow[l][1], 0u));
  s += ((int64_t)v < 0) ? T.cneg[l] : 0;          // s < 8*255*255 + 256 < 2^20: exact in fp32
  const int m = T.m[l];
  int q = __float2int_rz((float)s * T.invm[l]);
  int r = s - q * m;
  r += r < 0 ? m : 0;
  r -= r >= m ? m : 0;
  return r;
}

// ---- step 2: residue planes.  Thread = (row r, 16 consecutive logical k);
// plane l of row r lives at Q + l*qplane + r*ldq.  Columns k >= K are zero.
__global__ void __launch_bounds__(256) oz_split_kernel(const double* __restrict__ X, int64_t ld, RowMap rm,
                                                       RowMap km, int R, int K, const int* __restrict__ ex, int n,
                                                       int8_t* __restrict__ Q, int64_t ldq, int64_t qplane) {
  const int r = blockIdx.y;
  const int k0 = (blockIdx.x * blockDim.x + threadIdx.x) * 16;
  if (r >= R || k0 >= ldq) return;
  const OzTable& T = c_oz[n - OZ_MINN];
  const double* row = X + map_idx(rm, r) * ld;
  const int e = ex[r];
  int64_t v[16];
  const bool fast = km.idx == nullptr && (km.split >= k0 + 16 || km.split <= k0) && k0 + 16 <= K;
  if (fast) {
    const double* q = row + map_idx(km, k0);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __double2ll_rn(ldexp(q[i], e));
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = (k0 + i < K) ? __double2ll_rn(ldexp(row[map_idx(km, k0 + i)], e)) : 0;
  }
  int8_t* dst = Q + (int64_t)r * ldq + k0;
#pragma unroll 1
  for (int l = 0; l < n; ++l) {
    const int m = T.m[l];
    const int half = (m - 1) >> 1;
    uint32_t w[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint32_t pk = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        int x = oz_mod(T, l, (uint64_t)v[4 * g + b]);
        x -= x > half ? m : 0;                       // symmetric residue: |x| <= 128
        pk |= ((uint32_t)(x & 0xff)) << (8 * b);
      }
      w[g] = pk;
    }
    *reinterpret_cast<uint4*>(dst + (int64_t)l * qplane) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// ---- step 4: CRT + fused GEMM epilogue.
struct OzCrt {
  const uint8_t* R; int64_t ldr, rplane;    // residues [l][i][j]
  const int* ex; const int* ey;
  int n;            // moduli
  int M, ncols;     // rows of the output, columns of this chunk
  int j_off;        // logical column of chunk column 0
};

// Exact C' from n residues; returns C' · 2^-shift as FP64.
__device__ __forceinline__ double oz_crt_value(const OzTable& T, const uint32_t* rs, int byte, int shift) {
  int64_t acc[OZ_LIMBS];
#pragma unroll
  for (int k = 0; k < OZ_LIMBS; ++k) acc[k] = 0;
  double fq = 0.0;
#pragma unroll
  for (int l = 0; l < OZ_MAXN; ++l) {
    if (l < T.n) {
      const uint32_t r = (rs[l] >> (8 * byte)) & 0xffu;
#pragma unroll
      for (int k = 0; k < OZ_LIMBS; ++k) acc[k] += (int64_t)((uint64_t)r * T.w[l][k]);
      fq = fma((double)r, T.f[l], fq);
    }
  }
  const int64_t q = (int64_t)rint(fq);
#pragma unroll
  for (int k = 0; k < OZ_LIMBS; ++k) acc[k] -= q * (int64_t)T.P[k];
#pragma unroll
  for (int k = 0; k < OZ_LIMBS - 1; ++k) {
    acc[k + 1] += acc[k] >> 32;            // arithmetic shift: signed carry
    acc[k] &= 0xffffffffll;
  }
  uint32_t L[OZ_LIMBS];
#pragma unroll
  for (int k = 0; k < OZ_LIMBS; ++k) L[k] = (uint32_t)acc[k];
  const bool neg = (int32_t)L[OZ_LIMBS - 1] < 0;
  if (neg) {   // two's-complement negate the 192-bit value
    uint32_t carry = 1;
#pragma unroll
    for (int k = 0; k < OZ_LIMBS; ++k) {
      const uint64_t s = (uint64_t)(~L[k]) + carry;
      L[k] = (uint32_t)s;
      carry = (uint32_t)(s >> 32);
    }
  }
  double d = 0.0;
#pragma unroll
  for (int k = OZ_LIMBS - 1; k >= 0; --k) d = fma(d, 4294967296.0, (double)L[k]);
  return ldexp(neg ? -d : d, -shift);
}

// Block: 256 threads = 8 warps; tile 32 rows x 128 columns; thread = 4
// consecutive columns of 4 rows.  Mirror stores go through a shared-memory
// transpose so both stores are coalesced.
__global__ void __launch_bounds__(256) oz_crt_kernel(const GemmParams P, const OzCrt E) {
  __shared__ double tile[32][129];
  const OzTable& T = c_oz[E.n - OZ_MINN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 128;
  const int jl = j0 + 4 * lane;
  const bool diag_skip_all = P.lower && (E.j_off + j0) > (i0 + 31);
  if (diag_skip_all) return;
#pragma unroll 1
  for (int rr = 0; rr < 4; ++rr) {
    const int il = warp + 8 * rr;
    const int i = i0 + il;
    double v4[4] = {0.0, 0.0, 0.0, 0.0};
    bool ok4[4] = {false, false, false, false};
    if (i < E.M && jl < E.ncols) {
      uint32_t rs[OZ_MAXN];
      const uint8_t* src = E.R + (int64_t)i * E.ldr + jl;
#pragma unroll
      for (int l = 0; l < OZ_MAXN; ++l)
        rs[l] = l < E.n ? *reinterpret_cast<const uint32_t*>(src + (int64_t)l * E.rplane) : 0u;
      const int exi = E.ex[i];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int j = jl + b;
        if (j >= E.ncols) break;
        const int n = E.j_off + j;
        if (P.lower && i < n) continue;
        double v = P.alpha * oz_crt_value(T, rs, b, exi + E.ey[j]);
        if (P.beta != 0.0) v += P.beta * P.D[map_idx(P.dm, i) * P.ldd + map_idx(P.dn, n)];
        v4[b] = v;
        ok4[b] = true;
        if (P.direct) P.C[map_idx(P.cm, i) * P.ldc + map_idx(P.cn, n)] = v;
      }
    }
    if (P.mirror) {
#pragma unroll
      for (int b = 0; b < 4; ++b) tile[il][4 * lane + b] = ok4[b] ? v4[b] : __longlong_as_double(-1ll);
    }
  }
  if (!P.mirror) return;
  __syncthreads();
  // mirror: C2[c2n(n)][c2m(i)] for the 128 columns x 32 rows of the tile
  const int i = i0 + lane;
  if (i >= E.M) return;
  const int64_t mc = map_idx(P.c2m, i);
#pragma unroll 1
  for (int jj = warp; jj < 128; jj += 8) {
    const int j = j0 + jj;
    if (j >= E.ncols) break;
    const double v = tile[lane][jj];
    if (__double_as_longlong(v) == -1ll) continue;   // not computed (lower mask)
    P.C2[map_idx(P.c2n, E.j_off + j) * P.ldc2 + mc] = v;
  }
}

}  // namespace ibmi
