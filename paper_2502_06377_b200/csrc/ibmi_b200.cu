// libibmi_b200.so — B200-native IBMI sweep behind a C ABI (include/ibmi_b200.h).
//
// Device data layout (row-major FP64, leading dimension ld = roundup(p, 32),
// padding columns zero):
//   A        p × ld        the SPD input, read-only after set_matrix
//   Σ        p × ld        the approximation of A⁻¹, full symmetric storage
//   W_k      b_k × ld      A_II⁻¹ A_Ic in GLOBAL column coordinates (columns of
//                          I_k zero), one per set, cached for the whole solve
//                          (reference _BlockOp.w, solver.py:120)
//   ainv_k   b_k × ldb     A_II⁻¹ (exactly symmetric)
//   B        b_K × ldc     estimate matrix Σ_II A_Ic + Σ_Ic A_cc (solver.py:154)
//   G        n × n         its Gram matrix (B·Bᵀ or Bᵀ·B, whichever is smaller)
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <chrono>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ibmi_b200.h"
#include <nvtx3/nvToolsExt.h>
#include <cudaTypedefs.h>
#include "gemm_nt.cuh"
#include "gemm_tma.cuh"
#include "small_kernels.cuh"
#include "small_sweep.cuh"
#include "igemm_tc.cuh"
#include "ozaki.cuh"

using namespace ibmi;

namespace {

thread_local std::string g_err = "";

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      int code_ = (e_ == cudaErrorMemoryAllocation) ? IBMI_ERR_OOM : IBMI_ERR_CUDA;           \
      return fail(code_, std::string(#expr) + ": " + cudaGetErrorString(e_));                 \
    }                                                                                         \
  } while (0)

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ------------------------------------------------------ device block cache
// Every device buffer of a context (A, Σ, W_k, workspaces, residue planes) is
// a multi-GB cudaMalloc, and cudaMalloc/cudaFree of that size cost 10–700 ms
// each depending on what the driver has to map or unmap.  Freed blocks are
// therefore kept per device and handed to the next request of a similar size
// (a repeated solve of the same shape reuses every block), up to a cap of a
// quarter of the device's memory (IBMI_MEM_CACHE_MB overrides; 0 disables).
// release() synchronises the device first, as cudaFree does, so a cached block
// is never reused while kernels still touch it.  When cudaMalloc fails the
// device's cache is returned to the driver and the request retried;
// ibmi_release_cached_memory() does that on demand.
struct DevBlock { size_t bytes; int dev; };
std::mutex g_mem_mu;
struct MemCache {
  std::vector<std::pair<void*, DevBlock>> live;    // small: tens of blocks per context
  std::vector<std::pair<void*, DevBlock>> free;
  size_t free_bytes[64] = {};
};
MemCache g_mem;

size_t mem_cache_cap(int dev) {
  static long long env = [] {
    const char* v = getenv("IBMI_MEM_CACHE_MB");
    return v ? atoll(v) : -1ll;
  }();
  if (env >= 0) return (size_t)env << 20;
  static size_t caps[64] = {};
  if (dev < 0 || dev >= 64) return 0;
  if (!caps[dev]) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); return 0; }
    caps[dev] = tot / 4;
  }
  return caps[dev];
}

// Return every cached block of `dev` (or of all devices, dev < 0) to the driver.
void mem_flush_locked(int dev) {
  auto& fl = g_mem.free;
  for (size_t i = 0; i < fl.size();) {
    if (dev < 0 || fl[i].second.dev == dev) {
      (cudaFree)(fl[i].first);
      g_mem.free_bytes[fl[i].second.dev & 63] -= fl[i].second.bytes;
      fl[i] = fl.back();
      fl.pop_back();
    } else {
      ++i;
    }
  }
}

// Live contexts per device.  While none is left, the cache keeps at most
// 1/16 of the device's memory (IBMI_MEM_IDLE_CACHE_MB overrides): enough for
// the next solve of a c4-sized problem to reuse its blocks, without holding a
// quarter of HBM against torch (or another process) between solves.
int g_live_ctx[64] = {};

size_t mem_idle_cap(int dev) {
  static long long env = [] {
    const char* v = getenv("IBMI_MEM_IDLE_CACHE_MB");
    return v ? atoll(v) : -1ll;
  }();
  if (env >= 0) return (size_t)env << 20;
  return mem_cache_cap(dev) / 4;
}

// Return cached blocks of `dev`, largest first, until at most `keep` bytes stay.
void mem_trim_locked(int dev, size_t keep) {
  auto& fl = g_mem.free;
  while (g_mem.free_bytes[dev & 63] > keep) {
    int big = -1;
    for (int i = 0; i < (int)fl.size(); ++i)
      if (fl[i].second.dev == dev && (big < 0 || fl[i].second.bytes > fl[big].second.bytes)) big = i;
    if (big < 0) break;
    (cudaFree)(fl[big].first);
    g_mem.free_bytes[dev & 63] -= fl[big].second.bytes;
    fl[big] = fl.back();
    fl.pop_back();
  }
}

// IBMI_MEM_POISON=1: fill every block handed out with 0xFF bytes (NaN), so a
// kernel that reads memory it never wrote shows up in the parity tests.
cudaError_t mem_poison(void* p, size_t bytes) {
  static int on = getenv("IBMI_MEM_POISON") ? 1 : 0;
  if (!on) return cudaSuccess;
  cudaError_t e = cudaMemset(p, 0xFF, bytes);
  return e == cudaSuccess ? cudaDeviceSynchronize() : e;
}

cudaError_t mem_alloc_raw(void** out, size_t bytes);
cudaError_t mem_alloc(void** out, size_t bytes) {
  cudaError_t pe = mem_alloc_raw(out, bytes);
  if (pe == cudaSuccess && *out) pe = mem_poison(*out, bytes);
  return pe;
}

cudaError_t mem_alloc_raw(void** out, size_t bytes) {
  if (bytes == 0) return (cudaMalloc)(out, 0);
  const size_t need = (size_t)round_up((int64_t)bytes, 512);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(g_mem_mu);
  // best fit among cached blocks of this device no more than 1/8 larger
  int best = -1;
  for (int i = 0; i < (int)g_mem.free.size(); ++i) {
    const DevBlock& b = g_mem.free[i].second;
    if (b.dev == dev && b.bytes >= need && b.bytes - need <= need / 8 &&
        (best < 0 || b.bytes < g_mem.free[best].second.bytes))
      best = i;
  }
  if (best >= 0) {
    *out = g_mem.free[best].first;
    g_mem.free_bytes[dev & 63] -= g_mem.free[best].second.bytes;
    g_mem.live.push_back(g_mem.free[best]);
    g_mem.free[best] = g_mem.free.back();
    g_mem.free.pop_back();
    return cudaSuccess;
  }
  e = (cudaMalloc)(out, need);
  if (e == cudaErrorMemoryAllocation && g_mem.free_bytes[dev & 63] > 0) {
    cudaGetLastError();
    mem_flush_locked(dev);
    e = (cudaMalloc)(out, need);
  }
  if (e != cudaSuccess) return e;
  g_mem.live.push_back({*out, DevBlock{need, dev}});
  return cudaSuccess;
}

cudaError_t mem_release(void* p) {
  if (!p) return cudaSuccess;
  std::lock_guard<std::mutex> lock(g_mem_mu);
  int idx = -1;
  for (int i = (int)g_mem.live.size() - 1; i >= 0; --i)
    if (g_mem.live[i].first == p) { idx = i; break; }
  if (idx < 0) return (cudaFree)(p);        // not ours
  const DevBlock b = g_mem.live[idx].second;
  g_mem.live[idx] = g_mem.live.back();
  g_mem.live.pop_back();
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != b.dev) cudaSetDevice(b.dev);
  cudaError_t e = cudaDeviceSynchronize();   // cudaFree's implicit synchronisation
  if (e == cudaSuccess && g_mem.free_bytes[b.dev & 63] + b.bytes <= mem_cache_cap(b.dev)) {
    g_mem.free.push_back({p, b});
    g_mem.free_bytes[b.dev & 63] += b.bytes;
  } else {
    e = (cudaFree)(p);
  }
  if (cur != b.dev) cudaSetDevice(cur);
  return e;
}

// cudaMemGetInfo that counts this device's cached blocks as free.
cudaError_t mem_info(size_t* fr, size_t* tot) {
  cudaError_t e = cudaMemGetInfo(fr, tot);
  if (e != cudaSuccess) return e;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_mem_mu);
  *fr += g_mem.free_bytes[dev & 63];
  return cudaSuccess;
}

// Everything below allocates through the cache.  The IPC-exported panels
// (ibmi_device_alloc) call the driver directly as (cudaMalloc)/(cudaFree).
#define cudaMalloc(P, N) mem_alloc(reinterpret_cast<void**>(P), (size_t)(N))
#define cudaFree(P) mem_release((void*)(P))

// Every kernel this library launches bumps the counter (graph replays add the
// number of kernel nodes captured), so callers can report `gpu_launches`.
std::atomic<long long> g_launches{0};
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ---------------------------------------------------------------- GEMM launch
struct GemmOp {
  const double* X = nullptr; int64_t ldx = 0; RowMap xm = contig_map(0); bool xt = false;
  const double* Y = nullptr; int64_t ldy = 0; RowMap yn = contig_map(0); bool yt = false;
  int64_t M = 0, N = 0;
  int nseg = 0; KSeg seg[2];
  double* C = nullptr; int64_t ldc = 0; RowMap cm = contig_map(0), cn = contig_map(0);
  double alpha = 1.0, beta = 0.0;
  const double* D = nullptr; int64_t ldd = 0; RowMap dm = contig_map(0), dn = contig_map(0);
  bool mirror = false, lower = false;
  double* C2 = nullptr; int64_t ldc2 = 0; RowMap c2m = contig_map(0), c2n = contig_map(0);  // mirror target
  bool c2_set = false;           // false: mirror into C with (cm, cn)
  const int64_t* cidx = nullptr; // optional row index array for the direct store / δ
  bool direct = true;
  double* const* peers = nullptr; int64_t bc_panel = 0; int bc_world = 1, bc_rank = 0;  // fused exchange
  double* partial = nullptr;     // non-null -> Frobenius epilogue
  int splits = 1;                // split-K factor (needs ws: tiles*splits*128*128 doubles)
  double* ws = nullptr;
  // TMA eligibility: operand rows/cols below are the tensor-map extents; each
  // K segment gets maps whose inner extent ends at the segment end, so TMA
  // zero-fills every k slot past it.
  bool tma_ok = false;
  int64_t xrows = 0, xcols = 0, yrows = 0, ycols = 0;
  void add_seg(int64_t x0, int64_t y0, int64_t len) {
    if (len > 0) seg[nseg++] = KSeg{x0, y0, (int)len};
  }
};

// Split-K workspace: s partial tiles per output tile, then one int arrival counter per tile
// (the fused fix-up of the TMA kernel), in doubles.
inline int64_t split_ws_doubles(int64_t tiles, int s) { return tiles * s * GB_M * GB_N + (tiles + 1) / 2; }

// Tuning knobs (ibmi_tune): GEMM configuration of the hot NT kernels and
// split-K factors of the small-grid GEMMs.
int g_variant = 0;          // 0: CfgA (8 warps 64x32), 1: CfgB (16 warps 32x32), 2: CfgC (BK 32)
int g_split_diag = 0;       // split-K of the Σ_II GEMM (0 = auto)
int g_split_gram = 0;       // split-K of the Gram GEMM (0 = auto)
int g_split_panel = 0;      // split-K of the panel and estimate GEMMs (0 = auto)
int g_cluster_power = 1;    // small Gram power iteration on one 16-CTA cluster
int g_power_ll = 1;         // mid-size Gram power iteration with the flag-carrying exchange (no grid barrier)
int g_split_fused = 0;      // split-K partial tiles reduced by the last-arriving split inside the TMA GEMM (no reduction
                            // launch).  Measured slower than the separate reduction kernel (c4 274.2 vs 269.6 ms per sweep,
                            // profiles/r02_splitk_fused_ab.log): off by default
int g_small_fused = 1;      // p <= 1024: the whole sweep's GEMM phases in one cooperative kernel (small_sweep.cuh)
int g_split_min_kt = 4;     // split-K keeps at least this many k-tiles per split
int g_raster_group = 0;     // GEMM tile raster: bands of this many tile rows (0 = tm-major)
int g_tune_gen = 0;         // bumped by ibmi_tune: captured graphs are re-captured
int g_use_tma = 1;          // TMA/mbarrier kernel for eligible hot GEMMs

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
bool g_encode_tried = false;

bool tma_encoder() {
  if (!g_encode_tried) {
    g_encode_tried = true;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cudaGetLastError();
  }
  return g_encode != nullptr;
}

bool encode_map(CUtensorMap* m, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  if (!tma_encoder()) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int EPI, bool FIX = false>
cudaError_t launch_tma_inst(const GemmParams& P, const TmaMaps& maps, int grid, cudaStream_t s) {
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tma_kernel<EPI, FIX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)TMA_SMEM);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  gemm_tma_kernel<EPI, FIX><<<grid, 256, TMA_SMEM, s>>>(P, maps); note_launch();
  return cudaGetLastError();
}

template <class CF, bool XT, bool YT, bool V16, int EPI>
cudaError_t ensure_attr() {
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_nt_kernel<CF, XT, YT, V16, EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  return cudaSuccess;
}

template <class CF, bool XT, bool YT, bool V16, int EPI>
cudaError_t launch_inst(const GemmParams& P, int grid, cudaStream_t s) {
  cudaError_t e = ensure_attr<CF, XT, YT, V16, EPI>();
  if (e != cudaSuccess) return e;
  gemm_nt_kernel<CF, XT, YT, V16, EPI><<<grid, CF::THREADS, CF::SMEM, s>>>(P); note_launch();
  return cudaGetLastError();
}

// Set the dynamic-smem attribute of every instantiation up front (outside any
// graph capture).
cudaError_t prepare_gemm_attributes() {
#define PREP(CF, XT, YT, V, E) \
  { cudaError_t e = ensure_attr<CF, XT, YT, V, E>(); if (e != cudaSuccess) return e; }
#define PREP_NN(CF) \
  PREP(CF, false, false, true, EPI_STORE) PREP(CF, false, false, false, EPI_STORE) \
  PREP(CF, false, false, true, EPI_FROB) PREP(CF, false, false, false, EPI_FROB) \
  PREP(CF, false, false, true, EPI_PARTIAL) PREP(CF, false, false, false, EPI_PARTIAL)
  PREP_NN(CfgA) PREP_NN(CfgB) PREP_NN(CfgC)
  PREP(CfgA, false, true, true, EPI_STORE) PREP(CfgA, false, true, false, EPI_STORE)
  PREP(CfgA, true, true, true, EPI_STORE) PREP(CfgA, true, true, false, EPI_STORE)
  PREP(CfgA, true, false, true, EPI_STORE) PREP(CfgA, true, false, false, EPI_STORE)
#undef PREP_NN
#undef PREP
  for (int e : {EPI_STORE, EPI_FROB, EPI_PARTIAL}) {
    const void* f = e == EPI_STORE ? (const void*)gemm_tma_kernel<EPI_STORE>
                  : e == EPI_FROB ? (const void*)gemm_tma_kernel<EPI_FROB> : (const void*)gemm_tma_kernel<EPI_PARTIAL>;
    cudaError_t er = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TMA_SMEM);
    if (er != cudaSuccess) return er;
  }
  return cudaSuccess;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int gemm_tiles(const GemmOp& op) {
  const int tm = (int)((op.M + GB_M - 1) / GB_M), tn = (int)((op.N + GB_N - 1) / GB_N);
  return op.lower ? tm * (tm + 1) / 2 : tm * tn;
}
int gemm_grid(const GemmOp& op) { return gemm_tiles(op); }

template <class CF, bool V16>
cudaError_t launch_nn(const GemmParams& P, int grid, int epi, cudaStream_t s) {
  if (epi == EPI_FROB) return launch_inst<CF, false, false, V16, EPI_FROB>(P, grid, s);
  if (epi == EPI_PARTIAL) return launch_inst<CF, false, false, V16, EPI_PARTIAL>(P, grid, s);
  return launch_inst<CF, false, false, V16, EPI_STORE>(P, grid, s);
}

cudaError_t launch_gemm_impl(const GemmOp& op, cudaStream_t s, int* path);

// IBMI_PROFILE=1: device-synchronised phase timings of the host entry points
// on stderr (diagnostic only; the syncs change nothing but timing).
// NVTX ranges around the host-side phases (setup, block update k, estimate, sweep, solve loop)
// so a timeline (nsys, ncu --nvtx) shows the algorithm's structure.  Header-only NVTX v3:
// the calls are no-ops unless a tool injects itself; IBMI_NVTX=0 skips even those.
struct NvtxRange {
  bool on;
  explicit NvtxRange(const char* name) {
    static int en = -1;
    if (en < 0) { const char* e = getenv("IBMI_NVTX"); en = (e && e[0] == '0') ? 0 : 1; }
    on = en != 0;
    if (on) nvtxRangePushA(name);
  }
  ~NvtxRange() { if (on) nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct PhaseTimer {
  bool on;
  const char* fn;
  std::chrono::steady_clock::time_point t;
  explicit PhaseTimer(const char* f) : fn(f) {
    static int en = -1;
    if (en < 0) en = getenv("IBMI_PROFILE") ? 1 : 0;
    on = en != 0;
    if (on) { cudaDeviceSynchronize(); t = std::chrono::steady_clock::now(); }
  }
  void mark(const char* what) {
    if (!on) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[ibmi] %s: %s %.1f ms\n", fn, what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// IBMI_DEBUG_SYNC=1: synchronise after every GEMM and report the failing one.
cudaError_t launch_gemm(const GemmOp& op, cudaStream_t s) {
  static int dbg = -1;
  if (dbg < 0) dbg = getenv("IBMI_DEBUG_SYNC") ? 1 : 0;
  int path = -1;
  cudaError_t e = launch_gemm_impl(op, s, &path);
  if (dbg) {
    cudaError_t e2 = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = e2;
    fprintf(stderr, "[ibmi] gemm path=%d M=%lld N=%lld nseg=%d seg0=(%lld,%lld,%d) xt=%d yt=%d lower=%d mirror=%d "
            "splits=%d tma_ok=%d xrows=%lld yrows=%lld -> %s\n", path, (long long)op.M, (long long)op.N, op.nseg,
            (long long)op.seg[0].x0, (long long)op.seg[0].y0, op.nseg ? op.seg[0].len : 0, op.xt, op.yt, op.lower,
            op.mirror, op.splits, op.tma_ok, (long long)op.xrows, (long long)op.yrows, cudaGetErrorString(e));
  }
  return e;
}

cudaError_t launch_gemm_impl(const GemmOp& op, cudaStream_t s, int* path) {
  if (op.M <= 0 || op.N <= 0) return cudaSuccess;
  GemmParams P;
  memset(&P, 0, sizeof(P));
  P.X = op.X; P.ldx = op.ldx; P.xm = op.xm;
  P.Y = op.Y; P.ldy = op.ldy; P.yn = op.yn;
  P.M = (int)op.M; P.N = (int)op.N;
  P.nseg = op.nseg;
  P.kt0 = 0; P.kt_total = 0;
  const bool nn = !op.xt && !op.yt;
  const int bk = (nn && g_variant == 2) ? CfgC::BK : 16;
  for (int i = 0; i < op.nseg; ++i) {
    P.seg[i] = op.seg[i];
    const int kt = (op.seg[i].len + bk - 1) / bk;
    if (i == 0) P.kt0 = kt;
    P.kt_total += kt;
  }
  if (op.nseg == 1) P.seg[1] = op.seg[0];
  P.C = op.C; P.ldc = op.ldc; P.cm = op.cm; P.cn = op.cn;
  P.alpha = op.alpha; P.beta = op.beta;
  P.D = op.D ? op.D : op.C; P.ldd = op.D ? op.ldd : op.ldc; P.dm = op.dm; P.dn = op.dn;
  P.mirror = op.mirror; P.lower = op.lower;
  if (op.c2_set) { P.C2 = op.C2; P.ldc2 = op.ldc2; P.c2m = op.c2m; P.c2n = op.c2n; }
  else { P.C2 = op.C; P.ldc2 = op.ldc; P.c2m = op.cm; P.c2n = op.cn; }
  P.cidx = op.cidx;
  P.direct = op.direct ? 1 : 0;
  P.peers = op.peers; P.bc_panel = op.bc_panel; P.bc_world = op.bc_world; P.bc_rank = op.bc_rank;
  P.tiles_m = (P.M + GB_M - 1) / GB_M;
  P.tiles_n = (P.N + GB_N - 1) / GB_N;
  P.group_m = g_raster_group;
  const int tiles = gemm_tiles(op);
  // 16-byte cp.async only when every operand address it forms is 16B aligned
  bool v16 = aligned16(op.X) && aligned16(op.Y) && (op.ldx % 2 == 0) && (op.ldy % 2 == 0);
  for (int i = 0; i < op.nseg; ++i) v16 = v16 && (op.seg[i].x0 % 2 == 0) && (op.seg[i].y0 % 2 == 0);
  if (op.xt) v16 = v16 && (op.xm.off0 % 2 == 0);
  if (op.yt) v16 = v16 && (op.yn.off0 % 2 == 0);
  int epi = op.partial ? EPI_FROB : EPI_STORE;
  int grid = tiles;
  const bool split = nn && op.splits > 1 && op.ws != nullptr && !op.partial && P.kt_total >= op.splits;
  if (split) {
    epi = EPI_PARTIAL;
    P.splits = op.splits;
    P.partial = op.ws;
    grid = tiles * op.splits;
  } else {
    P.splits = 1;
    P.partial = op.partial;
  }
  cudaError_t err;
  bool use_tma = nn && op.tma_ok && g_use_tma && g_variant != 2 && tma_encoder() && aligned16(op.X) &&
                 aligned16(op.Y) && (op.ldx * 8) % 16 == 0 && (op.ldy * 8) % 16 == 0;
  auto gap_ok = [](const RowMap& m, int64_t rows) { return m.split >= rows || (m.split % 8) == 0; };
  use_tma = use_tma && gap_ok(op.xm, op.M) && gap_ok(op.yn, op.N) && !op.xm.idx && !op.yn.idx;
  // the innermost TMA coordinate must be 16-byte aligned: even K starts only
  for (int i = 0; i < op.nseg; ++i) use_tma = use_tma && (op.seg[i].x0 % 2 == 0) && (op.seg[i].y0 % 2 == 0);
  if (use_tma) {
    // k-tiles are 16 wide on this path
    P.kt0 = 0; P.kt_total = 0;
    for (int i = 0; i < op.nseg; ++i) {
      const int kt = (op.seg[i].len + 15) / 16;
      if (i == 0) P.kt0 = kt;
      P.kt_total += kt;
    }
    TmaMaps maps;
    bool ok = true;
    for (int sg = 0; sg < 2 && ok; ++sg) {
      const KSeg& k = P.seg[sg];   // P.seg[1] duplicates seg 0 when there is one segment
      const int64_t xend = std::min<int64_t>(op.xcols, k.x0 + k.len), yend = std::min<int64_t>(op.ycols, k.y0 + k.len);
      ok = encode_map(&maps.xb[sg], op.X, op.xrows, std::max<int64_t>(xend, 1), op.ldx, 128) &&
           encode_map(&maps.xs[sg], op.X, op.xrows, std::max<int64_t>(xend, 1), op.ldx, 8) &&
           encode_map(&maps.yb[sg], op.Y, op.yrows, std::max<int64_t>(yend, 1), op.ldy, 128) &&
           encode_map(&maps.ys[sg], op.Y, op.yrows, std::max<int64_t>(yend, 1), op.ldy, 8);
    }
    if (ok) {
      *path = 1;
      if (epi == EPI_PARTIAL && g_split_fused) {
        // arrival counters behind the partial tiles; the last split of a tile reduces it in the kernel
        P.tile_count = reinterpret_cast<int*>(op.ws + (size_t)tiles * op.splits * GB_M * GB_N);
        err = cudaMemsetAsync(P.tile_count, 0, (size_t)tiles * sizeof(int), s);
        if (err != cudaSuccess) return err;
        return launch_tma_inst<EPI_PARTIAL, true>(P, maps, grid, s);
      }
      if (epi == EPI_PARTIAL) err = launch_tma_inst<EPI_PARTIAL>(P, maps, grid, s);
      else if (epi == EPI_FROB) err = launch_tma_inst<EPI_FROB>(P, maps, grid, s);
      else err = launch_tma_inst<EPI_STORE>(P, maps, grid, s);
      if (err != cudaSuccess || !split) return err;
      splitk_reduce_kernel<<<tiles * (GB_M / 32), 256, 0, s>>>(P); note_launch();
      return cudaGetLastError();
    }
  }
  *path = 0;
  if (nn) {
    if (g_variant == 0) err = v16 ? launch_nn<CfgA, true>(P, grid, epi, s) : launch_nn<CfgA, false>(P, grid, epi, s);
    else if (g_variant == 2) err = v16 ? launch_nn<CfgC, true>(P, grid, epi, s) : launch_nn<CfgC, false>(P, grid, epi, s);
    else err = v16 ? launch_nn<CfgB, true>(P, grid, epi, s) : launch_nn<CfgB, false>(P, grid, epi, s);
  } else if (!op.xt && op.yt) {
    err = v16 ? launch_inst<CfgA, false, true, true, EPI_STORE>(P, grid, s)
              : launch_inst<CfgA, false, true, false, EPI_STORE>(P, grid, s);
  } else if (op.xt && op.yt) {
    err = v16 ? launch_inst<CfgA, true, true, true, EPI_STORE>(P, grid, s)
              : launch_inst<CfgA, true, true, false, EPI_STORE>(P, grid, s);
  } else {
    err = v16 ? launch_inst<CfgA, true, false, true, EPI_STORE>(P, grid, s)
              : launch_inst<CfgA, true, false, false, EPI_STORE>(P, grid, s);
  }
  if (err != cudaSuccess || !split) return err;
  splitk_reduce_kernel<<<tiles * (GB_M / 32), 256, 0, s>>>(P); note_launch();
  return cudaGetLastError();
}

// Split factor that fills the SMs: smallest s with tiles*s >= 0.9 * waves * SMs.
// Split-K factor minimising modelled time: whole waves of 128×128×16 k-tiles
// (2.1 µs each at the DMMA peak) plus the partial-tile traffic of the
// fixed-order reduction (write s tiles, read them back, write the result).
int auto_split(int tiles, int kt_total, int sms) {
  const double t_k = 2.1e-6, tile_bytes = 128.0 * 128.0 * 8.0, hbm = 6.0e12;
  int best = 1;
  double best_t = 1e300;
  for (int s = 1; s <= 16; ++s) {
    if (s > 1 && kt_total / s < g_split_min_kt) break;
    const int64_t ctas = (int64_t)tiles * s;
    const int64_t waves = (ctas + sms - 1) / sms;
    const double t = (double)waves * ((kt_total + s - 1) / s) * t_k +
                     (s > 1 ? (double)tiles * (2.0 * s + 1.0) * tile_bytes / hbm + 5e-6 : 0.0);
    if (t < best_t * 0.995) { best_t = t; best = s; }
  }
  return best;
}

// ------------------------------------------------ Ozaki-II FP64 emulation
// (ozaki.cuh).  g_oz_n = 0 keeps every GEMM on the FP64 DMMA kernels; 8..20
// routes the eligible hot GEMMs through n INT8 residue GEMMs on tcgen05.
int g_oz_n = 0;
int g_oz_pair = 1;             // 1: CTA-pair INT8 GEMM (cta_group::2, 256x256 tiles); 0: one CTA per 128x256 tile
int g_sms_hint = 148;          // SM count of the device in use (bounded persistent grids)
bool g_oz_timing = false;      // ibmi_tune(9): event-time every INT8 GEMM launch (eager paths only)
struct OzEvent { cudaEvent_t a, b; double ops; };
std::vector<OzEvent> g_oz_events;
double g_oz_budget = 6e9;      // bytes of Y residue planes per N chunk
const int kOzModuli[OZ_MAXN] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227,
                                223, 217, 211, 199, 197, 193, 191, 181, 179, 173};
OzTable g_oz_host[OZ_MAXN - OZ_MINN + 1];
bool g_oz_host_ready = false;
uint64_t g_oz_dev_ready = 0;   // bit per device: constant tables uploaded

struct Big {   // 192-bit unsigned, 32-bit limbs
  uint32_t l[OZ_LIMBS] = {0, 0, 0, 0, 0, 0};
  void mul(uint32_t m) {
    uint64_t carry = 0;
    for (int k = 0; k < OZ_LIMBS; ++k) {
      const uint64_t v = (uint64_t)l[k] * m + carry;
      l[k] = (uint32_t)v;
      carry = v >> 32;
    }
  }
  uint32_t mod(uint32_t m) const {
    uint64_t r = 0;
    for (int k = OZ_LIMBS - 1; k >= 0; --k) r = ((r << 32) | l[k]) % m;
    return (uint32_t)r;
  }
  double to_double() const {
    double d = 0.0;
    for (int k = OZ_LIMBS - 1; k >= 0; --k) d = d * 4294967296.0 + (double)l[k];
    return d;
  }
};

void oz_build_tables() {
  if (g_oz_host_ready) return;
  for (int n = OZ_MINN; n <= OZ_MAXN; ++n) {
    OzTable& T = g_oz_host[n - OZ_MINN];
    memset(&T, 0, sizeof(T));
    T.n = n;
    Big P;
    P.l[0] = 1;
    T.log2P = 0.0;
    for (int i = 0; i < n; ++i) {
      P.mul((uint32_t)kOzModuli[i]);
      T.log2P += std::log2((double)kOzModuli[i]);
    }
    memcpy(T.P, P.l, sizeof(T.P));
    const double Pd = P.to_double();
    for (int i = 0; i < n; ++i) {
      const uint32_t m = (uint32_t)kOzModuli[i];
      T.m[i] = (int)m;
      T.invm[i] = 1.0f / (float)m;
      T.k21[i] = (uint32_t)((1ull << 21) % m);
      T.k42[i] = (uint32_t)((1ull << 42) % m);
      int sh = 0;
      while ((2u << sh) <= m) ++sh;                  // sh = floor(log2 m)
      if ((m & (m - 1)) == 0) --sh;                  // power of two: magic 2^(32+sh)/m exact, < 2^32
      T.sh[i] = sh;
      T.magic[i] = (uint32_t)(((1ull << (32 + sh)) + m - 1) / m);
      T.bias[i] = (int)(m * (((1u << 30) + m - 1) / m));
      Big Pl;
      Pl.l[0] = 1;
      for (int j = 0; j < n; ++j)
        if (j != i) Pl.mul((uint32_t)kOzModuli[j]);
      const uint32_t a = Pl.mod(m);
      uint32_t y = 0;
      for (uint32_t t = 1; t < m; ++t)
        if ((uint64_t)a * t % m == 1) { y = t; break; }
      Pl.mul(y);
      memcpy(T.w[i], Pl.l, sizeof(T.w[i]));
      T.f[i] = (float)(Pl.to_double() / Pd);
    }
  }
  g_oz_host_ready = true;
}

cudaError_t oz_upload_tables() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 64 && (g_oz_dev_ready >> dev) & 1) return cudaSuccess;
  oz_build_tables();
  e = cudaMemcpyToSymbol(c_oz, g_oz_host, sizeof(g_oz_host));
  if (e == cudaSuccess && dev < 64) g_oz_dev_ready |= (uint64_t)1 << dev;
  return e;
}

// bits per scaled operand entry: K·2^(2t) <= P/4, capped at 62 (int64 path)
int oz_bits(int n, int64_t K) {
  oz_build_tables();
  const double lp = g_oz_host[n - OZ_MINN].log2P;
  const int t = (int)std::floor((lp - 2.0 - std::log2((double)std::max<int64_t>(K, 1))) * 0.5 - 1e-9);
  return std::min(62, t);
}

bool encode_map_u8(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  if (!tma_encoder()) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)IG_BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct OzWork {
  int8_t* xq = nullptr; int64_t xq_cap = 0;
  int8_t* yq = nullptr; int64_t yq_cap = 0;
  uint8_t* rq = nullptr; int64_t rq_cap = 0;
  int* ex = nullptr; int64_t ex_cap = 0;
  int* ey = nullptr; int64_t ey_cap = 0;
  void release() {
    for (void* q : {(void*)xq, (void*)yq, (void*)rq, (void*)ex, (void*)ey})
      if (q) cudaFree(q);
    xq = yq = nullptr; rq = nullptr; ex = ey = nullptr;
    xq_cap = yq_cap = rq_cap = ex_cap = ey_cap = 0;
  }
};

// Workspace of one emulated GEMM: X planes (n·M·ldq), Y planes of one chunk
// of nc rows (n·nc·ldq), residues (n·M·ldr).
struct OzPlan {
  int nch = 1;
  int64_t K = 0, ldq = 0, nc = 0, ldr = 0;
  int64_t xq = 0, yq = 0, rq = 0, ex = 0, ey = 0;
};
// N chunks: at most the budget's worth of Y planes each; with pipelining
// (g_oz_chunks > 1) at least g_oz_chunks chunks of >= 2 tiles, double-buffered
// so the conversion of chunk j+1 and the CRT of chunk j-1 run on the aux stream
// while the INT8 GEMM of chunk j runs on the main one.
int g_oz_chunks = 1;
OzPlan oz_plan(const GemmOp& op, int n) {
  OzPlan pl;
  for (int i = 0; i < op.nseg; ++i) pl.K += op.seg[i].len;
  pl.ldq = round_up(std::max<int64_t>(pl.K, 1), 16);
  int64_t nc = (int64_t)(g_oz_budget / ((double)n * pl.ldq));
  nc = std::max<int64_t>(IG_BN, nc / IG_BN * IG_BN);
  if (g_oz_chunks > 1) {
    const int64_t want = round_up((op.N + g_oz_chunks - 1) / g_oz_chunks, IG_BN);
    if (want >= 2 * IG_BN) nc = std::min(nc, want);
  }
  if (op.lower) nc = op.N;              // the lower-tile mask needs the whole N range
  pl.nc = std::min<int64_t>(op.N, nc);
  pl.nch = (int)((op.N + pl.nc - 1) / pl.nc);
  const int nbuf = pl.nch > 1 ? 2 : 1;
  pl.ldr = round_up(pl.nc, 16);
  pl.xq = n * op.M * pl.ldq;
  pl.yq = nbuf * n * pl.nc * pl.ldq;
  pl.rq = nbuf * n * op.M * pl.ldr;
  pl.ex = op.M;
  pl.ey = nbuf * pl.nc;
  return pl;
}
bool oz_eligible(const GemmOp& op) {
  return !op.xt && !op.yt && !op.peers && !op.cidx && !op.partial && op.nseg >= 1 && op.M > 0 && op.N > 0;
}
template <class T>
int oz_grow(T** p, int64_t* cap, int64_t need, size_t* bytes) {
  if (need <= *cap) return IBMI_OK;
  if (*p) { cudaFree(*p); *bytes -= (size_t)(*cap) * sizeof(T); }
  *p = nullptr;
  *cap = 0;
  CUDA_TRY(cudaMalloc(p, (size_t)need * sizeof(T)));
  *cap = need;
  *bytes += (size_t)need * sizeof(T);
  return IBMI_OK;
}
int oz_reserve(OzWork& w, const OzPlan& pl, size_t* bytes) {
  if (oz_grow(&w.xq, &w.xq_cap, pl.xq, bytes) || oz_grow(&w.yq, &w.yq_cap, pl.yq, bytes) ||
      oz_grow(&w.rq, &w.rq_cap, pl.rq, bytes) || oz_grow(&w.ex, &w.ex_cap, pl.ex, bytes) ||
      oz_grow(&w.ey, &w.ey_cap, pl.ey, bytes))
    return IBMI_ERR_OOM;
  return IBMI_OK;
}

RowMap map_shift(const RowMap& m, int64_t j0) {
  if (m.idx) return list_map(m.idx + j0);
  if (j0 >= m.split) return RowMap{INT_MAX, m.off1 + (j0 - m.split), 0, nullptr};
  return RowMap{(int)(m.split - j0), m.off0 + j0, m.off1, nullptr};
}

cudaError_t oz_convert(const double* X, int64_t ld, RowMap rm, RowMap km, int64_t R, int64_t K, int t, int* ex,
                       int n, int8_t* Q, int64_t ldq, cudaStream_t s, int64_t qplane = -1) {
  if (qplane < 0) qplane = R * ldq;
  // bounded grids (2 blocks per SM) only when the conversion should co-reside with an INT8 GEMM
  const int gmul = g_oz_chunks > 1 ? 2 : 32;
  const int64_t rx = std::min<int64_t>((R * 32 + 255) / 256, (int64_t)gmul * g_sms_hint);
  oz_carveout(oz_rowexp_kernel);
  oz_rowexp_kernel<<<(unsigned)rx, 256, 0, s>>>(X, ld, rm, km, (int)R, (int)K, t, ex);
  note_launch();
  // persistent split: two 256-thread blocks per SM at most (co-resident with the INT8 GEMM)
  const int64_t items = R * ((ldq + OZ_SPLIT_V * 256 - 1) / (OZ_SPLIT_V * 256));
  dim3 grid((unsigned)std::min<int64_t>(items, (int64_t)gmul * g_sms_hint));
  OZ_DISPATCH(n, oz_split_launch, grid, s, X, ld, rm, km, (int)R, (int)K, ex, Q, ldq, qplane);
  note_launch();
  return cudaGetLastError();
}

GemmParams oz_epilogue(const GemmOp& op) {
  GemmParams P;
  memset(&P, 0, sizeof(P));
  P.M = (int)op.M; P.N = (int)op.N;
  P.C = op.C; P.ldc = op.ldc; P.cm = op.cm; P.cn = op.cn;
  P.alpha = op.alpha; P.beta = op.beta;
  P.D = op.D ? op.D : op.C; P.ldd = op.D ? op.ldd : op.ldc; P.dm = op.dm; P.dn = op.dn;
  P.mirror = op.mirror; P.lower = op.lower;
  if (op.c2_set) { P.C2 = op.C2; P.ldc2 = op.ldc2; P.c2m = op.c2m; P.c2n = op.c2n; }
  else { P.C2 = op.C; P.ldc2 = op.ldc; P.c2m = op.cm; P.c2n = op.cn; }
  P.direct = op.direct ? 1 : 0;
  return P;
}

// Residue planes of one GEMM operand as the INT8 GEMM addresses them:
// plane l, row r, column k at q[(l*rows + r)*ldq + k]; the tensor map spans
// `rows` x `cols`; ig_gap mappings (IgemmParams) for rows and K columns; e
// (exponent per row) indexed through emap (all-zero = identity).
struct OzOperand {
  const int8_t* q = nullptr;
  const int* e = nullptr;
  RowMap emap{0, 0, 0, nullptr};
  int64_t ldq = 0, rows = 0, cols = 0;
  int row_off = 0, split = 0, off1 = 0;     // X: row_off; Y: row gap
  int ksplit = 0, koff1 = 0;
};
inline OzOperand oz_plain(const int8_t* q, const int* e, int64_t ldq, int64_t rows, int64_t cols) {
  OzOperand o;
  o.q = q; o.e = e; o.ldq = ldq; o.rows = rows; o.cols = cols;
  return o;
}

// INT8 residue GEMMs of one N chunk [j0, j0 + nc) into rq.
cudaError_t oz_igemm(const GemmOp& op, int n, const OzOperand& X, const OzOperand& Y, int64_t K, int64_t j0,
                     int64_t nc, uint8_t* rq, int sms, cudaStream_t s) {
  static bool attr = false;
  cudaError_t e;
  if (!attr) {
    e = cudaFuncSetAttribute(igemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)IG_SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(igemm_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)IG2_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const bool pair = g_oz_pair != 0;
  CUtensorMap mx, my;
  if (!encode_map_u8(&mx, X.q, n * X.rows, X.cols, X.ldq, IG_BM) || !encode_map_u8(&my, Y.q, n * Y.rows, Y.cols, Y.ldq, 128))
    return cudaErrorInvalidValue;
  const int64_t ldr = round_up(nc, 16);
  IgemmParams G;
  memset(&G, 0, sizeof(G));
  G.M = (int)op.M; G.N = (int)nc; G.K = (int)K;
  G.tiles_m = (int)((op.M + IG_BM - 1) / IG_BM);
  G.tiles_n = (int)((nc + IG_BN - 1) / IG_BN);
  G.planes = n;
  G.R = rq; G.ldr = ldr; G.r_plane = op.M * ldr;
  for (int l = 0; l < n; ++l) G.mod[l] = g_oz_host[n - OZ_MINN].m[l];
  G.rows_per_plane_x = (int)X.rows;
  G.rows_per_plane_y = (int)Y.rows;
  G.lower = (op.lower && j0 == 0) ? 1 : 0;
  G.x_row_off = X.row_off;
  G.y_split = Y.split; G.y_off1 = Y.off1;
  G.xk_split = X.ksplit; G.xk_off1 = X.koff1;
  G.yk_split = Y.ksplit; G.yk_off1 = Y.koff1;
  int total = G.tiles_m * G.tiles_n * n;
  if (pair) total = 2 * (int)((op.M + IG2_BM - 1) / IG2_BM) * (int)((nc + IG2_BN - 1) / IG2_BN) * n;
  int grid = std::min(total, sms);
  if (pair) grid = std::max(2, grid & ~1);
  cudaEvent_t tev[2] = {nullptr, nullptr};
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  const bool timing = g_oz_timing && cap == cudaStreamCaptureStatusNone;
  if (timing) {   // per-launch CUDA events on the launching stream (never during graph capture)
    cudaEventCreate(&tev[0]);
    cudaEventCreate(&tev[1]);
    cudaEventRecord(tev[0], s);
  }
  if (pair) igemm_tc2_kernel<<<grid, IG_THREADS, IG2_SMEM, s>>>(mx, my, G);
  else igemm_tc_kernel<<<grid, IG_THREADS, IG_SMEM, s>>>(mx, my, G);
  note_launch();
  if (timing) {
    cudaEventRecord(tev[1], s);
    // algorithmic INT8 ops of the launch (lower mode: the tiles it runs)
    double ops = 2.0 * (double)op.M * (double)nc * (double)K * n;
    if (G.lower) {
      const int bm = pair ? IG2_BM : IG_BM, bn = pair ? IG2_BN : IG_BN;
      const int tmm = (int)((op.M + bm - 1) / bm), tnn = (int)((nc + bn - 1) / bn);
      int64_t run = 0;
      for (int tm = 0; tm < tmm; ++tm)
        for (int tn = 0; tn < tnn; ++tn)
          if (!(tn * bn > tm * bm + bm - 1)) ++run;
      ops *= (double)run / (double)(tmm * tnn);
    }
    g_oz_events.push_back({tev[0], tev[1], ops});
  }
  return cudaGetLastError();
}

// CRT + fused epilogue of one N chunk.
cudaError_t oz_crt(const GemmOp& op, const GemmParams& P, int n, const OzOperand& X, const OzOperand& Y, int64_t j0,
                   int64_t nc, const uint8_t* rq, cudaStream_t s) {
  const int64_t ldr = round_up(nc, 16);
  OzCrt E;
  memset(&E, 0, sizeof(E));
  E.R = rq; E.ldr = ldr; E.rplane = op.M * ldr;
  E.ex = X.e; E.ey = Y.e; E.exm = X.emap; E.eym = Y.emap;
  E.n = n; E.M = (int)op.M; E.ncols = (int)nc; E.j_off = (int)j0;
  const int64_t ctiles = ((nc + 127) / 128) * ((op.M + 15) / 16);
  dim3 cg((unsigned)std::min<int64_t>(ctiles, (int64_t)(g_oz_chunks > 1 ? 2 : 32) * g_sms_hint));
  OZ_DISPATCH(n, oz_crt_launch, cg, s, P, E);
  note_launch();
  return cudaGetLastError();
}

cudaError_t oz_chunk(const GemmOp& op, const GemmParams& P, int n, const int8_t* xq, const int* ex, const int8_t* yq,
                     const int* ey, int64_t K, int64_t ldq, int64_t j0, int64_t nc, uint8_t* rq, int sms,
                     cudaStream_t s) {
  const OzOperand X = oz_plain(xq, ex, ldq, op.M, K), Y = oz_plain(yq, ey, ldq, nc, K);
  cudaError_t e = oz_igemm(op, n, X, Y, K, j0, nc, rq, sms, s);
  if (e != cudaSuccess) return e;
  return oz_crt(op, P, n, X, Y, j0, nc, rq, s);
}

bool oz_fits(const GemmOp& op, const OzWork& w, int n) {
  const OzPlan pl = oz_plan(op, n);
  return oz_eligible(op) && pl.xq <= w.xq_cap && pl.yq <= w.yq_cap && pl.rq <= w.rq_cap && pl.ex <= w.ex_cap &&
         pl.ey <= w.ey_cap && op.M <= 65535 && pl.nc <= 65535;
}

// Residue planes converted earlier (a cache or the previous GEMM's operand):
// plane l of row r at q + (l*rows + r)*ldq, exponents e[r].
struct OzPre {
  const int8_t* q = nullptr;
  const int* e = nullptr;
};

// K map of an operand: logical k -> column, from the GEMM's K segments.
inline RowMap oz_kmap(const GemmOp& op, bool y) {
  if (op.nseg == 2) return RowMap{op.seg[0].len, y ? op.seg[0].y0 : op.seg[0].x0, y ? op.seg[1].y0 : op.seg[1].x0, nullptr};
  return RowMap{INT_MAX, y ? op.seg[0].y0 : op.seg[0].x0, 0, nullptr};
}

__global__ void oz_stamp_kernel(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}

// Aux stream + events of the chunk pipeline (owned by a context).
constexpr int OZ_EVENTS = 64;
struct OzStreams {
  cudaStream_t aux = nullptr;
  cudaEvent_t ev[OZ_EVENTS] = {};
  bool ready = false;
  bool init() {
    if (ready) return true;
    if (cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking) != cudaSuccess) return false;
    for (auto& e : ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return false;
    ready = true;
    return true;
  }
  void release() {
    if (!ready) return;
    for (auto& e : ev) cudaEventDestroy(e);
    cudaStreamDestroy(aux);
    ready = false;
  }
};

// C = epilogue(X·Yᵀ) through n INT8 residue GEMMs.  The caller reserved the
// workspace (nothing is allocated here: graph capture).  xp / yp: operand
// planes already converted (same n, K map and K); x_in_ybuf: convert X into
// the Y buffers (when yp points at the X buffers of the previous call).
cudaError_t oz_gemm(const GemmOp& op, OzWork& w, int n, int sms, cudaStream_t s, OzPre xp = OzPre(),
                    OzPre yp = OzPre(), bool x_in_ybuf = false, OzStreams* ps = nullptr) {
  if (!oz_eligible(op) || n < OZ_MINN || n > OZ_MAXN || !tma_encoder()) return cudaErrorInvalidValue;
  const OzPlan pl = oz_plan(op, n);
  if (op.M > 65535 || op.N > 65535) return cudaErrorInvalidValue;
  const int64_t xneed = n * op.M * pl.ldq;
  if (!xp.q) {
    if (x_in_ybuf ? (xneed > w.yq_cap || op.M > w.ey_cap) : (xneed > w.xq_cap || op.M > w.ex_cap))
      return cudaErrorInvalidValue;
  }
  if (yp.q ? (n * op.M * round_up(op.N, 16) > w.rq_cap)
           : (x_in_ybuf || pl.yq > w.yq_cap || pl.ey > w.ey_cap || pl.rq > w.rq_cap))
    return cudaErrorInvalidValue;
  cudaError_t e = oz_upload_tables();
  if (e != cudaSuccess) return e;
  const int t = oz_bits(n, pl.K);
  const GemmParams P = oz_epilogue(op);
  if (!xp.q) {
    int8_t* q = x_in_ybuf ? w.yq : w.xq;
    int* ex = x_in_ybuf ? w.ey : w.ex;
    e = oz_convert(op.X, op.ldx, op.xm, oz_kmap(op, false), op.M, pl.K, t, ex, n, q, pl.ldq, s);
    if (e != cudaSuccess) return e;
    xp.q = q;
    xp.e = ex;
  }
  if (yp.q) return oz_chunk(op, P, n, xp.q, xp.e, yp.q, yp.e, pl.K, pl.ldq, 0, op.N, w.rq, sms, s);
  // (the two-stream pipeline is used with the single-CTA GEMM only: with CTA
  // pairs, a pipelined c4 sweep stalled on the box — not diagnosed)
  if (ps && ps->ready && pl.nch > 1 && 1 + 3 * pl.nch <= OZ_EVENTS && !g_oz_pair) {
    // two-stream pipeline: aux = conv(0) conv(1) crt(0) conv(2) crt(1) ...; main = gemm(0) gemm(1) ...
    cudaEvent_t* fork = &ps->ev[0];
    cudaEvent_t* evc = &ps->ev[1];
    cudaEvent_t* evg = evc + pl.nch;
    cudaEvent_t* evr = evg + pl.nch;
    const int64_t ybuf = n * pl.nc * pl.ldq, rbuf = n * op.M * pl.ldr;
    cudaStream_t a = ps->aux;
    if ((e = cudaEventRecord(*fork, s)) != cudaSuccess || (e = cudaStreamWaitEvent(a, *fork, 0)) != cudaSuccess)
      return e;
    auto conv = [&](int j) -> cudaError_t {
      const int64_t j0 = (int64_t)j * pl.nc, nc = std::min<int64_t>(pl.nc, op.N - j0);
      cudaError_t r = oz_convert(op.Y, op.ldy, map_shift(op.yn, j0), oz_kmap(op, true), nc, pl.K, t,
                                 w.ey + (j & 1) * pl.nc, n, w.yq + (j & 1) * ybuf, pl.ldq, a);
      if (r == cudaSuccess) r = cudaEventRecord(evc[j], a);
      return r;
    };
    // IBMI_OZ_TRACE=1 (eager calls only): print a per-stream timeline of the pipeline
    static int trace = -1;
    if (trace < 0) trace = getenv("IBMI_OZ_TRACE") ? 1 : 0;
    cudaStreamCaptureStatus capst = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &capst);
    std::vector<std::string> tl;
    static unsigned long long* tbuf = nullptr;
    if (trace && !tbuf) cudaMalloc(&tbuf, 256 * sizeof(unsigned long long));
    auto mark = [&](const std::string& name, cudaStream_t st) {
      if (!trace || capst != cudaStreamCaptureStatusNone || tl.size() >= 256) return;
      oz_stamp_kernel<<<1, 1, 0, st>>>(tbuf + tl.size());
      tl.push_back(name);
    };
    mark("start", s);
    if ((e = conv(0)) != cudaSuccess) return e;
    mark("aux conv0 done", a);
    for (int j = 0; j < pl.nch; ++j) {
      const int64_t j0 = (int64_t)j * pl.nc, nc = std::min<int64_t>(pl.nc, op.N - j0);
      const int b = j & 1;
      if ((e = cudaStreamWaitEvent(s, evc[j], 0)) != cudaSuccess) return e;
      if (j >= 2 && (e = cudaStreamWaitEvent(s, evr[j - 2], 0)) != cudaSuccess) return e;
      mark("main gemm" + std::to_string(j) + " start", s);
      const OzOperand Xo = oz_plain(xp.q, xp.e, pl.ldq, op.M, pl.K);
      const OzOperand Yo = oz_plain(w.yq + b * ybuf, w.ey + b * pl.nc, pl.ldq, nc, pl.K);
      e = oz_igemm(op, n, Xo, Yo, pl.K, j0, nc, w.rq + b * rbuf, sms, s);
      if (e != cudaSuccess || (e = cudaEventRecord(evg[j], s)) != cudaSuccess) return e;
      mark("main gemm" + std::to_string(j) + " done", s);
      if (j + 1 < pl.nch && (e = conv(j + 1)) != cudaSuccess) return e;
      mark("aux conv" + std::to_string(j + 1) + " done", a);
      if ((e = cudaStreamWaitEvent(a, evg[j], 0)) != cudaSuccess) return e;
      mark("aux crt" + std::to_string(j) + " start", a);
      e = oz_crt(op, P, n, Xo, Yo, j0, nc, w.rq + b * rbuf, a);
      if (e != cudaSuccess || (e = cudaEventRecord(evr[j], a)) != cudaSuccess) return e;
      mark("aux crt" + std::to_string(j) + " done", a);
    }
    e = cudaStreamWaitEvent(s, evr[pl.nch - 1], 0);
    if (!tl.empty()) {
      cudaStreamSynchronize(s);
      unsigned long long h[256];
      cudaMemcpy(h, tbuf, tl.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      for (size_t i = 0; i < tl.size(); ++i)
        fprintf(stderr, "[oz] %8.3f ms  %s\n", (double)(h[i] - h[0]) * 1e-6, tl[i].c_str());
    }
    return e;
  }
  for (int64_t j0 = 0; j0 < op.N; j0 += pl.nc) {
    const int64_t nc = std::min<int64_t>(pl.nc, op.N - j0);
    e = oz_convert(op.Y, op.ldy, map_shift(op.yn, j0), oz_kmap(op, true), nc, pl.K, t, w.ey, n, w.yq, pl.ldq, s);
    if (e != cudaSuccess) return e;
    e = oz_chunk(op, P, n, xp.q, xp.e, w.yq, w.ey, pl.K, pl.ldq, j0, nc, w.rq, sms, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Residue planes of a constant operand (W_k, rows of A), kept across sweeps.
struct OzCache {
  int8_t* q = nullptr;
  int* e = nullptr;
  int n = 0;
  size_t bytes = 0;
  void release() {
    if (q) cudaFree(q);
    if (e) cudaFree(e);
    q = nullptr;
    e = nullptr;
    n = 0;
    bytes = 0;
  }
  OzPre pre() const { OzPre p; p.q = q; p.e = e; return p; }
};

// Residue planes of the whole Σ (p x p, one exponent per row), kept in step
// with Σ by the emulated block updates: each step re-converts the set's rows
// and rewrites the set's columns of the other rows (oz_update_cols_kernel);
// a full conversion refreshes every row's exponent at the start of a sweep.
struct OzSigma {
  int8_t* q = nullptr;
  int* e = nullptr;
  int* flags = nullptr;
  int64_t ldq = 0;
  int n = 0, t = 0;
  bool valid = false;
  size_t bytes = 0;
  void release() {
    if (q) cudaFree(q);
    if (e) cudaFree(e);
    if (flags) cudaFree(flags);
    q = nullptr; e = nullptr; flags = nullptr;
    n = 0; valid = false; bytes = 0;
  }
};

// Convert op's X (y = false) or Y (y = true) operand into a cache if the
// device has `margin` bytes to spare afterwards.  Returns false (no cache) otherwise.
bool oz_cache_build(OzCache& cc, const GemmOp& op, bool y, int n, size_t margin, cudaStream_t s, size_t* ctx_bytes) {
  const OzPlan pl = oz_plan(op, n);
  const int64_t rows = y ? op.N : op.M;
  const size_t need = (size_t)n * rows * pl.ldq + (size_t)rows * sizeof(int);
  size_t fr = 0, tot = 0;
  if (mem_info(&fr, &tot) != cudaSuccess || fr < need + margin) { cudaGetLastError(); return false; }
  if (cudaMalloc(&cc.q, (size_t)n * rows * pl.ldq) != cudaSuccess) { cudaGetLastError(); cc.q = nullptr; return false; }
  if (cudaMalloc(&cc.e, (size_t)rows * sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(cc.q);
    cc.q = nullptr;
    cc.e = nullptr;
    return false;
  }
  if (oz_upload_tables() != cudaSuccess) { cc.release(); return false; }
  const int t = oz_bits(n, pl.K);
  cudaError_t e = y ? oz_convert(op.Y, op.ldy, op.yn, oz_kmap(op, true), rows, pl.K, t, cc.e, n, cc.q, pl.ldq, s)
                    : oz_convert(op.X, op.ldx, op.xm, oz_kmap(op, false), rows, pl.K, t, cc.e, n, cc.q, pl.ldq, s);
  if (e != cudaSuccess) { cc.release(); return false; }
  cc.n = n;
  cc.bytes = need;
  *ctx_bytes += need;
  return true;
}

// ------------------------------------------------------ host <-> device staging
// Large host copies go through a pool of pinned slots, several threads at a
// time: each thread copies its row chunks into its own pinned slots (touching
// and, for fresh destinations, faulting pages in parallel) while its stream
// moves the previous chunk over PCIe.
struct PinnedPool {
  std::mutex mu;
  std::vector<void*> slots;
  size_t slot_bytes = 0;
};
PinnedPool g_pool;
constexpr size_t STAGE_SLOT = 16u << 20;   // 16 MiB per slot, 2 slots per thread

// `hrows` (optional): host row of each device row (a row permutation applied
// while the rows pass through the pinned slots; the sharded Σ gather uses it).
int staged_copy(double* dev, int64_t ldd, double* host, int64_t ldh, int64_t rows, int64_t cols, bool to_device,
                int device, cudaStream_t stream, const int64_t* hrows = nullptr) {
  const size_t row_bytes = (size_t)cols * 8;
  const size_t total = row_bytes * (size_t)rows;
  if (row_bytes > STAGE_SLOT && hrows) return fail(IBMI_ERR_INVALID, "staged copy: row too long for a row map");
  if (!hrows && (total < (64u << 20) || row_bytes > STAGE_SLOT)) {
    // async on the caller's stream + sync: a pageable cudaMemcpy may return
    // before its DMA lands, and the context stream does not wait for stream 0
    CUDA_TRY(cudaMemcpy2DAsync(to_device ? (void*)dev : (void*)host, (to_device ? ldd : ldh) * 8,
                               to_device ? (const void*)host : (const void*)dev, (to_device ? ldh : ldd) * 8,
                               row_bytes, rows, to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    return IBMI_OK;
  }
  const int64_t chunk_rows = std::max<int64_t>(1, (int64_t)(STAGE_SLOT / row_bytes));
  const int64_t nchunks = (rows + chunk_rows - 1) / chunk_rows;
  unsigned hc = std::thread::hardware_concurrency();
  static const unsigned cap = [] {
    const char* v = getenv("IBMI_STAGE_THREADS");
    return v ? (unsigned)std::max(1, atoi(v)) : 12u;
  }();
  const int nthreads = (int)std::min<int64_t>(nchunks, std::max(1u, std::min(cap, hc ? hc : 1u)));
  std::lock_guard<std::mutex> lock(g_pool.mu);
  while ((int)g_pool.slots.size() < 2 * nthreads) {
    void* p = nullptr;
    CUDA_TRY(cudaMallocHost(&p, STAGE_SLOT));
    g_pool.slots.push_back(p);
  }
  std::vector<int> rc(nthreads, IBMI_OK);
  std::vector<std::string> msg(nthreads);
  auto work = [&](int t) {
    cudaSetDevice(device);
    cudaStream_t st;
    cudaEvent_t ev[2];
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) { rc[t] = IBMI_ERR_CUDA; return; }
    cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
    bool used[2] = {false, false};
    int64_t pending_r0[2] = {0, 0}, pending_n[2] = {0, 0};
    int s = 0;
    auto drain = [&](int slot) {   // D2H: wait for the slot's copy, move it to the destination
      if (!used[slot]) return;
      cudaEventSynchronize(ev[slot]);
      if (!to_device) {
        const char* src = (const char*)g_pool.slots[2 * t + slot];
        for (int64_t r = 0; r < pending_n[slot]; ++r) {
          const int64_t hr = hrows ? hrows[pending_r0[slot] + r] : pending_r0[slot] + r;
          memcpy(host + hr * ldh, src + r * row_bytes, row_bytes);
        }
      }
      used[slot] = false;
    };
    for (int64_t c = t; c < nchunks; c += nthreads) {
      const int64_t r0 = c * chunk_rows, n = std::min(chunk_rows, rows - r0);
      drain(s);
      char* slot = (char*)g_pool.slots[2 * t + s];
      cudaError_t e;
      if (to_device) {
        for (int64_t r = 0; r < n; ++r)
          memcpy(slot + r * row_bytes, host + (hrows ? hrows[r0 + r] : r0 + r) * ldh, row_bytes);
        e = cudaMemcpy2DAsync(dev + r0 * ldd, ldd * 8, slot, row_bytes, row_bytes, n, cudaMemcpyHostToDevice, st);
      } else {
        e = cudaMemcpy2DAsync(slot, row_bytes, dev + r0 * ldd, ldd * 8, row_bytes, n, cudaMemcpyDeviceToHost, st);
      }
      if (e != cudaSuccess) { rc[t] = IBMI_ERR_CUDA; msg[t] = cudaGetErrorString(e); break; }
      cudaEventRecord(ev[s], st);
      used[s] = true;
      pending_r0[s] = r0;
      pending_n[s] = n;
      s ^= 1;
    }
    drain(s);
    drain(s ^ 1);
    cudaStreamSynchronize(st);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    cudaStreamDestroy(st);
  };
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t) th.emplace_back(work, t);
  for (auto& x : th) x.join();
  for (int t = 0; t < nthreads; ++t)
    if (rc[t]) return fail(rc[t], "staged copy: " + msg[t]);
  return IBMI_OK;
}

// ------------------------------------------------------ IBMI1 files <-> HBM
// IBMI1 (reference matio.py:3-47): 8-byte magic "IBMI1\0\0\0", rows and cols as
// u64 LE, then rows*cols f64 LE row-major.  Rows stream between the file and
// device memory through the pinned slots, several threads doing pread/pwrite.
const char kMagic[8] = {'I', 'B', 'M', 'I', '1', 0, 0, 0};

int staged_file(double* dev, int64_t ldd, int fd, int64_t base, int64_t rows, int64_t cols, bool to_device,
                int device) {
  const size_t row_bytes = (size_t)cols * 8;
  const int64_t chunk_rows = std::max<int64_t>(1, (int64_t)(STAGE_SLOT / std::max<size_t>(row_bytes, 1)));
  if (row_bytes > STAGE_SLOT) return fail(IBMI_ERR_UNSUPPORTED, "row larger than a staging slot");
  const int64_t nchunks = (rows + chunk_rows - 1) / chunk_rows;
  unsigned hc = std::thread::hardware_concurrency();
  const int nthreads = (int)std::max<int64_t>(1, std::min<int64_t>(nchunks, std::max(1u, std::min(8u, hc ? hc : 1u))));
  std::lock_guard<std::mutex> lock(g_pool.mu);
  while ((int)g_pool.slots.size() < 2 * nthreads) {
    void* p = nullptr;
    CUDA_TRY(cudaMallocHost(&p, STAGE_SLOT));
    g_pool.slots.push_back(p);
  }
  std::vector<int> rc(nthreads, IBMI_OK);
  std::vector<std::string> msg(nthreads);
  auto work = [&](int t) {
    cudaSetDevice(device);
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) { rc[t] = IBMI_ERR_CUDA; return; }
    char* slot = (char*)g_pool.slots[2 * t];
    for (int64_t c = t; c < nchunks && rc[t] == IBMI_OK; c += nthreads) {
      const int64_t r0 = c * chunk_rows, n = std::min(chunk_rows, rows - r0);
      const size_t bytes = (size_t)n * row_bytes;
      const off_t off = (off_t)(base + (int64_t)r0 * (int64_t)row_bytes);
      if (to_device) {
        size_t got = 0;
        while (got < bytes) {
          ssize_t k = pread(fd, slot + got, bytes - got, off + (off_t)got);
          if (k <= 0) { rc[t] = IBMI_ERR_IO; msg[t] = "short read"; break; }
          got += (size_t)k;
        }
        if (rc[t]) break;
        if (cudaMemcpy2DAsync(dev + r0 * ldd, ldd * 8, slot, row_bytes, row_bytes, n, cudaMemcpyHostToDevice, st) !=
                cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
          rc[t] = IBMI_ERR_CUDA; msg[t] = "copy"; break;
        }
      } else {
        if (cudaMemcpy2DAsync(slot, row_bytes, dev + r0 * ldd, ldd * 8, row_bytes, n, cudaMemcpyDeviceToHost, st) !=
                cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
          rc[t] = IBMI_ERR_CUDA; msg[t] = "copy"; break;
        }
        size_t put = 0;
        while (put < bytes) {
          ssize_t k = pwrite(fd, slot + put, bytes - put, off + (off_t)put);
          if (k <= 0) { rc[t] = IBMI_ERR_IO; msg[t] = "short write"; break; }
          put += (size_t)k;
        }
      }
    }
    cudaStreamDestroy(st);
  };
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t) th.emplace_back(work, t);
  for (auto& x : th) x.join();
  for (int t = 0; t < nthreads; ++t)
    if (rc[t]) return fail(rc[t], "IBMI1 transfer: " + msg[t]);
  return IBMI_OK;
}

dim3 grid2d(int64_t rows, int64_t cols) {
  const int gx = (int)std::max<int64_t>(1, (cols + 255) / 256);
  const int gy = (int)std::min<int64_t>(std::max<int64_t>(rows, 1), 65535);
  return dim3(gx, gy);
}

// ------------------------------------------------------ blocked SPD inverse
// Scratch for one factorisation of order n.
struct CholScratch {
  double* ws = nullptr; int64_t ldw = 0;      // n × ldw  (matrix, then factor, then L⁻¹)
  double* dinv = nullptr;                      // nblocks × 64 × 64 diagonal-block inverses
  double* tmp = nullptr;                       // n × 64
  int* info = nullptr;
  int cap = 0;
  size_t bytes = 0;
  // potri only (allocated by ensure_potri_scratch): Lᵀ, L⁻ᵀ and the transposed solution, n × ldw each
  double *lt = nullptr, *yt = nullptr, *pt = nullptr;
  int potri_cap = 0;
  void release() {
    if (ws) cudaFree(ws);
    if (dinv) cudaFree(dinv);
    if (tmp) cudaFree(tmp);
    if (info) cudaFree(info);
    if (lt) cudaFree(lt);
    if (yt) cudaFree(yt);
    if (pt) cudaFree(pt);
    ws = dinv = tmp = lt = yt = pt = nullptr; info = nullptr; cap = 0; potri_cap = 0; bytes = 0;
  }
};

int ensure_scratch(CholScratch& cs, int n) {
  if (n <= cs.cap) return IBMI_OK;
  cs.release();
  const int64_t ldw = round_up(n, 32);
  const int nb = (n + CHOL_NB - 1) / CHOL_NB;
  CUDA_TRY(cudaMalloc(&cs.ws, (size_t)n * ldw * sizeof(double)));
  CUDA_TRY(cudaMalloc(&cs.dinv, (size_t)nb * CHOL_NB * CHOL_NB * sizeof(double)));
  CUDA_TRY(cudaMalloc(&cs.tmp, (size_t)n * CHOL_NB * sizeof(double)));
  CUDA_TRY(cudaMalloc(&cs.info, sizeof(int)));
  cs.ldw = ldw;
  cs.cap = n;
  cs.bytes = (size_t)n * ldw * 8 + (size_t)nb * CHOL_NB * CHOL_NB * 8 + (size_t)n * CHOL_NB * 8 + 4;
  return IBMI_OK;
}

// Enqueue the blocked Cholesky of cs.ws on stream s; the first failing pivot
// lands in *info (caller initialises it to INT_MAX).  No host sync.
int potrf_enqueue(CholScratch& cs, int n, cudaStream_t s, int* info);

// Factor the n×n SPD matrix whose LOWER triangle is in cs.ws (upper zero):
// blocked right-looking Cholesky (LAPACK dpotrf lower, linalg.py:104).
// Returns IBMI_ERR_NOT_SPD with *pivot = first failing elimination step.
int potrf_blocked(CholScratch& cs, int n, cudaStream_t s, int64_t* pivot) {
  const int init = INT_MAX;
  CUDA_TRY(cudaMemcpyAsync(cs.info, &init, sizeof(int), cudaMemcpyHostToDevice, s));
  int rc = potrf_enqueue(cs, n, s, cs.info);
  if (rc) return rc;
  int h = INT_MAX;
  CUDA_TRY(cudaMemcpyAsync(&h, cs.info, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (h != INT_MAX) {
    *pivot = h;
    return fail(IBMI_ERR_NOT_SPD, "non-positive pivot at elimination step " + std::to_string(h));
  }
  return IBMI_OK;
}

int potrf_enqueue(CholScratch& cs, int n, cudaStream_t s, int* info) {
  double* a = cs.ws;
  const int64_t ld = cs.ldw;
  for (int j0 = 0, blk = 0; j0 < n; j0 += CHOL_NB, ++blk) {
    const int jb = std::min(CHOL_NB, n - j0);
    const int j1 = j0 + jb;
    double* dblk = cs.dinv + (size_t)blk * CHOL_NB * CHOL_NB;
    potf2_trti2_kernel<<<1, 256, 0, s>>>(a + (int64_t)j0 * ld + j0, ld, jb, dblk, CHOL_NB, info, j0); note_launch();
    CUDA_TRY(cudaGetLastError());
    if (j1 >= n) break;
    // panel: L[j1:, j0:j1] = A[j1:, j0:j1] · L_jj⁻ᵀ   (in place, one N tile)
    GemmOp pn;
    pn.X = a; pn.ldx = ld; pn.xm = contig_map(j1);
    pn.Y = dblk; pn.ldy = CHOL_NB; pn.yn = contig_map(0);
    pn.M = n - j1; pn.N = jb;
    pn.add_seg(j0, 0, jb);
    pn.C = a; pn.ldc = ld; pn.cm = contig_map(j1); pn.cn = contig_map(j0);
    pn.tma_ok = true; pn.xrows = n; pn.xcols = n; pn.yrows = jb; pn.ycols = jb;
    CUDA_TRY(launch_gemm(pn, s));
    // trailing: A[j1:, j1:] -= P Pᵀ  (lower tiles only)
    GemmOp tr;
    tr.X = a; tr.ldx = ld; tr.xm = contig_map(j1);
    tr.Y = a; tr.ldy = ld; tr.yn = contig_map(j1);
    tr.M = n - j1; tr.N = n - j1;
    tr.add_seg(j0, j0, jb);
    tr.C = a; tr.ldc = ld; tr.cm = contig_map(j1); tr.cn = contig_map(j1);
    tr.alpha = -1.0; tr.beta = 1.0; tr.D = a; tr.ldd = ld; tr.dm = contig_map(j1); tr.dn = contig_map(j1);
    tr.lower = true;
    tr.tma_ok = true; tr.xrows = n; tr.xcols = n; tr.yrows = n; tr.ycols = n;
    CUDA_TRY(launch_gemm(tr, s));
  }
  return IBMI_OK;
}

// In-place L -> L⁻¹ (LAPACK dtrtri lower, blocked right-to-left), then
// out = L⁻ᵀ L⁻¹ (lower tiles, mirrored: exactly symmetric, like the
// reference's 0.5(inv + invᵀ), linalg.py:130).
int trtri_blocked(CholScratch& cs, int n, cudaStream_t s) {
  double* a = cs.ws;
  const int64_t ld = cs.ldw;
  const int nblk = (n + CHOL_NB - 1) / CHOL_NB;
  for (int blk = nblk - 1; blk >= 0; --blk) {
    const int j0 = blk * CHOL_NB;
    const int jb = std::min(CHOL_NB, n - j0);
    const int j1 = j0 + jb;
    double* dblk = cs.dinv + (size_t)blk * CHOL_NB * CHOL_NB;
    if (j1 < n) {
      // T = X[j1:, j1:] · L[j1:, j0:j1]
      GemmOp t1;
      t1.X = a; t1.ldx = ld; t1.xm = contig_map(j1);
      t1.Y = a; t1.ldy = ld; t1.yn = contig_map(j0); t1.yt = true;
      t1.M = n - j1; t1.N = jb;
      t1.add_seg(j1, j1, n - j1);
      t1.C = cs.tmp; t1.ldc = CHOL_NB;
      CUDA_TRY(launch_gemm(t1, s));
      // X[j1:, j0:j1] = −T · L_jj⁻¹
      GemmOp t2;
      t2.X = cs.tmp; t2.ldx = CHOL_NB;
      t2.Y = dblk; t2.ldy = CHOL_NB; t2.yt = true;
      t2.M = n - j1; t2.N = jb;
      t2.add_seg(0, 0, jb);
      t2.C = a; t2.ldc = ld; t2.cm = contig_map(j1); t2.cn = contig_map(j0);
      t2.alpha = -1.0;
      CUDA_TRY(launch_gemm(t2, s));
    }
    copy2d_kernel<<<grid2d(jb, jb), 256, 0, s>>>(dblk, CHOL_NB, contig_map(0), contig_map(0),
                                                 a + (int64_t)j0 * ld + j0, ld, jb, jb, 0); note_launch();
    CUDA_TRY(cudaGetLastError());
  }
  return IBMI_OK;
}

int ensure_potri_scratch(CholScratch& cs, int n) {
  if (n <= cs.potri_cap && cs.lt) return IBMI_OK;
  for (double** q : {&cs.lt, &cs.yt, &cs.pt}) {
    if (*q) cudaFree(*q);
    *q = nullptr;
  }
  cs.potri_cap = 0;
  const size_t bytes = (size_t)cs.cap * cs.ldw * sizeof(double);     // same shape as ws
  CUDA_TRY(cudaMalloc(&cs.lt, bytes));
  CUDA_TRY(cudaMalloc(&cs.yt, bytes));
  CUDA_TRY(cudaMalloc(&cs.pt, bytes));
  cs.potri_cap = cs.cap;
  cs.bytes += 3 * bytes;
  return IBMI_OK;
}

// out = A⁻¹ from the Cholesky factor in cs.ws, the way LAPACK's dpotrs(L, I) gets it
// (the reference's spd_inverse, linalg.py:122-130): Y = L⁻¹ (blocked dtrtri), then
// Lᵀ X = Y by blocked BACK SUBSTITUTION against L itself, then ½(X + Xᵀ).
//
// The earlier version formed X = L⁻ᵀ·L⁻¹ as a product of the explicit triangular
// inverse.  Both have the same residual ‖A X − I‖, but the product's errors are not
// backward-stable with respect to L, and the sweep is sensitive to exactly that: at c4
// the error estimate stalled at 9.5e-7 with the product and reaches 2.3e-8 with the
// substitution (reference CPU run: 3.3e-8; profiles/r02_c4_floor_probe*.log).
//
// Block row j (bottom-up), with P = Xᵀ so that every operand is K-contiguous:
//   Vᵀ[n][m] = Yᵀ[n][j0+m] − Σ_{k ≥ j1} P[n][k] · Lᵀ[j0+m][k]        (n × 64, K = n − j1)
//   P[n][j0+m] = Σ_i Vᵀ[n][i] · (L_jj⁻¹)[i][m]                        (n × 64, K = 64)
int potri_blocked(CholScratch& cs, int n, double* out, int64_t ldo, cudaStream_t s) {
  int rc = ensure_potri_scratch(cs, n);
  if (rc) return rc;
  double* a = cs.ws;
  const int64_t ld = cs.ldw;
  const dim3 tb(32, 8), tg((n + 31) / 32, (n + 31) / 32);
  transpose2d_kernel<<<tg, tb, 0, s>>>(a, ld, cs.lt, ld, n); note_launch();     // Lᵀ, before trtri overwrites L
  CUDA_TRY(cudaGetLastError());
  rc = trtri_blocked(cs, n, s);
  if (rc) return rc;
  transpose2d_kernel<<<tg, tb, 0, s>>>(a, ld, cs.yt, ld, n); note_launch();     // Yᵀ = L⁻ᵀ (upper triangular)
  CUDA_TRY(cudaGetLastError());
  const int nblk = (n + CHOL_NB - 1) / CHOL_NB;
  for (int blk = nblk - 1; blk >= 0; --blk) {
    const int j0 = blk * CHOL_NB;
    const int jb = std::min(CHOL_NB, n - j0);
    const int j1 = j0 + jb;
    double* dblk = cs.dinv + (size_t)blk * CHOL_NB * CHOL_NB;
    if (j1 < n) {
      GemmOp g;
      g.X = cs.pt; g.ldx = ld;
      g.Y = cs.lt; g.ldy = ld; g.yn = contig_map(j0);
      g.M = n; g.N = jb;
      g.add_seg(j1, j1, n - j1);
      g.C = cs.tmp; g.ldc = CHOL_NB;
      g.alpha = -1.0; g.beta = 1.0; g.D = cs.yt; g.ldd = ld; g.dn = contig_map(j0);
      g.tma_ok = true; g.xrows = n; g.xcols = n; g.yrows = n; g.ycols = n;
      CUDA_TRY(launch_gemm(g, s));
    } else {
      copy2d_kernel<<<grid2d(n, jb), 256, 0, s>>>(cs.yt, ld, contig_map(0), contig_map(j0), cs.tmp, CHOL_NB, n, jb, 0);
      note_launch();
      CUDA_TRY(cudaGetLastError());
    }
    GemmOp h;
    h.X = cs.tmp; h.ldx = CHOL_NB;
    h.Y = dblk; h.ldy = CHOL_NB; h.yt = true;
    h.M = n; h.N = jb;
    h.add_seg(0, 0, jb);
    h.C = cs.pt; h.ldc = ld; h.cn = contig_map(j0);
    CUDA_TRY(launch_gemm(h, s));
  }
  sym_avg_kernel<<<tg, tb, 0, s>>>(cs.pt, ld, out, ldo, n); note_launch();
  CUDA_TRY(cudaGetLastError());
  return IBMI_OK;
}



// Monte Carlo guess (solver.py:167-181): A = L Lᵀ (blocked Cholesky), Z = L⁻ᵀ w,
// out[orow(m)][ocol(n)] = (1/n) Σ_s Z[cmap(m)][s] Z[cmap(n)][s] for m, n < c0.
int mc_guess_into(const double* A, int64_t lda, int64_t p, const double* w_src, int on_device, int64_t n,
                  RowMap cmap, int64_t c0, double* out, int64_t ldo, RowMap orow, RowMap ocol, cudaStream_t st) {
  CholScratch cs;
  int rc = ensure_scratch(cs, (int)p);
  if (rc) { cs.release(); return rc; }
  double *w = nullptr, *z = nullptr;
  cudaError_t e = cudaMalloc(&w, (size_t)p * n * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&z, (size_t)p * n * sizeof(double));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(w, w_src, (size_t)p * n * sizeof(double),
                        on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) { cs.release(); cudaFree(w); cudaFree(z); return fail(IBMI_ERR_OOM, cudaGetErrorString(e)); }
  copy2d_kernel<<<grid2d(p, p), 256, 0, st>>>(A, lda, contig_map(0), contig_map(0), cs.ws, cs.ldw, (int)p, (int)p, 1); note_launch();
  int64_t piv = -1;
  rc = potrf_blocked(cs, (int)p, st, &piv);
  if (!rc) rc = trtri_blocked(cs, (int)p, st);
  if (!rc) {
    GemmOp gz;   // Z[i][s] = Σ_k L⁻¹[k][i] w[k][s]   (both operands transposed)
    gz.X = cs.ws; gz.ldx = cs.ldw; gz.xt = true;
    gz.Y = w; gz.ldy = n; gz.yt = true;
    gz.M = p; gz.N = n;
    gz.add_seg(0, 0, p);
    gz.C = z; gz.ldc = n;
    e = launch_gemm(gz, st);
    GemmOp gg;   // out = Z_c Z_cᵀ / n  (lower tiles, mirrored)
    gg.X = z; gg.ldx = n; gg.xm = cmap;
    gg.Y = z; gg.ldy = n; gg.yn = cmap;
    gg.M = c0; gg.N = c0;
    gg.add_seg(0, 0, n);
    gg.C = out; gg.ldc = ldo; gg.cm = orow; gg.cn = ocol;
    gg.alpha = 1.0 / (double)n;
    gg.lower = true; gg.mirror = true;
    if (e == cudaSuccess) e = launch_gemm(gg, st);
    if (e != cudaSuccess) rc = fail(IBMI_ERR_CUDA, cudaGetErrorString(e));
  }
  cudaStreamSynchronize(st);
  cs.release();
  cudaFree(w);
  cudaFree(z);
  return rc;
}

}  // namespace

// ------------------------------------------------------------------ context
struct SetDev {
  int64_t lo = 0, hi = 0;
  int b = 0;
  bool general = false;          // non-contiguous set: index lists below
  int64_t* idx = nullptr;        // device, b entries (ascending)
  int64_t* comp = nullptr;       // device, p - b entries (ascending complement)
  RowMap rows() const { return general ? list_map(idx) : contig_map(lo); }
  RowMap cmap() const { return general ? list_map(comp) : complement_map(lo, hi); }
  double* W = nullptr;      // b × ld
  double* ainv = nullptr;   // b × ldb
  int64_t ldb = 0;
  bool ready = false;
};

struct ibmi_ctx {
  int device = 0;
  int64_t p = 0, ld = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool counted = false;      // included in g_live_ctx[device]
  double* A = nullptr;
  double* S = nullptr;
  bool a_set = false;
  std::vector<SetDev> sets;
  CholScratch cs;
  // estimate buffers
  double* Bm = nullptr; int64_t ldB = 0; int64_t B_cap = 0;
  double* Gm = nullptr; int64_t ldG = 0; int64_t G_cap = 0;
  double* vec = nullptr; int64_t vec_cap = 0;
  double* part = nullptr; int part_cap = 0;
  double* vr = nullptr; int64_t vr_n = 0;
  double* frob_part = nullptr; int frob_cap = 0;
  double* splitws = nullptr; int64_t splitws_cap = 0;   // split-K partial tiles
  OzWork oz;                      // Ozaki-II planes / residues (oz_n > 0)
  int oz_n = 0;                   // 0: FP64 DMMA GEMMs; 8..20: Ozaki-II with oz_n moduli
  std::vector<OzCache> oz_w;      // per set: residue planes of W_k (K = complement)
  OzCache oz_a;                   // residue planes of A[c_K, :] (error estimate of the last set)
  int oz_a_set = -1;
  OzStreams ozs;                  // aux stream + events of the chunk pipeline
  OzSigma oz_s;                   // residue planes of Σ (incremental block updates)
  int graph_gen = -1;
  long long graph_launches = 0;   // kernel nodes in the captured sweep
  double* dscal = nullptr;        // [0..2] power out, [3..4] frob, [8..9] symcheck (u64)
  double* hpin = nullptr;         // pinned mirror of dscal
  int sms = 148;
  int power_blocks = 148;
  int power_threads = 512;
  size_t power_smem_cap = 200 * 1024;
  cudaGraphExec_t graph = nullptr;
  bool graph_tried = false, graph_ok = false;
  double graph_rtol = -1.0;
  int graph_max = -1;
  size_t bytes = 0;
};

namespace {

int ensure_buf(double** p, int64_t* cap, int64_t need, size_t* bytes) {
  if (need <= *cap) return IBMI_OK;
  if (*p) { cudaFree(*p); *bytes -= (size_t)(*cap) * 8; }
  *p = nullptr;
  *cap = 0;
  CUDA_TRY(cudaMalloc(p, (size_t)need * sizeof(double)));
  *cap = need;
  *bytes += (size_t)need * 8;
  return IBMI_OK;
}

void oz_drop_caches(ibmi_ctx* c) {
  for (auto& w : c->oz_w) {
    c->bytes -= w.bytes;
    w.release();
  }
  c->oz_w.clear();
  c->bytes -= c->oz_a.bytes;
  c->oz_a.release();
  c->oz_a_set = -1;
  c->bytes -= c->oz_s.bytes;
  c->oz_s.release();
}

void invalidate_graph(ibmi_ctx* c) {
  if (c->graph) cudaGraphExecDestroy(c->graph);
  c->graph = nullptr;
  c->graph_tried = false;
  c->graph_ok = false;
}

int symcheck(ibmi_ctx* c, RowMap map, int64_t n, const char* what) {
  unsigned long long* d = reinterpret_cast<unsigned long long*>(c->dscal + 8);
  CUDA_TRY(cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), c->stream));
  const int nt = (int)((n + 31) / 32);
  symcheck_kernel<<<dim3(nt, nt), dim3(32, 8), 0, c->stream>>>(c->A, c->ld, map, (int)n, d); note_launch();
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(c->hpin + 8, c->dscal + 8, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const double mabs = c->hpin[8], skew = c->hpin[9];
  if (mabs == 0.0) return IBMI_OK;
  if (!(skew <= 1e-12 * mabs)) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%s is not symmetric: max |a - a.T| = %.3e exceeds 1.0e-12 * max|a| = %.3e", what,
             skew, 1e-12 * mabs);
    return fail(IBMI_ERR_NOT_SYMMETRIC, buf);
  }
  return IBMI_OK;
}

// Split-K factor and workspace (doubles) for a GEMM on this context.
int plan_split(const ibmi_ctx* c, const GemmOp& op, int forced, int64_t* ws_need) {
  const int tiles = gemm_tiles(op);
  int64_t klen = 0;
  for (int i = 0; i < op.nseg; ++i) klen += op.seg[i].len;
  const int bk = g_variant == 2 ? 32 : 16;
  const int s = forced > 0 ? forced : auto_split(tiles, (int)((klen + bk - 1) / bk), c->sms);
  if (ws_need) *ws_need = s > 1 ? split_ws_doubles(tiles, s) : 0;
  return s;
}

// ---- one block update: the hot path (solver.py:122-129)
// `mid` (optional) is recorded between the two GEMMs (for ibmi_sweep_timed).
// Contiguous sets whose start is a multiple of 128 (no TMA box of the
// planes straddles the set) and whose end is 16-byte aligned.
bool oz_global_set_ok(const SetDev& s) { return !s.general && s.lo % 128 == 0 && s.hi % 16 == 0; }

// Emulated block update on the residue planes of Σ (OzSigma): no per-step
// conversion of Σ[c, c]; see OzSigma.
int enqueue_block_update_ozg(ibmi_ctx* c, int k, cudaEvent_t mid) {
  const SetDev& s = c->sets[k];
  OzSigma& G = c->oz_s;
  const OzCache& W = c->oz_w[k];
  const int n = c->oz_n;
  const int64_t p = c->p, lo = s.lo, hi = s.hi, b = s.b, cc = p - b;
  const int64_t qplane = p * G.ldq;
  cudaStream_t st = c->stream;
  CUDA_TRY(oz_upload_tables());
  if (k == 0 || !G.valid) {
    CUDA_TRY(oz_convert(c->S, c->ld, contig_map(0), contig_map(0), p, p, G.t, G.e, n, G.q, G.ldq, st, qplane));
    G.valid = true;
  }
  const int64_t ldw = round_up(cc, 16);
  // K1: Σ[I, c] = −W Σ[c, c] (mirrored), Y = the planes' rows c over columns c
  GemmOp k1;
  k1.M = b; k1.N = cc;
  k1.C = c->S; k1.ldc = c->ld; k1.cm = contig_map(lo); k1.cn = complement_map(lo, hi);
  k1.alpha = -1.0; k1.mirror = true;
  const OzOperand X1 = oz_plain(W.q, W.e, ldw, b, cc);
  OzOperand Y1;
  Y1.q = G.q; Y1.e = G.e; Y1.emap = complement_map(lo, hi);
  Y1.ldq = G.ldq; Y1.rows = p; Y1.cols = p;
  Y1.split = (int)lo; Y1.off1 = (int)hi; Y1.ksplit = (int)lo; Y1.koff1 = (int)hi;
  CUDA_TRY(oz_igemm(k1, n, X1, Y1, cc, 0, cc, c->oz.rq, c->sms, st));
  CUDA_TRY(oz_crt(k1, oz_epilogue(k1), n, X1, Y1, 0, cc, c->oz.rq, st));
  if (mid) CUDA_TRY(cudaEventRecord(mid, st));
  // the set's rows of the planes (fresh exponents; their own columns follow K2)
  CUDA_TRY(oz_convert(c->S, c->ld, contig_map(lo), contig_map(0), b, p, G.t, G.e + lo, n, G.q + lo * G.ldq, G.ldq,
                      st, qplane));
  // K2: Σ[I, I] = A_II⁻¹ − Σ[I, c] Wᵀ, X = the planes' rows I over columns c
  GemmOp k2;
  k2.M = b; k2.N = b;
  k2.C = c->S; k2.ldc = c->ld; k2.cm = contig_map(lo); k2.cn = contig_map(lo);
  k2.alpha = -1.0; k2.beta = 1.0; k2.D = s.ainv; k2.ldd = s.ldb;
  k2.lower = true; k2.mirror = true;
  OzOperand X2;
  X2.q = G.q; X2.e = G.e + lo;
  X2.ldq = G.ldq; X2.rows = p; X2.cols = p;
  X2.row_off = (int)lo; X2.ksplit = (int)lo; X2.koff1 = (int)hi;
  const OzOperand Y2 = oz_plain(W.q, W.e, ldw, b, cc);
  CUDA_TRY(oz_igemm(k2, n, X2, Y2, cc, 0, b, c->oz.rq, c->sms, st));
  CUDA_TRY(oz_crt(k2, oz_epilogue(k2), n, X2, Y2, 0, b, c->oz.rq, st));
  // the set's columns in every row, then full re-conversion of rows whose
  // exponent no longer covers them
  const int64_t items = p * ((b + 7) / 8);
  dim3 ug((unsigned)std::min<int64_t>((items + 255) / 256, 32LL * c->sms));
  OZ_DISPATCH(n, oz_update_cols_launch, ug, st, c->S, c->ld, (int)p, lo, (int)b, G.e, G.t, G.q, G.ldq, qplane,
              G.flags);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  dim3 fg((unsigned)std::min<int64_t>(p, 4LL * c->sms));
  OZ_DISPATCH(n, oz_fix_rows_launch, fg, st, c->S, c->ld, (int)p, (int)p, G.e, G.t, G.q, G.ldq, qplane, G.flags);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return IBMI_OK;
}

bool ozg_ready(const ibmi_ctx* c, int k) {
  return c->oz_n > 0 && c->oz_s.q && c->oz_s.n == c->oz_n && k < (int)c->oz_w.size() && c->oz_w[k].q &&
         c->oz_w[k].n == c->oz_n && oz_global_set_ok(c->sets[k]) &&
         (int64_t)c->oz_n * c->sets[k].b * round_up(c->p - c->sets[k].b, 16) <= c->oz.rq_cap;
}

int enqueue_block_update(ibmi_ctx* c, int k, cudaEvent_t mid = nullptr) {
  NvtxRange nvtx_("block_update");
  if (ozg_ready(c, k)) return enqueue_block_update_ozg(c, k, mid);
  c->oz_s.valid = false;             // Σ changes outside the planes' bookkeeping
  const SetDev& s = c->sets[k];
  const int64_t p = c->p, lo = s.lo, hi = s.hi, b = s.b, cc = p - b;
  if (s.general) {
    // K loop over all p columns: W is exactly zero on I, so the extra b
    // columns contribute nothing (p/c more flops, no gather of Σ_cc).
    GemmOp k1;
    k1.X = s.W; k1.ldx = c->ld;
    k1.Y = c->S; k1.ldy = c->ld; k1.yn = s.cmap();
    k1.M = b; k1.N = cc;
    k1.add_seg(0, 0, p);
    k1.C = c->S; k1.ldc = c->ld; k1.cm = s.rows(); k1.cn = s.cmap();
    k1.alpha = -1.0; k1.mirror = true;
    {
      int64_t need = 0;
      k1.splits = plan_split(c, k1, g_split_panel, &need);
      if (need > c->splitws_cap) k1.splits = 1;
      k1.ws = c->splitws;
    }
    CUDA_TRY(launch_gemm(k1, c->stream));
    if (mid) CUDA_TRY(cudaEventRecord(mid, c->stream));
    GemmOp k2;
    k2.X = c->S; k2.ldx = c->ld; k2.xm = s.rows();
    k2.Y = s.W; k2.ldy = c->ld;
    k2.M = b; k2.N = b;
    k2.add_seg(0, 0, p);
    k2.C = c->S; k2.ldc = c->ld; k2.cm = s.rows(); k2.cn = s.rows();
    k2.alpha = -1.0; k2.beta = 1.0; k2.D = s.ainv; k2.ldd = s.ldb;
    k2.lower = true; k2.mirror = true;
    int64_t need = 0;
    k2.splits = plan_split(c, k2, g_split_diag, &need);
    if (need > c->splitws_cap) k2.splits = 1;
    k2.ws = c->splitws;
    CUDA_TRY(launch_gemm(k2, c->stream));
    return IBMI_OK;
  }
  // K1: Σ[I, c] = −W Σ[c, c];  Σ[c, I] = its transpose (mirror store)
  GemmOp k1;
  k1.X = s.W; k1.ldx = c->ld; k1.xm = contig_map(0);
  k1.Y = c->S; k1.ldy = c->ld; k1.yn = complement_map(lo, hi);
  k1.M = b; k1.N = cc;
  k1.add_seg(0, 0, lo);
  k1.add_seg(hi, hi, p - hi);
  k1.C = c->S; k1.ldc = c->ld; k1.cm = contig_map(lo); k1.cn = complement_map(lo, hi);
  k1.alpha = -1.0; k1.mirror = true;
  k1.tma_ok = true; k1.xrows = b; k1.xcols = p; k1.yrows = p; k1.ycols = p;
  const bool wcache = c->oz_n > 0 && k < (int)c->oz_w.size() && c->oz_w[k].q && c->oz_w[k].n == c->oz_n;
  if (c->oz_n > 0) {
    CUDA_TRY(oz_gemm(k1, c->oz, c->oz_n, c->sms, c->stream, wcache ? c->oz_w[k].pre() : OzPre(), OzPre(), false,
                     &c->ozs));
  } else {
    int64_t need = 0;
    k1.splits = plan_split(c, k1, g_split_panel, &need);
    if (need > c->splitws_cap) k1.splits = 1;
    k1.ws = c->splitws;
    CUDA_TRY(launch_gemm(k1, c->stream));
  }
  if (mid) CUDA_TRY(cudaEventRecord(mid, c->stream));
  // K2: Σ[I, I] = A_II⁻¹ − Σ[I, c] W_cᵀ   (= ainv + M Wᵀ), lower tiles mirrored
  GemmOp k2;
  k2.X = c->S; k2.ldx = c->ld; k2.xm = contig_map(lo);
  k2.Y = s.W; k2.ldy = c->ld; k2.yn = contig_map(0);
  k2.M = b; k2.N = b;
  k2.add_seg(0, 0, lo);
  k2.add_seg(hi, hi, p - hi);
  k2.C = c->S; k2.ldc = c->ld; k2.cm = contig_map(lo); k2.cn = contig_map(lo);
  k2.alpha = -1.0; k2.beta = 1.0; k2.D = s.ainv; k2.ldd = s.ldb;
  k2.lower = true; k2.mirror = true;
  k2.tma_ok = true; k2.xrows = p; k2.xcols = p; k2.yrows = b; k2.ycols = p;
  if (c->oz_n > 0) {   // W's residue planes (cache, or K1's X buffers) are K2's Y
    if (wcache) {
      CUDA_TRY(oz_gemm(k2, c->oz, c->oz_n, c->sms, c->stream, OzPre(), c->oz_w[k].pre()));
    } else {
      OzPre wp;
      wp.q = c->oz.xq;
      wp.e = c->oz.ex;
      CUDA_TRY(oz_gemm(k2, c->oz, c->oz_n, c->sms, c->stream, OzPre(), wp, /*x_in_ybuf=*/true));
    }
    return IBMI_OK;
  }
  int64_t need = 0;
  k2.splits = plan_split(c, k2, g_split_diag, &need);
  if (need > c->splitws_cap) k2.splits = 1;    // workspace is planned by plan_workspace()
  k2.ws = c->splitws;
  CUDA_TRY(launch_gemm(k2, c->stream));
  return IBMI_OK;
}

int ensure_estimate_buffers(ibmi_ctx* c, int64_t b, int64_t cc) {
  const int64_t ldB = round_up(std::max<int64_t>(cc, 1), 32);
  if (ensure_buf(&c->Bm, &c->B_cap, b * ldB, &c->bytes)) return IBMI_ERR_OOM;
  c->ldB = ldB;
  const int64_t n = std::min(b, cc);
  const int64_t ldG = round_up(n, 32);
  if (ensure_buf(&c->Gm, &c->G_cap, n * ldG, &c->bytes)) return IBMI_ERR_OOM;
  c->ldG = ldG;
  if (ensure_buf(&c->vec, &c->vec_cap, 2 * std::max(b, cc), &c->bytes)) return IBMI_ERR_OOM;
  int64_t pc = c->part_cap;
  if (ensure_buf(&c->part, &pc, (4 + 32) * (int64_t)c->power_blocks, &c->bytes)) return IBMI_ERR_OOM;  // + LL lines
  c->part_cap = (int)pc;
  return IBMI_OK;
}

// Allocate the split-K workspace for every split GEMM of a sweep (before any
// graph capture: nothing is allocated while capturing).
int plan_workspace(ibmi_ctx* c) {
  int64_t need = 0;
  for (const SetDev& s : c->sets) {
    GemmOp k1;
    k1.M = s.b; k1.N = c->p - s.b;
    if (s.general) {
      k1.add_seg(0, 0, c->p);
    } else {
      k1.add_seg(0, 0, s.lo);
      k1.add_seg(s.hi, s.hi, c->p - s.hi);
    }
    int64_t w1 = 0;
    plan_split(c, k1, g_split_panel, &w1);
    need = std::max(need, w1);
    GemmOp k2;
    k2.M = s.b; k2.N = s.b; k2.lower = true;
    if (s.general) {
      k2.add_seg(0, 0, c->p);
    } else {
      k2.add_seg(0, 0, s.lo);
      k2.add_seg(s.hi, s.hi, c->p - s.hi);
    }
    int64_t w = 0;
    plan_split(c, k2, g_split_diag, &w);
    need = std::max(need, w);
  }
  if (!c->sets.empty()) {
    const SetDev& s = c->sets.back();
    const int64_t cc = c->p - s.b;
    GemmOp gb;
    gb.M = s.b; gb.N = cc;
    gb.add_seg(0, 0, c->p);
    int64_t wb = 0;
    plan_split(c, gb, g_split_panel, &wb);
    need = std::max(need, wb);
    if (s.b <= cc) {
      GemmOp gg;
      gg.M = s.b; gg.N = s.b; gg.lower = true;
      gg.add_seg(0, 0, cc);
      int64_t w = 0;
      plan_split(c, gg, g_split_gram, &w);
      need = std::max(need, w);
    }
  }
  if (need > c->splitws_cap) {
    if (ensure_buf(&c->splitws, &c->splitws_cap, need, &c->bytes)) return IBMI_ERR_OOM;
  }
  if (c->oz_n > 0) {
    const int n = c->oz_n;
    if (!c->ozs.init()) return fail(IBMI_ERR_CUDA, "cannot create the emulation pipeline stream");
    OzPlan tot;
    for (const SetDev& s : c->sets) {
      if (s.general) continue;
      GemmOp k1;
      k1.M = s.b; k1.N = c->p - s.b;
      k1.add_seg(0, 0, s.lo);
      k1.add_seg(s.hi, s.hi, c->p - s.hi);
      const OzPlan pl = oz_plan(k1, n);
      tot.xq = std::max(tot.xq, pl.xq); tot.yq = std::max(tot.yq, pl.yq); tot.rq = std::max(tot.rq, pl.rq);
      tot.ex = std::max(tot.ex, pl.ex); tot.ey = std::max(tot.ey, pl.ey);
      // K2 (y_pre): X = Σ[I, c] into the Y buffers, residues b × b
      tot.yq = std::max(tot.yq, n * s.b * pl.ldq);
      tot.ey = std::max(tot.ey, (int64_t)s.b);
      tot.rq = std::max(tot.rq, n * s.b * round_up(s.b, 16));
    }
    if (!c->sets.empty() && !c->sets.back().general) {
      const SetDev& s = c->sets.back();
      GemmOp gb;
      gb.M = s.b; gb.N = c->p - s.b;
      gb.add_seg(0, 0, c->p);
      const OzPlan pl = oz_plan(gb, n);
      tot.xq = std::max(tot.xq, pl.xq); tot.yq = std::max(tot.yq, pl.yq); tot.rq = std::max(tot.rq, pl.rq);
      tot.ex = std::max(tot.ex, pl.ex); tot.ey = std::max(tot.ey, pl.ey);
    }
    int rc = oz_reserve(c->oz, tot, &c->bytes);
    if (rc) return rc;
    // constant operands: W_k (all sets) and A[c_K, :] keep their planes when
    // the device has room (margin 4 GB); otherwise they are converted per use
    if (c->oz_w.size() != c->sets.size()) {
      for (auto& w : c->oz_w) w.release();
      c->oz_w.assign(c->sets.size(), OzCache());
    }
    const size_t margin = (size_t)4 << 30;
    for (size_t k = 0; k < c->sets.size(); ++k) {
      const SetDev& s = c->sets[k];
      OzCache& wc = c->oz_w[k];
      if (s.general || !s.ready || (wc.q && wc.n == n)) continue;
      c->bytes -= wc.bytes;
      wc.release();
      GemmOp k1;
      k1.X = s.W; k1.ldx = c->ld; k1.xm = contig_map(0);
      k1.M = s.b; k1.N = c->p - s.b;
      k1.add_seg(0, 0, s.lo);
      k1.add_seg(s.hi, s.hi, c->p - s.hi);
      if (!oz_cache_build(wc, k1, false, n, margin, c->stream, &c->bytes)) break;
    }
    const int last = (int)c->sets.size() - 1;
    if (last >= 0 && !c->sets[last].general && !(c->oz_a.q && c->oz_a.n == n && c->oz_a_set == last)) {
      c->bytes -= c->oz_a.bytes;
      c->oz_a.release();
      c->oz_a_set = -1;
      const SetDev& s = c->sets[last];
      GemmOp gb;
      gb.Y = c->A; gb.ldy = c->ld; gb.yn = s.cmap();
      gb.M = s.b; gb.N = c->p - s.b;
      gb.add_seg(0, 0, c->p);
      if (oz_cache_build(c->oz_a, gb, true, n, margin, c->stream, &c->bytes)) c->oz_a_set = last;
    }
    // residue planes of Σ for the incremental block updates (all sets eligible,
    // W planes cached, room for n·p² bytes)
    bool all_ok = c->p <= 65535;
    for (size_t k = 0; k < c->sets.size(); ++k)
      all_ok = all_ok && oz_global_set_ok(c->sets[k]) && k < c->oz_w.size() && c->oz_w[k].q;
    if (all_ok && !(c->oz_s.q && c->oz_s.n == n)) {
      c->bytes -= c->oz_s.bytes;
      c->oz_s.release();
      const int64_t ldq = round_up(c->p, 16);
      const size_t need = (size_t)n * c->p * ldq + 2 * (size_t)c->p * sizeof(int);
      size_t fr = 0, tot_mem = 0;
      if (mem_info(&fr, &tot_mem) == cudaSuccess && fr >= need + margin &&
          cudaMalloc(&c->oz_s.q, (size_t)n * c->p * ldq) == cudaSuccess &&
          cudaMalloc(&c->oz_s.e, (size_t)c->p * sizeof(int)) == cudaSuccess &&
          cudaMalloc(&c->oz_s.flags, (size_t)c->p * sizeof(int)) == cudaSuccess &&
          cudaMemset(c->oz_s.flags, 0, (size_t)c->p * sizeof(int)) == cudaSuccess) {
        c->oz_s.ldq = ldq;
        c->oz_s.n = n;
        c->oz_s.t = oz_bits(n, c->p);     // valid for every GEMM of the solve (K <= p)
        c->oz_s.valid = false;
        c->oz_s.bytes = need;
        c->bytes += need;
      } else {
        cudaGetLastError();
        c->oz_s.release();
      }
    }
    if (c->oz_s.q) {   // K1 of the planes path runs as one N chunk: residues b × c
      OzPlan more;
      for (const SetDev& s : c->sets) more.rq = std::max(more.rq, n * s.b * round_up(c->p - s.b, 16));
      rc = oz_reserve(c->oz, more, &c->bytes);
      if (rc) return rc;
    }
    if (c->oz_a.q) {   // the cached estimate runs as one N chunk: residues b × c
      const SetDev& s = c->sets[last];
      OzPlan more;
      more.rq = n * s.b * round_up(c->p - s.b, 16);
      rc = oz_reserve(c->oz, more, &c->bytes);
      if (rc) return rc;
    }
  }
  return IBMI_OK;
}

// ---- ‖B‖₂ of a device matrix by the Gram-form power iteration
// (linalg.py:223-274).  Buffers: G (n×ldG, n = min(rows, cols)), vec (2·max),
// part (4·blocks), out (3 doubles), vr (cols, normalised restart vector).
struct NormBufs {
  double* G; int64_t ldG;
  double* vec;
  double* part;
  double* out;
  const double* vr;
  int blocks, threads;
  size_t smem_cap;
  double* ws;           // split-K workspace for the Gram GEMM (may be null)
  int64_t ws_cap;
  int sms;
  OzWork* oz = nullptr;  // Ozaki-II emulation of the Gram GEMM (context with emulation on)
  int oz_n = 0;
};

// Flag-exchange power iteration (power_gram_ll_kernel) when the Gram matrix fits its
// shape: even n, ≤ 15 rows per CTA, ≤ 3072 columns, rows resident in registers + shared
// memory.  Returns false when not applicable (the grid-barrier kernel runs instead).
template <int RR, int Q>
bool power_ll_inst(PowerParams& P, const NormBufs& nb, int grid, int rpc, size_t smem, cudaStream_t st) {
  static bool attr[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    if (cudaFuncSetAttribute(power_gram_ll_kernel<RR, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024) !=
        cudaSuccess) { cudaGetLastError(); return false; }
    attr[dev & 63] = true;
  }
  double* msg = nb.part + 4 * (size_t)nb.blocks;
  if (cudaMemsetAsync(msg, 0, (size_t)32 * nb.blocks * sizeof(double), st) != cudaSuccess) { cudaGetLastError(); return false; }
  void* args[] = {&P, &msg, &rpc};
  if (cudaLaunchCooperativeKernel((const void*)power_gram_ll_kernel<RR, Q>, dim3(grid), dim3(512), args, smem, st) !=
      cudaSuccess) { cudaGetLastError(); return false; }
  note_launch();
  return true;
}

bool power_ll_launch(PowerParams& P, const NormBufs& nb, cudaStream_t st) {
  const int n = P.n;
  if (n < 512 || (n & 1) || n > 3072 || (P.ldg & 1) || !aligned16(P.G) || nb.threads != 512) return false;
  const int rpc = (n + nb.blocks - 1) / nb.blocks;
  if (rpc > LL_ROWS) return false;
  const int grid = (n + rpc - 1) / rpc;
  if (grid > 192) return false;                  // the kernel polls at most 3 rounds of 64 lines
  const int q = (n / 2 + 511) / 512;
  const int rr = q == 1 ? 8 : (q == 2 ? 6 : 4);
  const size_t smem = ((size_t)((grid * rpc + 1) & ~1) + 256 + 64 + (size_t)std::max(0, rpc - rr) * n) * sizeof(double);
  if (smem > 220 * 1024) return false;
  if (q == 1) return power_ll_inst<8, 1>(P, nb, grid, rpc, smem, st);
  if (q == 2) return power_ll_inst<6, 2>(P, nb, grid, rpc, smem, st);
  return power_ll_inst<4, 3>(P, nb, grid, rpc, smem, st);
}

int enqueue_two_norm(const double* Bm, int64_t ldB, int64_t b, int64_t cc, double rtol, int max_iters,
                     const NormBufs& nb, cudaStream_t st, cudaEvent_t ev_gram = nullptr, bool have_gram = false) {
  const int mode = (b <= cc) ? 0 : 1;
  const int64_t n = mode == 0 ? b : cc;
  if (have_gram && mode != 0) return fail(IBMI_ERR_INVALID, "precomputed Gram matrix needs the row form");
  GemmOp gg;
  if (mode == 0) {   // G = B Bᵀ
    gg.X = Bm; gg.ldx = ldB;
    gg.Y = Bm; gg.ldy = ldB;
    gg.add_seg(0, 0, cc);
    gg.tma_ok = true; gg.xrows = b; gg.xcols = cc; gg.yrows = b; gg.ycols = cc;
  } else {           // H = Bᵀ B
    gg.X = Bm; gg.ldx = ldB; gg.xt = true;
    gg.Y = Bm; gg.ldy = ldB; gg.yt = true;
    gg.add_seg(0, 0, b);
  }
  gg.M = n; gg.N = n;
  gg.C = nb.G; gg.ldc = nb.ldG;
  gg.lower = true; gg.mirror = true;
  // emulated Gram product (context in emulation mode, workspace large enough)
  const bool emu = mode == 0 && nb.oz && nb.oz_n > 0 && n <= 65535 && n <= nb.oz->ex_cap &&
                   (int64_t)nb.oz_n * n * round_up(n, 16) <= nb.oz->rq_cap &&
                   (int64_t)nb.oz_n * n * round_up(cc, 16) <= nb.oz->xq_cap;
  if (have_gram) {
    // G and y₁ were written by the fused small-problem sweep kernel
  } else if (emu) {
    // G = B Bᵀ: X and Y are the same rows, one conversion serves both
    OzPre same;
    same.q = nb.oz->xq;
    same.e = nb.oz->ex;
    CUDA_TRY(oz_gemm(gg, *nb.oz, nb.oz_n, nb.sms, st, OzPre(), same));
  } else {
    if (nb.ws && mode == 0) {
      const int bk = g_variant == 2 ? 32 : 16;
      gg.splits = g_split_gram > 0 ? g_split_gram : auto_split(gemm_tiles(gg), (int)((cc + bk - 1) / bk), nb.sms);
      if (split_ws_doubles(gemm_tiles(gg), gg.splits) > nb.ws_cap) gg.splits = 1;
      gg.ws = nb.ws;
    }
    CUDA_TRY(launch_gemm(gg, st));
  }
  if (mode == 0 && !have_gram) {
    const int threads = 256;
    const int blocks = (int)((b * 32 + threads - 1) / threads);
    rowsum_scaled_kernel<<<blocks, threads, 0, st>>>(Bm, ldB, (int)b, (int)cc, 1.0 / std::sqrt((double)cc), nb.vec); note_launch();
    CUDA_TRY(cudaGetLastError());
  }
  if (ev_gram) CUDA_TRY(cudaEventRecord(ev_gram, st));
  PowerParams P;
  P.G = nb.G; P.ldg = nb.ldG; P.n = (int)n;
  P.B = Bm; P.ldb = ldB; P.brows = (int)b; P.bcols = (int)cc;
  P.vr = nb.vr;
  P.vec = nb.vec;
  P.part = nb.part;
  P.rtol = rtol;
  P.max_iters = max_iters;
  P.mode = mode;
  P.out = nb.out;
  P.smem_cap = (int)(nb.smem_cap / sizeof(double));
  if (n <= CLUSTER_MAX_N && g_cluster_power) {
    // small Gram: one 16-CTA cluster, G resident in shared memory, DSMEM exchange
    const size_t csm = power_cluster_smem((int)n);
    static bool attr[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr[dev & 63]) {
      CUDA_TRY(cudaFuncSetAttribute(power_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      CUDA_TRY(cudaFuncSetAttribute(power_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      attr[dev & 63] = true;
    }
    power_cluster_kernel<<<CLUSTER_CTAS, 256, csm, st>>>(P); note_launch();
    if (cudaGetLastError() == cudaSuccess) return IBMI_OK;
    // cluster not schedulable here: fall through to the grid-wide kernel
  }
  if (g_power_ll && power_ll_launch(P, nb, st)) return IBMI_OK;
  // rows of G kept resident in each CTA's shared memory, after the staged iterate
  const int64_t rpc = (n + nb.blocks - 1) / nb.blocks;
  P.resident = 0;
  if (n <= P.smem_cap) P.resident = (int)std::max<int64_t>(0, std::min<int64_t>(rpc, (P.smem_cap - n) / n));
  const size_t smem = ((size_t)std::min<int64_t>(n, P.smem_cap) + (size_t)P.resident * n) * sizeof(double);
  void* args[] = {&P};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)power_gram_kernel, dim3(nb.blocks), dim3(nb.threads), args, smem,
                                       st));
  note_launch();
  return IBMI_OK;
}

void power_launch_shape(int device, int* blocks, int* threads, size_t* smem_cap) {
  int sms = 148, maxb = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  *threads = 512;
  *smem_cap = 220 * 1024;
  cudaFuncSetAttribute(power_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem_cap);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, power_gram_kernel, *threads, *smem_cap);
  *blocks = sms * std::max(1, std::min(maxb, 1));
}

// ---- error estimate for set k (solver.py:147-155 + linalg.py:223-274)
// ev (optional): [0] after the B GEMM, [1] after the Gram GEMM.
int enqueue_error_estimate(ibmi_ctx* c, int k, double rtol, int max_iters, cudaEvent_t* ev = nullptr,
                           bool copy_out = true) {
  NvtxRange nvtx_("error_estimate");
  const SetDev& s = c->sets[k];
  const int64_t p = c->p, b = s.b, cc = p - b;
  if (cc <= 0) return fail(IBMI_ERR_DIM, "set covers every index: empty complement");
  int rc = ensure_estimate_buffers(c, b, cc);
  if (rc) return rc;
  if (c->vr == nullptr || c->vr_n != cc) {
    return fail(IBMI_ERR_STATE, "restart vector of length " + std::to_string(cc) + " not set");
  }
  // B[m][n] = Σ_k Σ[I_m][k] A[c_n][k]   (A symmetric: A[k][c_n] = A[c_n][k])
  GemmOp gb;
  gb.X = c->S; gb.ldx = c->ld; gb.xm = s.rows();
  gb.Y = c->A; gb.ldy = c->ld; gb.yn = s.cmap();
  gb.M = b; gb.N = cc;
  gb.add_seg(0, 0, p);
  gb.C = c->Bm; gb.ldc = c->ldB;
  gb.tma_ok = true; gb.xrows = p; gb.xcols = p; gb.yrows = p; gb.ycols = p;
  const bool acache_ok = c->oz_n > 0 && !s.general && c->oz_a_set == k && c->oz_a.q && c->oz_a.n == c->oz_n &&
                         c->oz_n * b * round_up(cc, 16) <= c->oz.rq_cap;
  if (acache_ok && c->oz_s.q && c->oz_s.valid && c->oz_s.n == c->oz_n && b <= 65535 && cc <= 65535) {
    // X = the planes' rows I (all columns), Y = cached planes of A[c, :]
    OzOperand X;
    X.q = c->oz_s.q; X.e = c->oz_s.e + s.lo;
    X.ldq = c->oz_s.ldq; X.rows = p; X.cols = p; X.row_off = (int)s.lo;
    const OzOperand Y = oz_plain(c->oz_a.q, c->oz_a.e, round_up(p, 16), cc, p);
    CUDA_TRY(oz_upload_tables());
    CUDA_TRY(oz_igemm(gb, c->oz_n, X, Y, p, 0, cc, c->oz.rq, c->sms, c->stream));
    CUDA_TRY(oz_crt(gb, oz_epilogue(gb), c->oz_n, X, Y, 0, cc, c->oz.rq, c->stream));
  } else if (c->oz_n > 0 && !s.general && oz_fits(gb, c->oz, c->oz_n)) {
    const bool acache = acache_ok;
    CUDA_TRY(oz_gemm(gb, c->oz, c->oz_n, c->sms, c->stream, OzPre(), acache ? c->oz_a.pre() : OzPre(), false,
                     &c->ozs));
  } else {
    int64_t need = 0;
    gb.splits = plan_split(c, gb, g_split_panel, &need);
    if (need > c->splitws_cap) gb.splits = 1;
    gb.ws = c->splitws;
    CUDA_TRY(launch_gemm(gb, c->stream));
  }
  if (ev) CUDA_TRY(cudaEventRecord(ev[0], c->stream));
  NormBufs nb{c->Gm, c->ldG, c->vec, c->part, c->dscal, c->vr, c->power_blocks, c->power_threads,
              c->power_smem_cap, c->splitws, c->splitws_cap, c->sms};
  if (c->oz_n > 0 && !s.general) {
    nb.oz = &c->oz;
    nb.oz_n = c->oz_n;
  }
  rc = enqueue_two_norm(c->Bm, c->ldB, b, cc, rtol, max_iters, nb, c->stream, ev ? ev[1] : nullptr);
  if (rc) return rc;
  if (copy_out) CUDA_TRY(cudaMemcpyAsync(c->hpin, c->dscal, 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  return IBMI_OK;
}

int read_power(ibmi_ctx* c, double* err, int* iters, int* conv) {
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (err) *err = c->hpin[0];
  if (conv) *conv = c->hpin[1] != 0.0 ? 1 : 0;
  if (iters) *iters = (int)c->hpin[2];
  return IBMI_OK;
}

// Σ is allocated on first use (a sharded rank that only borrows the setup
// never pays for a p×p Σ).
int ensure_sigma(ibmi_ctx* c) {
  if (c->S) return IBMI_OK;
  const size_t mat = (size_t)c->p * c->ld * sizeof(double);
  CUDA_TRY(cudaMalloc(&c->S, mat));
  CUDA_TRY(cudaMemsetAsync(c->S, 0, mat, c->stream));
  c->bytes += mat;
  return IBMI_OK;
}

int check_ready(ibmi_ctx* c) {
  if (!c) return fail(IBMI_ERR_INVALID, "null context");
  if (!c->a_set) return fail(IBMI_ERR_STATE, "matrix not set");
  if (c->sets.empty()) return fail(IBMI_ERR_STATE, "partition not set");
  CUDA_TRY(cudaSetDevice(c->device));
  return ensure_sigma(c);
}

}  // namespace

// ======================================================================= ABI
extern "C" {

const char* ibmi_last_error(void) { return g_err.c_str(); }
const char* ibmi_version(void) { return "ibmi_b200 0.1.0 sm_100a (FP64 DMMA)"; }

int ibmi_create(ibmi_ctx** out, int device, int64_t p, void* stream) {
  if (!out) return fail(IBMI_ERR_INVALID, "out is null");
  *out = nullptr;
  if (p < 2) return fail(IBMI_ERR_DIM, "matrix order must be >= 2");
  CUDA_TRY(cudaSetDevice(device));
  PhaseTimer pt("create");
  ibmi_ctx* c = new ibmi_ctx();
  c->device = device;
  c->p = p;
  c->ld = round_up(p, 32);
  if (stream) {
    c->stream = (cudaStream_t)stream;
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) { delete c; return fail(IBMI_ERR_CUDA, cudaGetErrorString(e)); }
    c->own_stream = true;
  }
  if (device >= 0 && device < 64) {
    std::lock_guard<std::mutex> lock(g_mem_mu);
    ++g_live_ctx[device];
    c->counted = true;
  }
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  c->oz_n = g_oz_n;
  g_sms_hint = c->sms;
  prepare_gemm_attributes();
  power_launch_shape(device, &c->power_blocks, &c->power_threads, &c->power_smem_cap);
  const size_t mat = (size_t)p * c->ld * sizeof(double);
  cudaError_t e1 = cudaMalloc(&c->A, mat);
  cudaError_t e3 = e1 == cudaSuccess ? cudaMalloc(&c->dscal, 16 * sizeof(double)) : e1;
  cudaError_t e4 = e3 == cudaSuccess ? cudaMallocHost(&c->hpin, 16 * sizeof(double)) : e3;
  if (e4 != cudaSuccess) {
    ibmi_destroy(c);
    return fail(e4 == cudaErrorMemoryAllocation ? IBMI_ERR_OOM : IBMI_ERR_CUDA,
                std::string("allocating A/Σ: ") + cudaGetErrorString(e4));
  }
  c->bytes = mat + 16 * 8;
  *out = c;
  pt.mark("context + A allocation");
  return IBMI_OK;
}

int ibmi_destroy(ibmi_ctx* c) {
  if (!c) return IBMI_OK;
  cudaSetDevice(c->device);
  PhaseTimer pt("destroy");
  if (c->stream) cudaStreamSynchronize(c->stream);
  invalidate_graph(c);
  pt.mark("sync + graph");
  for (auto& s : c->sets) {
    if (s.W) cudaFree(s.W);
    if (s.ainv) cudaFree(s.ainv);
    if (s.idx) cudaFree(s.idx);
    if (s.comp) cudaFree(s.comp);
  }
  c->cs.release();
  c->oz.release();
  for (auto& w : c->oz_w) w.release();
  c->oz_a.release();
  c->oz_s.release();
  c->ozs.release();
  for (double* q : {c->A, c->S, c->Bm, c->Gm, c->vec, c->part, c->vr, c->frob_part, c->dscal, c->splitws})
    if (q) cudaFree(q);
  if (c->hpin) cudaFreeHost(c->hpin);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  const int dev = c->device;
  const bool counted = c->counted;
  delete c;
  {
    std::lock_guard<std::mutex> lock(g_mem_mu);
    if (counted && dev >= 0 && dev < 64 && --g_live_ctx[dev] == 0) mem_trim_locked(dev, mem_idle_cap(dev));
  }
  pt.mark("free");
  return IBMI_OK;
}

int ibmi_set_matrix(ibmi_ctx* c, const double* a, int64_t lda, int on_device) {
  NvtxRange nvtx_("set_matrix");
  if (!c || !a) return fail(IBMI_ERR_INVALID, "null argument");
  if (lda < c->p) return fail(IBMI_ERR_DIM, "lda < p");
  CUDA_TRY(cudaSetDevice(c->device));
  const int64_t p = c->p;
  PhaseTimer pt("set_matrix");
  CUDA_TRY(cudaMemsetAsync(c->A, 0, (size_t)p * c->ld * sizeof(double), c->stream));
  if (on_device) {
    CUDA_TRY(cudaMemcpy2DAsync(c->A, c->ld * sizeof(double), a, lda * sizeof(double), p * sizeof(double), p,
                               cudaMemcpyDeviceToDevice, c->stream));
  } else {
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    int rc = staged_copy(c->A, c->ld, const_cast<double*>(a), lda, p, p, true, c->device, c->stream);
    if (rc) return rc;
  }
  c->a_set = true;
  for (auto& s : c->sets) s.ready = false;
  invalidate_graph(c);
  c->bytes -= c->oz_a.bytes;
  c->oz_a.release();
  c->oz_a_set = -1;
  pt.mark("upload");
  int rc = symcheck(c, contig_map(0), p, "matrix");
  if (rc) { c->a_set = false; return rc; }
  pt.mark("symmetry check");
  return IBMI_OK;
}

int ibmi_set_partition(ibmi_ctx* c, int k, const int64_t* lo, const int64_t* hi) {
  if (!c || !lo || !hi) return fail(IBMI_ERR_INVALID, "null argument");
  if (k < 1) return fail(IBMI_ERR_INVALID, "need at least one set");
  CUDA_TRY(cudaSetDevice(c->device));
  for (int j = 0; j < k; ++j) {
    if (lo[j] < 0 || hi[j] > c->p || lo[j] >= hi[j])
      return fail(IBMI_ERR_INDEX, "set " + std::to_string(j) + " has indices outside [0, p)");
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  for (auto& s : c->sets) {
    if (s.W) cudaFree(s.W);
    if (s.ainv) cudaFree(s.ainv);
    if (s.idx) cudaFree(s.idx);
    if (s.comp) cudaFree(s.comp);
    if (s.W) c->bytes -= (size_t)s.b * c->ld * 8 + (size_t)s.b * s.ldb * 8;
  }
  oz_drop_caches(c);
  c->sets.assign(k, SetDev());
  for (int j = 0; j < k; ++j) {
    c->sets[j].lo = lo[j];
    c->sets[j].hi = hi[j];
    c->sets[j].b = (int)(hi[j] - lo[j]);
    c->sets[j].ldb = round_up(c->sets[j].b, 32);
  }
  invalidate_graph(c);
  return IBMI_OK;
}

int ibmi_set_partition_general(ibmi_ctx* c, int k, const int64_t* set_ptr, const int64_t* set_idx) {
  if (!c || !set_ptr || !set_idx) return fail(IBMI_ERR_INVALID, "null argument");
  if (k < 1) return fail(IBMI_ERR_INVALID, "need at least one set");
  const int64_t p = c->p;
  std::vector<int64_t> lo(k), hi(k);
  std::vector<bool> run(k);
  for (int j = 0; j < k; ++j) {
    const int64_t n = set_ptr[j + 1] - set_ptr[j];
    if (n < 1) return fail(IBMI_ERR_INVALID, "set " + std::to_string(j) + " is empty");
    const int64_t* s = set_idx + set_ptr[j];
    bool r = true;
    for (int64_t i = 0; i < n; ++i) {
      if (s[i] < 0 || s[i] >= p) return fail(IBMI_ERR_INDEX, "set " + std::to_string(j) + " has indices outside [0, p)");
      if (i && s[i] <= s[i - 1]) return fail(IBMI_ERR_INVALID, "set " + std::to_string(j) + " must be strictly ascending");
      if (s[i] != s[0] + i) r = false;
    }
    lo[j] = s[0];
    hi[j] = s[n - 1] + 1;
    run[j] = r;
  }
  int rc = ibmi_set_partition(c, k, lo.data(), hi.data());
  if (rc) return rc;
  for (int j = 0; j < k; ++j) {
    if (run[j]) continue;
    SetDev& sd = c->sets[j];
    const int64_t n = set_ptr[j + 1] - set_ptr[j];
    const int64_t* s = set_idx + set_ptr[j];
    std::vector<int64_t> comp;
    comp.reserve(p - n);
    for (int64_t i = 0, q = 0; i < p; ++i) {
      if (q < n && s[q] == i) { ++q; continue; }
      comp.push_back(i);
    }
    sd.general = true;
    sd.b = (int)n;
    sd.ldb = round_up(n, 32);
    CUDA_TRY(cudaMalloc(&sd.idx, n * sizeof(int64_t)));
    CUDA_TRY(cudaMemcpyAsync(sd.idx, s, n * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    if (!comp.empty()) {
      CUDA_TRY(cudaMalloc(&sd.comp, comp.size() * sizeof(int64_t)));
      CUDA_TRY(cudaMemcpyAsync(sd.comp, comp.data(), comp.size() * sizeof(int64_t), cudaMemcpyHostToDevice,
                               c->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  return IBMI_OK;
}

int ibmi_setup(ibmi_ctx* c, int first, int count, int* fail_set, int64_t* fail_pivot) {
  NvtxRange nvtx_("ibmi_setup");
  if (!c) return fail(IBMI_ERR_INVALID, "null context");
  if (c) c->oz_s.valid = false;   // Σ (or W) changes outside the residue planes' bookkeeping
  if (!c->a_set) return fail(IBMI_ERR_STATE, "matrix not set");
  if (c->sets.empty()) return fail(IBMI_ERR_STATE, "partition not set");
  CUDA_TRY(cudaSetDevice(c->device));
  if (fail_set) *fail_set = -1;
  if (fail_pivot) *fail_pivot = -1;
  const int K = (int)c->sets.size();
  if (count < 0) count = K - first;
  if (first < 0 || first + count > K) return fail(IBMI_ERR_INVALID, "set range out of bounds");
  if (count == 0) return IBMI_OK;
  const int64_t p = c->p;
  cudaStream_t st = c->stream;
  PhaseTimer pt("setup");
  for (int j = first; j < first + count && j < (int)c->oz_w.size(); ++j) {
    c->bytes -= c->oz_w[j].bytes;
    c->oz_w[j].release();
  }

  // 1. symmetry of every A_II (linalg.py:68-77), one sync for all sets
  unsigned long long* dsym = nullptr;
  CUDA_TRY(cudaMalloc(&dsym, (size_t)2 * count * sizeof(unsigned long long)));
  CUDA_TRY(cudaMemsetAsync(dsym, 0, (size_t)2 * count * sizeof(unsigned long long), st));
  for (int j = 0; j < count; ++j) {
    const SetDev& s = c->sets[first + j];
    const int nt = (s.b + 31) / 32;
    symcheck_kernel<<<dim3(nt, nt), dim3(32, 8), 0, st>>>(c->A, c->ld, s.rows(), s.b, dsym + 2 * j); note_launch();
  }
  std::vector<unsigned long long> hsym(2 * count);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(hsym.data(), dsym, hsym.size() * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(dsym);
  if (e != cudaSuccess) return fail(IBMI_ERR_CUDA, cudaGetErrorString(e));
  pt.mark("block symmetry checks");

  // 2. factor / invert / W for all sets, up to 8 sets in flight on their own streams
  for (int j = 0; j < count; ++j) {
    SetDev& s = c->sets[first + j];
    if (!s.W) {
      CUDA_TRY(cudaMalloc(&s.W, (size_t)s.b * c->ld * sizeof(double)));
      CUDA_TRY(cudaMalloc(&s.ainv, (size_t)s.b * s.ldb * sizeof(double)));
      c->bytes += (size_t)s.b * c->ld * 8 + (size_t)s.b * s.ldb * 8;
    }
  }
  pt.mark("W / ainv allocation");
  const int S = std::min(count, 8);
  std::vector<cudaStream_t> ss(S, nullptr);
  std::vector<CholScratch> scr(S);
  std::vector<double*> gather(S, nullptr);
  std::vector<int> infos(count, INT_MAX);
  int* dinfo = nullptr;
  cudaEvent_t ready = nullptr;
  int rc = IBMI_OK;
  auto cleanup = [&]() {
    for (int q = 0; q < S; ++q) {
      if (ss[q]) { cudaStreamSynchronize(ss[q]); cudaStreamDestroy(ss[q]); }
      scr[q].release();
      if (gather[q]) cudaFree(gather[q]);
    }
    if (dinfo) cudaFree(dinfo);
    if (ready) cudaEventDestroy(ready);
  };
#define SETUP_TRY(expr)                                                             \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess) { cleanup(); return fail(e_ == cudaErrorMemoryAllocation \
        ? IBMI_ERR_OOM : IBMI_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); } \
  } while (0)
  SETUP_TRY(cudaMalloc(&dinfo, (size_t)count * sizeof(int)));
  SETUP_TRY(cudaMemcpyAsync(dinfo, infos.data(), (size_t)count * sizeof(int), cudaMemcpyHostToDevice, st));
  SETUP_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  SETUP_TRY(cudaEventRecord(ready, st));
  for (int q = 0; q < S; ++q) {
    SETUP_TRY(cudaStreamCreateWithFlags(&ss[q], cudaStreamNonBlocking));
    SETUP_TRY(cudaStreamWaitEvent(ss[q], ready, 0));
    int bmax = 0;
    for (int j = q; j < count; j += S) bmax = std::max(bmax, c->sets[first + j].b);
    rc = ensure_scratch(scr[q], bmax);
    // the inverse's scratch too, before any work is queued: a cudaMalloc inside the loop
    // below would synchronise the device and serialise the eight set pipelines
    if (!rc) rc = ensure_potri_scratch(scr[q], bmax);
    if (rc) { cleanup(); return rc; }
  }
  pt.mark("streams + scratch");
  const auto t_enq0 = std::chrono::steady_clock::now();
  for (int j = 0; j < count; ++j) {
    const int q = j % S;
    SetDev& s = c->sets[first + j];
    cudaStream_t sq = ss[q];
    CholScratch& cs = scr[q];
    const int64_t b = s.b, lo = s.lo, hi = s.hi;
    int* info = dinfo + j;
    copy2d_kernel<<<grid2d(b, b), 256, 0, sq>>>(c->A, c->ld, s.rows(), s.rows(), cs.ws, cs.ldw, (int)b, (int)b, 1); note_launch();
    SETUP_TRY(cudaGetLastError());
    rc = potrf_enqueue(cs, (int)b, sq, info);
    if (!rc) rc = potri_blocked(cs, (int)b, s.ainv, s.ldb, sq);
    if (rc) { cleanup(); return rc; }
    SETUP_TRY(cudaMemsetAsync(s.W, 0, (size_t)b * c->ld * sizeof(double), sq));
    if (s.general) {
      // A_I = A[I, :] gathered (b × p), W = ainv · A_I (transposed-Y GEMM), then zero W[:, I]
      if (!gather[q]) {
        int64_t gmax = 0;
        for (int jj = q; jj < count; jj += S)
          if (c->sets[first + jj].general) gmax = std::max<int64_t>(gmax, c->sets[first + jj].b);
        SETUP_TRY(cudaMalloc(&gather[q], (size_t)gmax * c->ld * sizeof(double)));
      }
      double* ai = gather[q];
      copy2d_kernel<<<grid2d(b, c->ld), 256, 0, sq>>>(c->A, c->ld, s.rows(), contig_map(0), ai, c->ld, (int)b,
                                                     (int)c->ld, 0); note_launch();
      GemmOp gw;
      gw.X = s.ainv; gw.ldx = s.ldb;
      gw.Y = ai; gw.ldy = c->ld; gw.yt = true;
      gw.M = b; gw.N = p;
      gw.add_seg(0, 0, b);
      gw.C = s.W; gw.ldc = c->ld;
      SETUP_TRY(launch_gemm(gw, sq));
      zero_cols_kernel<<<dim3((unsigned)((b + 255) / 256), (unsigned)std::min<int64_t>(b, 65535)), 256, 0, sq>>>(
          s.W, c->ld, (int)b, s.rows(), (int)b); note_launch();
      SETUP_TRY(cudaGetLastError());
    } else {
      GemmOp gw;
      gw.X = s.ainv; gw.ldx = s.ldb;
      gw.Y = c->A; gw.ldy = c->ld; gw.yn = complement_map(lo, hi);
      gw.M = b; gw.N = p - b;
      gw.add_seg(0, lo, b);
      gw.C = s.W; gw.ldc = c->ld; gw.cn = complement_map(lo, hi);
      // K tails end at the segment ends (the TMA maps stop there and zero-fill)
      gw.tma_ok = true; gw.xrows = b; gw.xcols = b; gw.yrows = p; gw.ycols = p;
      SETUP_TRY(launch_gemm(gw, sq));
    }
  }
  if (getenv("IBMI_PROFILE"))
    fprintf(stderr, "[ibmi] setup: host time to enqueue all sets %.1f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_enq0).count());
  for (int q = 0; q < S; ++q) SETUP_TRY(cudaStreamSynchronize(ss[q]));
  SETUP_TRY(cudaMemcpy(infos.data(), dinfo, (size_t)count * sizeof(int), cudaMemcpyDeviceToHost));
#undef SETUP_TRY
  pt.mark("factor + inverse + W");
  cleanup();
  pt.mark("scratch release");

  // 3. errors in the reference's order: set by set, symmetry before the pivot
  for (int j = 0; j < count; ++j) {
    const double mabs = __builtin_bit_cast(double, hsym[2 * j]);
    const double skew = __builtin_bit_cast(double, hsym[2 * j + 1]);
    if (mabs != 0.0 && !(skew <= 1e-12 * mabs)) {
      if (fail_set) *fail_set = first + j;
      char buf[256];
      snprintf(buf, sizeof(buf), "matrix is not symmetric: max |a - a.T| = %.3e exceeds 1.0e-12 * max|a| = %.3e",
               skew, 1e-12 * mabs);
      return fail(IBMI_ERR_NOT_SYMMETRIC, buf);
    }
    if (infos[j] != INT_MAX) {
      if (fail_set) *fail_set = first + j;
      if (fail_pivot) *fail_pivot = infos[j];
      return fail(IBMI_ERR_NOT_SPD, "non-positive pivot at elimination step " + std::to_string(infos[j]));
    }
  }
  for (int j = 0; j < count; ++j) c->sets[first + j].ready = true;
  invalidate_graph(c);
  return IBMI_OK;
}

int ibmi_init_sigma(ibmi_ctx* c, int kind, const double* guess, int64_t ldg, int on_device) {
  NvtxRange nvtx_("init_sigma");
  int rc = check_ready(c);
  if (c) c->oz_s.valid = false;   // Σ (or W) changes outside the residue planes' bookkeeping
  if (rc) return rc;
  const int64_t p = c->p;
  const SetDev& s0 = c->sets[0];
  const int64_t c0 = p - s0.b;
  cudaStream_t st = c->stream;
  fill2d_kernel<<<grid2d(p, c->ld), 256, 0, st>>>(c->S, c->ld, (int)p, (int)c->ld, 0.0, 1.0); note_launch();
  CUDA_TRY(cudaGetLastError());
  if (c0 == 0) return IBMI_OK;
  const RowMap cmap = s0.cmap();
  if (kind == IBMI_GUESS_IDENTITY) {
  } else if (kind == IBMI_GUESS_JACOBI) {
    jacobi_diag_kernel<<<(int)((c0 + 255) / 256), 256, 0, st>>>(c->A, c->ld, c->S, c->ld, cmap, (int)c0); note_launch();
    CUDA_TRY(cudaGetLastError());
  } else if (kind == IBMI_GUESS_MATRIX) {
    if (!guess || ldg < c0) return fail(IBMI_ERR_DIM, "guess must be c1 x c1");
    double* tmp = nullptr;
    CUDA_TRY(cudaMalloc(&tmp, (size_t)c0 * c0 * sizeof(double)));
    cudaError_t e = cudaMemcpy2DAsync(tmp, c0 * 8, guess, ldg * 8, c0 * 8, c0,
                                      on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
      scatter2d_kernel<<<grid2d(c0, c0), 256, 0, st>>>(tmp, c0, c->S, c->ld, cmap, cmap, (int)c0, (int)c0); note_launch();
      e = cudaGetLastError();
    }
    cudaStreamSynchronize(st);
    cudaFree(tmp);
    if (e != cudaSuccess) return fail(IBMI_ERR_CUDA, cudaGetErrorString(e));
  } else if (kind == IBMI_GUESS_LOCAL) {
    CholScratch cs;
    rc = ensure_scratch(cs, (int)c0);
    if (rc) { cs.release(); return rc; }
    double* inv = nullptr;
    cudaError_t e = cudaMalloc(&inv, (size_t)c0 * cs.ldw * sizeof(double));
    if (e != cudaSuccess) { cs.release(); return fail(IBMI_ERR_OOM, cudaGetErrorString(e)); }
    copy2d_kernel<<<grid2d(c0, c0), 256, 0, st>>>(c->A, c->ld, cmap, cmap, cs.ws, cs.ldw, (int)c0, (int)c0, 1); note_launch();
    int64_t piv = -1;
    rc = potrf_blocked(cs, (int)c0, st, &piv);
    if (!rc) rc = potri_blocked(cs, (int)c0, inv, cs.ldw, st);
    if (!rc) {
      scatter2d_kernel<<<grid2d(c0, c0), 256, 0, st>>>(inv, cs.ldw, c->S, c->ld, cmap, cmap, (int)c0, (int)c0); note_launch();
      cudaStreamSynchronize(st);
    }
    cudaFree(inv);
    cs.release();
    if (rc) return rc;
  } else if (kind == IBMI_GUESS_MC) {
    // Σ0[c,c] = Z_c Z_cᵀ / n, Z = L⁻ᵀ w, A = L Lᵀ (reference solver.py:167-181); w = p × ldg draws.
    if (!guess || ldg < 1) return fail(IBMI_ERR_INVALID, "mc guess needs the p x n sample matrix");
    rc = mc_guess_into(c->A, c->ld, p, guess, on_device, ldg, cmap, c0, c->S, c->ld, cmap, cmap, st);
    if (rc) return rc;
  } else if (kind == IBMI_GUESS_TAKAHASHI) {
    // (A⁻¹)[c,c] = S_c⁻¹, S_c = A_cc − A_cI W (W = A_II⁻¹ A_Ic of set 0): the block the
    // reference's LDLᵀ backward recurrence reproduces (solver.py:184-212).  Needs set 0 set up.
    if (!s0.ready) return fail(IBMI_ERR_STATE, "takahashi guess needs set 0 set up (call ibmi_setup first)");
    const int64_t b0 = s0.b;
    CholScratch cs;
    rc = ensure_scratch(cs, (int)c0);
    if (rc) { cs.release(); return rc; }
    double *aci = nullptr, *wc = nullptr, *inv = nullptr;
    const int64_t ldb0 = round_up(b0, 32), ldc0 = round_up(c0, 32);
    cudaError_t e = cudaMalloc(&aci, (size_t)c0 * ldb0 * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&wc, (size_t)b0 * ldc0 * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&inv, (size_t)c0 * cs.ldw * sizeof(double));
    if (e != cudaSuccess) {
      cs.release(); cudaFree(aci); cudaFree(wc); cudaFree(inv);
      return fail(IBMI_ERR_OOM, cudaGetErrorString(e));
    }
    const RowMap imap = s0.rows();
    copy2d_kernel<<<grid2d(c0, c0), 256, 0, st>>>(c->A, c->ld, cmap, cmap, cs.ws, cs.ldw, (int)c0, (int)c0, 1); note_launch();
    copy2d_kernel<<<grid2d(c0, b0), 256, 0, st>>>(c->A, c->ld, cmap, imap, aci, ldb0, (int)c0, (int)b0, 0); note_launch();
    copy2d_kernel<<<grid2d(b0, c0), 256, 0, st>>>(s0.W, c->ld, contig_map(0), cmap, wc, ldc0, (int)b0, (int)c0, 0); note_launch();
    GemmOp gs;   // S_c[m][n] = A_cc[m][n] − Σ_k A_cI[m][k] W_c[k][n]
    gs.X = aci; gs.ldx = ldb0;
    gs.Y = wc; gs.ldy = ldc0; gs.yt = true;
    gs.M = c0; gs.N = c0;
    gs.add_seg(0, 0, b0);
    gs.C = cs.ws; gs.ldc = cs.ldw;
    gs.alpha = -1.0; gs.beta = 1.0; gs.D = cs.ws; gs.ldd = cs.ldw;
    gs.lower = true;
    e = launch_gemm(gs, st);
    if (e != cudaSuccess) rc = fail(IBMI_ERR_CUDA, cudaGetErrorString(e));
    int64_t piv = -1;
    if (!rc) rc = potrf_blocked(cs, (int)c0, st, &piv);
    if (!rc) rc = potri_blocked(cs, (int)c0, inv, cs.ldw, st);
    if (!rc) {
      scatter2d_kernel<<<grid2d(c0, c0), 256, 0, st>>>(inv, cs.ldw, c->S, c->ld, cmap, cmap, (int)c0, (int)c0); note_launch();
      cudaStreamSynchronize(st);
    }
    cs.release();
    cudaFree(aci);
    cudaFree(wc);
    cudaFree(inv);
    if (rc) return rc;
  } else {
    return fail(IBMI_ERR_INVALID, "unknown guess kind " + std::to_string(kind));
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return IBMI_OK;
}

int ibmi_set_sigma(ibmi_ctx* c, const double* s, int64_t lds, int on_device) {
  if (!c || !s) return fail(IBMI_ERR_INVALID, "null argument");
  if (c) c->oz_s.valid = false;   // Σ (or W) changes outside the residue planes' bookkeeping
  if (lds < c->p) return fail(IBMI_ERR_DIM, "lds < p");
  CUDA_TRY(cudaSetDevice(c->device));
  if (int rc = ensure_sigma(c)) return rc;
  CUDA_TRY(cudaMemsetAsync(c->S, 0, (size_t)c->p * c->ld * sizeof(double), c->stream));
  if (on_device) {
    CUDA_TRY(cudaMemcpy2DAsync(c->S, c->ld * 8, s, lds * 8, c->p * 8, c->p, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    int rc = staged_copy(c->S, c->ld, const_cast<double*>(s), lds, c->p, c->p, true, c->device, c->stream);
    if (rc) return rc;
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return IBMI_OK;
}

int ibmi_get_sigma(ibmi_ctx* c, double* out, int64_t ldo, int on_device) {
  NvtxRange nvtx_("get_sigma");
  if (!c || !out) return fail(IBMI_ERR_INVALID, "null argument");
  if (ldo < c->p) return fail(IBMI_ERR_DIM, "ldo < p");
  CUDA_TRY(cudaSetDevice(c->device));
  if (int rc = ensure_sigma(c)) return rc;
  PhaseTimer pt("get_sigma");
  if (on_device) {
    CUDA_TRY(cudaMemcpy2DAsync(out, ldo * 8, c->S, c->ld * 8, c->p * 8, c->p, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    int rc = staged_copy(c->S, c->ld, out, ldo, c->p, c->p, false, c->device, c->stream);
    if (rc) return rc;
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  pt.mark("download");
  return IBMI_OK;
}

int ibmi_copy_rows(int device, double* dev, int64_t ldd, double* host, int64_t ldh, int64_t rows, int64_t cols,
                   const int64_t* host_rows, int to_device, void* stream) {
  if (!dev || !host || rows < 0 || cols < 0) return fail(IBMI_ERR_INVALID, "bad copy arguments");
  if (ldd < cols || ldh < cols) return fail(IBMI_ERR_DIM, "leading dimension < cols");
  if (rows == 0 || cols == 0) return IBMI_OK;
  CUDA_TRY(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaStreamSynchronize(st));   // the rows are produced on the caller's stream
  return staged_copy(dev, ldd, host, ldh, rows, cols, to_device != 0, device, st, host_rows);
}

int ibmi_set_restart_vector(ibmi_ctx* c, int64_t n, const double* v) {
  if (!c || !v || n < 1) return fail(IBMI_ERR_INVALID, "bad restart vector");
  CUDA_TRY(cudaSetDevice(c->device));
  if (c->vr_n != n) {
    if (c->vr) cudaFree(c->vr);
    c->vr = nullptr;
    c->vr_n = 0;
    CUDA_TRY(cudaMalloc(&c->vr, (size_t)n * sizeof(double)));
    c->vr_n = n;
    invalidate_graph(c);
  }
  CUDA_TRY(cudaMemcpyAsync(c->vr, v, (size_t)n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return IBMI_OK;
}

int ibmi_block_update(ibmi_ctx* c, int k) {
  int rc = check_ready(c);
  if (rc) return rc;
  if (k < 0 || k >= (int)c->sets.size()) return fail(IBMI_ERR_INVALID, "set index out of range");
  if (!c->sets[k].ready) return fail(IBMI_ERR_STATE, "set not set up");
  rc = plan_workspace(c);
  if (rc) return rc;
  rc = enqueue_block_update(c, k);
  if (rc) return rc;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return IBMI_OK;
}

int ibmi_error_estimate(ibmi_ctx* c, int k, double rtol, int max_iters, double* err, int* iters, int* conv) {
  int rc = check_ready(c);
  if (rc) return rc;
  if (k < 0 || k >= (int)c->sets.size()) return fail(IBMI_ERR_INVALID, "set index out of range");
  if (max_iters < 1) return fail(IBMI_ERR_INVALID, "max_iters must be >= 1");
  rc = plan_workspace(c);
  if (rc) return rc;
  rc = enqueue_error_estimate(c, k, rtol, max_iters);
  if (rc) return rc;
  return read_power(c, err, iters, conv);
}

// ---- small problems: the sweep's GEMM phases as one cooperative kernel (small_sweep.cuh)
bool small_fused_ok(const ibmi_ctx* c) {
  if (!g_small_fused || c->oz_n > 0 || c->p > 1024 || c->sets.empty() || (int)c->sets.size() > SS_MAX_SETS) return false;
  for (const SetDev& s : c->sets)
    if (s.general || !s.ready) return false;
  const SetDev& last = c->sets.back();
  return last.b <= c->p - last.b && c->Bm && c->Gm && c->vec && c->vr_n == c->p - last.b;
}

// All K block updates and, with `estimate`, B, G = B·Bᵀ and y₁ of the last set; then the power iteration.
// ev (optional): [0] after the fused kernel, [1] after the power iteration.
int enqueue_small_sweep(ibmi_ctx* c, double rtol, int max_iters, cudaEvent_t* ev, bool copy_out) {
  static bool attr[64] = {false};
  if (!attr[c->device & 63]) {
    CUDA_TRY(cudaFuncSetAttribute(small_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SS_SMEM));
    attr[c->device & 63] = true;
  }
  SmallSweepParams P;
  memset(&P, 0, sizeof(P));
  P.S = c->S; P.A = c->A; P.ld = c->ld; P.p = (int)c->p; P.K = (int)c->sets.size();
  int tiles = 1;
  for (int k = 0; k < P.K; ++k) {
    const SetDev& s = c->sets[k];
    P.set[k] = SmallSet{(int)s.lo, (int)s.hi, s.W, s.ainv, s.ldb};
    const int ntm = (s.b + SS_TM - 1) / SS_TM, ntn = (int)((c->p - s.b + SS_TILE - 1) / SS_TILE);
    tiles = std::max(tiles, ntm * ntn);
  }
  P.estimate = 1;
  P.B = c->Bm; P.ldB = c->ldB; P.G = c->Gm; P.ldG = c->ldG; P.y1 = c->vec;
  // IBMI_SS_TRACE=1 (eager launches only): per-phase %globaltimer stamps of block 0, printed to stderr
  static int trace_on = -1;
  if (trace_on < 0) trace_on = getenv("IBMI_SS_TRACE") ? 1 : 0;
  static unsigned long long* trace_dev = nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cap);
  const bool tracing = trace_on && cap == cudaStreamCaptureStatusNone;
  if (tracing) {
    if (!trace_dev) CUDA_TRY(cudaMalloc(&trace_dev, 128 * sizeof(unsigned long long)));
    P.trace = trace_dev;
  }
  const int grid = std::min(tiles, c->sms);
  void* args[] = {&P};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)small_sweep_kernel, dim3(grid), dim3(SS_THREADS), args, SS_SMEM,
                                       c->stream));
  note_launch();
  if (tracing) {
    unsigned long long h[128];
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    CUDA_TRY(cudaMemcpy(h, trace_dev, sizeof(h), cudaMemcpyDeviceToHost));
    const int stamps = 4 * P.K + 4;
    fprintf(stderr, "[ibmi] small_sweep phases (ns, block 0; phase, barrier, ...):");
    for (int i = 1; i < stamps && i < 128; ++i) fprintf(stderr, " %llu", h[i] - h[i - 1]);
    fprintf(stderr, "\n");
  }
  if (ev) CUDA_TRY(cudaEventRecord(ev[0], c->stream));
  const SetDev& last = c->sets.back();
  NormBufs nb{c->Gm, c->ldG, c->vec, c->part, c->dscal, c->vr, c->power_blocks, c->power_threads,
              c->power_smem_cap, c->splitws, c->splitws_cap, c->sms};
  int rc = enqueue_two_norm(c->Bm, c->ldB, last.b, c->p - last.b, rtol, max_iters, nb, c->stream, nullptr, true);
  if (rc) return rc;
  if (ev) CUDA_TRY(cudaEventRecord(ev[1], c->stream));
  if (copy_out) CUDA_TRY(cudaMemcpyAsync(c->hpin, c->dscal, 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  return IBMI_OK;
}

static int enqueue_sweep(ibmi_ctx* c, double rtol, int max_iters) {
  if (small_fused_ok(c)) return enqueue_small_sweep(c, rtol, max_iters, nullptr, true);
  for (int k = 0; k < (int)c->sets.size(); ++k) {
    int rc = enqueue_block_update(c, k);
    if (rc) return rc;
  }
  return enqueue_error_estimate(c, (int)c->sets.size() - 1, rtol, max_iters);
}

int ibmi_sweep(ibmi_ctx* c, double rtol, int max_iters, double* err, int* iters, int* conv) {
  NvtxRange nvtx_("ibmi_sweep");
  int rc = check_ready(c);
  if (rc) return rc;
  for (auto& s : c->sets)
    if (!s.ready) return fail(IBMI_ERR_STATE, "setup not complete");
  if (max_iters < 1) return fail(IBMI_ERR_INVALID, "max_iters must be >= 1");
  // make sure lazily-allocated buffers exist before any capture
  const SetDev& last = c->sets.back();
  rc = ensure_estimate_buffers(c, last.b, c->p - last.b);
  if (rc) return rc;
  rc = plan_workspace(c);
  if (rc) return rc;
  if (c->graph_gen != g_tune_gen) invalidate_graph(c);
  c->graph_gen = g_tune_gen;
  if (c->graph_tried && (c->graph_rtol != rtol || c->graph_max != max_iters)) invalidate_graph(c);
  if (!c->graph_tried) {
    c->graph_tried = true;
    c->graph_rtol = rtol;
    c->graph_max = max_iters;
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      const long long before = g_launches.load();
      int erc = enqueue_sweep(c, rtol, max_iters);
      c->graph_launches = g_launches.load() - before;
      g_launches.fetch_sub(c->graph_launches);     // captured, not launched
      cudaError_t ec = cudaStreamEndCapture(c->stream, &g);
      if (erc == IBMI_OK && ec == cudaSuccess && g) {
        if (cudaGraphInstantiate(&c->graph, g, 0) == cudaSuccess) c->graph_ok = true;
      }
      if (g) cudaGraphDestroy(g);
    }
    cudaGetLastError();   // clear any capture error; fall back to direct launches
    if (!c->graph_ok && c->graph) { cudaGraphExecDestroy(c->graph); c->graph = nullptr; }
  }
  if (c->graph_ok) {
    CUDA_TRY(cudaGraphLaunch(c->graph, c->stream));
    g_launches.fetch_add(c->graph_launches);
  } else {
    rc = enqueue_sweep(c, rtol, max_iters);
    if (rc) return rc;
  }
  return read_power(c, err, iters, conv);
}

int ibmi_sweep_timed(ibmi_ctx* c, double rtol, int max_iters, double* err, int* iters, int* conv, float* times) {
  NvtxRange nvtx_("ibmi_sweep_timed");
  int rc = check_ready(c);
  if (rc) return rc;
  for (auto& s : c->sets)
    if (!s.ready) return fail(IBMI_ERR_STATE, "setup not complete");
  const int K = (int)c->sets.size();
  rc = plan_workspace(c);
  if (rc) return rc;
  std::vector<cudaEvent_t> ev(2 * K + 4);
  for (auto& e : ev) CUDA_TRY(cudaEventCreate(&e));
  float t[6] = {0, 0, 0, 0, 0, 0};
  CUDA_TRY(cudaEventRecord(ev[0], c->stream));
  {
    const SetDev& last = c->sets.back();
    rc = ensure_estimate_buffers(c, last.b, c->p - last.b);
    if (rc) return rc;
  }
  if (small_fused_ok(c)) {
    // fused small-problem sweep: times[0] = the fused kernel (all GEMM phases), times[4] = power iteration
    rc = enqueue_small_sweep(c, rtol, max_iters, &ev[1], true);
    if (rc) return rc;
    rc = read_power(c, err, iters, conv);
    if (rc) return rc;
    float ms;
    CUDA_TRY(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    t[0] = ms;
    CUDA_TRY(cudaEventElapsedTime(&ms, ev[1], ev[2]));
    t[4] = ms;
    CUDA_TRY(cudaEventElapsedTime(&ms, ev[0], ev[2]));
    t[5] = ms;
    for (auto& e : ev) cudaEventDestroy(e);
    if (times) memcpy(times, t, sizeof(t));
    return IBMI_OK;
  }
  for (int k = 0; k < K; ++k) {
    rc = enqueue_block_update(c, k, ev[1 + 2 * k]);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(ev[2 + 2 * k], c->stream));
  }
  rc = enqueue_error_estimate(c, K - 1, rtol, max_iters, &ev[2 * K + 1]);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(ev[2 * K + 3], c->stream));
  rc = read_power(c, err, iters, conv);
  if (rc) return rc;
  float ms;
  for (int k = 0; k < K; ++k) {
    CUDA_TRY(cudaEventElapsedTime(&ms, ev[2 * k], ev[1 + 2 * k]));
    t[0] += ms;
    CUDA_TRY(cudaEventElapsedTime(&ms, ev[1 + 2 * k], ev[2 + 2 * k]));
    t[1] += ms;
  }
  CUDA_TRY(cudaEventElapsedTime(&ms, ev[2 * K], ev[2 * K + 1]));
  t[2] = ms;
  CUDA_TRY(cudaEventElapsedTime(&ms, ev[2 * K + 1], ev[2 * K + 2]));
  t[3] = ms;
  CUDA_TRY(cudaEventElapsedTime(&ms, ev[2 * K + 2], ev[2 * K + 3]));
  t[4] = ms;
  CUDA_TRY(cudaEventElapsedTime(&ms, ev[0], ev[2 * K + 3]));
  t[5] = ms;
  for (auto& e : ev) cudaEventDestroy(e);
  if (times) memcpy(times, t, sizeof(t));
  return IBMI_OK;
}

static int enqueue_frobenius(ibmi_ctx* c) {
  const int64_t p = c->p;
  GemmOp fr;
  fr.X = c->A; fr.ldx = c->ld;
  fr.Y = c->S; fr.ldy = c->ld;
  fr.M = p; fr.N = p;
  fr.add_seg(0, 0, p);
  fr.tma_ok = true; fr.xrows = p; fr.xcols = p; fr.yrows = p; fr.ycols = p;
  const int nparts = gemm_grid(fr);
  int64_t cap = c->frob_cap;
  if (ensure_buf(&c->frob_part, &cap, nparts, &c->bytes)) return IBMI_ERR_OOM;
  c->frob_cap = (int)cap;
  fr.partial = c->frob_part;
  CUDA_TRY(launch_gemm(fr, c->stream));
  reduce_partials_kernel<<<1, 1024, 0, c->stream>>>(c->frob_part, nparts, c->dscal + 3); note_launch();
  CUDA_TRY(cudaGetLastError());
  return IBMI_OK;
}

// Frobenius workspace sized before any capture.
static int ensure_frob_buffers(ibmi_ctx* c) {
  GemmOp fr;
  fr.M = c->p; fr.N = c->p;
  const int nparts = gemm_grid(fr);
  int64_t cap = c->frob_cap;
  if (ensure_buf(&c->frob_part, &cap, nparts, &c->bytes)) return IBMI_ERR_OOM;
  c->frob_cap = (int)cap;
  return IBMI_OK;
}

}  // extern "C"

// ---- device-side solve loop (conditional WHILE graph) -----------------------
namespace {

int frontier(cudaStream_t st, std::vector<cudaGraphNode_t>& out) {
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CUDA_TRY(cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd));
  out.assign(deps, deps + nd);
  return IBMI_OK;
}

int enqueue_sweep_body(ibmi_ctx* c, double rtol, int max_iters) {
  if (small_fused_ok(c)) return enqueue_small_sweep(c, rtol, max_iters, nullptr, false);
  for (int k = 0; k < (int)c->sets.size(); ++k) {
    int rc = enqueue_block_update(c, k);
    if (rc) return rc;
  }
  return enqueue_error_estimate(c, (int)c->sets.size() - 1, rtol, max_iters, nullptr, false);
}

// Builds: start -> WHILE(hw){ sweep; [gate -> IF(hi){ ‖I-AΣ‖_F }]; check }
int build_loop_graph(ibmi_ctx* c, const LoopState& L, double gate, double rtol, int max_iters, bool frob,
                     cudaGraph_t* out) {
  cudaStream_t st = c->stream;
  const auto mode = cudaStreamCaptureModeThreadLocal;
  cudaGraph_t g = nullptr;
  CUDA_TRY(cudaGraphCreate(&g, 0));
  *out = g;
  cudaGraphConditionalHandle hw;
  CUDA_TRY(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  std::vector<cudaGraphNode_t> deps;
  CUDA_TRY(cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0, mode));
  loop_start_kernel<<<1, 1, 0, st>>>(L); note_launch();
  int rc = frontier(st, deps);
  cudaGraph_t tmp = nullptr;
  CUDA_TRY(cudaStreamEndCapture(st, &tmp));
  if (rc) return rc;
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wnode;
  CUDA_TRY(cudaGraphAddNode(&wnode, g, deps.data(), deps.size(), &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];

  CUDA_TRY(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, mode));
  rc = enqueue_sweep_body(c, rtol, max_iters);
  if (!rc && !frob) {
    loop_check_kernel<<<1, 1, 0, st>>>(hw, L); note_launch();
  }
  cudaGraphConditionalHandle hi = 0;
  if (!rc && frob) {
    if (cudaGraphConditionalHandleCreate(&hi, g, 0, 0) != cudaSuccess) rc = fail(IBMI_ERR_CUDA, "if handle");
    if (!rc) {
      frob_gate_kernel<<<1, 1, 0, st>>>(hi, c->dscal, c->dscal + 3, gate); note_launch();
      rc = frontier(st, deps);
    }
  }
  cudaError_t ec = cudaStreamEndCapture(st, &tmp);
  if (rc) return rc;
  if (ec != cudaSuccess) return fail(IBMI_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(ec));
  if (frob) {
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hi;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t inode;
    CUDA_TRY(cudaGraphAddNode(&inode, body, deps.data(), deps.size(), &ip));
    CUDA_TRY(cudaStreamBeginCaptureToGraph(st, ip.conditional.phGraph_out[0], nullptr, nullptr, 0, mode));
    rc = enqueue_frobenius(c);
    ec = cudaStreamEndCapture(st, &tmp);
    if (rc) return rc;
    if (ec != cudaSuccess) return fail(IBMI_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(ec));
    CUDA_TRY(cudaStreamBeginCaptureToGraph(st, body, &inode, nullptr, 1, mode));
    loop_check_kernel<<<1, 1, 0, st>>>(hw, L); note_launch();
    ec = cudaStreamEndCapture(st, &tmp);
    if (ec != cudaSuccess) return fail(IBMI_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(ec));
  }
  return IBMI_OK;
}

}  // namespace

int ibmi_solve_loop(ibmi_ctx* c, double tol, int max_sweeps, double rtol, int max_iters, int stopping, int* sweeps,
                    int* converged, double* err_trace, int* pow_iters, int* pow_conv, double* resid_trace,
                    double* sweep_ms) {
  NvtxRange nvtx_("ibmi_solve_loop");
  int rc = check_ready(c);
  if (rc) return rc;
  for (auto& s : c->sets)
    if (!s.ready) return fail(IBMI_ERR_STATE, "setup not complete");
  if (max_sweeps < 1 || max_iters < 1) return fail(IBMI_ERR_INVALID, "max_sweeps and max_iters must be >= 1");
  if (stopping < 0 || stopping > 2) return fail(IBMI_ERR_INVALID, "stopping must be 0, 1 or 2");
  const SetDev& last = c->sets.back();
  if (c->p - last.b <= 0) return fail(IBMI_ERR_DIM, "last set covers every index");
  rc = ensure_estimate_buffers(c, last.b, c->p - last.b);
  if (!rc) rc = plan_workspace(c);
  if (!rc && stopping) rc = ensure_frob_buffers(c);
  if (rc) return rc;
  if (c->vr == nullptr || c->vr_n != c->p - last.b) return fail(IBMI_ERR_STATE, "restart vector not set");
  // device trace: err, res (doubles), pit, pconv (ints), ts (u64), it, converged
  const size_t n = (size_t)max_sweeps;
  const size_t bytes = n * 8 * 2 + n * 4 * 2 + (n + 1) * 8 + 16;
  char* buf = nullptr;
  CUDA_TRY(cudaMalloc(&buf, bytes));
  LoopState L;
  L.err = (double*)buf;
  L.res = L.err + n;
  L.ts = (unsigned long long*)(L.res + n);
  L.pit = (int*)(L.ts + n + 1);
  L.pconv = L.pit + n;
  L.it = L.pconv + n;
  L.converged = L.it + 1;
  L.pw = c->dscal;
  L.frob = stopping ? c->dscal + 3 : nullptr;
  L.tol = tol;
  L.max_sweeps = max_sweeps;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
    // mode 1 skips the residual while the estimate (a lower bound of it) is above tol
  const double gate = stopping == 2 ? HUGE_VAL : 1.01 * tol;
  rc = build_loop_graph(c, L, gate, rtol, max_iters, stopping != 0, &g);
  if (!rc) {
    cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
    if (e != cudaSuccess) rc = fail(IBMI_ERR_UNSUPPORTED, std::string("loop graph: ") + cudaGetErrorString(e));
  }
  cudaGetLastError();
  if (!rc) {
    cudaError_t e = cudaGraphLaunch(ge, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) rc = fail(IBMI_ERR_CUDA, cudaGetErrorString(e));
  }
  int h_it = 0, h_conv = 0;
  if (!rc) {
    std::vector<double> err(n), res(n);
    std::vector<int> pit(n), pcv(n);
    std::vector<unsigned long long> ts(n + 1);
    cudaError_t e = cudaMemcpy(&h_it, L.it, 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(&h_conv, L.converged, 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(err.data(), L.err, n * 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(res.data(), L.res, n * 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(pit.data(), L.pit, n * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(pcv.data(), L.pconv, n * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(ts.data(), L.ts, (n + 1) * 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      rc = fail(IBMI_ERR_CUDA, cudaGetErrorString(e));
    } else {
      // every sweep node of the loop ran h_it times
      for (int i = 0; i < h_it; ++i) {
        if (err_trace) err_trace[i] = err[i];
        if (resid_trace) resid_trace[i] = res[i];
        if (pow_iters) pow_iters[i] = pit[i];
        if (pow_conv) pow_conv[i] = pcv[i];
        if (sweep_ms) sweep_ms[i] = (double)(ts[i + 1] - ts[i]) * 1e-6;
      }
    }
  }
  if (ge) cudaGraphExecDestroy(ge);
  if (g) cudaGraphDestroy(g);
  cudaFree(buf);
  if (rc) return rc;
  if (sweeps) *sweeps = h_it;
  if (converged) *converged = h_conv;
  return IBMI_OK;
}

extern "C" {

int ibmi_frobenius_residual(ibmi_ctx* c, double* out) {
  NvtxRange nvtx_("frobenius_residual");
  int rc = check_ready(c);
  if (rc) return rc;
  rc = enqueue_frobenius(c);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(c->hpin + 3, c->dscal + 3, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (out) *out = c->hpin[3];
  return IBMI_OK;
}

int ibmi_device_bytes(ibmi_ctx* c, int64_t* bytes) {
  if (!c || !bytes) return fail(IBMI_ERR_INVALID, "null argument");
  *bytes = (int64_t)c->bytes;
  return IBMI_OK;
}

int ibmi_dgemm_nt(int64_t m, int64_t n, int64_t k, double alpha, const double* x, int64_t ldx, const double* y,
                  int64_t ldy, double beta, double* c, int64_t ldc, void* stream) {
  if (m < 0 || n < 0 || k < 0) return fail(IBMI_ERR_DIM, "negative dimension");
  if (!x || !y || !c) return fail(IBMI_ERR_INVALID, "null pointer");
  if (m > INT_MAX || n > INT_MAX || k > INT_MAX) return fail(IBMI_ERR_DIM, "dimension exceeds int32");
  GemmOp op;
  op.X = x; op.ldx = ldx;
  op.Y = y; op.ldy = ldy;
  op.M = m; op.N = n;
  op.add_seg(0, 0, k);
  op.C = c; op.ldc = ldc;
  op.alpha = alpha; op.beta = beta; op.D = c; op.ldd = ldc;
  CUDA_TRY(launch_gemm(op, (cudaStream_t)stream));
  return IBMI_OK;
}

int ibmi_dgemm_nt_ozaki(int64_t m, int64_t n, int64_t k, double alpha, const double* x, int64_t ldx,
                        const double* y, int64_t ldy, double* c, int64_t ldc, int moduli, void* stream) {
  if (m < 0 || n < 0 || k < 0) return fail(IBMI_ERR_DIM, "negative dimension");
  if (!x || !y || !c) return fail(IBMI_ERR_INVALID, "null pointer");
  if (moduli < OZ_MINN || moduli > OZ_MAXN) return fail(IBMI_ERR_INVALID, "moduli must be in [8, 20]");
  if (m > 65535 || n > INT_MAX || k > (1 << 17)) return fail(IBMI_ERR_DIM, "m <= 65535 and k <= 131072 required");
  if (m == 0 || n == 0) return IBMI_OK;
  GemmOp op;
  op.X = x; op.ldx = ldx;
  op.Y = y; op.ldy = ldy;
  op.M = m; op.N = n;
  op.add_seg(0, 0, k);
  op.C = c; op.ldc = ldc;
  op.alpha = alpha;
  if (k == 0) { op.nseg = 1; op.seg[0] = KSeg{0, 0, 0}; }
  static std::mutex mu;
  static OzWork work;
  static size_t bytes = 0;
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  int sms = 148;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaStreamSynchronize(st));
  int rc = oz_reserve(work, oz_plan(op, moduli), &bytes);
  if (rc) return rc;
  CUDA_TRY(oz_gemm(op, work, moduli, sms, st));
  CUDA_TRY(cudaStreamSynchronize(st));   // the shared workspace is reused by the next call
  return IBMI_OK;
}

int ibmi_emulation_timing(double* ms, double* int8_ops, int* launches) {
  double tms = 0.0, tops = 0.0;
  int nl = 0;
  int rc = IBMI_OK;
  for (auto& e : g_oz_events) {
    float m = 0.0f;
    if (cudaEventSynchronize(e.b) != cudaSuccess || cudaEventElapsedTime(&m, e.a, e.b) != cudaSuccess) rc = IBMI_ERR_CUDA;
    tms += m;
    tops += e.ops;
    ++nl;
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  g_oz_events.clear();
  if (ms) *ms = tms;
  if (int8_ops) *int8_ops = tops;
  if (launches) *launches = nl;
  return rc == IBMI_OK ? IBMI_OK : fail(rc, "event timing failed");
}

int ibmi_set_emulation(ibmi_ctx* c, int moduli) {
  if (!c) return fail(IBMI_ERR_INVALID, "null context");
  if (moduli != 0 && (moduli < OZ_MINN || moduli > OZ_MAXN))
    return fail(IBMI_ERR_INVALID, "moduli must be 0 (FP64 DMMA) or in [8, 20]");
  if (moduli == c->oz_n) return IBMI_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->oz_n = moduli;
  oz_drop_caches(c);
  invalidate_graph(c);
  return IBMI_OK;
}

int ibmi_get_emulation(ibmi_ctx* c, int* moduli) {
  if (!c || !moduli) return fail(IBMI_ERR_INVALID, "null argument");
  *moduli = c->oz_n;
  return IBMI_OK;
}

int ibmi_spd_inverse(int64_t n, const double* a, int64_t lda, double* out, int64_t ldo, int64_t* fail_pivot,
                     void* stream) {
  if (n < 1) return fail(IBMI_ERR_DIM, "matrix must be nonempty");
  if (!a || !out) return fail(IBMI_ERR_INVALID, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  CholScratch cs;
  int rc = ensure_scratch(cs, (int)n);
  if (rc) { cs.release(); return rc; }
  copy2d_kernel<<<grid2d(n, n), 256, 0, st>>>(a, lda, contig_map(0), contig_map(0), cs.ws, cs.ldw, (int)n, (int)n, 1); note_launch();
  int64_t piv = -1;
  rc = potrf_blocked(cs, (int)n, st, &piv);
  if (rc == IBMI_ERR_NOT_SPD && fail_pivot) *fail_pivot = piv;
  if (!rc) rc = potri_blocked(cs, (int)n, out, ldo, st);
  cudaStreamSynchronize(st);
  cs.release();
  return rc;
}

int ibmi_cholesky(int64_t n, const double* a, int64_t lda, double* l, int64_t ldl, int64_t* fail_pivot,
                  void* stream) {
  if (n < 1) return fail(IBMI_ERR_DIM, "matrix must be nonempty");
  if (!a || !l) return fail(IBMI_ERR_INVALID, "null pointer");
  if (lda < n || ldl < n) return fail(IBMI_ERR_DIM, "leading dimension < n");
  cudaStream_t st = (cudaStream_t)stream;
  CholScratch cs;
  int rc = ensure_scratch(cs, (int)n);
  if (rc) { cs.release(); return rc; }
  copy2d_kernel<<<grid2d(n, n), 256, 0, st>>>(a, lda, contig_map(0), contig_map(0), cs.ws, cs.ldw, (int)n, (int)n, 1); note_launch();
  int64_t piv = -1;
  rc = potrf_blocked(cs, (int)n, st, &piv);
  if (rc == IBMI_ERR_NOT_SPD && fail_pivot) *fail_pivot = piv;
  if (!rc) {   // lower factor, strict upper zeroed (dpotrf clean=1, linalg.py:104)
    copy2d_kernel<<<grid2d(n, n), 256, 0, st>>>(cs.ws, cs.ldw, contig_map(0), contig_map(0), l, ldl, (int)n, (int)n, 1);
    note_launch();
  }
  cudaError_t e = cudaStreamSynchronize(st);
  cs.release();
  if (!rc && e != cudaSuccess) return fail(IBMI_ERR_CUDA, cudaGetErrorString(e));
  return rc;
}

int ibmi_chol_solve(int64_t n, const double* l, int64_t ldl, int64_t nrhs, const double* b, int64_t ldb, double* x,
                    int64_t ldx, void* stream) {
  if (n < 1 || nrhs < 1) return fail(IBMI_ERR_DIM, "empty system");
  if (!l || !b || !x) return fail(IBMI_ERR_INVALID, "null pointer");
  if (ldl < n || ldb < nrhs || ldx < nrhs) return fail(IBMI_ERR_DIM, "leading dimension too small");
  cudaStream_t st = (cudaStream_t)stream;
  CholScratch cs;
  int rc = ensure_scratch(cs, (int)n);
  if (rc) { cs.release(); return rc; }
  double* y = nullptr;
  cudaError_t e = cudaMalloc(&y, (size_t)n * nrhs * sizeof(double));
  if (e != cudaSuccess) { cs.release(); return fail(IBMI_ERR_OOM, cudaGetErrorString(e)); }
  // L⁻¹ (lower): diagonal blocks by substitution, then the blocked trtri
  copy2d_kernel<<<grid2d(n, n), 256, 0, st>>>(l, ldl, contig_map(0), contig_map(0), cs.ws, cs.ldw, (int)n, (int)n, 1); note_launch();
  trti2_blocks_kernel<<<(unsigned)((n + CHOL_NB - 1) / CHOL_NB), 256, 0, st>>>(cs.ws, cs.ldw, (int)n, cs.dinv); note_launch();
  rc = trtri_blocked(cs, (int)n, st);
  if (!rc) {
    GemmOp g1;   // y = L⁻¹ b:  y[m][j] = Σ_k L⁻¹[m][k] b[k][j]
    g1.X = cs.ws; g1.ldx = cs.ldw;
    g1.Y = b; g1.ldy = ldb; g1.yt = true;
    g1.M = n; g1.N = nrhs;
    g1.add_seg(0, 0, n);
    g1.C = y; g1.ldc = nrhs;
    e = launch_gemm(g1, st);
    GemmOp g2;   // x = L⁻ᵀ y:  x[m][j] = Σ_k L⁻¹[k][m] y[k][j]
    g2.X = cs.ws; g2.ldx = cs.ldw; g2.xt = true;
    g2.Y = y; g2.ldy = nrhs; g2.yt = true;
    g2.M = n; g2.N = nrhs;
    g2.add_seg(0, 0, n);
    g2.C = x; g2.ldc = ldx;
    if (e == cudaSuccess) e = launch_gemm(g2, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(IBMI_ERR_CUDA, cudaGetErrorString(e));
  }
  cudaStreamSynchronize(st);
  cudaFree(y);
  cs.release();
  return rc;
}

int ibmi_gather(const double* a, int64_t lda, const int64_t* rows, int64_t nr, const int64_t* cols, int64_t nc,
                double* out, int64_t ldo, void* stream) {
  if (nr < 0 || nc < 0) return fail(IBMI_ERR_DIM, "negative index count");
  if (nr == 0 || nc == 0) return IBMI_OK;
  if (!a || !rows || !cols || !out) return fail(IBMI_ERR_INVALID, "null pointer");
  if (ldo < nc) return fail(IBMI_ERR_DIM, "ldo < number of columns");
  cudaStream_t st = (cudaStream_t)stream;
  copy2d_kernel<<<grid2d(nr, nc), 256, 0, st>>>(a, lda, list_map(rows), list_map(cols), out, ldo, (int)nr, (int)nc, 0);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  return IBMI_OK;
}

int ibmi_scatter(double* target, int64_t ldt, const int64_t* rows, int64_t nr, const int64_t* cols, int64_t nc,
                 const double* src, int64_t lds, int add, void* stream) {
  if (nr < 0 || nc < 0) return fail(IBMI_ERR_DIM, "negative index count");
  if (nr == 0 || nc == 0) return IBMI_OK;
  if (!target || !rows || !cols || !src) return fail(IBMI_ERR_INVALID, "null pointer");
  if (lds < nc) return fail(IBMI_ERR_DIM, "lds < number of columns");
  cudaStream_t st = (cudaStream_t)stream;
  scatter_add2d_kernel<<<grid2d(nr, nc), 256, 0, st>>>(src, lds, target, ldt, list_map(rows), list_map(cols), (int)nr,
                                                       (int)nc, add ? 1 : 0);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  return IBMI_OK;
}

int ibmi_sym_rows(const double* base, int64_t ldb, const double* low, int64_t ldl, const int64_t* rows, int64_t nrows,
                  int64_t n, double* dst, int64_t ldd, void* stream) {
  if (nrows < 0 || n < 0) return fail(IBMI_ERR_DIM, "negative size");
  if (nrows == 0 || n == 0) return IBMI_OK;
  if (!base || !low || !rows || !dst) return fail(IBMI_ERR_INVALID, "null pointer");
  if (nrows > INT_MAX || n > INT_MAX || ldd < n || ldb < n || ldl < n) return fail(IBMI_ERR_DIM, "bad leading dimension");
  cudaStream_t st = (cudaStream_t)stream;
  sym_rows_kernel<<<grid2d(nrows, n), 256, 0, st>>>(base, ldb, low, ldl, rows, dst, ldd, (int)nrows, (int)n);
  note_launch();
  CUDA_TRY(cudaGetLastError());
  return IBMI_OK;
}

// Buffers of the stand-alone two_norm, kept per device between calls (the
// sharded sweep calls it once per sweep; no cudaMalloc on that path).
struct NormCache {
  std::mutex mu;
  double *G = nullptr, *vec = nullptr, *part = nullptr, *out = nullptr, *vr = nullptr, *ws = nullptr;
  int64_t g_cap = 0, vec_cap = 0, vr_cap = 0, ws_cap = 0;
  int blocks = 0, threads = 0;
  size_t smem_cap = 0;
  double* host = nullptr;
};
NormCache g_norm[64];

int ibmi_two_norm(int64_t rows, int64_t cols, const double* b, int64_t ldb, const double* restart_v, double rtol,
                  int max_iters, double* sigma, int* iters, int* converged, void* stream) {
  if (rows < 1 || cols < 1) return fail(IBMI_ERR_DIM, "matrix must be nonempty");
  if (!b || !restart_v) return fail(IBMI_ERR_INVALID, "null pointer");
  if (max_iters < 1) return fail(IBMI_ERR_INVALID, "max_iters must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  NormCache& nc = g_norm[dev & 63];
  std::lock_guard<std::mutex> lock(nc.mu);
  if (!nc.blocks) {
    power_launch_shape(dev, &nc.blocks, &nc.threads, &nc.smem_cap);
    CUDA_TRY(cudaMalloc(&nc.part, (size_t)(4 + 32) * nc.blocks * sizeof(double)));   // partials + LL lines
    CUDA_TRY(cudaMalloc(&nc.out, 4 * sizeof(double)));
    CUDA_TRY(cudaMallocHost(&nc.host, 4 * sizeof(double)));
  }
  const int64_t n = std::min(rows, cols);
  const int64_t ldG = round_up(n, 32);
  size_t dummy = 0;
  if (ensure_buf(&nc.G, &nc.g_cap, n * ldG, &dummy)) return IBMI_ERR_OOM;
  if (ensure_buf(&nc.vec, &nc.vec_cap, 2 * std::max(rows, cols), &dummy)) return IBMI_ERR_OOM;
  if (ensure_buf(&nc.vr, &nc.vr_cap, cols, &dummy)) return IBMI_ERR_OOM;
  CUDA_TRY(cudaMemcpyAsync(nc.vr, restart_v, (size_t)cols * sizeof(double), cudaMemcpyHostToDevice, st));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (rows <= cols) {   // split-K workspace of the Gram GEMM G = B Bᵀ (same plan as enqueue_two_norm)
    GemmOp gg;
    gg.M = n; gg.N = n; gg.lower = true;
    gg.add_seg(0, 0, cols);
    const int bk = g_variant == 2 ? 32 : 16;
    const int sp = g_split_gram > 0 ? g_split_gram : auto_split(gemm_tiles(gg), (int)((cols + bk - 1) / bk), sms);
    if (sp > 1 && ensure_buf(&nc.ws, &nc.ws_cap, split_ws_doubles(gemm_tiles(gg), sp), &dummy))
      return IBMI_ERR_OOM;
  }
  NormBufs nb{nc.G, ldG, nc.vec, nc.part, nc.out, nc.vr, nc.blocks, nc.threads, nc.smem_cap, nc.ws, nc.ws_cap, sms};
  int rc = enqueue_two_norm(b, ldb, rows, cols, rtol, max_iters, nb, st);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(nc.host, nc.out, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (sigma) *sigma = nc.host[0];
  if (converged) *converged = nc.host[1] != 0.0;
  if (iters) *iters = (int)nc.host[2];
  return IBMI_OK;
}

static RowMap to_map(const ibmi_map& m) {
  RowMap r;
  r.split = (m.split < 0 || m.split > INT_MAX) ? INT_MAX : (int)m.split;
  r.off0 = m.off0;
  r.off1 = m.off1;
  r.idx = m.idx;
  return r;
}

int ibmi_two_norm_gram(int64_t rows, int64_t cols, const double* b, int64_t ldb, const double* g, int64_t ldg,
                       const double* y1, const double* restart_v, double rtol, int max_iters, double* sigma, int* iters,
                       int* converged, void* stream) {
  if (rows < 1 || cols < 1) return fail(IBMI_ERR_DIM, "matrix must be nonempty");
  if (rows > cols) return fail(IBMI_ERR_DIM, "two_norm_gram needs rows <= cols (row Gram form)");
  if (!b || !g || !y1 || !restart_v) return fail(IBMI_ERR_INVALID, "null pointer");
  if (ldg < rows) return fail(IBMI_ERR_DIM, "ldg < rows");
  if (max_iters < 1) return fail(IBMI_ERR_INVALID, "max_iters must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  NormCache& nc = g_norm[dev & 63];
  std::lock_guard<std::mutex> lock(nc.mu);
  if (!nc.blocks) {
    power_launch_shape(dev, &nc.blocks, &nc.threads, &nc.smem_cap);
    CUDA_TRY(cudaMalloc(&nc.part, (size_t)(4 + 32) * nc.blocks * sizeof(double)));   // partials + LL lines
    CUDA_TRY(cudaMalloc(&nc.out, 4 * sizeof(double)));
    CUDA_TRY(cudaMallocHost(&nc.host, 4 * sizeof(double)));
  }
  size_t dummy = 0;
  if (ensure_buf(&nc.vec, &nc.vec_cap, 2 * std::max(rows, cols), &dummy)) return IBMI_ERR_OOM;
  if (ensure_buf(&nc.vr, &nc.vr_cap, cols, &dummy)) return IBMI_ERR_OOM;
  CUDA_TRY(cudaMemcpyAsync(nc.vr, restart_v, (size_t)cols * sizeof(double), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(nc.vec, y1, (size_t)rows * sizeof(double), cudaMemcpyDeviceToDevice, st));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  NormBufs nb{const_cast<double*>(g), ldg, nc.vec, nc.part, nc.out, nc.vr, nc.blocks, nc.threads, nc.smem_cap,
              nullptr, 0, sms};
  int rc = enqueue_two_norm(b, ldb, rows, cols, rtol, max_iters, nb, st, nullptr, true);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(nc.host, nc.out, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (sigma) *sigma = nc.host[0];
  if (converged) *converged = nc.host[1] != 0.0;
  if (iters) *iters = (int)nc.host[2];
  return IBMI_OK;
}

static int desc_to_op(const ibmi_gemm_desc* d, GemmOp& op) {
  if (!d) return fail(IBMI_ERR_INVALID, "null descriptor");
  if (d->m < 0 || d->n < 0 || d->m > INT_MAX || d->n > INT_MAX) return fail(IBMI_ERR_DIM, "bad m/n");
  if (d->nseg < 0 || d->nseg > 2) return fail(IBMI_ERR_INVALID, "nseg must be 0, 1 or 2");
  if (!d->x || !d->y) return fail(IBMI_ERR_INVALID, "null operand");
  if (!d->frob_out && !d->c && d->direct) return fail(IBMI_ERR_INVALID, "null output");
  if (d->lower && d->m != d->n) return fail(IBMI_ERR_DIM, "lower requires m == n");
  op.X = d->x; op.ldx = d->ldx; op.xm = to_map(d->xm);
  op.Y = d->y; op.ldy = d->ldy; op.yn = to_map(d->yn);
  op.M = d->m; op.N = d->n;
  for (int i = 0; i < d->nseg; ++i) {
    if (d->seg_len[i] < 0 || d->seg_len[i] > INT_MAX) return fail(IBMI_ERR_DIM, "bad segment length");
    op.add_seg(d->seg_x0[i], d->seg_y0[i], d->seg_len[i]);
  }
  op.C = d->c; op.ldc = d->ldc; op.cm = to_map(d->cm); op.cn = to_map(d->cn);
  op.cidx = d->cidx; op.direct = d->direct != 0;
  if (d->mirror) {
    op.mirror = true;
    if (d->c2) { op.c2_set = true; op.C2 = d->c2; op.ldc2 = d->ldc2; op.c2m = to_map(d->c2m); op.c2n = to_map(d->c2n); }
  }
  op.alpha = d->alpha; op.beta = d->beta;
  op.D = d->d; op.ldd = d->ldd; op.dm = to_map(d->dm); op.dn = to_map(d->dn);
  op.lower = d->lower != 0;
  op.tma_ok = d->tma_safe != 0;
  op.xrows = d->xrows; op.xcols = d->xcols; op.yrows = d->yrows; op.ycols = d->ycols;
  op.xt = d->xt != 0;
  op.yt = d->yt != 0;
  if ((op.xt && (op.xm.idx || op.xm.split != INT_MAX)) || (op.yt && (op.yn.idx || op.yn.split != INT_MAX)))
    return fail(IBMI_ERR_INVALID, "transposed operands take contiguous maps only");
  if (d->peers) {
    if (d->bc_panel < 1 || d->bc_world < 1 || d->bc_rank < 0 || d->bc_rank >= d->bc_world || op.cidx)
      return fail(IBMI_ERR_INVALID, "bad peer-store layout");
    op.peers = d->peers; op.bc_panel = d->bc_panel; op.bc_world = d->bc_world; op.bc_rank = d->bc_rank;
  }
  // split-K: explicit factor, or (splits <= 0) the same wave model as the
  // context's own GEMMs; the fixed-order reduction kernel also runs the
  // mirrored and peer-store epilogues.  Not for transposed operands or the
  // Frobenius epilogue.
  if (op.xt || op.yt) op.tma_ok = false;
  if (op.xt || op.yt || d->frob_out) {
    op.splits = 1;
  } else if (d->splits > 0) {
    op.splits = d->splits;
  } else {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    static int sm_of[64] = {0};
    if (dev >= 0 && dev < 64) {
      if (!sm_of[dev]) cudaDeviceGetAttribute(&sm_of[dev], cudaDevAttrMultiProcessorCount, dev);
      sms = sm_of[dev] > 0 ? sm_of[dev] : 148;
    }
    int64_t klen = 0;
    for (int i = 0; i < op.nseg; ++i) klen += op.seg[i].len;
    const int bk = g_variant == 2 ? 32 : 16;
    op.splits = auto_split(gemm_tiles(op), (int)((klen + bk - 1) / bk), sms);
  }
  return IBMI_OK;
}

int ibmi_gemm_workspace(const ibmi_gemm_desc* d, int64_t* doubles) {
  GemmOp op;
  int rc = desc_to_op(d, op);
  if (rc) return rc;
  const int64_t tiles = gemm_tiles(op);
  int64_t need = 0;
  if (d->frob_out) need = tiles;
  else if (op.splits > 1) need = split_ws_doubles(tiles, op.splits);
  if (doubles) *doubles = need;
  return IBMI_OK;
}

int ibmi_gemm(const ibmi_gemm_desc* d, void* stream) {
  GemmOp op;
  int rc = desc_to_op(d, op);
  if (rc) return rc;
  int64_t need = 0;
  ibmi_gemm_workspace(d, &need);
  if (need > 0 && (!d->ws || d->ws_len < need)) return fail(IBMI_ERR_INVALID, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  if (d->frob_out) {
    op.partial = d->ws;
    CUDA_TRY(launch_gemm(op, st));
    reduce_partials_kernel<<<1, 1024, 0, st>>>(d->ws, (int)need, d->frob_out); note_launch();
    CUDA_TRY(cudaGetLastError());
    return IBMI_OK;
  }
  if (op.splits > 1) op.ws = d->ws;
  CUDA_TRY(launch_gemm(op, st));
  return IBMI_OK;
}

int ibmi_export(ibmi_ctx* c, int which, int k, double** ptr, int64_t* rows, int64_t* cols, int64_t* ld) {
  if (!c || !ptr) return fail(IBMI_ERR_INVALID, "null argument");
  if (which == 0) { *ptr = c->A; if (rows) *rows = c->p; if (cols) *cols = c->p; if (ld) *ld = c->ld; return IBMI_OK; }
  if (which == 1) {
    CUDA_TRY(cudaSetDevice(c->device));
    if (int rc = ensure_sigma(c)) return rc;
    *ptr = c->S; if (rows) *rows = c->p; if (cols) *cols = c->p; if (ld) *ld = c->ld; return IBMI_OK;
  }
  if (k < 0 || k >= (int)c->sets.size()) return fail(IBMI_ERR_INVALID, "set index out of range");
  const SetDev& s = c->sets[k];
  if (!s.ready) return fail(IBMI_ERR_STATE, "set not set up");
  if (which == 2) { *ptr = s.W; if (rows) *rows = s.b; if (cols) *cols = c->p; if (ld) *ld = c->ld; return IBMI_OK; }
  if (which == 3) { *ptr = s.ainv; if (rows) *rows = s.b; if (cols) *cols = s.b; if (ld) *ld = s.ldb; return IBMI_OK; }
  return fail(IBMI_ERR_INVALID, "unknown buffer");
}

int ibmi_context_stream(ibmi_ctx* c, void** stream) {
  if (!c || !stream) return fail(IBMI_ERR_INVALID, "null argument");
  *stream = (void*)c->stream;
  return IBMI_OK;
}

int ibmi_release_cached_memory(int device) {
  std::lock_guard<std::mutex> lock(g_mem_mu);
  mem_flush_locked(device);
  return IBMI_OK;
}

int ibmi_cached_bytes(int device, int64_t* bytes) {
  if (!bytes) return fail(IBMI_ERR_INVALID, "null argument");
  std::lock_guard<std::mutex> lock(g_mem_mu);
  size_t t = 0;
  for (int d = 0; d < 64; ++d)
    if (device < 0 || d == device) t += g_mem.free_bytes[d];
  *bytes = (int64_t)t;
  return IBMI_OK;
}

int ibmi_device_alloc(int device, int64_t bytes, void** ptr) {
  if (!ptr || bytes < 0) return fail(IBMI_ERR_INVALID, "bad argument");
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY((cudaMalloc)(ptr, bytes > 0 ? bytes : 8));   // not cached: exported over CUDA IPC
  CUDA_TRY(cudaMemset(*ptr, 0, bytes > 0 ? bytes : 8));
  return IBMI_OK;
}

int ibmi_device_free(void* ptr) {
  if (ptr) CUDA_TRY((cudaFree)(ptr));
  return IBMI_OK;
}

int ibmi_ipc_handle(void* ptr, void* handle) {
  if (!ptr || !handle) return fail(IBMI_ERR_INVALID, "null argument");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, ptr));
  memcpy(handle, &h, sizeof(h));
  return IBMI_OK;
}

int ibmi_ipc_open(int device, const void* handle, void** ptr) {
  if (!ptr || !handle) return fail(IBMI_ERR_INVALID, "null argument");
  CUDA_TRY(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return IBMI_OK;
}

int ibmi_ipc_close(void* ptr) {
  if (ptr) CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return IBMI_OK;
}

int ibmi_load_ibmi1(ibmi_ctx* c, const char* path) {
  if (!c || !path) return fail(IBMI_ERR_INVALID, "null argument");
  int fd = open(path, O_RDONLY);
  if (fd < 0) return fail(IBMI_ERR_IO, std::string(path) + ": cannot open");
  char magic[8];
  uint64_t hdr[2] = {0, 0};
  if (pread(fd, magic, 8, 0) != 8 || memcmp(magic, kMagic, 8) != 0) {
    close(fd);
    return fail(IBMI_ERR_IO, std::string(path) + ": bad magic, expected IBMI1");
  }
  if (pread(fd, hdr, 16, 8) != 16) { close(fd); return fail(IBMI_ERR_IO, std::string(path) + ": truncated header"); }
  const off_t size = lseek(fd, 0, SEEK_END);
  if ((int64_t)hdr[0] != c->p || (int64_t)hdr[1] != c->p) {
    close(fd);
    return fail(IBMI_ERR_DIM, std::string(path) + ": matrix is " + std::to_string(hdr[0]) + "x" +
                                  std::to_string(hdr[1]) + ", context expects " + std::to_string(c->p));
  }
  if ((int64_t)size - 24 != (int64_t)(hdr[0] * hdr[1] * 8)) {
    close(fd);
    return fail(IBMI_ERR_IO, std::string(path) + ": payload size does not match the header");
  }
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaMemsetAsync(c->A, 0, (size_t)c->p * c->ld * sizeof(double), c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  int rc = staged_file(c->A, c->ld, fd, 24, c->p, c->p, true, c->device);
  close(fd);
  if (rc) return rc;
  c->a_set = true;
  for (auto& s : c->sets) s.ready = false;
  invalidate_graph(c);
  rc = symcheck(c, contig_map(0), c->p, "matrix");
  if (rc) { c->a_set = false; return rc; }
  return IBMI_OK;
}

int ibmi_save_sigma_ibmi1(ibmi_ctx* c, const char* path) {
  if (!c || !path) return fail(IBMI_ERR_INVALID, "null argument");
  CUDA_TRY(cudaSetDevice(c->device));
  if (int rc = ensure_sigma(c)) return rc;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  int fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) return fail(IBMI_ERR_IO, std::string(path) + ": cannot create");
  uint64_t hdr[2] = {(uint64_t)c->p, (uint64_t)c->p};
  if (pwrite(fd, kMagic, 8, 0) != 8 || pwrite(fd, hdr, 16, 8) != 16) {
    close(fd);
    return fail(IBMI_ERR_IO, std::string(path) + ": write failed");
  }
  int rc = staged_file(c->S, c->ld, fd, 24, c->p, c->p, false, c->device);
  if (close(fd) != 0 && !rc) rc = fail(IBMI_ERR_IO, std::string(path) + ": close failed");
  return rc;
}

long long ibmi_launch_count(void) { return g_launches.load(); }

int ibmi_tune(int key, int value) {
  switch (key) {
    case 0:
      if (value < 0 || value > 2) return fail(IBMI_ERR_INVALID, "gemm variant must be 0, 1 or 2");
      g_variant = value;
      break;
    case 1:
      if (value < 0 || value > 16) return fail(IBMI_ERR_INVALID, "split must be in [0, 16]");
      g_split_diag = value;
      break;
    case 2:
      if (value < 0 || value > 16) return fail(IBMI_ERR_INVALID, "split must be in [0, 16]");
      g_split_gram = value;
      break;
    case 3:
      g_use_tma = value ? 1 : 0;
      break;
    case 4:
      if (value < 0 || value > 16) return fail(IBMI_ERR_INVALID, "split must be in [0, 16]");
      g_split_panel = value;
      break;
    case 5:
      g_cluster_power = value ? 1 : 0;
      break;
    case 6:
      if (value < 1 || value > 64) return fail(IBMI_ERR_INVALID, "min k-tiles per split must be in [1, 64]");
      g_split_min_kt = value;
      break;
    case 7:
      if (value != 0 && (value < OZ_MINN || value > OZ_MAXN))
        return fail(IBMI_ERR_INVALID, "Ozaki moduli must be 0 (FP64 DMMA) or in [8, 20]");
      g_oz_n = value;
      break;
    case 11:
      g_oz_pair = value ? 1 : 0;
      break;
    case 13:
      g_power_ll = value ? 1 : 0;
      break;
    case 14:
      g_small_fused = value ? 1 : 0;
      break;
    case 15:
      g_split_fused = value ? 1 : 0;
      break;
    case 12:
      if (value < 0 || value > 1024) return fail(IBMI_ERR_INVALID, "raster group must be in [0, 1024]");
      g_raster_group = value;
      break;
    case 10:
      if (value < 1 || value > 16) return fail(IBMI_ERR_INVALID, "Ozaki pipeline chunks must be in [1, 16]");
      g_oz_chunks = value;
      break;
    case 9:
      g_oz_timing = value != 0;
      return IBMI_OK;          // no graph re-capture: timing applies to eager launches only
    case 8:
      if (value < 64) return fail(IBMI_ERR_INVALID, "Ozaki chunk budget must be >= 64 MB");
      g_oz_budget = (double)value * 1048576.0;
      break;
    default:
      return fail(IBMI_ERR_INVALID, "unknown tuning key");
  }
  ++g_tune_gen;
  return IBMI_OK;
}


int ibmi_mc_guess(int64_t p, const double* a, int64_t lda, const double* w, int64_t n, const int64_t* comp,
                  int64_t c, double* out, int64_t ldo, void* stream) {
  if (p < 1 || n < 1 || c < 1) return fail(IBMI_ERR_DIM, "bad sizes");
  if (!a || !w || !comp || !out) return fail(IBMI_ERR_INVALID, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t* dcomp = nullptr;
  CUDA_TRY(cudaMalloc(&dcomp, c * sizeof(int64_t)));
  CUDA_TRY(cudaMemcpyAsync(dcomp, comp, c * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  int rc = mc_guess_into(a, lda, p, w, 0, n, list_map(dcomp), c, out, ldo, contig_map(0), contig_map(0), st);
  cudaFree(dcomp);
  return rc;
}

int ibmi_probe_fp64_peak(int device, double* tflops) {
  if (!tflops) return fail(IBMI_ERR_INVALID, "null argument");
  CUDA_TRY(cudaSetDevice(device));
  int sms = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  const int warps = 8, iters = 20000;
  dmma_probe_kernel<<<sms * 2, warps * 32>>>(d, 200, 1.0000001, 0.999999); note_launch();
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    CUDA_TRY(cudaEventRecord(e0));
    dmma_probe_kernel<<<sms * 2, warps * 32>>>(d, iters, 1.0000001, 0.999999); note_launch();
    CUDA_TRY(cudaEventRecord(e1));
    CUDA_TRY(cudaEventSynchronize(e1));
    float ms;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const double flops = 2.0 * 256 * 8 * (double)iters * warps * sms * 2;
  *tflops = flops / (best * 1e-3) / 1e12;
  return IBMI_OK;
}

}  // extern "C"
