/*
 * ibmi_b200.h — C ABI of the B200-native IBMI sweep (libibmi_b200.so).
 *
 * The reference (arxiv 2502.06377, package `ibmi`, pure Python) has no FFI:
 * its boundary is the Python API re-exported at
 * /root/reference/pkg/src/ibmi/__init__.py:57-77 and the internal seam
 * linalg.py ("the only place that talks to LAPACK/BLAS", linalg.py:1-8)
 * together with the per-set operator _BlockOp (solver.py:109-129).  Each entry
 * point below names the reference function it replaces.  The Python host
 * package `paper_2502_06377_b200` binds these with ctypes and re-exposes the
 * reference's names; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - every function returns an ibmi_status (0 = OK); the message of the last
 *     failure on the calling thread is ibmi_last_error();
 *   - matrices are float64, row-major, leading dimension in elements;
 *     `on_device` = 1 means the pointer is CUDA device memory on the context's
 *     device, 0 means host memory (pinned or pageable);
 *   - a context is one solve: not re-entrant, all work on its stream.
 */
#ifndef IBMI_B200_H
#define IBMI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  IBMI_OK = 0,
  IBMI_ERR_INVALID = 1,        /* bad argument                      -> ValueError            */
  IBMI_ERR_DIM = 2,            /* shapes disagree                   -> DimensionMismatch     */
  IBMI_ERR_INDEX = 3,          /* set outside [0, p)                -> IndexOutOfRange       */
  IBMI_ERR_NOT_SPD = 4,        /* non-positive Cholesky pivot       -> NotPositiveDefinite   */
  IBMI_ERR_NOT_SYMMETRIC = 5,  /* max|a-aT| > 1e-12 max|a|          -> ValueError            */
  IBMI_ERR_CUDA = 6,           /* CUDA runtime failure              -> DeviceError           */
  IBMI_ERR_OOM = 7,            /* device allocation failed          -> OutOfMemoryBudget     */
  IBMI_ERR_STATE = 8,          /* call out of order (e.g. sweep before setup)                */
  IBMI_ERR_UNSUPPORTED = 9,    /* not implemented on this path                               */
  IBMI_ERR_IO = 10             /* file unreadable / malformed       -> IoError               */
} ibmi_status;

typedef enum {
  IBMI_GUESS_IDENTITY = 0,     /* solver.py:158-159                                         */
  IBMI_GUESS_JACOBI = 1,       /* BASELINE c1/c2: Σ0[c1,c1] = diag(1/A_ii) (not in reference) */
  IBMI_GUESS_MATRIX = 2,       /* caller-supplied c1×c1 block (any host-side guess)         */
  IBMI_GUESS_LOCAL = 3,        /* solver.py:162-164: spd_inverse(A[c1,c1]) on the device     */
  IBMI_GUESS_MC = 4,           /* solver.py:167-181: guess = p x ldg standard-normal draws      */
  IBMI_GUESS_TAKAHASHI = 5     /* solver.py:184-212: (A^-1)[c1,c1] = S_c^-1 (needs ibmi_setup)  */
} ibmi_guess;

typedef struct ibmi_ctx ibmi_ctx;

/* Thread-local message of the last failure (never NULL). */
const char* ibmi_last_error(void);
/* Library version string, e.g. "ibmi_b200 0.1.0 sm_100a". */
const char* ibmi_version(void);

/* Create a context for a p×p problem on `device`; `stream` is a cudaStream_t
 * (NULL: the library creates its own non-blocking stream).
 * Replaces the allocation half of solve() (solver.py:233-251). */
int ibmi_create(ibmi_ctx** out, int device, int64_t p, void* stream);
int ibmi_destroy(ibmi_ctx* ctx);

/* Copy A in (host or device), zero the padding, and check symmetry of the
 * whole matrix with the reference's tolerance (linalg.py:68-77).
 * Replaces np.asarray(a, float64) at solver.py:234. */
int ibmi_set_matrix(ibmi_ctx* ctx, const double* a, int64_t lda, int on_device);

/* A straight from an IBMI1 file (reference matio.py:3-47 layout) into HBM:
 * parallel pread into pinned slots, async copies; same checks as set_matrix.
 * Replaces matio.load_matrix (matio.py:74-77) on the `invert` path (cli.py:146). */
int ibmi_load_ibmi1(ibmi_ctx* ctx, const char* path);
/* Σ from HBM straight to an IBMI1 file (replaces matio.save_matrix, cli.py:150). */
int ibmi_save_sigma_ibmi1(ibmi_ctx* ctx, const char* path);

/* K contiguous sets [lo[j], hi[j]); complement of set j is [0,lo) ∪ [hi,p).
 * Replaces the comps/ops construction at solver.py:241-242 (the index
 * validation of partition.py:102-121 stays on the host). */
int ibmi_set_partition(ibmi_ctx* ctx, int k, const int64_t* lo, const int64_t* hi);

/* General partition: set j is set_idx[set_ptr[j] .. set_ptr[j+1]) (ascending,
 * any index sets, overlapping or not — reference partition.py:124-141).  Runs
 * use the contiguous kernels; other sets use device index lists and a K loop
 * over all p columns (W is exactly zero on I). */
int ibmi_set_partition_general(ibmi_ctx* ctx, int k, const int64_t* set_ptr, const int64_t* set_idx);

/* Per set: symmetry check of A_II, Cholesky (dpotrf, linalg.py:104), inverse
 * (dpotrs against I + symmetrise, linalg.py:119,130) and W = A_II⁻¹ A_Ic
 * (solver.py:119-120).  On IBMI_ERR_NOT_SPD, *fail_set / *fail_pivot hold the
 * set and the block-local elimination step (LAPACK info-1, linalg.py:105-106).
 * `first`/`count` select sets (count < 0: all). */
int ibmi_setup(ibmi_ctx* ctx, int first, int count, int* fail_set, int64_t* fail_pivot);

/* Σ = I, then Σ[c1,c1] = guess (solver.py:244-251; JACOBI is the BASELINE
 * extension).  For IBMI_GUESS_MATRIX `guess` is c1×c1 with leading dim ldg. */
int ibmi_init_sigma(ibmi_ctx* ctx, int guess_kind, const double* guess, int64_t ldg, int on_device);

/* Overwrite / read Σ (p×p). get_sigma replaces SolveReport.result (solver.py:277). */
int ibmi_set_sigma(ibmi_ctx* ctx, const double* s, int64_t lds, int on_device);
int ibmi_get_sigma(ibmi_ctx* ctx, double* out, int64_t ldo, int on_device);

/* Host <-> device row copy through the pinned staging pool (several threads),
 * device row r <-> host row host_rows[r] (NULL: r).  Used by the sharded solve
 * to gather Σ's block-cyclic row panels straight into SolveReport.result
 * (solver.py:277) without a host-side permutation pass.  Synchronises `stream`
 * first (the rows are produced on it). */
int ibmi_copy_rows(int device, double* dev, int64_t ldd, double* host, int64_t ldh, int64_t rows, int64_t cols,
                   const int64_t* host_rows, int to_device, void* stream);

/* The normalised default_rng(0x5EED) restart vector of length n used when the
 * power iteration collapses to σ = 0 (linalg.py:237-244). */
int ibmi_set_restart_vector(ibmi_ctx* ctx, int64_t n, const double* v);

/* One block update of set k: M = W Σ_cc; Σ_Ic = −M; Σ_cI = −Mᵀ;
 * Σ_II = A_II⁻¹ + M Wᵀ (symmetric).  Replaces _BlockOp.apply (solver.py:122-129). */
int ibmi_block_update(ibmi_ctx* ctx, int k);

/* ‖Σ_II A_Ic + Σ_Ic A_cc‖₂ for set k by power iteration with the reference's
 * stopping rule.  Replaces error_estimate (solver.py:147-155) and two_norm /
 * _power_sigma_max (linalg.py:223-274).  *converged = 0 means the cap was hit
 * (the caller emits NoConvergenceWarning, linalg.py:267-273). */
int ibmi_error_estimate(ibmi_ctx* ctx, int k, double rtol, int max_iters, double* err, int* iters,
                        int* converged);

/* One sweep: block updates of all sets in order, then the estimate on the last
 * set (solver.py:257-265).  Replayed from a captured CUDA graph. */
int ibmi_sweep(ibmi_ctx* ctx, double rtol, int max_iters, double* err, int* iters, int* converged);

/* As ibmi_sweep without the graph, with per-kernel-class device times in ms
 * (CUDA events on the context stream):
 * times[0] panel GEMMs M=WΣcc, [1] Σ_II GEMMs, [2] estimate GEMM B,
 * [3] Gram GEMM, [4] power iteration, [5] whole sweep. */
int ibmi_sweep_timed(ibmi_ctx* ctx, double rtol, int max_iters, double* err, int* iters, int* converged,
                     float* times);

/* The whole solve loop on the device (solver.py:257-270): a CUDA graph whose
 * conditional WHILE node replays one sweep plus a one-thread check kernel
 * until the estimate (stopping 0) or ‖I − AΣ‖_F (stopping 1, evaluated under a
 * nested IF node only when the estimate allows it; stopping 2, every sweep)
 * is below tol, or max_sweeps.
 * Outputs (host, max_sweeps entries, the first *sweeps valid): the estimate,
 * power iterations / convergence flags, residuals (stopping 1/2; NaN = skipped)
 * and per-sweep device time (ms, %globaltimer).  IBMI_ERR_UNSUPPORTED if the
 * driver cannot build the graph (callers fall back to ibmi_sweep). */
int ibmi_solve_loop(ibmi_ctx* ctx, double tol, int max_sweeps, double rtol, int max_iters, int stopping,
                    int* sweeps, int* converged, double* err_trace, int* pow_iters, int* pow_conv,
                    double* resid_trace, double* sweep_ms);

/* ‖I − AΣ‖_F (BASELINE c2 stopping norm), fused GEMM + reduction. */
int ibmi_frobenius_residual(ibmi_ctx* ctx, double* out);

/* Bytes of device memory held by the context. */
int ibmi_device_bytes(ibmi_ctx* ctx, int64_t* bytes);

/* ---- stand-alone dense building blocks (linalg.py seam), device pointers ---- */

/* C = alpha · X · Yᵀ + beta · C ; X m×k (ldx), Y n×k (ldy), C m×n (ldc).
 * Replaces the `@` products of solver.py:120,124-125,154. */
int ibmi_dgemm_nt(int64_t m, int64_t n, int64_t k, double alpha, const double* x, int64_t ldx,
                  const double* y, int64_t ldy, double beta, double* c, int64_t ldc, void* stream);

/* C = alpha · X · Yᵀ by Ozaki-II emulation: `moduli` (8..20) exact INT8
 * tcgen05 GEMMs of the residues of the row-scaled operands, Chinese
 * remaindering to the exact integer product, one FP64 rounding.  Accurate to
 * 2^-t of each row's largest entry, t = min(62, (log2 Π m - 2 - log2 k) / 2).
 * m <= 65535, k <= 131072.  Synchronises `stream` (shared workspace). */
int ibmi_dgemm_nt_ozaki(int64_t m, int64_t n, int64_t k, double alpha, const double* x, int64_t ldx,
                        const double* y, int64_t ldy, double* c, int64_t ldc, int moduli, void* stream);

/* FP64 emulation of the context's hot GEMMs (panel, Σ_II and error-estimate
 * GEMMs of contiguous sets): moduli = 0 keeps the FP64 DMMA kernels (default);
 * 8..20 runs each of them as that many exact INT8 tcgen05 GEMMs of residues
 * (Ozaki-II, see ibmi_dgemm_nt_ozaki).  Residue planes of the constant
 * operands (W_k, rows of A) are cached when HBM allows. */
int ibmi_set_emulation(ibmi_ctx* ctx, int moduli);
int ibmi_get_emulation(ibmi_ctx* ctx, int* moduli);
/* With ibmi_tune(9, 1), every eagerly launched INT8 residue GEMM is bracketed
 * by CUDA events on its stream; this returns (and clears) their summed device
 * time, algorithmic INT8 ops and launch count (the emulated roofline). */
int ibmi_emulation_timing(double* ms, double* int8_ops, int* launches);

/* out = A⁻¹ for SPD A (n×n) via blocked Cholesky; replaces spd_inverse
 * (linalg.py:122-130).  On IBMI_ERR_NOT_SPD *fail_pivot = elimination step. */
int ibmi_spd_inverse(int64_t n, const double* a, int64_t lda, double* out, int64_t ldo, int64_t* fail_pivot,
                     void* stream);

/* Lower Cholesky factor of SPD A (device n×n) into l (strict upper zeroed);
 * replaces cholesky (linalg.py:96-109, dpotrf lower clean=1).  Reads only the
 * lower triangle (the caller checks symmetry, linalg.py:68-77).  On
 * IBMI_ERR_NOT_SPD *fail_pivot = the failing elimination step (info − 1). */
int ibmi_cholesky(int64_t n, const double* a, int64_t lda, double* l, int64_t ldl, int64_t* fail_pivot,
                  void* stream);

/* x = (L Lᵀ)⁻¹ b for a lower factor l (device n×n) and b (device n×nrhs);
 * replaces chol_solve (linalg.py:112-119, dpotrs): L⁻¹ by blocked trtri, then
 * two GEMMs. */
int ibmi_chol_solve(int64_t n, const double* l, int64_t ldl, int64_t nrhs, const double* b, int64_t ldb, double* x,
                    int64_t ldx, void* stream);

/* out[i][j] = a[rows[i]][cols[j]] (device arrays); replaces gather
 * (linalg.py:186-191).  Indices are checked by the caller (_check_indices). */
int ibmi_gather(const double* a, int64_t lda, const int64_t* rows, int64_t nr, const int64_t* cols, int64_t nc,
                double* out, int64_t ldo, void* stream);

/* target[rows[i]][cols[j]] = (add ? target[..] : 0) + src[i][j] (device arrays);
 * replaces scatter_add_assign (linalg.py:194-211).  The grid must not repeat an
 * element: the caller resolves repeated indices to their last occurrence, which
 * is what NumPy's fancy assignment keeps. */
int ibmi_scatter(double* target, int64_t ldt, const int64_t* rows, int64_t nr, const int64_t* cols, int64_t nc,
                 const double* src, int64_t lds, int add, void* stream);

/* Monte Carlo guess block (solver.py:167-181) for any ordering: A (device, p×p),
 * w (host, p×n standard-normal draws of default_rng(mc_seed)), comp (host, c
 * ascending indices); out (device, c×c) = (L⁻ᵀw)_c (L⁻ᵀw)_cᵀ / n. */
int ibmi_mc_guess(int64_t p, const double* a, int64_t lda, const double* w, int64_t n, const int64_t* comp,
                  int64_t c, double* out, int64_t ldo, void* stream);

/* ‖B‖₂ of a device matrix (rows×cols, ldb) by power iteration with the
 * reference's stopping rule; replaces two_norm (linalg.py:256-274).
 * `restart_v` (host, length cols) is the normalised default_rng(0x5EED) draw. */
int ibmi_two_norm(int64_t rows, int64_t cols, const double* b, int64_t ldb, const double* restart_v, double rtol,
                  int max_iters, double* sigma, int* iters, int* converged, void* stream);

/* The same power iteration on a Gram matrix the caller already holds (rows <= cols):
 * g = b·bᵀ (device rows × rows, full symmetric storage) and y1 = b·(1/√cols)·1 (device, rows).
 * The sharded sweep forms g from per-rank partial products over column chunks of b and one
 * all-reduce instead of a replicated rows² × cols product; b itself is only
 * read on the σ = 0 restart path (linalg.py:237-244). */
int ibmi_two_norm_gram(int64_t rows, int64_t cols, const double* b, int64_t ldb, const double* g, int64_t ldg,
                       const double* y1, const double* restart_v, double rtol, int max_iters, double* sigma, int* iters,
                       int* converged, void* stream);

/* ---- composable pieces for the sharded (multi-GPU) sweep ---- */

/* One-gap index map: logical i -> (i < split ? off0 + i : off1 + (i - split)),
 * or, when idx != NULL, logical i -> idx[i] (device array, rows only on the
 * cp.async path).  A contiguous run starting at o is {INT64_MAX, o, 0, NULL}. */
typedef struct {
  int64_t split, off0, off1;
  const int64_t* idx;
} ibmi_map;

/* General NT GEMM on device pointers (the kernels behind every call above):
 *   v(m,n) = alpha * sum_k X(xm(m), k) * Y(yn(n), k) + beta * D(dm(m), dn(n))
 * over up to two K segments [x0, x0+len) (in X) paired with [y0, y0+len) (in Y);
 *   direct: C[cidx ? cidx[m] : cm(m)][cn(n)] = v;   mirror: C2[c2n(n)][c2m(m)] = v;
 *   lower: only the lower triangle (M == N);  frob_out != NULL: instead of storing,
 *   frob_out[0] = sqrt(sum (delta(row(m), cn(n)) - acc)^2), frob_out[1] = the sum.
 * xrows/xcols/yrows/ycols are the operands' physical extents; tma_safe = 1 allows
 * the TMA kernel (per-segment tensor maps end at the segment end, so boxes
 * past it are zero-filled by the hardware).  `ws` (ws_len doubles, may be NULL) is
 * scratch for split-K / reduction partials; ibmi_gemm_workspace gives the size. */
typedef struct {
  const double* x; int64_t ldx; ibmi_map xm; int64_t xrows, xcols;
  const double* y; int64_t ldy; ibmi_map yn; int64_t yrows, ycols;
  int64_t m, n;
  int nseg; int64_t seg_x0[2], seg_y0[2], seg_len[2];
  double* c; int64_t ldc; ibmi_map cm, cn; const int64_t* cidx; int direct;
  double* c2; int64_t ldc2; ibmi_map c2m, c2n; int mirror;
  double alpha, beta; const double* d; int64_t ldd; ibmi_map dm, dn;
  int lower, tma_safe, splits;   /* splits: split-K factor, <= 0 = automatic (wave model) */
  double* frob_out;
  double* ws; int64_t ws_len;
  /* fused exchange (sharded sweep): when peers != NULL every element (m, n) is
   * also stored to peers[h][lr * ldc2 + gc] with r = c2m(m) (global row),
   * h = (r/T)%G, lr = (r/(T*G))*T + r%T, l = c2n(n) (local row of bc_rank),
   * gc = ((l/T)*G + bc_rank)*T + l%T, T = bc_panel, G = bc_world — straight
   * into the owner's row panel through NVLink peer pointers (IPC-mapped). */
  double* const* peers; int64_t bc_panel; int bc_world, bc_rank;
  /* transposed operands: X(m, k) = x[(x0 + k) * ldx + xm.off0 + m] (likewise Y);
   * contiguous maps only, cp.async kernel. */
  int xt, yt;
} ibmi_gemm_desc;

int ibmi_gemm(const ibmi_gemm_desc* desc, void* stream);
int ibmi_gemm_workspace(const ibmi_gemm_desc* desc, int64_t* doubles);

/* Rows of the symmetric block update from an all-reduced lower triangle (the
 * sharded Σ_II = sym(A_II⁻¹ + M·Wᵀ), solver.py:125-127):
 * dst[i][j] = base[r][j] + (j <= r ? low[r][j] : low[j][r]), r = rows[i] (device int64).
 * Stream-ordered, no synchronisation (graph-capturable). */
int ibmi_sym_rows(const double* base, int64_t ldb, const double* low, int64_t ldl, const int64_t* rows, int64_t nrows,
                  int64_t n, double* dst, int64_t ldd, void* stream);

/* The CUDA stream the context's work is ordered on (its own non-blocking
 * stream, or the one passed to ibmi_create). */
int ibmi_context_stream(ibmi_ctx* ctx, void** stream);

/* Device pointer, shape and leading dimension of a context buffer:
 * which = 0 A, 1 Σ, 2 W_k (b_k × ld, global columns), 3 A_II⁻¹ of set k. */
int ibmi_export(ibmi_ctx* ctx, int which, int k, double** ptr, int64_t* rows, int64_t* cols, int64_t* ld);

/* Device memory for peer-visible buffers and its CUDA IPC handle (64 bytes),
 * opened by the other ranks of the node for the fused exchange. */
int ibmi_device_alloc(int device, int64_t bytes, void** ptr);
int ibmi_device_free(void* ptr);
int ibmi_ipc_handle(void* ptr, void* handle64);
int ibmi_ipc_open(int device, const void* handle64, void** ptr);
int ibmi_ipc_close(void* ptr);

/* Device block cache (the library's allocator): buffers freed by destroyed
 * contexts stay reserved per device and are reused by the next context of a
 * similar shape, instead of paying cudaFree/cudaMalloc of GB-sized blocks per
 * solve.  Capped at a quarter of device memory (env IBMI_MEM_CACHE_MB; 0 turns
 * it off).  No reference counterpart: the reference allocates with NumPy
 * (solver.py:250, :120).  release: return device `device`'s cached blocks to
 * the driver (device < 0: all devices); cached: bytes currently held. */
int ibmi_release_cached_memory(int device);
int ibmi_cached_bytes(int device, int64_t* bytes);

/* Number of kernels this library has launched in the process (graph replays
 * count their kernel nodes) — the `gpu_launches` of bench.py. */
long long ibmi_launch_count(void);

/* Tuning knobs (process-wide; contexts re-capture their sweep graph):
 * key 0: GEMM configuration of the hot NT kernels (0: 8 warps 64x32, BK16;
 *        1: 16 warps 32x32, BK16 [default]; 2: 16 warps 32x32, BK32);
 * key 1: split-K factor of the Σ_II GEMM (0 = auto); key 2: of the Gram GEMM;
 * key 3: TMA/mbarrier kernel on/off; key 4: split-K of the panel and estimate GEMMs;
 * key 5: cluster (DSMEM) power iteration for Gram order <= 640 on/off;
 * key 6: minimum k-tiles per split-K slice (default 4);
 * key 7: default of ibmi_set_emulation for contexts created afterwards
 *        (0 = FP64 DMMA, 8..20 = Ozaki-II moduli);
 * key 8: Ozaki residue-plane budget per N chunk, MB (default 5722 = 6e9 B);
 * key 9: event-time the INT8 GEMM launches (ibmi_emulation_timing) on/off;
 * key 10: N chunks of the two-stream emulated GEMM pipeline (default 1 = no overlap:
 *         the conversion shares the L1/shared-memory datapath with the INT8
 *         GEMM's operand reads, so overlapping them gained nothing);
 * key 11: INT8 GEMM on CTA pairs (cta_group::2, default 1) or single CTAs (0);
 * key 12: FP64 GEMM tile raster: bands of this many 128-row tile rows walked column by
 *         column (default 0 = tile-row-major);
 * key 13: power iteration of mid-size Gram matrices (512 <= n <= 2220) with the
 *         flag-carrying line exchange instead of a grid barrier per iteration (default 1);
 * key 14: p <= 1024 (FP64 DMMA, contiguous sets): ibmi_sweep / ibmi_solve_loop run the K block updates,
 *         the estimate matrix and its Gram form as one cooperative kernel (default 1);
 * key 15: split-K GEMMs on the TMA kernel reduce their partial tiles inside the GEMM (the split
 *         that arrives last at a tile sums them in split order and runs the epilogue) instead of
 *         a separate reduction launch (default 0: measured 1-4% slower than the reduction kernel,
 *         DESIGN.md §3; same bits either way). */
int ibmi_tune(int key, int value);

/* Measured FP64 DMMA throughput of `device` (TFLOP/s), the roofline denominator. */
int ibmi_probe_fp64_peak(int device, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* IBMI_B200_H */
