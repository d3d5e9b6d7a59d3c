// Standalone probe of the tcgen05 INT8 GEMM (csrc/igemm_tc.cuh): exactness
// against a scalar int32 reference and throughput at the c4 panel shape.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -o tools/igemm_probe tools/igemm_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2502_06377_b200/csrc/igemm_tc.cuh"
#include "../paper_2502_06377_b200/csrc/ozaki.cuh"

using namespace ibmi;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;

static void make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)IG_BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
}

__global__ void ref_kernel(const int8_t* x, const int8_t* y, int M, int N, int K, int64_t ld, int32_t* c) {
  int n = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
  if (n >= N) return;
  int32_t s = 0;
  for (int k = 0; k < K; ++k) s += (int32_t)x[(int64_t)m * ld + k] * (int32_t)y[(int64_t)n * ld + k];
  c[(int64_t)m * N + n] = s;
}

__global__ void fill_kernel(int8_t* p, int64_t n, uint32_t seed) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    p[i] = (int8_t)(h & 0xff);
  }
}

int g_pair = 0;
int run(int M, int N, int K, int planes, int mod, bool check, int reps) {
  const int64_t ld = (K + 15) / 16 * 16;
  const int64_t rx = (int64_t)(M + 255) / 256 * 256, ry = (int64_t)(N + IG_BN - 1) / IG_BN * IG_BN;
  int8_t *x, *y;
  CK(cudaMalloc(&x, rx * ld * planes));
  CK(cudaMalloc(&y, ry * ld * planes));
  CK(cudaMemset(x, 0, rx * ld * planes));
  CK(cudaMemset(y, 0, ry * ld * planes));
  fill_kernel<<<1024, 256>>>(x, rx * ld * planes, 1234);
  fill_kernel<<<1024, 256>>>(y, ry * ld * planes, 99);
  // zero K padding columns and padding rows of every plane so planes are exact
  CK(cudaDeviceSynchronize());
  {
    std::vector<int8_t> hx(rx * ld * planes), hy(ry * ld * planes);
    CK(cudaMemcpy(hx.data(), x, hx.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hy.data(), y, hy.size(), cudaMemcpyDeviceToHost));
    for (int l = 0; l < planes; ++l) {
      for (int64_t r = 0; r < rx; ++r)
        for (int64_t k = 0; k < ld; ++k)
          if (r >= M || k >= K) hx[(l * rx + r) * ld + k] = 0;
      for (int64_t r = 0; r < ry; ++r)
        for (int64_t k = 0; k < ld; ++k)
          if (r >= N || k >= K) hy[(l * ry + r) * ld + k] = 0;
    }
    CK(cudaMemcpy(x, hx.data(), hx.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(y, hy.data(), hy.size(), cudaMemcpyHostToDevice));
  }
  CUtensorMap mx, my;
  make_map(&mx, x, rx * planes, K, ld, IG_BM);
  make_map(&my, y, ry * planes, K, ld, 128);
  IgemmParams P{};
  P.M = M;
  P.N = N;
  P.K = K;
  P.tiles_m = (M + IG_BM - 1) / IG_BM;
  P.tiles_n = (N + IG_BN - 1) / IG_BN;
  P.planes = planes;
  P.rows_per_plane_x = (int)rx;
  P.rows_per_plane_y = (int)ry;
  const int64_t ldr = (N + 15) / 16 * 16;
  uint8_t* R;
  int32_t* C32;
  CK(cudaMalloc(&R, (int64_t)M * ldr * planes));
  CK(cudaMalloc(&C32, (int64_t)M * N * 4));
  P.R = R;
  P.ldr = ldr;
  P.r_plane = (int64_t)M * ldr;
  P.C32 = C32;
  P.ldc32 = N;
  for (int l = 0; l < planes; ++l) P.mod[l] = mod;
  CK(cudaFuncSetAttribute(igemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)IG_SMEM));
  CK(cudaFuncSetAttribute(igemm_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)IG2_SMEM));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int total = P.tiles_m * P.tiles_n * planes;
  if (g_pair) total = 2 * ((M + 255) / 256) * ((N + 255) / 256) * planes;
  int grid = total < sms ? total : sms;
  if (g_pair) grid = grid < 2 ? 2 : (grid & ~1);
  auto launch = [&]() {
    if (g_pair) igemm_tc2_kernel<<<grid, IG_THREADS, IG2_SMEM>>>(mx, my, P);
    else igemm_tc_kernel<<<grid, IG_THREADS, IG_SMEM>>>(mx, my, P);
  };
  launch();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  int bad = 0;
  if (check) {
    int32_t* Cr;
    CK(cudaMalloc(&Cr, (int64_t)M * N * 4));
    ref_kernel<<<dim3((N + 127) / 128, M), 128>>>(x, y, M, N, K, ld, Cr);
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> a((int64_t)M * N), b((int64_t)M * N);
    CK(cudaMemcpy(b.data(), Cr, b.size() * 4, cudaMemcpyDeviceToHost));
    if (mod == 0) {
      CK(cudaMemcpy(a.data(), C32, a.size() * 4, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < (int64_t)M * N; ++i)
        if (a[i] != b[i]) {
          if (bad < 5) printf("  mismatch at %lld,%lld: %d vs %d\n", (long long)(i / N), (long long)(i % N), a[i], b[i]);
          ++bad;
        }
    } else {
      std::vector<uint8_t> rr((int64_t)M * ldr);
      CK(cudaMemcpy(rr.data(), R, rr.size(), cudaMemcpyDeviceToHost));
      for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
          int e = b[m * N + n] % mod;
          if (e < 0) e += mod;
          if (rr[m * ldr + n] != e) {
            if (bad < 5) printf("  mismatch at %lld,%lld: %d vs %d\n", (long long)m, (long long)n, rr[m * ldr + n], e);
            ++bad;
          }
        }
    }
    CK(cudaFree(Cr));
  }
  float ms = 0;
  if (reps > 0) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int i = 0; i < 2; ++i) launch();
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
  }
  const double ops = 2.0 * M * N * (double)K * planes;
  printf("%s M=%d N=%d K=%d planes=%d mod=%d grid=%d: %s%d bad; %.3f ms  %.1f TOPS\n", g_pair ? "pair" : "1cta", M, N, K, planes, mod, grid,
         check ? "" : "(unchecked) ", bad, ms, reps > 0 ? ops / ms * 1e-9 : 0.0);
  CK(cudaFree(x));
  CK(cudaFree(y));
  CK(cudaFree(R));
  CK(cudaFree(C32));
  return bad;
}

// concurrency check: INT8 GEMM on one stream, residue split (ALU-bound) on another
void concurrency() {
  const int M = 2560, N = 14080, K = 14080, planes = 16;
  const int64_t ld = K;
  int8_t *x, *y;
  CK(cudaMalloc(&x, (int64_t)M * ld * planes));
  CK(cudaMalloc(&y, (int64_t)N * ld * planes));
  CK(cudaMemset(x, 1, (int64_t)M * ld * planes));
  CK(cudaMemset(y, 1, (int64_t)N * ld * planes));
  CUtensorMap mx, my;
  make_map(&mx, x, (int64_t)M * planes, K, ld, IG_BM);
  make_map(&my, y, (int64_t)N * planes, K, ld, IG_BN);
  IgemmParams P{};
  P.M = M; P.N = N; P.K = K;
  P.tiles_m = M / IG_BM; P.tiles_n = (N + IG_BN - 1) / IG_BN; P.planes = planes;
  P.rows_per_plane_x = M; P.rows_per_plane_y = N;
  uint8_t* R;
  CK(cudaMalloc(&R, (int64_t)M * N * planes));
  P.R = R; P.ldr = N; P.r_plane = (int64_t)M * N;
  for (int l = 0; l < planes; ++l) P.mod[l] = 251;
  // split workload: 198M doubles -> 16 planes
  const int64_t rows = 14080, cols = 14080;
  double* src;
  int8_t* q;
  int* ex;
  CK(cudaMalloc(&src, rows * cols * 8));
  CK(cudaMemset(src, 0, rows * cols * 8));
  CK(cudaMalloc(&q, rows * cols * 16));
  CK(cudaMalloc(&ex, rows * 4));
  CK(cudaMemset(ex, 0, rows * 4));
  CK(cudaFuncSetAttribute(igemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)IG_SMEM));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  RowMap rm{INT_MAX, 0, 0, nullptr};
  auto gemm = [&](cudaStream_t s) { igemm_tc_kernel<<<148, IG_THREADS, IG_SMEM, s>>>(mx, my, P); };
  auto split = [&](cudaStream_t s, dim3 sg) {
    oz_split_kernel<16><<<sg, 256, 0, s>>>(src, cols, rm, rm, (int)rows, (int)cols, ex, q, cols, rows * cols);
  };
  CK(cudaFuncSetAttribute(oz_split_kernel<16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  for (int bps : {2, 3, 4}) {
  dim3 sg(148 * bps);
  printf("split grid %d blocks\n", 148 * bps);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float t;
  for (int w = 0; w < 2; ++w) { gemm(s1); split(s1, sg); }
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a, s1)); gemm(s1); CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&t, a, b)); printf("igemm alone: %.3f ms\n", t);
  CK(cudaEventRecord(a, s1)); split(s1, sg); CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&t, a, b)); printf("split alone: %.3f ms\n", t);
  CK(cudaEventRecord(a, s1)); gemm(s1); split(s1, sg); CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&t, a, b)); printf("serial: %.3f ms\n", t);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a, s1)); CK(cudaStreamWaitEvent(s2, a, 0));
  gemm(s1); split(s2, sg);
  cudaEvent_t c2; CK(cudaEventCreate(&c2)); CK(cudaEventRecord(c2, s2)); CK(cudaStreamWaitEvent(s1, c2, 0));
  CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&t, a, b)); printf("concurrent (gemm first): %.3f ms\n", t);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a, s1)); CK(cudaStreamWaitEvent(s2, a, 0));
  split(s2, sg); gemm(s1);
  CK(cudaEventRecord(c2, s2)); CK(cudaStreamWaitEvent(s1, c2, 0));
  CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&t, a, b)); printf("concurrent (split first): %.3f ms\n", t);
  CK(cudaDeviceSynchronize());
  }
}

int main(int argc, char** argv) {
  if (argc > 1) { cudaDriverEntryPointQueryResult q0; CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q0)); concurrency(); return 0; }
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  int bad = 0;
  for (g_pair = 0; g_pair < 2; ++g_pair) {
  bad += run(128, 256, 128, 1, 0, true, 0);
  bad += run(256, 512, 1024, 1, 0, true, 0);
  bad += run(300, 700, 1000, 1, 0, true, 0);
  bad += run(1000, 1100, 2000, 2, 251, true, 0);
  bad += run(640, 1280, 4096, 3, 256, true, 0);
  printf("correctness: %s\n", bad ? "FAIL" : "ok");
  run(2560, 14080, 14080, 1, 251, false, 5);
  run(2560, 14080, 14080, 4, 251, false, 3);
  run(8192, 8192, 8192, 1, 0, false, 5);
  run(8192, 8192, 8192, 1, 251, false, 5);
  }
  return bad ? 1 : 0;
}
