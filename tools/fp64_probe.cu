// FP64 throughput probe for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) vs DFMA vs mixed.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; i++) { c[i][0] = threadIdx.x; c[i][1] = i; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
template <int CH>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double c[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) c[i] = threadIdx.x + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += c[i];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  for (int warps : {4, 8, 16}) {
    for (int rep = 0; rep < 2; rep++) {
      int iters = 20000;
      k_dmma<8><<<sms * 2, warps * 32>>>(d, 100, 1.0000001, 0.999999);
      cudaEventRecord(e0);
      k_dmma<8><<<sms * 2, warps * 32>>>(d, iters, 1.0000001, 0.999999);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)iters * warps * sms * 2;  // 8x8x4=256 FMA
      printf("DMMA warps/CTA=%d 2CTA/SM: %.2f TFLOP/s (%.3f ms)\n", warps, flops / ms / 1e9, ms);
    }
  }
  for (int warps : {8, 16, 32}) {
    int iters = 20000;
    k_dfma<8><<<sms * 2, warps * 32>>>(d, 100, 1.0000001, 0.999999);
    cudaEventRecord(e0);
    k_dfma<8><<<sms * 2, warps * 32>>>(d, iters, 1.0000001, 0.999999);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * warps * 32 * sms * 2;
    printf("DFMA warps/CTA=%d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
