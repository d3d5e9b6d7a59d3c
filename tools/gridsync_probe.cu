// Grid-barrier cost on B200 (the floor of the power iteration).
//   A: grid.sync() only;  B: partial write + grid.sync() + warp-0 read of all
//   partials (what one power iteration does besides the matvec);
//   C: the same exchange with clusters of 4: DSMEM reduce inside the cluster,
//   cluster leaders' partials through L2, cooperative launch with clusters.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gridsync_probe tools/gridsync_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(512, 1) k_sync(int iters, double* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

__global__ void __launch_bounds__(512, 1) k_exchange(int iters, double* part, double* sink) {
  cg::grid_group g = cg::this_grid();
  __shared__ double bc;
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    double* pp = part + (i & 1) * gridDim.x;
    if (threadIdx.x == 0) pp[blockIdx.x] = acc + blockIdx.x;
    g.sync();
    if (threadIdx.x < 32) {
      double s = 0.0;
      for (int j = threadIdx.x; j < (int)gridDim.x; j += 32) s += __ldcg(pp + j);
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (threadIdx.x == 0) bc = s;
    }
    __syncthreads();
    acc = bc * 1e-9;
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = acc;
}

__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(512, 1) k_cluster(int iters, double* part, double* sink) {
  cg::grid_group g = cg::this_grid();
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double mine, bc;
  const int nl = gridDim.x / 4;
  const int leader = blockIdx.x / 4;
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    double* pp = part + (i & 1) * nl;
    if (threadIdx.x == 0) mine = acc + blockIdx.x;
    cl.sync();
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
      double s = 0.0;
      for (int r = 0; r < 4; ++r) s += *cl.map_shared_rank(&mine, r);
      pp[leader] = s;
    }
    g.sync();
    if (threadIdx.x < 32) {
      double s = 0.0;
      for (int j = threadIdx.x; j < nl; j += 32) s += __ldcg(pp + j);
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (threadIdx.x == 0) bc = s;
    }
    __syncthreads();
    acc = bc * 1e-9;
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *part, *sink;
  cudaMalloc(&part, 4096 * sizeof(double));
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  float ms;
  {
    int it = iters;
    void* args[] = {&it, &sink};
    cudaLaunchCooperativeKernel((void*)k_sync, sms, 512, args, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_sync, sms, 512, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("A grid.sync only, %d CTAs: %.3f us/iter (%s)\n", sms, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  {
    int it = iters;
    void* args[] = {&it, &part, &sink};
    cudaLaunchCooperativeKernel((void*)k_exchange, sms, 512, args, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_exchange, sms, 512, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("B partials + grid.sync + read, %d CTAs: %.3f us/iter (%s)\n", sms, ms * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  {
    int ncl = 0;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = 4; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
    cfg.blockDim = dim3(512);
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cfg.gridDim = dim3(sms / 4 * 4);
    cudaOccupancyMaxActiveClusters(&ncl, (void*)k_cluster, &cfg);
    cfg.gridDim = dim3(ncl * 4);
    cfg.numAttrs = 1;   // cluster dims come from __cluster_dims__
    int it = iters;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cluster, it, part, sink);
    cudaEventRecord(e0);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, k_cluster, it, part, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("C clusters of 4 (%d clusters, %d CTAs): %.3f us/iter (%s / %s)\n", ncl, ncl * 4, ms * 1e3 / iters,
           cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
