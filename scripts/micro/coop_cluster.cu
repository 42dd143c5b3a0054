// Can a persistent kernel with compile-time clusters be launched cooperatively (the
// co-residency guarantee the grid-wide spin-waits of K1/K2 need), and what does the
// occupancy API report? Build: nvcc -gencode arch=compute_100a,code=sm_100a -o coop_cluster coop_cluster.cu
#include <cooperative_groups.h>
#include <cstdio>

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) k_cluster(int* ctr, int n) {
  if (threadIdx.x == 0) {
    atomicAdd(ctr, 1);
    long long t0 = clock64();
    while (atomicAdd(ctr, 0) < n) {
      if (clock64() - t0 > 4000000000ll) { atomicAdd(ctr + 1, 1); break; }
    }
  }
}

__global__ void __launch_bounds__(256, 1) k_plain(int* ctr, int n) {
  if (threadIdx.x == 0) {
    atomicAdd(ctr, 1);
    long long t0 = clock64();
    while (atomicAdd(ctr, 0) < n) {
      if (clock64() - t0 > 4000000000ll) { atomicAdd(ctr + 1, 1); break; }
    }
  }
}

template <class K>
void run(const char* name, K k, int grid, int smem, bool coop, bool cluster_attr) {
  int* ctr;
  cudaMalloc(&ctr, 8);
  cudaMemset(ctr, 0, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (coop) {
    at[n].id = cudaLaunchAttributeCooperative;
    at[n].val.cooperative = 1;
    ++n;
  }
  if (cluster_attr) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = 2;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, ctr, grid);
  cudaError_t e2 = cudaDeviceSynchronize();
  int h[2] = {0, 0};
  cudaMemcpy(h, ctr, 8, cudaMemcpyDeviceToHost);
  printf("%-8s grid=%4d smem=%6d coop=%d clattr=%d launch=%s sync=%s arrived=%d timeouts=%d\n", name, grid, smem,
         coop, cluster_attr, cudaGetErrorString(e), cudaGetErrorString(e2), h[0], h[1]);
  cudaGetLastError();
  cudaFree(ctr);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  int clusters = -1;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&clusters, k_cluster, &cfg);
  printf("SMs=%d maxActiveClusters(2-CTA, %d B smem)=%d (%s)\n", sms, smem, clusters, cudaGetErrorString(e));
  int blocks = -1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_plain, 256, smem);
  printf("plain blocks/SM=%d\n", blocks);
  run("cluster", k_cluster, 2 * clusters, smem, true, false);
  run("cluster", k_cluster, 2 * clusters, smem, true, true);
  run("cluster", k_cluster, 2 * clusters, smem, false, false);
  run("cluster", k_cluster, 2 * clusters + 2, smem, true, false);
  run("plain", k_plain, sms, smem, true, false);
  run("plain", k_plain, sms + 1, smem, true, false);
  // two cooperative grids on two streams, each sized to the whole device: must serialize, not deadlock
  {
    int *c1, *c2;
    cudaMalloc(&c1, 8);
    cudaMalloc(&c2, 8);
    cudaMemset(c1, 0, 8);
    cudaMemset(c2, 0, 8);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cudaLaunchConfig_t c{};
    c.gridDim = dim3(2 * clusters);
    c.blockDim = dim3(256);
    c.dynamicSmemBytes = smem;
    c.attrs = at;
    c.numAttrs = 1;
    c.stream = s1;
    cudaError_t a = cudaLaunchKernelEx(&c, k_cluster, c1, 2 * clusters);
    c.stream = s2;
    cudaError_t b = cudaLaunchKernelEx(&c, k_cluster, c2, 2 * clusters);
    cudaError_t d = cudaDeviceSynchronize();
    int h1[2], h2[2];
    cudaMemcpy(h1, c1, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2, c2, 8, cudaMemcpyDeviceToHost);
    printf("two coop grids on two streams: %s %s sync=%s timeouts %d %d\n", cudaGetErrorString(a),
           cudaGetErrorString(b), cudaGetErrorString(d), h1[1], h2[1]);
    c.attrs = nullptr;
    c.numAttrs = 0;
    cudaMemset(c1, 0, 8);
    cudaMemset(c2, 0, 8);
    c.stream = s1;
    a = cudaLaunchKernelEx(&c, k_cluster, c1, 2 * clusters);
    c.stream = s2;
    b = cudaLaunchKernelEx(&c, k_cluster, c2, 2 * clusters);
    d = cudaDeviceSynchronize();
    cudaMemcpy(h1, c1, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2, c2, 8, cudaMemcpyDeviceToHost);
    printf("two NON-coop grids on two streams: %s %s sync=%s timeouts %d %d\n", cudaGetErrorString(a),
           cudaGetErrorString(b), cudaGetErrorString(d), h1[1], h2[1]);
  }
  return 0;
}
