// Microbenchmark: cost of barrier.cluster (arrive.release + wait.acquire) and of
// __syncthreads, 256 threads per CTA, cluster sizes 1..8, one cluster per GPC-ish.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_bar tools/cluster_bar.cu
#include <cstdio>
__global__ void bar_kernel(long long* out, int n, int mode) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (mode == 0)
      __syncthreads();
    else
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}
int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int mode = 0; mode < 2; ++mode)
    for (int c : {1, 2, 4, 8}) {
      if (mode == 0 && c > 1) continue;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(c * 8);
      cfg.blockDim = dim3(256);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 2000;
      void* args[] = {&d, &n, &mode};
      cudaLaunchKernelExC(&cfg, (const void*)bar_kernel, args);
      cudaLaunchKernelExC(&cfg, (const void*)bar_kernel, args);
      cudaError_t e = cudaDeviceSynchronize();
      long long h = 0;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%s cluster=%d: %.1f cycles per barrier %s\n", mode ? "barrier.cluster" : "__syncthreads", c,
             (double)h / n, e ? cudaGetErrorString(e) : "");
    }
  return 0;
}
