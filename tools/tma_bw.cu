// Microbenchmark: per-SM throughput of 1-D TMA bulk copies (global -> shared) through a
// ring of `stages` x `chunk` bytes, as the chain kernel streams its weights.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bw tools/tma_bw.cu
//   tools/tma_bw <ctas> <chunk_bytes> <stages> <MB_per_cta> <src_MB>
#include <cstdio>
#include <cstdlib>

#include "../paper_1611_09482_b200/csrc/tc_ptx.cuh"

using namespace fw::ptx;

__global__ void stream_kernel(const uint8_t* src, size_t src_bytes, int chunk, int stages,
                              long long total, unsigned long long* cycles, int lane_mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * chunk);
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // issuer k (threads 0, 32, 64, ...) owns stages [k*stages/issuers, (k+1)*stages/issuers)
  // lane_mode = issuing lanes per warp (0 or 1: lane 0 of each warp)
  const int lpw = lane_mode > 1 ? lane_mode : 1;
  const int issuers = (blockDim.x / 32) * lpw;
  if (threadIdx.x % 32 >= lpw) return;
  const int k = (threadIdx.x / 32) * lpw + threadIdx.x % 32;
  const int my = stages / issuers;
  const long long n = total / chunk / issuers;
  long long t0 = clock64();
  size_t off = ((size_t)blockIdx.x * 7919 + k * 131) * 1024 % src_bytes;
  for (long long i = 0; i < n + my; ++i) {
    const int s = k * my + (int)(i % my);
    if (i >= my) mbar_wait(&full[s], ((i / my) - 1) & 1);
    if (i < n) {
      mbar_arrive_expect_tx(&full[s], chunk);
      bulk_g2s(smem + (size_t)s * chunk, src + off, chunk, &full[s]);
      off += chunk;
      if (off + chunk > src_bytes) off = 0;
    }
  }
  if (k == 0) cycles[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 32;
  const int chunk = argc > 2 ? atoi(argv[2]) : 16384;
  const int stages = argc > 3 ? atoi(argv[3]) : 4;
  const long long per_cta = (argc > 4 ? atoll(argv[4]) : 64) << 20;
  const int issuers = argc > 6 ? atoi(argv[6]) : 1;
  const int lane_mode = argc > 7 ? atoi(argv[7]) : 0;
  const size_t src_bytes = (size_t)(argc > 5 ? atoll(argv[5]) : 8) << 20;
  uint8_t* src;
  unsigned long long* cyc;
  cudaMalloc(&src, src_bytes);
  cudaMemset(src, 1, src_bytes);
  cudaMalloc(&cyc, sizeof(unsigned long long) * ctas);
  const size_t smem = (size_t)stages * chunk + 1024;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  stream_kernel<<<ctas, 32 * (issuers / (lane_mode > 1 ? lane_mode : 1)), smem>>>(src, src_bytes, chunk, stages, per_cta, cyc, lane_mode);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  stream_kernel<<<ctas, 32 * (issuers / (lane_mode > 1 ? lane_mode : 1)), smem>>>(src, src_bytes, chunk, stages, per_cta, cyc, lane_mode);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long* h = new unsigned long long[ctas];
  cudaMemcpy(h, cyc, sizeof(unsigned long long) * ctas, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < ctas; ++i) mean += h[i];
  mean /= ctas;
  printf("ctas=%d chunk=%d stages=%d src=%zuMB: %.3f ms, per-SM %.1f B/clk, %.1f GB/s/SM, total %.0f GB/s (%s)\n",
         ctas, chunk, stages, src_bytes >> 20, ms, per_cta / mean, per_cta / (ms * 1e6),
         ctas * per_cta / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
