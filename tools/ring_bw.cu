// Microbenchmark of a weight ring as the chain kernel uses it: `stages` x `chunk` bytes,
// a consumer thread that holds each stage ~`hold` cycles after it lands (an MMA), and one
// of several producer layouts:
//   mode 0: one thread issues every stage
//   mode 1: lanes 0..k-1 of 2 warps, one stage each (k = stages / 2)
//   mode 2: lane 0 of `stages` warps, one stage each
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ring_bw tools/ring_bw.cu
//   tools/ring_bw <mode> <stages> <chunk> <hold_cycles> <MB>
#include <cstdio>
#include <cstdlib>

#include "../paper_1611_09482_b200/csrc/tc_ptx.cuh"

using namespace fw::ptx;

__device__ int g_poll;
__device__ long long g_ts[2][4096];  // CTA 0: [0]=issue time, [1]=consumer-saw time  // 1: spin on mbarrier.test_wait instead of try_wait
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t parity) {
  if (!g_poll) {
    mbar_wait(bar, parity);
    return;
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}

__global__ void ring_kernel(const uint8_t* src, size_t src_bytes, int mode, int stages, int chunk,
                            int hold, long long n, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * chunk);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int cons_warp = blockDim.x / 32 - 1;
  auto issue = [&](long long i) {
    const int s = (int)(i % stages);
    wait_bar(&empty[s], ((i / stages) & 1) ^ 1);
    mbar_arrive_expect_tx(&full[s], chunk);
    size_t off = ((size_t)blockIdx.x * 7919 * 1024 + (size_t)i * chunk) % (src_bytes - chunk);
    off &= ~(size_t)15;
    if (blockIdx.x == 0 && i < 4096) g_ts[0][i] = clock64();
    bulk_g2s(smem + (size_t)s * chunk, src + off, chunk, &full[s]);
  };
  if (warp == cons_warp) {
    if (mode == 3) {  // no consumer: producers re-issue on their own full barriers
      if (lane == 0) out[blockIdx.x] = 0;
      return;
    }
    if (lane == 0) {
      const long long t0 = clock64();
      for (long long i = 0; i < n; ++i) {
        const int s = (int)(i % stages);
        wait_bar(&full[s], (i / stages) & 1);
        const long long h0 = clock64();
        if (blockIdx.x == 0 && i < 4096) g_ts[1][i] = h0;
        while (clock64() - h0 < hold) {
        }
        mbar_arrive(&empty[s]);
      }
      out[blockIdx.x] = clock64() - t0;
    }
    return;
  }
  if (mode == 0) {
    if (warp == 0 && lane == 0)
      for (long long i = 0; i < n; ++i) issue(i);
  } else if (mode == 1) {
    const int k = stages / 2;
    if (warp < 2 && lane < k) {
      const int p = warp * k + lane;
      for (long long i = p; i < n; i += stages) issue(i);
    }
  } else if (mode == 2) {
    if (lane == 0 && warp < stages)
      for (long long i = warp; i < n; i += stages) issue(i);
  } else {
    if (lane == 0 && warp < stages) {
      const long long t0 = clock64();
      for (long long i = warp; i < n; i += stages) {
        const int s = (int)(i % stages);
        if (i >= stages) mbar_wait(&full[s], ((i / stages) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], chunk);
        size_t off = ((size_t)blockIdx.x * 7919 * 1024 + (size_t)i * chunk) % (src_bytes - chunk);
        off &= ~(size_t)15;
        bulk_g2s(smem + (size_t)s * chunk, src + off, chunk, &full[s]);
      }
      const int s = warp;
      mbar_wait(&full[s], ((n - 1 - ((n - 1 - warp) % stages)) / stages) & 1);
      if (warp == 0) out[blockIdx.x] = clock64() - t0;
    }
  }
}

int main(int argc, char** argv) {
  const int mode = atoi(argv[1]), stages = atoi(argv[2]), chunk = atoi(argv[3]), hold = atoi(argv[4]);
  const long long bytes = (long long)atoi(argv[5]) << 20;
  const long long n = bytes / chunk;
  const int poll = argc > 6 ? atoi(argv[6]) : 0;
  cudaMemcpyToSymbol(g_poll, &poll, sizeof(int));
  const int ctas = 32;
  const size_t src_bytes = 8 << 20;
  uint8_t* src;
  unsigned long long* out;
  cudaMalloc(&src, src_bytes);
  cudaMalloc(&out, 8 * ctas);
  const int warps = (mode >= 2 ? stages : 2) + 1;
  const size_t smem = (size_t)stages * chunk + 1024;
  cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  ring_kernel<<<ctas, 32 * warps, smem>>>(src, src_bytes, mode, stages, chunk, hold, n, out);
  cudaDeviceSynchronize();
  ring_kernel<<<ctas, 32 * warps, smem>>>(src, src_bytes, mode, stages, chunk, hold, n, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[32];
  cudaMemcpy(h, out, 8 * ctas, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < ctas; ++i) mean += h[i];
  mean /= ctas;
  static long long ts[2][4096];
  cudaMemcpyFromSymbol(ts, g_ts, sizeof(ts));
  double lat = 0, hand = 0; int cnt = 0;
  for (int i = 100; i < 1000 && i + stages < n; ++i) { lat += ts[1][i] - ts[0][i]; hand += ts[0][i + stages] - ts[1][i]; ++cnt; }
  printf("load latency (issue->seen) %.0f, handoff (seen->reissue) %.0f cycles; ", lat / cnt, hand / cnt);
  printf("poll=%d ", poll);
  printf("mode=%d stages=%d chunk=%d hold=%d: %.1f cycles/chunk, %.1f B/clk (%s)\n", mode, stages,
         chunk, hold, mean / n, n * (double)chunk / mean, cudaGetErrorString(e));
  return 0;
}
