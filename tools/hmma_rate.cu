// Warp-level HMMA (mma.sync m16n8k16 f16 -> f32) on sm_100a: latency of a dependent chain and
// throughput with independent accumulators, per SM (8 warps). nvcc -arch=sm_100a -o /tmp/h hmma_rate.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
template <int NACC>
__global__ void k(float* out, long long* cyc, int iters) {
  uint32_t a[4] = {0x3c003c00u ^ threadIdx.x, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u};
  uint32_t b[2] = {0x3c003c00u, 0x3c00u ^ threadIdx.x};
  float c[NACC][4] = {};
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < NACC; ++j) mma(c[j], a, b);
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < NACC; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* o; long long* cy; cudaMalloc(&o, 1 << 20); cudaMalloc(&cy, 8 * 1024);
  const int iters = 4096;
  for (int warps : {1, 4, 8, 16}) {
    auto run = [&](auto kern, int nacc) {
      kern<<<1, 32 * warps>>>(o, cy, iters); cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cy, 8, cudaMemcpyDeviceToHost);
      printf("warps %2d acc %d: %.1f cycles per HMMA per warp, SM rate %.2f HMMA/clk\n", warps, nacc,
             (double)c / (iters * nacc), (double)iters * nacc * warps / c);
    };
    run(k<1>, 1); run(k<4>, 4); run(k<8>, 8);
  }
  return 0;
}
