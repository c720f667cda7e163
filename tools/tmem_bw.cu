// Microbenchmark: per-SM throughput of tcgen05.ld / tcgen05.st for several shapes, with
// 1 / 4 / 8 warps (warp w on lane quadrant w % 4), as the chain kernel's gate and queue
// warps use them. Each load is 4 KB per warp (32 registers per thread) unless noted.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bw tools/tmem_bw.cu
#include <cstdio>

#include "../paper_1611_09482_b200/csrc/tc_ptx.cuh"

using namespace fw::ptx;

#define R32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"
#define O32(r)                                                                                    \
  "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),    \
      "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),  \
      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),  \
      "=r"(r[29]), "=r"(r[30]), "=r"(r[31])

template <int SHAPE>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t (&r)[32]) {
  if (SHAPE == 0)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " R32 ", [%32];" : O32(r) : "r"(taddr));
  else if (SHAPE == 1)
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 " R32 ", [%32];" : O32(r) : "r"(taddr));
  else if (SHAPE == 2)
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 " R32 ", [%32];" : O32(r) : "r"(taddr));
  else if (SHAPE == 3)
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 " R32 ", [%32];" : O32(r) : "r"(taddr));
  else if (SHAPE == 4)  // 32 lanes x 64 columns of 16-bit pairs packed: reads 8 KB, 32 regs
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 " R32 ", [%32];"
                 : O32(r)
                 : "r"(taddr));
}

// MODE 0: ld (shape S) x NL per iteration then wait; MODE 1: st 32x32b.x32 x2 then wait
template <int MODE, int S, int NL>
__global__ void probe(int iters, uint32_t* out, long long* cyc) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder + ((uint32_t)((warp & 3) * 32) << 16);
  const uint32_t col = 128 * ((warp >> 2) & 3);
  uint32_t v[NL][32];
#pragma unroll
  for (int k = 0; k < NL; ++k)
#pragma unroll
    for (int j = 0; j < 32; ++j) v[k][j] = threadIdx.x + j + k;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int k = 0; k < NL; ++k) ld<S>(tmem + col + 32 * k, v[k]);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < NL; ++k) acc += v[k][k] ^ v[k][31 - k];
    } else {
      v[0][0] += 1;
      tmem_st32(tmem + col, *reinterpret_cast<float(*)[32]>(v[0]));
      tmem_st32(tmem + col + 32, *reinterpret_cast<float(*)[32]>(v[0]));
      tmem_wait_st();
    }
  }
  const long long t1 = clock64();
  out[threadIdx.x] = acc + v[0][3];
  if ((threadIdx.x & 31) == 0) cyc[warp] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(holder, 512);
}

template <int M, int S, int NL>
void run(const char* name, int warps, int bytes_per_ld) {
  const int iters = 512;
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 4 * 32 * warps);
  cudaMalloc(&cyc, 8 * warps);
  probe<M, S, NL><<<1, 32 * warps>>>(iters, out, cyc);
  probe<M, S, NL><<<1, 32 * warps>>>(iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[32];
  cudaMemcpy(h, cyc, 8 * warps, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < warps; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes = (double)warps * iters * NL * bytes_per_ld;
  printf("%-22s x%d warps %2d: %7lld cycles, %6.1f cycles/iter, %6.1f B/clk/SM %s\n", name, NL,
         warps, mx, (double)mx / iters, bytes / mx, e ? cudaGetErrorString(e) : "");
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 4, 8, 16}) {
    run<0, 0, 1>("ld 32x32b.x32", w, 4096);
    run<0, 0, 2>("ld 32x32b.x32", w, 4096);
    run<0, 0, 4>("ld 32x32b.x32", w, 4096);
    run<0, 1, 2>("ld 16x256b.x8", w, 4096);
    run<0, 2, 2>("ld 16x128b.x16", w, 4096);
    run<0, 3, 2>("ld 16x64b.x32", w, 4096);
    run<0, 4, 2>("ld 32x32b.x32.pack16", w, 4096);
    run<1, 0, 2>("st 32x32b.x32", w, 4096);
  }
  return 0;
}
