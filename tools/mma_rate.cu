// Microbenchmark: tcgen05.mma kind::f16 issue-to-completion rate for M = 128 and
// N in {32, 64, 128, 256}, A from shared memory (SS) or from TMEM (TS), one CTA.
// Operand contents are irrelevant (zeros); only timing is reported.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu
#include <cstdio>

#include "../paper_1611_09482_b200/csrc/tc_ptx.cuh"

using namespace fw::ptx;

// rot >= 8: elect-issued; bit 16 of rot: random operand data; bit 17: 4 extra warps stream
// tcgen05.ld from TMEM columns 256..447 while the MMAs run
__global__ void probe(int n, int ts, int count, long long* out, int rot, int mrows) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  const bool rnd = (rot >> 16) & 1, ldload = (rot >> 17) & 1;
  const int rot_all = rot;
  rot &= 0xFFFF;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) {
    uint32_t x = rnd ? (uint32_t)i * 2654435761u + 12345u : 0u;
    auto h = [&](uint32_t v) { v ^= v >> 13; v *= 0x5bd1e995u; v ^= v >> 15; return (v & 0x3bff3bffu); };
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(h(x), h(x + 1), h(x + 2), h(x + 3));
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&holder, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // bit 18 of rot: accumulator and TMEM A operand in plane P1 (lane offset 16, M = 64)
  const uint32_t tmem = holder + (((rot >> 18) & 1) ? (16u << 16) : 0u);
  const bool elect_mode = rot >= 8;
  __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (ldload && warp >= 4 && warp < 8) {
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t acc = 0;
    while (!*(volatile int*)&stop) {
      float v[32];
      tmem_ld32(trow + 256 + 64 * (warp & 1), v);
      tmem_wait_ld();
      acc += __float_as_uint(v[0]) ^ __float_as_uint(v[31]);
    }
    if (acc == 0x12345678u) out[2] = acc;
  }
  if (elect_mode ? warp == 0 : threadIdx.x == 0) {
    const uint32_t id = idesc_f16(mrows, n);
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    // warm-up
    if (!elect_mode || (threadIdx.x & 31) == 0)
    for (int i = 0; i < 8; ++i)
      mma_bf16(tmem, sdesc_sw128(sa + (i & 3) * 32), sdesc_sw128(sb + (i & 3) * 32), id, 1u);
    if (!elect_mode || (threadIdx.x & 31) == 0) mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t0 = clock64();
    const uint64_t da0 = sdesc_sw128(sa), da1 = sdesc_sw128(sa + 32), db0 = sdesc_sw128(sb),
                   db1 = sdesc_sw128(sb + 32);
    // rot: accumulators rotate over `rot` disjoint 64-column TMEM regions
    const uint32_t d1 = rot > 1 ? 64u : 0u, d2 = rot > 2 ? 128u : 0u, d3 = rot > 2 ? 192u : d1;
    for (int i = 0; i < count; i += 4) {
      if (elect_mode) {
        uint32_t pred;
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(pred));
        if (pred) {
          if (ts) {
            mma_bf16_ta(tmem, tmem + 448, db0, id, 1u);
            mma_bf16_ta(tmem, tmem + 456, db1, id, 1u);
            mma_bf16_ta(tmem, tmem + 464, db0, id, 1u);
            mma_bf16_ta(tmem, tmem + 472, db1, id, 1u);
          } else {
            mma_bf16(tmem, da0, db0, id, 1u);
            mma_bf16(tmem, da1, db1, id, 1u);
            mma_bf16(tmem, da0, db0, id, 1u);
            mma_bf16(tmem, da1, db1, id, 1u);
          }
        }
        __syncwarp();
      } else if (ts) {
        mma_bf16_ta(tmem, tmem + 448, db0, id, 1u);
        mma_bf16_ta(tmem + d1, tmem + 456, db1, id, 1u);
        mma_bf16_ta(tmem + d2, tmem + 464, db0, id, 1u);
        mma_bf16_ta(tmem + d3, tmem + 472, db1, id, 1u);
      } else {
        mma_bf16(tmem, da0, db0, id, 1u);
        mma_bf16(tmem + d1, da1, db1, id, 1u);
        mma_bf16(tmem + d2, da0, db0, id, 1u);
        mma_bf16(tmem + d3, da1, db1, id, 1u);
      }
    }
    const long long t1 = clock64();
    if (!elect_mode || (threadIdx.x & 31) == 0) mma_commit(&bar);
    mbar_wait(&bar, 1);
    const long long t2 = clock64();
    if ((threadIdx.x & 31) == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
      *(volatile int*)&stop = 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 32);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  for (int mrows : {64})
  for (int rot : {8, 0x40008})
  for (int ts = 0; ts < 2; ++ts)
    for (int n : {32, 64, 128, 256}) {

      const int count = 512;
      probe<<<1, 256, 65536 + 1024>>>(n, ts, count, d, rot, mrows);
      probe<<<1, 256, 65536 + 1024>>>(n, ts, count, d, rot, mrows);
      long long h[2] = {0, 0};
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("mode %x %s M=%d N=%3d K=16: issue %6.1f cyc/mma, complete %6.1f cyc/mma (floor %d) %s\n",
             rot, ts ? "TS" : "SS", mrows, n, (double)h[0] / count, (double)h[1] / count, 128 * n / 256,
             e ? cudaGetErrorString(e) : "");
    }
  return 0;
}
