// Microbenchmark: latency from issuing k back-to-back tcgen05.mma (M=128, N=128, K=16 each,
// issued under elect.sync by one converged warp) plus tcgen05.commit to the mbarrier
// completing, as seen by (a) the issuing warp and (b) a second warp waiting on the barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_latency tools/mma_latency.cu
#include <cstdio>

#include "../paper_1611_09482_b200/csrc/tc_ptx.cuh"

using namespace fw::ptx;

// pre > 0: the timed burst follows `pre` untimed MMAs into another accumulator (busy pipe)
__global__ void probe(int k, int ts, long long* out, int pre) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, go;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&go, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&holder, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  const uint32_t id = idesc_f16(128, 128);
  const uint32_t sa = smem_u32(smem), sb = sa + 16384;
  const int reps = 16;
  long long sum_issue = 0, sum_self = 0, sum_other = 0;
  for (int rep = 0; rep < reps; ++rep) {
    if (warp == 0) {
      // let the waiter park on the barrier first
      __nanosleep(2000);
      if (pre > 0) {
        if (elect_one())
          for (int i = 0; i < pre; ++i)
            mma_bf16_ta(tmem + 256, tmem + 448 + (i & 7) * 8, sdesc_sw128(sb + (i & 3) * 32), id, 1u);
        __syncwarp();
      }
      const long long t0 = clock64();
      if (elect_one()) {
        for (int i = 0; i < k; ++i) {
          if (ts)
            mma_bf16_ta(tmem, tmem + 448 + (i & 7) * 8, sdesc_sw128(sb + (i & 3) * 32), id, 1u);
          else
            mma_bf16(tmem, sdesc_sw128(sa + (i & 3) * 32), sdesc_sw128(sb + (i & 3) * 32), id, 1u);
        }
        mma_commit(&bar);
      }
      __syncwarp();
      const long long t1 = clock64();
      mbar_wait(&bar, rep & 1);
      const long long t2 = clock64();
      sum_issue += t1 - t0;
      sum_self += t2 - t0;
      if (lane == 0) {
        out[8] = t0;  // publish t0 for the other warp through global memory
      }
      if (lane == 0) mbar_arrive(&go);
    } else if (warp == 1) {
      mbar_wait(&bar, rep & 1);
      const long long t2 = clock64();
      mbar_wait(&go, rep & 1);
      __threadfence_block();
      const long long t0 = *(volatile long long*)&out[8];
      sum_other += t2 - t0;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = sum_issue / reps;
    out[1] = sum_self / reps;
  }
  if (threadIdx.x == 32) out[2] = sum_other / reps;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 128);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  for (int pre : {0, 2, 16})
  for (int ts = 1; ts < 2; ++ts)
    for (int k : {1, 4, 8}) {
      probe<<<1, 64, 32768 + 1024>>>(k, ts, d, pre);
      probe<<<1, 64, 32768 + 1024>>>(k, ts, d, pre);
      long long h[3] = {0, 0, 0};
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
      printf("pre %2d %s k=%2d N=128: issue %5lld, done (issuer) %5lld, done (other warp) %5lld cycles %s\n",
             pre, ts ? "TS" : "SS", k, h[0], h[1], h[2], e ? cudaGetErrorString(e) : "");
    }
  return 0;
}
