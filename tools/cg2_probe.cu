// Probe: 2-SM tcgen05.mma (cta_group::2), M = 128 = 64 rows per CTA, kind::f16 -- where D
// lands in each CTA's TMEM, how B is split between the pair, and the MMA rate against the
// 1-SM M = 64 MMA the cfg4 chain uses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cg2_probe tools/cg2_probe.cu
// Layout hypothesis: CTA r's SMEM holds A rows [64r, 64r+64) and B rows (N) [N/2 r, N/2 (r+1))
// (SW128 K-major), the MMA is issued by rank 0 only, and CTA r's TMEM receives D rows
// [64r, 64r+64) x all N columns.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_fp16.h>

#include "../paper_1611_09482_b200/csrc/tc_ptx.cuh"

using namespace fw::ptx;

__device__ __forceinline__ void mma_cg2(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_cg2_ta(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_cg2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// img: per CTA [A 64 rows x 64 K SW128 (8 KB)][B N/2 rows x 64 K SW128 (N/2 x 128 B)]
__global__ void probe(const uint8_t* img, int N, float* dump, long long* cyc, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const int bytes = 8192 + N / 2 * 128;
  for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = reinterpret_cast<const uint4*>(img + (size_t)rank * bytes)[i];
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = holder;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  {
    float z[32];
    for (int j = 0; j < 32; ++j) z[j] = -7.f;
    for (int c = 0; c < 512; c += 32) tmem_st32(trow + c, z);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t id = idesc_f16(128, N);
  if (rank == 0 && warp == 0) {
    if (elect_one()) {
      for (int kk = 0; kk < 4; ++kk)
        mma_cg2(tmem, sdesc_sw128(smem_u32(smem) + kk * 32), sdesc_sw128(smem_u32(smem) + 8192 + kk * 32), id,
                kk != 0);
      commit_cg2(&bar);
    }
    __syncwarp();
  }
  mbar_wait_cluster(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 32) {
    float v[32];
    tmem_ld32(trow + c, v);
    for (int j = 0; j < 32; ++j) dump[((size_t)rank * 128 + warp * 32 + lane) * N + c + j] = v[j];
  }
  // timing: back-to-back 2-SM MMAs (K = 16 each), then one commit
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (rank == 0 && warp == 0) {
    long long t0 = 0;
    if (elect_one()) {
      t0 = clock64();
      for (int r = 0; r < reps; ++r)
        mma_cg2(tmem + 256, sdesc_sw128(smem_u32(smem) + (r & 3) * 32), sdesc_sw128(smem_u32(smem) + 8192 + (r & 3) * 32),
                idesc_f16(128, N), 1u);
      commit_cg2(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 1);
    if (lane == 0) cyc[0] = clock64() - t0;
  } else {
    mbar_wait_cluster(&bar, 1);
  }
  // same with A from TMEM (the A operand at columns [384, 416) of each CTA's TMEM: zeros)
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (rank == 0 && warp == 0) {
    long long t0 = 0;
    if (elect_one()) {
      t0 = clock64();
      for (int r = 0; r < reps; ++r)
        mma_cg2_ta(tmem + 256, tmem + 384 + (r & 3) * 8, sdesc_sw128(smem_u32(smem) + 8192 + (r & 3) * 32),
                   idesc_f16(128, N), 1u);
      commit_cg2(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    if (lane == 0) cyc[1] = clock64() - t0;
  } else {
    mbar_wait_cluster(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

static uint16_t h16(float v) {
  __half h = __float2half_rn(v);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}
static void pack(uint8_t* dst, int nrows, const std::vector<float>& M, int ld, int row0) {
  for (int r = 0; r < nrows; ++r)
    for (int k = 0; k < 64; ++k) {
      const size_t off = (size_t)(r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 3) ^ (r & 7))) << 4) + (k & 7) * 2;
      const uint16_t b = h16(M[(size_t)(row0 + r) * ld + k]);
      memcpy(dst + off, &b, 2);
    }
}

int main() {
  for (int N : {64, 128, 256}) {
    std::vector<float> A(128 * 64), B((size_t)N * 64);
    for (int i = 0; i < 128 * 64; ++i) A[i] = (float)((i * 7) % 13 - 6) / 8.f;
    for (int i = 0; i < N * 64; ++i) B[i] = (float)((i * 5) % 11 - 5) / 8.f;
    const int bytes = 8192 + N / 2 * 128;
    std::vector<uint8_t> img(2 * bytes, 0);
    for (int r = 0; r < 2; ++r) {
      pack(img.data() + (size_t)r * bytes, 64, A, 64, 64 * r);
      pack(img.data() + (size_t)r * bytes + 8192, N / 2, B, 64, N / 2 * r);
    }
    uint8_t* dimg;
    float* ddump;
    long long* dcyc;
    cudaMalloc(&dimg, img.size());
    cudaMemcpy(dimg, img.data(), img.size(), cudaMemcpyHostToDevice);
    cudaMalloc(&ddump, 2 * 128 * N * 4);
    cudaMalloc(&dcyc, 16);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 64 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int reps = 512;
    cudaError_t e = cudaLaunchKernelEx(&cfg, probe, (const uint8_t*)dimg, N, ddump, dcyc, reps);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("N=%d: launch failed: %s\n", N, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> dump(2 * 128 * N);
    long long cyc[2];
    cudaMemcpy(dump.data(), ddump, dump.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(cyc, dcyc, 16, cudaMemcpyDeviceToHost);
    // where does D[m][n] land? search each (rank, lane, col) for the reference value pattern
    int hits = 0, checked = 0;
    std::vector<int> lane_of_row(128, -1), rank_of_row(128, -1);
    for (int m = 0; m < 128; ++m) {
      // find a (rank, lane) whose row equals D[m][:]
      for (int r = 0; r < 2 && lane_of_row[m] < 0; ++r)
        for (int ln = 0; ln < 128; ++ln) {
          bool ok = true;
          for (int n = 0; n < N && ok; ++n) {
            double ref = 0;
            for (int k = 0; k < 64; ++k) ref += (double)A[m * 64 + k] * B[(size_t)n * 64 + k];
            ok = fabs(dump[((size_t)r * 128 + ln) * N + n] - ref) < 1e-3;
          }
          if (ok) {
            lane_of_row[m] = ln;
            rank_of_row[m] = r;
            break;
          }
        }
      ++checked;
      if (lane_of_row[m] >= 0) ++hits;
    }
    if (N == 128) {
      auto ref = [&](int m, int n) {
        double r = 0;
        for (int k = 0; k < 64; ++k) r += (double)A[m * 64 + k] * B[(size_t)n * 64 + k];
        return r;
      };
      for (int r = 0; r < 2; ++r)
        for (int ln : {0, 1, 15, 16, 17, 31, 32, 33, 48, 63, 64, 96, 127}) {
          printf("  r%d lane%3d:", r, ln);
          for (int n = 0; n < 6; ++n) printf(" %8.3f", dump[((size_t)r * 128 + ln) * N + n]);
          printf("  | n=64..65: %8.3f %8.3f\n", dump[((size_t)r * 128 + ln) * N + 64], dump[((size_t)r * 128 + ln) * N + 65]);
        }
      for (int m : {0, 1, 16, 32, 63, 64, 65, 127}) {
        printf("  ref m%3d:", m);
        for (int n = 0; n < 6; ++n) printf(" %8.3f", ref(m, n));
        printf("  | n=64..65: %8.3f %8.3f\n", ref(m, 64), ref(m, 65));
      }
    }
    printf("N=%d: %d/%d rows of D found;", N, hits, checked);
    for (int m : {0, 1, 15, 16, 31, 32, 63, 64, 65, 127})
      printf(" m%d->r%d:l%d", m, rank_of_row[m], lane_of_row[m]);
    printf("\n  2-SM MMA M=128 N=%d K=16: SS %.1f cycles, TS %.1f cycles (per MMA, %d back to back)\n", N,
           (double)cyc[0] / reps, (double)cyc[1] / reps, reps);
    cudaFree(dimg);
    cudaFree(ddump);
    cudaFree(dcyc);
  }
  return 0;
}
