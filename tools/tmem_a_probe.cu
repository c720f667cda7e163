// Probe: tcgen05.mma kind::f16 with the A operand in TMEM vs in shared memory.
// A [128 x 64] bf16, B [128 x 64] bf16; D = A . B^T (128 x 128 fp32).
// Path S: A as a SW128 K-major smem image. Path T: A in TMEM, lane = row, 32-bit column j
// holding (A[r][2j], A[r][2j+1]) -- the layout this probe checks.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_a_probe tools/tmem_a_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1611_09482_b200/csrc/tc_ptx.cuh"

using namespace fw::ptx;

__device__ __forceinline__ void mma_bf16_tmem_a(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}

__global__ void probe(const uint8_t* a_img, const uint8_t* b_img, const uint32_t* a_packed,
                      float* out_s, float* out_t) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* As = smem;
  uint8_t* Bs = smem + 16384;
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 16384 / 16; i += blockDim.x) {
    reinterpret_cast<uint4*>(As)[i] = reinterpret_cast<const uint4*>(a_img)[i];
    reinterpret_cast<uint4*>(Bs)[i] = reinterpret_cast<const uint4*>(b_img)[i];
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
  const uint32_t tmem = holder;
  // A into TMEM columns [256, 288): thread (warp w, lane) = row 32w + lane
  {
    const int r = warp * 32 + lane;
    float v[32];
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(a_packed[r * 32 + j]);
    tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 256, v);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_bf16(128, 128);
    for (int kk = 0; kk < 4; ++kk)
      mma_bf16(tmem + 0, sdesc_sw128(smem_u32(As) + kk * 32), sdesc_sw128(smem_u32(Bs) + kk * 32),
               id, kk != 0);
    for (int kk = 0; kk < 4; ++kk)
      mma_bf16_tmem_a(tmem + 128, tmem + 256 + kk * 8, sdesc_sw128(smem_u32(Bs) + kk * 32), id,
                      kk != 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  {
    const int r = warp * 32 + lane;
    for (int q = 0; q < 4; ++q) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 32 * q, v);
      tmem_wait_ld();
      for (int j = 0; j < 32; ++j) out_s[r * 128 + 32 * q + j] = v[j];
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 128 + 32 * q, v);
      tmem_wait_ld();
      for (int j = 0; j < 32; ++j) out_t[r * 128 + 32 * q + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

static uint16_t bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)((u + 0x7FFF + ((u >> 16) & 1)) >> 16);
}
static float unbf(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main() {
  std::vector<uint16_t> A(128 * 64), B(128 * 64);
  srand(1);
  for (auto& v : A) v = bf((rand() % 17 - 8) / 8.0f);
  for (auto& v : B) v = bf((rand() % 13 - 6) / 4.0f);
  std::vector<uint8_t> ai(16384), bi(16384);
  auto img = [](std::vector<uint8_t>& dst, const std::vector<uint16_t>& m) {
    for (int r = 0; r < 128; ++r)
      for (int k = 0; k < 64; ++k) {
        size_t off = (r >> 3) * 1024 + (r & 7) * 128 + (((k >> 3) ^ (r & 7)) << 4) + (k & 7) * 2;
        memcpy(&dst[off], &m[r * 64 + k], 2);
      }
  };
  img(ai, A);
  img(bi, B);
  std::vector<uint32_t> ap(128 * 32);
  for (int r = 0; r < 128; ++r)
    for (int j = 0; j < 32; ++j) ap[r * 32 + j] = A[r * 64 + 2 * j] | ((uint32_t)A[r * 64 + 2 * j + 1] << 16);
  uint8_t *da, *db;
  uint32_t* dp;
  float *ds, *dt;
  cudaMalloc(&da, 16384);
  cudaMalloc(&db, 16384);
  cudaMalloc(&dp, ap.size() * 4);
  cudaMalloc(&ds, 128 * 128 * 4);
  cudaMalloc(&dt, 128 * 128 * 4);
  cudaMemcpy(da, ai.data(), 16384, cudaMemcpyHostToDevice);
  cudaMemcpy(db, bi.data(), 16384, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, ap.data(), ap.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  probe<<<1, 128, 32768 + 1024>>>(da, db, dp, ds, dt);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> hs(128 * 128), ht(128 * 128);
  cudaMemcpy(hs.data(), ds, hs.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(ht.data(), dt, ht.size() * 4, cudaMemcpyDeviceToHost);
  double es = 0, et = 0;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < 128; ++n) {
      double ref = 0;
      for (int k = 0; k < 64; ++k) ref += (double)unbf(A[r * 64 + k]) * unbf(B[n * 64 + k]);
      es = fmax(es, fabs(hs[r * 128 + n] - ref));
      et = fmax(et, fabs(ht[r * 128 + n] - ref));
    }
  printf("probe: %s  smem-A max err %.3g  tmem-A max err %.3g\n", cudaGetErrorString(e), es, et);
  return 0;
}
