// Microbenchmark: throughput of the f32 -> f16x2 pack (F2FP) next to MUFU.TANH, one SM,
// 16 warps, 8 independent chains per thread (does F2FP share the SFU with MUFU?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cvt_probe tools/cvt_probe.cu
#include <cstdio>
#include <cstdint>

template <int KIND>
__global__ void probe(int iters, uint32_t* out, long long* cyc) {
  float f[8];
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) f[j] = 0.001f * (threadIdx.x + j);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t v;
      if (KIND == 0) {  // F2FP only (fed by the previous result, no folding)
        asm volatile("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(v) : "f"(f[j]), "f"(f[(j + 1) & 7]));
        f[j] = __uint_as_float(v);
      } else if (KIND == 1) {  // MUFU.TANH f32 only
        asm volatile("tanh.approx.f32 %0, %0;" : "+f"(f[j]));
      } else if (KIND == 2) {  // one F2FP + two MUFU.TANH f32 per element pair
        float a, b;
        asm volatile("tanh.approx.f32 %0, %1;" : "=f"(a) : "f"(f[j]));
        asm volatile("tanh.approx.f32 %0, %1;" : "=f"(b) : "f"(f[(j + 1) & 7]));
        asm volatile("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(v) : "f"(a), "f"(b));
        f[j] = __uint_as_float(v);
      } else {  // FMUL only (baseline of the dependency chain)
        asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(f[j]) : "f"(f[(j + 1) & 7]));
      }
    }
  }
  const long long t1 = clock64();
#pragma unroll
  for (int j = 0; j < 8; ++j) acc ^= __float_as_uint(f[j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int KIND>
void run(const char* name, int warps) {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 4 * 1024);
  cudaMalloc(&cyc, 8);
  const int iters = 1024;
  probe<KIND><<<1, 32 * warps>>>(iters, out, cyc);
  probe<KIND><<<1, 32 * warps>>>(iters, out, cyc);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double inst = (double)iters * 8 * warps;
  printf("%-22s warps %2d: %8lld cycles, %.3f warp-inst/clk/SM\n", name, warps, c, inst / c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {8, 16}) {
    run<0>("cvt.f16x2.f32 (F2FP)", w);
    run<1>("tanh.approx.f32", w);
    run<2>("2 tanh + 1 F2FP", w);
    run<3>("mul.f32", w);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
