// Microbenchmark: issue throughput of the gate's special-function and conversion
// instructions on one SM (8 warps, 8 independent chains per thread).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/xu_probe tools/xu_probe.cu
//   tools/xu_probe
#include <cstdio>
#include <cstdint>

#define OP_LOOP(BODY)                                                  \
  for (int it = 0; it < iters; ++it) {                                 \
    _Pragma("unroll") for (int j = 0; j < 8; ++j) { BODY; }            \
  }

template <int KIND>
__global__ void probe(int iters, uint32_t* out, long long* cyc) {
  uint32_t v[8];
  float f[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    v[j] = 0x3c003c00u + threadIdx.x * 7 + j;
    f[j] = 0.001f * (threadIdx.x + j);
  }
  __syncthreads();
  const long long t0 = clock64();
  if (KIND == 0) {  // tanh.approx.f32
    OP_LOOP(asm volatile("tanh.approx.f32 %0, %0;" : "+f"(f[j])));
  } else if (KIND == 1) {  // tanh.approx.f16x2
    OP_LOOP(asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(v[j])));
  } else if (KIND == 2) {  // ex2.approx.f32
    OP_LOOP(asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[j])));
  } else if (KIND == 3) {  // ex2.approx.f16x2
    OP_LOOP(asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[j])));
  } else if (KIND == 4) {  // rcp.approx.f32
    OP_LOOP(asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(f[j])));
  } else if (KIND == 5) {  // cvt f32 pair -> f16x2
    OP_LOOP(asm volatile("cvt.rn.satfinite.f16x2.f32 %0, %1, %1;" : "+r"(v[j]) : "f"(f[j])));
  } else if (KIND == 6) {  // fma.rn.f16x2
    OP_LOOP(asm volatile("fma.rn.f16x2 %0, %0, %0, %0;" : "+r"(v[j])));
  } else if (KIND == 7) {  // fma.rn.f32
    OP_LOOP(asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f[j])));
  } else if (KIND == 8) {  // tanh.approx.bf16x2
    OP_LOOP(asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(v[j])));
  } else if (KIND == 9) {  // cvt f16x2 -> two f32 (unpack via cvt.f32.f16)
    OP_LOOP({
      float a;
      asm volatile("{.reg .b16 lo, hi; mov.b32 {lo, hi}, %1; cvt.f32.f16 %0, lo;}" : "=f"(a) : "r"(v[j]));
      f[j] += a;
    });
  } else if (KIND == 10) {  // min/max clamp f16x2
    OP_LOOP(asm volatile("min.f16x2 %0, %0, %0;" : "+r"(v[j])));
  } else if (KIND == 11) {  // mul f16x2
    OP_LOOP(asm volatile("mul.rn.f16x2 %0, %0, %0;" : "+r"(v[j])));
  }
  const long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc ^= v[j] ^ __float_as_uint(f[j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x % 32 == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0;
}

template <int K>
void run(const char* name, int warps) {
  const int iters = 256;
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 4 * 32 * warps);
  cudaMalloc(&cyc, 8 * warps);
  probe<K><<<1, 32 * warps>>>(iters, out, cyc);
  probe<K><<<1, 32 * warps>>>(iters, out, cyc);
  cudaDeviceSynchronize();
  long long h[64];
  cudaMemcpy(h, cyc, 8 * warps, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < warps; ++i) mx = h[i] > mx ? h[i] : mx;
  const double winst = (double)warps * iters * 8;
  printf("%-22s warps %2d: %8lld cycles, %.3f warp-inst/clk/SM (%.1f thread-ops/clk/SM)\n", name,
         warps, mx, winst / mx, 32 * winst / mx);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {8, 16}) {
    run<0>("tanh.approx.f32", w);
    run<1>("tanh.approx.f16x2", w);
    run<8>("tanh.approx.bf16x2", w);
    run<2>("ex2.approx.f32", w);
    run<3>("ex2.approx.f16x2", w);
    run<4>("rcp.approx.f32", w);
    run<5>("cvt.f16x2.f32", w);
    run<9>("cvt.f32.f16(+fadd)", w);
    run<6>("fma.rn.f16x2", w);
    run<11>("mul.rn.f16x2", w);
    run<10>("min.f16x2", w);
    run<7>("fma.rn.f32", w);
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
