// FP32 CUDA-core peak on this device: the denominator of the fp32 configs' roofline
// ("FP32 CUDA-core peak ... not measured. Measure it.").
//
// Every thread runs 8 independent FFMA chains (enough to cover the FMA pipe latency at
// 4 warps per SMSP), 2 flops per FFMA, grid = 4 x SMs blocks of 512 threads; best of 10
// launches timed with CUDA events. Clocks are not touched (the driver owns them); the
// SM clock during the run is reported beside the result by the caller (nvidia-smi).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp32_peak tools/fp32_peak.cu
//   tools/fp32_peak            -> one JSON line
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(512) ffma_loop(float* out, float a, float b) {
  float v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = threadIdx.x * 1e-3f + c;
#pragma unroll 4
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = fmaf(v[c], a, b);
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 12345.678f) out[threadIdx.x] = s;  // keeps the chains alive
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 4096);
  const int blocks = 4 * sms, threads = 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ffma_loop<<<blocks, threads>>>(out, 0.999f, 1e-4f);  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    ffma_loop<<<blocks, threads>>>(out, 0.999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * kChains * kIters * (double)blocks * threads;
  const double tflops = flops / (best * 1e-3) / 1e12;
  const double nominal = 2.0 * 128 * sms * (clk_khz * 1e3) / 1e12;
  printf("{\"fp32_tflops\": %.2f, \"best_ms\": %.4f, \"sms\": %d, \"max_clock_mhz\": %.0f, "
         "\"nominal_tflops_at_max_clock\": %.2f, \"how\": \"FFMA, 8 independent chains per thread, "
         "%d blocks x %d threads, best of 10 (CUDA events)\", \"error\": \"%s\"}\n",
         tflops, best, sms, clk_khz / 1e3, nominal, blocks, threads,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
