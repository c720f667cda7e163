// Microbenchmark: the fused selection epilogue (epi_select, pre-noise TMEM columns) alone on
// one CTA -- 8 epilogue warps over 128 rows x 256 classes, timed per phase with globaltimer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -o tools/sel_probe tools/sel_probe.cu
#include "../paper_1611_09482_b200/csrc/cell_tc.cu"
using namespace fw;
using namespace fw::ptx;
namespace fw { void set_error(const std::string& s) { fprintf(stderr, "%s\n", s.c_str()); } }

__global__ void __launch_bounds__(480, 1) probe(ChainArgs a, SelectArgs sel, int reps, int busy) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  if (warp >= 2 && warp < 10) {
    const int sub = warp & 3, hf = (warp - 2) >> 2, r = sub * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(sub * 32) << 16);
    // fill logits and bias+noise columns
    for (int c = hf * 256; c < hf * 256 + 256; c += 32) {
      float v[32];
      for (int j = 0; j < 32; ++j) v[j] = (float)((r * 131 + (c + j) * 17) % 97) * 0.01f;
      tmem_st32(trow + c, v);
    }
    tc_fence_before();
    named_bar_sync(1, 256);
    tc_fence_after();
    const bool t2 = warp == 2 && lane == 0;
    for (int it = 0; it < reps; ++it) {
      named_bar_sync(1, 256);
      trace_g(a, t2, 28);
      epi_select(trow, r, hf, r, sel, reinterpret_cast<float*>(smem), 256, true, t2 ? &a : nullptr);
      named_bar_sync(1, 256);
      trace_g(a, t2, 24);
    }
  } else if (busy && warp >= 10 && warp < 14) {
    // optional: polling warps as in the tail (relaxed loads + nanosleep)
    for (int i = 0; i < 2000; ++i) {
      (void)ld_relaxed_gpu(a.zflag);
      __nanosleep(64);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* tr;
  cudaMalloc(&tr, 64 * 8);
  cudaMemset(tr, 0, 64 * 8);
  float* bias;
  cudaMalloc(&bias, 256 * 4);
  cudaMemset(bias, 0, 1024);
  int32_t *oc, *cn;
  cudaMalloc(&oc, 1024);
  cudaMalloc(&cn, 1024);
  uint32_t* flag;
  cudaMalloc(&flag, 64);
  cudaMemset(flag, 0, 64);
  ChainArgs a;
  memset(&a, 0, sizeof(a));
  a.trace = tr;
  a.L = 0;
  a.zflag = flag;
  SelectArgs s;
  memset(&s, 0, sizeof(s));
  s.bias = bias;
  s.out_cls = oc;
  s.cls_next = cn;
  s.A = 256;
  s.mode = FW_SAMPLE_GUMBEL;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  for (int busy = 0; busy < 2; ++busy) {
    probe<<<1, 480, 8192>>>(a, s, 3, busy);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[32];
    cudaMemcpy(h, tr, 32 * 8, cudaMemcpyDeviceToHost);
    printf("busy=%d %s: start->ld %lld ns, cc0 %lld, cc1 %lld, cc2 %lld, loop %lld, exch %lld, done %lld ns\n", busy,
           cudaGetErrorString(e), h[29] - h[28], h[21] - h[29], h[22] - h[21], h[23] - h[22],
           h[26] - h[23], h[27] - h[26], h[24] - h[28]);
  }
  return 0;
}
