// Selection rules of the SIMT kernels and of fw_cell_select (one warp per stream), shared
// by cell_simt.cu and prefill.cu. The rules of oracle/cell.py's select_*: argmax takes the first maximum (numpy argmax); Gumbel-max adds -log(-log u) of the
// counter hash (internal.h); inverse CDF takes the smallest i whose running sum of
// exp(l - max) exceeds u * total.
#pragma once

#include "internal.h"

namespace fw {
namespace {

__device__ __forceinline__ float sigmoidf_(float x) { return 1.f / (1.f + expf(-x)); }

// Warp-wide (value, index) maximum; ties go to the lower index (numpy argmax).
__device__ __forceinline__ void warp_argmax(float& v, int& i) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, v, off);
    int oi = __shfl_xor_sync(0xffffffffu, i, off);
    if (ov > v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
}

// Selection for one stream by one warp over A logits in smem.
__device__ int select_class(const float* lg, int A, int mode, uint32_t prefix) {
  const int lane = threadIdx.x & 31;
  if (mode == FW_SAMPLE_INVCDF) {
    float m = -INFINITY;
    for (int a = lane; a < A; a += 32) m = fmaxf(m, lg[a]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    // contiguous chunk per lane, sequential inside, scan across lanes
    const int chunk = (A + 31) / 32;
    const int a0 = min(A, lane * chunk), a1 = min(A, a0 + chunk);
    float part = 0.f;
    for (int a = a0; a < a1; ++a) part += expf(lg[a] - m);
    float incl = part;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      float o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    const float total = __shfl_sync(0xffffffffu, incl, 31);
    const float thr = noise_uniform(prefix, kUniformClass) * total;
    float run = incl - part;
    int found = A;
    for (int a = a0; a < a1; ++a) {
      run += expf(lg[a] - m);
      if (run > thr) {
        found = a;
        break;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) found = min(found, __shfl_xor_sync(0xffffffffu, found, off));
    return found < A ? found : A - 1;
  }
  float best = -INFINITY;
  int bi = A;
  for (int a = lane; a < A; a += 32) {
    float v = lg[a];
    if (mode == FW_SAMPLE_GUMBEL) v += -logf(-logf(noise_uniform(prefix, (uint32_t)a)));
    if (v > best) {
      best = v;
      bi = a;
    }
  }
  warp_argmax(best, bi);
  return bi;
}


}  // namespace
}  // namespace fw
