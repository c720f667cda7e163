// K3: plain-mode step kernel -- the reference's own stack in float64.
//
// Literal-parity path for the unmodified reference:
// every node is evaluated in the reference's pinned order (kernel.py:45-56):
// taps k ascending, input channels ascending, each product and sum rounded
// separately (__dmul_rn/__dadd_rn, so no FMA contraction), bias after the taps,
// tanh last. Ring queues follow SURVEY App. A.2 (capacity (w-1)*d; tap k reads
// slot (t - k*d) mod cap; the layer input is written to slot t mod cap after
// all taps are read, which is ConvQueue.peek/pop/push of fast.py:57-88).
// One CTA per stream; the step loop runs on the device.
#include "internal.h"
#include "libm_tanh.cuh"

namespace fw {
namespace {

constexpr int NT = 128;

struct PlainParams {
  PlainDev p;
  int B;
  int64_t t0;
};

__device__ __forceinline__ int64_t ring_slot(int64_t t, int k, int d, int cap) {
  int64_t v = (t - (int64_t)k * d) % cap;
  return v < 0 ? v + cap : v;
}

// Evaluates one layer for stream `sidx`: prev = [h | taps 1..w-1] in smem,
// writes act(...) into hout[0..cout).
__device__ void eval_layer(const PlainDev& p, int l, const double* prev, double* hout) {
  const int cin = p.cin[l], cout = p.cout[l], w = p.w;
  const double* taps = p.taps + p.woff[l];
  const double* bias = p.bias + p.boff[l];
  for (int o = threadIdx.x; o < cout; o += NT) {
    double acc = 0.0;
    for (int k = 0; k < w; ++k) {
      const double* row = taps + ((size_t)k * cout + o) * cin;
      const double* v = prev + (size_t)k * p.cmax;
      for (int c = 0; c < cin; ++c) acc = __dadd_rn(acc, __dmul_rn(row[c], v[c]));
    }
    acc = __dadd_rn(acc, bias[o]);
    if (p.act == 1) acc = libm_tanh(acc);
    hout[o] = acc;
  }
}

__global__ void __launch_bounds__(NT) plain_generate_kernel(PlainParams pp, const double* inputs,
                                                            int n_inputs, int n_steps,
                                                            double* out) {
  extern __shared__ double sm[];
  const PlainDev& p = pp.p;
  const int w = p.w, cmax = p.cmax, B = pp.B;
  double* prev = sm;              // [w][cmax]
  double* hnext = sm + w * cmax;  // [cmax]
  const int sidx = blockIdx.x;
  double x = inputs[sidx];
  for (int i = 0; i < n_steps; ++i) {
    const int64_t t = pp.t0 + i;
    if (threadIdx.x == 0) prev[0] = x;
    __syncthreads();
    for (int l = 0; l < p.n_layers; ++l) {
      const int cin = p.cin[l], d = p.dil[l];
      const int cap = (w - 1) * d;
      double* q = p.queue + p.qoff[l];
      for (int e = threadIdx.x; e < (w - 1) * cin; e += NT) {
        const int k = 1 + e / cin, c = e % cin;
        prev[k * cmax + c] = q[(ring_slot(t, k, d, cap) * B + sidx) * cin + c];
      }
      __syncthreads();
      for (int c = threadIdx.x; c < cin; c += NT)
        q[(ring_slot(t, 0, d, cap) * B + sidx) * cin + c] = prev[c];
      eval_layer(p, l, prev, hnext);
      __syncthreads();
      for (int c = threadIdx.x; c < p.cout[l]; c += NT) prev[c] = hnext[c];
      __syncthreads();
    }
    const double y = prev[0];
    if (threadIdx.x == 0) out[(size_t)i * B + sidx] = y;
    x = (i + 1 < n_inputs) ? inputs[(size_t)(i + 1) * B + sidx] : y;
    __syncthreads();
  }
}

// rec layout: rows roff[l] + (k-1)*cin + c, column = stream.
__global__ void plain_pop_kernel(PlainParams pp, double* rec) {
  const PlainDev& p = pp.p;
  const int B = pp.B, w = p.w;
  const int sidx = blockIdx.x;
  for (int l = 0; l < p.n_layers; ++l) {
    const int cin = p.cin[l], d = p.dil[l], cap = (w - 1) * d;
    const double* q = p.queue + p.qoff[l];
    for (int e = threadIdx.x; e < (w - 1) * cin; e += blockDim.x) {
      const int k = 1 + e / cin, c = e % cin;
      rec[(p.roff[l] + e) * B + sidx] = q[(ring_slot(pp.t0, k, d, cap) * B + sidx) * cin + c];
    }
  }
}

__global__ void __launch_bounds__(NT) plain_compute_kernel(PlainParams pp, const double* in,
                                                           const double* rec, double* out,
                                                           double* states) {
  extern __shared__ double sm[];
  const PlainDev& p = pp.p;
  const int w = p.w, cmax = p.cmax, B = pp.B;
  double* prev = sm;
  double* hnext = sm + w * cmax;
  const int sidx = blockIdx.x;
  if (threadIdx.x == 0) prev[0] = in[sidx];
  __syncthreads();
  for (int l = 0; l < p.n_layers; ++l) {
    const int cin = p.cin[l];
    for (int e = threadIdx.x; e < (w - 1) * cin; e += NT) {
      const int k = 1 + e / cin, c = e % cin;
      prev[k * cmax + c] = rec[(p.roff[l] + e) * B + sidx];
    }
    for (int c = threadIdx.x; c < cin; c += NT) states[(p.soff[l] + c) * B + sidx] = prev[c];
    __syncthreads();
    eval_layer(p, l, prev, hnext);
    __syncthreads();
    for (int c = threadIdx.x; c < p.cout[l]; c += NT) prev[c] = hnext[c];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[sidx] = prev[0];
}

__global__ void plain_push_kernel(PlainParams pp, const double* states) {
  const PlainDev& p = pp.p;
  const int B = pp.B, w = p.w;
  const int sidx = blockIdx.x;
  for (int l = 0; l < p.n_layers; ++l) {
    const int cin = p.cin[l], d = p.dil[l], cap = (w - 1) * d;
    double* q = p.queue + p.qoff[l];
    for (int c = threadIdx.x; c < cin; c += blockDim.x)
      q[(ring_slot(pp.t0, 0, d, cap) * B + sidx) * cin + c] = states[(p.soff[l] + c) * B + sidx];
  }
}

// Naive step: every node of the demand plan of the output at T = n-1, layer by layer, each
// in the same pinned order as eval_layer (so the result equals the queue-cached output bit
// for bit; pre-history inputs are zero, as the cached path's zero-filled queues).
__global__ void __launch_bounds__(NT) plain_naive_kernel(PlainDev p, NaivePlan plan, int B,
                                                         const double* hist, int n, double* out) {
  const int sidx = blockIdx.x, w = p.w;
  double* vals = plan.vals + (size_t)sidx * plan.vals_per_stream;
  const int T = n - 1;
  for (int l = 0; l < p.n_layers; ++l) {
    const int cin = p.cin[l], cout = p.cout[l], cnt = plan.count[l];
    const double* taps = p.taps + p.woff[l];
    const double* bias = p.bias + p.boff[l];
    const int* g = plan.gather + plan.goff[l];
    const int* gs = plan.gsrc + plan.goff[l];
    double* dst = vals + plan.voff[l];
    const double* src = l > 0 ? vals + plan.voff[l - 1] : nullptr;
    for (int e = threadIdx.x; e < cnt * cout; e += NT) {
      const int node = e / cout, o = e % cout;
      double acc = 0.0;
      for (int k = 0; k < w; ++k) {
        const double* row = taps + ((size_t)k * cout + o) * cin;
        const int gi = g[node * w + k];
        if (l == 0) {
          const int tau = T - gi;  // the scalar input of that time step, zero before it
          const double v = tau >= 0 ? hist[(size_t)tau * B + sidx] : 0.0;
          acc = __dadd_rn(acc, __dmul_rn(row[0], v));
        } else if (T - gs[node * w + k] >= 0) {
          const double* v = src + (size_t)gi * cin;
          for (int c = 0; c < cin; ++c) acc = __dadd_rn(acc, __dmul_rn(row[c], v[c]));
        } else {  // a layer output before the history began: the cached path reads zeros
          for (int c = 0; c < cin; ++c) acc = __dadd_rn(acc, __dmul_rn(row[c], 0.0));
        }
      }
      acc = __dadd_rn(acc, bias[o]);
      if (p.act == 1) acc = libm_tanh(acc);
      dst[(size_t)node * cout + o] = acc;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[sidx] = vals[plan.voff[p.n_layers - 1]];
}

PlainParams params(const Handle& h) {
  PlainParams pp;
  pp.p = h.p;
  pp.B = h.batch;
  pp.t0 = h.t;
  return pp;
}

size_t smem(const Handle& h) { return sizeof(double) * (size_t)(h.p.w + 1) * h.p.cmax; }

cudaError_t prep(const void* fn, size_t sm) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
}

}  // namespace

cudaError_t launch_plain_generate(const Handle& h, const double* inputs, int n_inputs,
                                  int n_steps, double* out, cudaStream_t st) {
  const size_t sm = smem(h);
  cudaError_t e = prep((const void*)plain_generate_kernel, sm);
  if (e != cudaSuccess) return e;
  plain_generate_kernel<<<h.batch, NT, sm, st>>>(params(h), inputs, n_inputs, n_steps, out);
  return cudaGetLastError();
}

cudaError_t launch_plain_pop(const Handle& h, double* rec, cudaStream_t st) {
  plain_pop_kernel<<<h.batch, NT, 0, st>>>(params(h), rec);
  return cudaGetLastError();
}

cudaError_t launch_plain_compute(const Handle& h, const double* in, const double* rec,
                                 double* out, double* states, cudaStream_t st) {
  const size_t sm = smem(h);
  cudaError_t e = prep((const void*)plain_compute_kernel, sm);
  if (e != cudaSuccess) return e;
  plain_compute_kernel<<<h.batch, NT, sm, st>>>(params(h), in, rec, out, states);
  return cudaGetLastError();
}

cudaError_t launch_plain_naive(const Handle& h, const double* history, int n, double* out,
                               cudaStream_t st) {
  plain_naive_kernel<<<h.batch, NT, 0, st>>>(h.p, h.naive, h.batch, history, n, out);
  return cudaGetLastError();
}

cudaError_t launch_plain_push(const Handle& h, const double* states, cudaStream_t st) {
  plain_push_kernel<<<h.batch, NT, 0, st>>>(params(h), states);
  return cudaGetLastError();
}

}  // namespace fw
