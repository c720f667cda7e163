// K1: persistent fp32 CUDA-core step kernel for the gated cell.
//
// One CTA owns a tile of BT streams for the whole generate call and loops on
// the device over steps and layers (no launch per step or per layer; SURVEY
// section 3 "Host<->device crossings"). Per layer it performs the reference's
// pop -> compute -> push cycle (fast.py:131-213) for its streams:
//   pop/push : one HBM slot (t mod d_l) of the layer's ring queue is read
//              (x_l[t-d]) and overwritten with the layer input x_l[t] by the
//              same thread, so read-before-write needs no barrier;
//   compute  : a = W0 x_l[t] + W1 x_l[t-d] + b, z = tanh(a[:D]) * sigmoid(a[D:]),
//              s += W_skip z + b_skip, x_{l+1} = x_l + W_res z + b_res;
// then the ReLU-1x1-ReLU-1x1 head, the selection rule and the re-embedding.
// Activations stay in shared memory; weights (fp32, transposed to [in][out]
// for coalescing) stream from L2, each weight load reused BT times.
// Narrow layers split K across thread groups and reduce through smem so a
// batch-1 stream still uses all 256 threads.
//
// This kernel serves every configuration (fp32 cfg1/2/3/5 and, with
// bf16-rounded weights and fp32 math, cfg4); the tcgen05 kernel (cell_tc.cu)
// replaces it for large batches.
#include <cstdlib>

#include "internal.h"
#include "tc_ptx.cuh"
#include "select.cuh"

namespace fw {
namespace {

// threads per CTA: a template parameter, 256 (1024 at one stream per CTA measured slower:
// the barriers cost more than the extra loads in flight gain)

struct SimtParams {
  CellDims d;
  int B;
  int pre_pop;  // all layers' pops at the top of each step ([L][BT][R] floats of smem)
  const int* dil;
  const int64_t* qoff;
  float* queue;
  SimtWeights w;
  CellRun run;
};

// out[b][o] = epi(b, o, sum_c WT[c][o] * in[b][c]) for o < N, b < BT.
template <int NT, int BT, typename Epi>
__device__ __forceinline__ void gemv(const float* __restrict__ WT, int K, int N,
                                     const float* in, int ldin, float* red, Epi epi) {
  const int tid = threadIdx.x;
  if (N >= NT) {
    for (int o = tid; o < N; o += NT) {
      float acc[BT];
#pragma unroll
      for (int b = 0; b < BT; ++b) acc[b] = 0.f;
      int c = 0;
      // 16 independent weight loads in flight per thread: at batch 1 the loop is a chain of
      // L2 round trips, not FMA-bound (same summation order as the 4-wide loop below)
      for (; c + 16 <= K; c += 16) {
        float w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) w[j] = __ldg(WT + (size_t)(c + j) * N + o);
#pragma unroll
        for (int b = 0; b < BT; ++b) {
          const float* x = in + b * ldin + c;
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[b] = fmaf(w[j], x[j], acc[b]);
        }
      }
      for (; c + 4 <= K; c += 4) {
        float w0 = __ldg(WT + (size_t)(c + 0) * N + o);
        float w1 = __ldg(WT + (size_t)(c + 1) * N + o);
        float w2 = __ldg(WT + (size_t)(c + 2) * N + o);
        float w3 = __ldg(WT + (size_t)(c + 3) * N + o);
#pragma unroll
        for (int b = 0; b < BT; ++b) {
          const float* x = in + b * ldin + c;
          acc[b] = fmaf(w0, x[0], acc[b]);
          acc[b] = fmaf(w1, x[1], acc[b]);
          acc[b] = fmaf(w2, x[2], acc[b]);
          acc[b] = fmaf(w3, x[3], acc[b]);
        }
      }
      for (; c < K; ++c) {
        float w0 = __ldg(WT + (size_t)c * N + o);
#pragma unroll
        for (int b = 0; b < BT; ++b) acc[b] = fmaf(w0, in[b * ldin + c], acc[b]);
      }
#pragma unroll
      for (int b = 0; b < BT; ++b) epi(b, o, acc[b]);
    }
    return;
  }
  // Split K over G groups of N threads, reduce partials in a fixed order.
  const int G = NT / N;
  const int o = tid % N, g = tid / N;
  const int kc = (K + G - 1) / G;
  const int k0 = g * kc, k1 = min(K, k0 + kc);
  float acc[BT];
#pragma unroll
  for (int b = 0; b < BT; ++b) acc[b] = 0.f;
  if (g < G) {
    int c = k0;
    for (; c + 16 <= k1; c += 16) {
      float w[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) w[j] = __ldg(WT + (size_t)(c + j) * N + o);
#pragma unroll
      for (int b = 0; b < BT; ++b)
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[b] = fmaf(w[j], in[b * ldin + c + j], acc[b]);
    }
    for (; c < k1; ++c) {
      float w0 = __ldg(WT + (size_t)c * N + o);
#pragma unroll
      for (int b = 0; b < BT; ++b) acc[b] = fmaf(w0, in[b * ldin + c], acc[b]);
    }
#pragma unroll
    for (int b = 0; b < BT; ++b) red[(g * BT + b) * N + o] = acc[b];
  }
  __syncthreads();
  for (int e = tid; e < BT * N; e += NT) {
    const int b = e / N, oo = e % N;
    float v = 0.f;
    for (int gg = 0; gg < G; ++gg) v += red[(gg * BT + b) * N + oo];
    epi(b, oo, v);
  }
}

// the pre-pop buffer follows the class ids (16-byte aligned)
__device__ __forceinline__ float* cls_end(int* cls, int bt) {
  return reinterpret_cast<float*>(cls + ((bt + 3) & ~3));
}

template <int BT, int NT>
__global__ void __launch_bounds__(NT) cell_simt_kernel(SimtParams p) {
  extern __shared__ float smem[];
  const CellDims d = p.d;
  const int R = d.R, D = d.D, S = d.S, H = d.H, A = d.A, L = d.L;
  float* xx = smem;                 // [BT][2R]: x_l[t] | x_l[t-d]
  float* a = xx + BT * 2 * R;       // [BT][2D]
  float* z = a + BT * 2 * D;        // [BT][D]
  float* s = z + BT * D;            // [BT][S]
  float* hb = s + BT * S;           // [BT][H]
  float* lg = hb + BT * H;          // [BT][A]
  float* red = lg + BT * A;         // [NT * BT] K-split partials
  int* cls = reinterpret_cast<int*>(red + NT * BT);  // [BT]

  const int tid = threadIdx.x;
  const int s0 = blockIdx.x * BT;
  const int nb = min(BT, p.B - s0);
  const CellRun& run = p.run;
  const int B = p.B;

  if (tid < BT) cls[tid] = (tid < nb) ? run.inputs[s0 + tid] : 0;
  __syncthreads();
  // pops of all layers at the top of the step, when they fit: x_l[t-d] does not depend on
  // the step's chain, so the ring reads leave the per-layer dependency chain (at small batch
  // each was an L2/HBM round trip per layer)
  const bool pre_pop = p.pre_pop != 0;
  float* xd_all = cls_end(cls, BT);  // [L][BT][R] when pre_pop
  const int Rp = (R + 3) & ~3;       // channels padded to whole 16-byte chunks
  const size_t slot_elems = (size_t)((B + 127) / 128) * 128 * Rp;

  for (int i = 0; i < run.n_steps; ++i) {
    const int64_t t = run.t0 + i;
    // x_0 = E[c_t]; s = 0
    for (int e = tid; e < BT * R; e += NT) {
      const int b = e / R, r = e % R;
      xx[b * 2 * R + r] = __ldg(p.w.embed + (size_t)clamp_class(cls[b], A) * R + r);
    }
    for (int e = tid; e < BT * S; e += NT) s[e] = 0.f;
    if (pre_pop) {
      for (int e = tid; e < L * nb * R; e += NT) {
        const int l = e / (nb * R), rest = e % (nb * R);
        const int b = rest / R, r = rest % R;
        const int st = s0 + b;
        const float* q = p.queue + p.qoff[l] + (size_t)(t % p.dil[l]) * slot_elems;
        xd_all[(l * BT + b) * R + r] = q[((size_t)((st >> 7) * (Rp / 4) + (r >> 2)) * 128 + (st & 127)) * 4 + (r & 3)];
      }
    }
    __syncthreads();

    for (int l = 0; l < L; ++l) {
      // pop + push on slot t mod d_l: read x_l[t-d], cache x_l[t] (fast.py:192)
      // slot layout [ceil(B/128)][R/4][128][4] (shared with the tcgen05 path): element
      // (stream s, channel r) at ((s/128 * R/4 + r/4) * 128 + s%128) * 4 + r%4; e walks the
      // tile's streams contiguously per 16-byte channel chunk.
      const int dl = p.dil[l];
      float* q = p.queue + p.qoff[l] + (size_t)(t % dl) * slot_elems;
      for (int e = tid; e < nb * Rp; e += NT) {
        const int j = e & 3, rest = e >> 2;
        const int b = rest % nb, c4 = rest / nb;
        const int r = c4 * 4 + j;
        if (r >= R) continue;
        const int s = s0 + b;
        float* slot = q + ((size_t)((s >> 7) * (Rp / 4) + c4) * 128 + (s & 127)) * 4 + j;
        const float old = pre_pop ? xd_all[(l * BT + b) * R + r] : *slot;
        *slot = xx[b * 2 * R + r];
        xx[b * 2 * R + R + r] = old;
      }
      __syncthreads();
      const float* db = p.w.dil_b + (size_t)l * 2 * D;
      gemv<NT, BT>(p.w.dilT + (size_t)l * 2 * R * 2 * D, 2 * R, 2 * D, xx, 2 * R, red,
               [&](int b, int o, float v) { a[b * 2 * D + o] = v + db[o]; });
      __syncthreads();
      for (int e = tid; e < BT * D; e += NT) {
        const int b = e / D, j = e % D;
        z[e] = tanhf(a[b * 2 * D + j]) * sigmoidf_(a[b * 2 * D + D + j]);
      }
      __syncthreads();
      const float* sb = p.w.skip_b + (size_t)l * S;
      gemv<NT, BT>(p.w.skipT + (size_t)l * D * S, D, S, z, D, red,
               [&](int b, int o, float v) { s[b * S + o] += v + sb[o]; });
      if (l + 1 < L) {
        __syncthreads();
        const float* rb = p.w.res_b + (size_t)l * R;
        gemv<NT, BT>(p.w.resT + (size_t)l * D * R, D, R, z, D, red,
                 [&](int b, int o, float v) { xx[b * 2 * R + o] += v + rb[o]; });
      }
      __syncthreads();
    }
    // head: logits = W2 relu(W1 relu(s) + b1) + b2
    for (int e = tid; e < BT * S; e += NT) s[e] = fmaxf(s[e], 0.f);
    __syncthreads();
    gemv<NT, BT>(p.w.h1T, S, H, s, S, red,
             [&](int b, int o, float v) { hb[b * H + o] = fmaxf(v + p.w.h1_b[o], 0.f); });
    __syncthreads();
    gemv<NT, BT>(p.w.h2T, H, A, hb, H, red,
             [&](int b, int o, float v) { lg[b * A + o] = v + p.w.h2_b[o]; });
    __syncthreads();

    if (run.logits != nullptr && i < run.n_logit_steps) {
      float* dst = run.logits + ((size_t)i * B + s0) * A;
      for (int e = tid; e < nb * A; e += NT) dst[e] = lg[e];
    }
    const int warp = tid >> 5;
    for (int b = warp; b < nb; b += NT / 32) {
      const uint32_t gs = (uint32_t)(run.stream_offset + s0 + b);
      const uint32_t prefix = noise_prefix(run.seed, gs, (uint32_t)t);
      const int c = select_class(lg + b * A, A, run.mode, prefix);
      if ((tid & 31) == 0) {
        run.out[(size_t)i * B + s0 + b] = c;
        cls[b] = (i + 1 < run.n_inputs) ? run.inputs[(size_t)(i + 1) * B + s0 + b] : c;
      }
    }
    __syncthreads();
  }
}

// Cluster size for a stream count (0: no cluster kernel): the small-batch kernel
// (cell_lat.cu) splits every GEMV's outputs over the C CTAs of a cluster, so every slice
// must divide evenly
int cluster_for(const CellDims& d, int B) {
  if (const char* e = getenv("FW_SIMT_CLUSTER")) return atoi(e);
  // one stream per cluster while the clusters fit the SMs side by side (B * C <= 148: up to
  // 9 streams at 16 CTAs ... 74 at 2); past that the weight-staged kernel shares each weight
  // load between several streams
  for (int c = 16; c >= 2; c /= 2)
    if ((int64_t)B * c <= 148 && lat_supported(d, c)) return c;
  return 0;
}


// ---- K1s: weight-staged fp32 kernel (mid batches, fp32 configs 3 and 5) -----------------
// The per-CTA kernel above reads every weight with __ldg and spends most of a layer waiting on
// L2 round trips (cfg5: 13 us per layer for 8 streams, < 10 % of the FP32 pipe). Here a
// producer warp streams the step's weight matrices, in consumption order, through a ring of
// shared-memory stages with 1-D bulk copies (TMA engine, mbarrier completion), a GEMV or more
// ahead of the 8 compute warps, so the L2 latency leaves the layer chain. The compute warps
// read each weight from shared memory once for all BT streams of the CTA (4 consecutive
// outputs x BT streams per thread, K split across thread groups and reduced in a fixed order).
// The ring pops are prefetched two layers ahead by the threads that push the same elements
// (cp.async: program order covers the slot reuse, as in the tcgen05 chain). Same cell, same
// pop -> compute -> push order per layer as cell_simt_kernel (fast.py:131-213).
constexpr int kStNT = 256;                 // compute threads (8 warps; 16 measured slower: 908 vs 721 us/step on cfg5)
constexpr int kStThreads = kStNT + 32;     // + the weight producer warp
constexpr int kStStagesMax = 8;            // weight ring depth (runtime, <= 8)
constexpr int kStBarId = 1;                // named barrier of the compute warps

struct StagedLayout {
  int stage_bytes;  // one weight stage
  int issuers;      // producer lanes issuing a chunk's bulk copies
  int stages;       // ring depth
  // float offsets of the activation buffers from the start of dynamic smem
  int xx, z, s, hb, lg, red, pops, bias, hbias, lcon, cls, ring, bars;
  size_t total;
};

// rows of a [K][N] fp32 weight matrix per stage (a multiple of 4)
__host__ __device__ __forceinline__ int st_rows(int K, int N, int stage_bytes) {
  const int r = (stage_bytes / (N * 4)) & ~3;
  return r < K ? r : K;
}

struct StageRing {
  uint64_t* full;
  uint64_t* empty;
  float* buf;
  int stage_floats;
  int slot;
  uint32_t ph;
  int nst;                // stages in the ring
  __device__ __forceinline__ void advance() {
    if (++slot == nst) {
      slot = 0;
      ph ^= 1u;
    }
  }
};

// Producer side of one GEMV: its K-chunks into the ring, run by the whole producer warp.
// A chunk is split into `issuers` bulk copies issued by different lanes (one thread's bulk
// copies execute one after another). (TMA multicast of each stage across a 2/4/8-CTA cluster
// was measured slower, DESIGN.md section 4 K1s.)
__device__ __forceinline__ void st_produce(StageRing& rg, const float* W, int K, int N,
                                           int stage_bytes, int issuers) {
  const int lane = threadIdx.x & 31;
  const int kc = st_rows(K, N, stage_bytes);
  for (int k0 = 0; k0 < K; k0 += kc) {
    const int rows = min(kc, K - k0);
    const uint32_t bytes = (uint32_t)rows * N * 4;
    if (lane == 0) {
      ptx::mbar_wait(&rg.empty[rg.slot], rg.ph ^ 1u);  // every compute warp released it
      ptx::mbar_arrive_expect_tx(&rg.full[rg.slot], bytes);
    }
    __syncwarp();
    const uint32_t slice = (bytes + 16 * issuers - 1) / (16 * issuers) * 16;
    const uint32_t off = (uint32_t)lane * slice;
    if (lane < issuers && off < bytes)
      ptx::bulk_g2s(reinterpret_cast<uint8_t*>(rg.buf + (size_t)rg.slot * rg.stage_floats) + off,
                    reinterpret_cast<const uint8_t*>(W + (size_t)k0 * N) + off,
                    min(slice, bytes - off), &rg.full[rg.slot]);
    rg.advance();
  }
}

// (a0, a1) += (w0, w1) * x on the packed FP32x2 pipe: one FFMA2 with x as a broadcast
// scalar operand; each lane is the same fused multiply-add as fmaf (bit-identical)
__device__ __forceinline__ void ffma2(float& a0, float& a1, float w0, float w1, float x) {
  unsigned long long acc, w;
  asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(w) : "f"(w0), "f"(w1));
  unsigned long long xx;
  asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(x));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(w), "l"(xx));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc));
}

// Consumer side, part 1: partial sums of out[b][o] = sum_k W[k][o] in[b][k] (b < BT, o < N,
// N % 4 == 0, K % 4 == 0, ldin % 4 == 0) into red[g][b][o], one slice per K group g of the
// thread groups (4 consecutive outputs x BT streams per thread). Returns the group count;
// ends with a barrier of the compute warps.
template <int BT, int OB>
__device__ __forceinline__ int st_partial_ob(StageRing& rg, const float* in, int ldin, int K, int N,
                                          int stage_bytes, float* red) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int NQ = N / OB;
  const int G = NQ >= kStNT ? 1 : kStNT / NQ;
  float acc[OB][BT];
#pragma unroll
  for (int j = 0; j < OB; ++j)
#pragma unroll
    for (int b = 0; b < BT; ++b) acc[j][b] = 0.f;
  const int kc = st_rows(K, N, stage_bytes);
  for (int qq = tid; qq < NQ * G; qq += kStNT) {  // one pass unless N > 4 * kStNT
    const int q = qq % NQ, g = qq / NQ;
    for (int k0 = 0; k0 < K; k0 += kc) {
      const int rows = min(kc, K - k0);
      const int rpg = ((rows + G - 1) / G + 3) & ~3;
      if (qq == tid) ptx::mbar_wait(&rg.full[rg.slot], rg.ph);
      const float* w = rg.buf + (size_t)rg.slot * rg.stage_floats;
      const int ka = g * rpg, kb = min(rows, ka + rpg);
      for (int k = ka; k < kb; k += 4) {
        float wv[4][OB];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float* wr = w + (size_t)(k + u) * N + OB * q;
          if constexpr (OB == 4) {
            const float4 t4 = *reinterpret_cast<const float4*>(wr);
            wv[u][0] = t4.x, wv[u][1] = t4.y, wv[u][2] = t4.z, wv[u][3] = t4.w;
          } else if constexpr (OB == 2) {
            const float2 t2 = *reinterpret_cast<const float2*>(wr);
            wv[u][0] = t2.x, wv[u][1] = t2.y;
          } else {
            wv[u][0] = *wr;
          }
        }
#pragma unroll
        for (int b = 0; b < BT; ++b) {
          const float4 x = *reinterpret_cast<const float4*>(in + b * ldin + k0 + k);
          const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if constexpr (OB % 2 == 0) {
              // output pairs on the packed FP32x2 pipe (FFMA2, the stream's input broadcast):
              // half the issue slots, the same fused multiply-add per output and order
#pragma unroll
              for (int j = 0; j < OB; j += 2) ffma2(acc[j][b], acc[j + 1][b], wv[u][j], wv[u][j + 1], xs[u]);
            } else {
#pragma unroll
              for (int j = 0; j < OB; ++j) acc[j][b] = fmaf(wv[u][j], xs[u], acc[j][b]);
            }
          }
        }
      }
      if (qq == tid) {
        // (CTA-scope release: a cluster-scope one would wait for the ring-push stores)
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&rg.empty[rg.slot]);
        rg.advance();
      }
    }
#pragma unroll
    for (int b = 0; b < BT; ++b) {
#pragma unroll
      for (int j = 0; j < OB; ++j) {
        red[((size_t)g * BT + b) * N + OB * q + j] = acc[j][b];
        acc[j][b] = 0.f;
      }
    }
  }
  if (NQ * G < kStNT && tid >= NQ * G) {
    // idle threads still walk the ring
    for (int k0 = 0; k0 < K; k0 += kc) {
      ptx::mbar_wait(&rg.full[rg.slot], rg.ph);
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&rg.empty[rg.slot]);
      rg.advance();
    }
  }
  ptx::named_bar_sync(kStBarId, kStNT);
  return G;
}

// outputs per thread: 4 (fewest shared-memory loads per FMA) once BT >= 4 streams share each
// weight; at 1-2 streams the phase is latency-bound and as few outputs as keep N / OB <= kStNT
// leave fewer K groups to reduce (measured: cfg5 729 vs 790 us/step at BT = 8)
template <int BT>
__device__ __forceinline__ int st_partial(StageRing& rg, const float* in, int ldin, int K, int N,
                                          int stage_bytes, float* red) {
  if (BT >= 4) return st_partial_ob<BT, 4>(rg, in, ldin, K, N, stage_bytes, red);
  if (N <= kStNT) return st_partial_ob<BT, 1>(rg, in, ldin, K, N, stage_bytes, red);
  if (N <= 2 * kStNT) return st_partial_ob<BT, 2>(rg, in, ldin, K, N, stage_bytes, red);
  return st_partial_ob<BT, 4>(rg, in, ldin, K, N, stage_bytes, red);
}

// fixed-order sum of the K groups' partials of the 4 elements at e4 = b * N + 4 q
__device__ __forceinline__ float4 st_sum4(const float* red, int G, int BTN, int e4) {
  float4 v = *reinterpret_cast<const float4*>(red + e4);
  for (int g = 1; g < G; ++g) {
    const float4 u = *reinterpret_cast<const float4*>(red + (size_t)g * BTN + e4);
    v.x += u.x;
    v.y += u.y;
    v.z += u.z;
    v.w += u.w;
  }
  return v;
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 relu4(float4 a) {
  return make_float4(fmaxf(a.x, 0.f), fmaxf(a.y, 0.f), fmaxf(a.z, 0.f), fmaxf(a.w, 0.f));
}
#define ST_F4(p) (*reinterpret_cast<float4*>(p))
#define ST_C4(p) (*reinterpret_cast<const float4*>(p))

// Part 2 for the head GEMVs: reduce + epilogue over 4 outputs at a time, then a barrier.
template <int BT, typename Epi>
__device__ __forceinline__ void st_gemv(StageRing& rg, const float* in, int ldin, int K, int N,
                                        int stage_bytes, float* red, Epi epi) {
  const int G = st_partial<BT>(rg, in, ldin, K, N, stage_bytes, red);
  const int NQ = N >> 2;
  for (int e = threadIdx.x; e < BT * NQ; e += kStNT) {
    const int b = e / NQ, o = 4 * (e - b * NQ);
    epi(b, o, st_sum4(red, G, BT * N, b * N + o));
  }
  ptx::named_bar_sync(kStBarId, kStNT);
}

template <int BT>
StagedLayout staged_layout(const CellDims& d, int stages = 3) {
  StagedLayout y{};
  y.stages = stages;
  int o = 0;
  auto take = [&](int floats) {
    const int at = o;
    o += (floats + 31) & ~31;  // 128-byte aligned buffers
    return at;
  };
  y.xx = take(2 * BT * 2 * d.R);  // two layer buffers
  y.z = take(BT * d.D);
  y.s = take(BT * d.S);
  y.hb = take(BT * d.H);
  y.lg = take(BT * d.A);
  y.red = take(kStNT * 4 * BT);
  y.pops = take(4 * BT * d.R);
  y.bias = take(4 * (2 * d.D + d.S + d.R));  // per-layer biases, prefetched with the pops
  y.hbias = take(d.H + d.A);
  y.lcon = take(4 * d.L);                    // ring offsets (int64), slots of steps t, t+1
  y.cls = take(BT);
  y.bars = take(2 * 2 * kStStagesMax);
  y.ring = take(0);
  const size_t budget = 227 * 1024 - 1024;
  const size_t used = (size_t)y.ring * 4;
  y.stage_bytes = used >= budget ? 0 : (int)(((budget - used) / stages) & ~(size_t)1023);
  y.total = used + (size_t)stages * y.stage_bytes;
  return y;
}

// Per layer (gg = step * L + l, layer buffers xx[gg & 1] = x_l[t] | x_l[t-d]):
//   push x_l[t] -> slot; dil partials; [bar] reduce + gate -> z, the pop of layer gg+1 into the
//   other buffer, prefetch of layer gg+3; [bar] skip|res partials over z (one [D][S+R] weight
//   matrix); [bar] s += .., x_{l+1} -> the other buffer; [bar]
// Sh: the shape at compile time (kFixed) for BASELINE config 5, so the GEMV loops see
// constant trip counts; StAnyShape reads it at run time.
struct StAnyShape {
  static constexpr bool kFixed = false;
  static constexpr int R = 0, D = 0, S = 0, H = 0, A = 0;
};
template <int R_, int D_, int S_, int H_, int A_>
struct StShape {
  static constexpr bool kFixed = true;
  static constexpr int R = R_, D = D_, S = S_, H = H_, A = A_;
};
template <int BT, class Sh = StAnyShape>
__global__ void __launch_bounds__(kStThreads, 1) cell_staged_kernel(SimtParams p, StagedLayout y) {
  extern __shared__ __align__(1024) float smf[];
  const CellDims d = p.d;
  const int R = Sh::kFixed ? Sh::R : d.R, D = Sh::kFixed ? Sh::D : d.D, S = Sh::kFixed ? Sh::S : d.S,
            H = Sh::kFixed ? Sh::H : d.H, A = Sh::kFixed ? Sh::A : d.A, L = d.L;
  const int SR = S + R;
  float* xx = smf + y.xx;  // [2][BT][2R]
  float* z = smf + y.z;    // [BT][D]
  float* s = smf + y.s;    // [BT][S]
  float* hb = smf + y.hb;  // [BT][H]
  float* lg = smf + y.lg;  // [BT][A]
  float* red = smf + y.red;
  float* pops = smf + y.pops;  // [4][BT][R]: prefetched x_{t-d} of layers gg % 4
  // [4][2D | S | R]: dil / skip / res biases of the prefetched layers (global loads in the
  // epilogues would put an L2 round trip per GEMV on the chain)
  float* bias = smf + y.bias;
  float* hbias = smf + y.hbias;  // h1 | h2 biases
  int64_t* qoff_s = reinterpret_cast<int64_t*>(smf + y.lcon);
  int* slot_s = reinterpret_cast<int*>(qoff_s + L);  // [2][L]: slots of steps t, t+1
  int* cls = reinterpret_cast<int*>(smf + y.cls);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smf + y.bars);
  StageRing rg{bars, bars + kStStagesMax, smf + y.ring, y.stage_bytes / 4, 0, 0u,
               y.stages};
  const int NB = 2 * D + S + R;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int s0 = blockIdx.x * BT;
  const int nb = min(BT, p.B - s0);
  const CellRun& run = p.run;
  const int B = p.B;
  const int sb = y.stage_bytes;
  const int GL = run.n_steps * L;
  if (tid == 0) {
    for (int i = 0; i < rg.nst; ++i) {
      ptx::mbar_init(&rg.full[i], 1);
      ptx::mbar_init(&rg.empty[i], kStNT / 32);
    }
    ptx::fence_mbar_init();
  }
  if (tid < BT) cls[tid] = (tid < nb) ? run.inputs[s0 + tid] : 0;
  for (int e = tid; e < L; e += blockDim.x) {
    qoff_s[e] = p.qoff[e];
    slot_s[e] = (int)(run.t0 % p.dil[e]);
    slot_s[L + e] = (int)((run.t0 + 1) % p.dil[e]);
  }
  for (int e = tid; e < H + A; e += blockDim.x) hbias[e] = e < H ? p.w.h1_b[e] : p.w.h2_b[e - H];
  __syncthreads();

  if (warp == kStNT / 32) {
    // ---- weight producer: the step's GEMVs in the compute warps' order ----
    const int is = y.issuers;
    for (int i = 0; i < run.n_steps; ++i) {
      for (int l = 0; l < L; ++l) {
        st_produce(rg, p.w.dilT + (size_t)l * 2 * R * 2 * D, 2 * R, 2 * D, sb, is);
        st_produce(rg, p.w.catT + (size_t)l * D * SR, D, SR, sb, is);
      }
      st_produce(rg, p.w.h1T, S, H, sb, is);
      st_produce(rg, p.w.h2T, H, A, sb, is);
    }
    return;
  }

  // ring pops: thread e owns (stream b, 4-channel chunk c4) for every layer -- it pushes the
  // chunk and prefetches the same chunk three layers ahead (program order covers slot reuse)
  const int Rp = (R + 3) & ~3;
  const int R4 = R >> 2;  // R % 4 == 0 here
  const size_t slot_elems = (size_t)((B + 127) / 128) * 128 * Rp;
  // layer gg of step i0 + (0 | 1): slot from the table of step t or t+1
  auto slot_ptr = [&](int gg, int i0, int b, int c4) {
    const int l = gg % L;
    const int st = s0 + b;
    return p.queue + qoff_s[l] + (size_t)slot_s[(gg / L - i0) * L + l] * slot_elems +
           ((size_t)((st >> 7) * (Rp / 4) + c4) * 128 + (st & 127)) * 4;
  };
  auto prefetch = [&](int gg, int i0) {
    if (gg < GL) {
      for (int e = tid; e < nb * R4; e += kStNT) {
        const int b = e / R4, c4 = e % R4;
        ptx::cp_async16(ptx::smem_u32(pops + ((gg % 4) * BT + b) * R + 4 * c4), slot_ptr(gg, i0, b, c4));
      }
      const int l = gg % L;
      float* bb = bias + (gg % 4) * NB;
      for (int e = tid; e < NB / 4; e += kStNT) {
        const int o = 4 * e;
        const float* src = o < 2 * D ? p.w.dil_b + (size_t)l * 2 * D + o
                         : o < 2 * D + S ? p.w.skip_b + (size_t)l * S + (o - 2 * D)
                                         : p.w.res_b + (size_t)l * R + (o - 2 * D - S);
        ptx::cp_async16(ptx::smem_u32(bb + o), src);
      }
    }
    ptx::cp_async_commit();
  };
  auto take_pops = [&](int gg) {  // prefetched x_{t-d} of layer gg -> xx[gg & 1][.][R..2R)
    float* xd = xx + (gg & 1) * BT * 2 * R + R;
    for (int e = tid; e < nb * R4; e += kStNT) {
      const int b = e / R4, c4 = e % R4;
      *reinterpret_cast<float4*>(xd + b * 2 * R + 4 * c4) =
          *reinterpret_cast<const float4*>(pops + ((gg % 4) * BT + b) * R + 4 * c4);
    }
  };
  prefetch(0, 0);
  prefetch(1, 0);
  prefetch(2, 0);
  ptx::cp_async_wait<2>();
  take_pops(0);

  for (int i = 0; i < run.n_steps; ++i) {
    const int64_t t = run.t0 + i;
    float* x0 = xx + ((i * L) & 1) * BT * 2 * R;
    for (int e = tid; e < BT * R; e += kStNT) {
      const int b = e / R, r = e % R;
      x0[b * 2 * R + r] = __ldg(p.w.embed + (size_t)clamp_class(cls[b], A) * R + r);
    }
    for (int e = tid; e < BT * S; e += kStNT) s[e] = 0.f;
    if (i > 0)
      for (int e = tid; e < L; e += kStNT) {  // slot tables of steps t, t+1
        slot_s[e] = slot_s[L + e];
        slot_s[L + e] = (int)((t + 1) % p.dil[e]);
      }
    ptx::named_bar_sync(kStBarId, kStNT);
    for (int l = 0; l < L; ++l) {
      const int gg = i * L + l;
      float* xc = xx + (gg & 1) * BT * 2 * R;
      float* xn = xx + ((gg + 1) & 1) * BT * 2 * R;
      const float* bl = bias + (gg % 4) * NB;  // (the prefetch of gg + 3 fills another)
      // push x_l[t] into slot t mod d_l (fast.py:200-213; its pop, x_l[t-d], was read ahead)
      for (int e = tid; e < nb * R4; e += kStNT) {
        const int b = e / R4, c4 = e % R4;
        *reinterpret_cast<float4*>(slot_ptr(gg, i, b, c4)) =
            *reinterpret_cast<const float4*>(xc + b * 2 * R + 4 * c4);
      }
      const int G1 = st_partial<BT>(rg, xc, 2 * R, 2 * R, 2 * D, sb, red);
      // gate: z = tanh(a[:D]) * sigmoid(a[D:]), a = partial sums + bias
      for (int e = tid; e < BT * (D >> 1); e += kStNT) {
        const int b = e / (D >> 1), j = 2 * (e - b * (D >> 1));
        const int ea = b * 2 * D + j;
        float2 va = *reinterpret_cast<const float2*>(red + ea);
        float2 vs = *reinterpret_cast<const float2*>(red + ea + D);
        for (int g = 1; g < G1; ++g) {
          const float2 ua = *reinterpret_cast<const float2*>(red + (size_t)g * BT * 2 * D + ea);
          const float2 us = *reinterpret_cast<const float2*>(red + (size_t)g * BT * 2 * D + ea + D);
          va.x += ua.x, va.y += ua.y, vs.x += us.x, vs.y += us.y;
        }
        *reinterpret_cast<float2*>(z + b * D + j) =
            make_float2(tanhf(va.x + bl[j]) * sigmoidf_(vs.x + bl[D + j]),
                        tanhf(va.y + bl[j + 1]) * sigmoidf_(vs.y + bl[D + j + 1]));
      }
      ptx::cp_async_wait<1>();  // this thread's prefetch of layer gg + 1
      if (gg + 1 < GL) take_pops(gg + 1);
      prefetch(gg + 3, i);
      ptx::named_bar_sync(kStBarId, kStNT);
      const int G2 = st_partial<BT>(rg, z, D, D, SR, sb, red);
      const bool res = l + 1 < L;
      for (int e = tid; e < BT * (SR >> 2); e += kStNT) {
        const int b = e / (SR >> 2), o = 4 * (e - b * (SR >> 2));
        const float4 v = add4(st_sum4(red, G2, BT * SR, b * SR + o), ST_C4(bl + 2 * D + o));
        if (o < S) ST_F4(s + b * S + o) = add4(ST_F4(s + b * S + o), v);
        else if (res) ST_F4(xn + b * 2 * R + (o - S)) = add4(ST_F4(xc + b * 2 * R + (o - S)), v);
      }
      ptx::named_bar_sync(kStBarId, kStNT);
    }
    // head: logits = W2 relu(W1 relu(s) + b1) + b2
    for (int e = tid; e < BT * S / 4; e += kStNT) ST_F4(s + 4 * e) = relu4(ST_F4(s + 4 * e));
    ptx::named_bar_sync(kStBarId, kStNT);
    st_gemv<BT>(rg, s, S, S, H, sb, red,
                [&](int b, int o, float4 v) { ST_F4(hb + b * H + o) = relu4(add4(v, ST_F4(hbias + o))); });
    st_gemv<BT>(rg, hb, H, H, A, sb, red,
                [&](int b, int o, float4 v) { ST_F4(lg + b * A + o) = add4(v, ST_F4(hbias + H + o)); });
    if (run.logits != nullptr && i < run.n_logit_steps) {
      float* dst = run.logits + ((size_t)i * B + s0) * A;
      for (int e = tid; e < nb * A; e += kStNT) dst[e] = lg[e];
    }
    for (int b = warp; b < nb; b += kStNT / 32) {
      const uint32_t gs = (uint32_t)(run.stream_offset + s0 + b);
      const uint32_t prefix = noise_prefix(run.seed, gs, (uint32_t)t);
      const int c = select_class(lg + b * A, A, run.mode, prefix);
      if ((tid & 31) == 0) {
        run.out[(size_t)i * B + s0 + b] = c;
        cls[b] = (i + 1 < run.n_inputs) ? run.inputs[(size_t)(i + 1) * B + s0 + b] : c;
      }
    }
    ptx::named_bar_sync(kStBarId, kStNT);
  }
  ptx::cp_async_wait<0>();
}

bool staged_supported(const CellDims& d) {
  auto m4 = [](int v) { return v % 4 == 0; };
  return d.L >= 3 && m4(d.R) && m4(d.D) && m4(d.S) && m4(d.H) && m4(d.A) && 2 * d.D <= 1024 &&
         d.S + d.R <= 1024 && d.H <= 1024 && d.A <= 1024 && d.R <= 1024 &&
         staged_layout<8>(d).stage_bytes >= 4 * 4 * 1024;
}

template <int BT, class Sh = StAnyShape>
cudaError_t launch_staged(const SimtParams& p, cudaStream_t st) {
  int stages = 3;
  if (const char* ev = getenv("FW_SIMT_STAGES")) stages = max(2, min(kStStagesMax, atoi(ev)));
  StagedLayout y = staged_layout<BT>(p.d, stages);
  if (y.stage_bytes < 4 * 4 * 1024) y = staged_layout<BT>(p.d, 3);
  y.issuers = 4;
  if (const char* ev = getenv("FW_SIMT_ISSUERS")) y.issuers = max(1, min(32, atoi(ev)));
  cudaError_t e = cudaFuncSetAttribute(cell_staged_kernel<BT, Sh>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)y.total);
  if (e != cudaSuccess) return e;
  const int grid = (p.B + BT - 1) / BT;
  cell_staged_kernel<BT, Sh><<<grid, kStThreads, y.total, st>>>(p, y);
  return cudaGetLastError();
}

constexpr size_t kPrePopMax = 64 * 1024;  // bytes of smem the pre-pop buffer may take

template <int BT>
size_t pre_pop_bytes(const CellDims& d) {
  return sizeof(float) * (size_t)d.L * BT * d.R;
}
template <int BT, int NT>
size_t smem_bytes(const CellDims& d) {
  const size_t pp = pre_pop_bytes<BT>(d);
  return sizeof(float) * (size_t)(BT * (2 * d.R + 2 * d.D + d.D + d.S + d.H + d.A) + NT * BT) +
         sizeof(int) * ((BT + 3) & ~3) + (pp <= kPrePopMax ? pp : 0);
}

template <int BT, int NT = 256>
cudaError_t launch_bt(const SimtParams& p, cudaStream_t st) {
  const size_t sm = smem_bytes<BT, NT>(p.d);
  SimtParams q = p;
  q.pre_pop = pre_pop_bytes<BT>(p.d) <= kPrePopMax ? 1 : 0;
  cudaError_t e = cudaFuncSetAttribute(cell_simt_kernel<BT, NT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  const int grid = (p.B + BT - 1) / BT;
  cell_simt_kernel<BT, NT><<<grid, NT, sm, st>>>(q);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_cell_simt(Handle& h, const CellRun& run, cudaStream_t st,
                             int64_t* launches) {
  SimtParams p;
  p.d = h.dims;
  p.B = h.batch;
  p.dil = h.d_dil;
  p.qoff = h.d_qoff;
  p.queue = h.d_queue;
  p.w = h.w;
  p.run = run;
  *launches = 1;
  // Streams per CTA: enough CTAs to cover the SMs, up to 8 streams sharing
  // each weight load.
  const int B = h.batch;
  // small batches: one cluster of 2..16 CTAs per stream (FW_SIMT_CLUSTER overrides)
  if (const int c = cluster_for(h.dims, B)) {
    const cudaError_t e = launch_cell_lat(h, run, c, st);
    if (e != cudaErrorNotSupported) return e;
  }
  // the fp32 configs' shape (3, 5) past the cluster kernel's batches: the warp-MMA kernel
  // (cell_hmma.cu; FW_SIMT_HMMA=0 selects the SIMT kernels below)
  const char* he = getenv("FW_SIMT_HMMA");
  if (hmma_supported(h.dims) && !(he != nullptr && atoi(he) == 0)) {
    const cudaError_t e = launch_cell_hmma(h, run, st);
    if (e != cudaErrorNotSupported) return e;
  }
  // mid/large batches: the weight-staged kernel (FW_SIMT_STAGED=0 selects the __ldg kernel)
  const char* se = getenv("FW_SIMT_STAGED");
  if (staged_supported(h.dims) && !(se != nullptr && atoi(se) == 0)) {
    int bt = 8;
    for (int c : {1, 2, 4, 6, 7, 8})
      if ((B + c - 1) / c <= 148) {
        bt = c;
        break;
      }
    if (const char* e = getenv("FW_SIMT_BT")) bt = atoi(e);
    switch (bt) {
      case 1: return launch_staged<1>(p, st);
      case 2: return launch_staged<2>(p, st);
      case 4: return launch_staged<4>(p, st);
      case 6: return launch_staged<6>(p, st);
      case 7:  // BASELINE config 5 (1,024 streams) at its shape: the specialised kernel
        if (h.dims.R == 64 && h.dims.D == 64 && h.dims.S == 256 && h.dims.H == 256 &&
            h.dims.A == 256 && !getenv("FW_LAT_GENERIC"))
          return launch_staged<7, StShape<64, 64, 256, 256, 256>>(p, st);
        return launch_staged<7>(p, st);
      default: return launch_staged<8>(p, st);
    }
  }
  if (const char* e = getenv("FW_SIMT_BT")) {  // streams per CTA override (measurements)
    switch (atoi(e)) {
      case 8: return launch_bt<8>(p, st);
      case 4: return launch_bt<4>(p, st);
      case 2: return launch_bt<2>(p, st);
      case 1: return launch_bt<1>(p, st);
      default: break;
    }
  }
  if (B >= 148 * 8) return launch_bt<8>(p, st);
  if (B >= 148 * 4) return launch_bt<4>(p, st);
  if (B >= 148 * 2) return launch_bt<2>(p, st);
  return launch_bt<1>(p, st);
}

}  // namespace fw
