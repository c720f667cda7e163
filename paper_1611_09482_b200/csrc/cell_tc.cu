// K2: tcgen05 step kernels for large batches (BASELINE config 4).
//
// One generation step of B streams = four launches on the caller's stream:
//
//  1. chain  (B/128 CTAs, chain_tc.cuh): per 128-stream tile, the dependent chain of all
//     L layers. Per layer: pop of the tile's ring slot (the fp16 x_{t-d} operand, loaded a
//     layer ahead into registers and stored into TMEM), the dilated GEMM
//     [128 x 256] += [128 x 256] . [256 x 256]^T in two N-halves into TMEM, the
//     tanh*sigmoid gate in the TMEM->register epilogue, z -> smem operand (+ a z stash in
//     HBM for the skip GEMM), the residual MMA [128 x 128] += z . W_res^T accumulating
//     straight onto x, which lives in TMEM for the whole step, and the push of x_t.
//  2. skip   GEMM  s = [z_0 .. z_{L-1}] . W_skip_cat^T + sum_l b_skip_l, ReLU
//     (K = L*D = 5120): the skip sum of every layer done as ONE big-K GEMM on
//     (B/128) x (S/128) CTAs instead of S more TMEM columns per layer.
//  3. head1  GEMM  h = ReLU(s . W1^T + b1)
//  4. head2  GEMM  logits = h . W2^T + b2, fused selection (argmax / inverse
//     CDF / Gumbel-max with the counter hash) and teacher/feedback of the next
//     input class.
//
// Numerics: the bf16 weights exactly as fp16 MMA operands, activations rounded to fp16
// operands, fp32 accumulation, fp32 residual stream (TMEM); queue slots hold the fp16
// operand image of x (the precision the MMA consumes). DESIGN.md, "Numerics".
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "internal.h"
#include "tc_ptx.cuh"

namespace fw {

struct TcState {
  int ntile = 0;
  uint8_t* wchain = nullptr;  // per layer: 10 chunks [128][64] in MMA issue order
  uint8_t* wskip = nullptr;   // [S/128][L*D/64] chunks of [128][64] (unfused skip GEMM)
  uint8_t* wskip2 = nullptr;  // [S/SK][L][2][SK][64] (fused skip role of the step kernel)
  uint32_t* zflag = nullptr;  // [5][B/128] fused counters: z stash | s | h | selections | z reads
  int64_t* d_qoff = nullptr;  // [L] byte offset of each layer's ring
  int fused = 0, SK = 256, nchain = 0, nskip = 0;
  int split = 0;              // chain tiles split over 2-CTA clusters (small batches)
  int fold = 0;               // folded chain (chain_fold.cuh): 128-row tiles over 2-CTA clusters
  uint8_t* wfold = nullptr;   // [L][14 chunks][128 n][64 k] SW128 (chain_fold.cuh)
  float* fold_b = nullptr;    // [L][2D] dilated bias + W0_l b_res,l-1
  int fold_has_bias = 0;
  int cg2 = 0;                // 2-SM chain (chain_2sm.cuh): tile pairs as 2-CTA clusters
  uint8_t* w2sm = nullptr;    // [L][2 CTAs][5 stages][64 n][128 k] SW128
  int heads = 0;              // head1 / head2 fused into the skip blocks (needs fused)
  uint8_t* wh1b = nullptr;    // [nsk][S/64][H/nsk rows][128 B] (fused head1)
  uint8_t* wh1 = nullptr;     // [H/128][S/64] chunks of [128][64]
  uint8_t* wh2 = nullptr;     // [H/64] chunks of [A=256][64]
  float* skip_bsum = nullptr;  // [S]
  uint8_t* zimg = nullptr;    // [ntile][L*D/64][16 KB]
  uint8_t* simg = nullptr;    // [ntile][S/64][16 KB]
  uint8_t* himg = nullptr;    // [ntile][H/64][16 KB]
  int32_t* cls = nullptr;     // [B]
  int has_dil_bias = 1, has_res_bias = 1;
  long long* trace = nullptr;  // device buffer [L][kTraceSlots] (debug)
};

void tc_set_trace(Handle& h, long long* trace) {
  if (h.tc) h.tc->trace = trace;
}

int64_t tc_debug_buffer(Handle& h, int which, const void** src) {
  TcState* tc = h.tc;
  if (!tc) return 0;
  const int64_t tile_bytes = 16384;
  if (which == 1) {
    *src = tc->zimg;
    return (int64_t)tc->ntile * h.dims.L * h.dims.D / 64 * tile_bytes;
  }
  if (which == 2) {
    *src = tc->simg;
    return (int64_t)tc->ntile * h.dims.S / 64 * tile_bytes;
  }
  if (which == 3) {
    *src = tc->himg;
    return (int64_t)tc->ntile * h.dims.H / 64 * tile_bytes;
  }
  return 0;
}

namespace {

using namespace ptx;

constexpr uint32_t kChunk = 16384;  // one [128 rows][64] bf16 operand image
constexpr int kChunksPerLayer = 10;  // 8 dil (2 N-halves x 4 K-chunks) + 2 res
constexpr uint32_t kLayerBytes = kChunksPerLayer * kChunk;
constexpr uint32_t kTile = 16384;    // [128 rows][64] bf16 activation chunk
constexpr int kR = 128, kD = 128;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

constexpr int kMaxChainLayers = 128;

// Device-side phase trace (CTA 0 only, clock64 cycles), enabled by fw_debug_trace.
// Per layer kTraceSlots entries; see tools/trace_chain.py for the slot meanings.
constexpr int kTraceSlots = 48;
enum TraceSlot {
  T_MMA_XD = 0, T_MMA_XT, T_MMA_ACC0, T_MMA_ACC1, T_MMA_Z0, T_MMA_Z1, T_MMA_XFULL, T_MMA_WWAIT,
  T_EPI_A, T_EPI_XFULL, T_EPI_XT, T_EPI_ACC0, T_EPI_Z0, T_EPI_ACC1, T_EPI_Z1, T_H0_EARLY,
  T_Q_XD, T_Q_LOAD, T_PROD_A0, T_PROD_A1, T_PROD_B, T_PROD_C, T_G0_LD, T_G0_MATH,
  T_G0_STS, T_PUSHED, T_G1_LD, T_G1_MATH, T_G1_STS, T_SP1, T_SP2, T_SP3
};

// head2 + selection of one step (shared by the head2 GEMM kernel and the fused tail)
struct SelectArgs {
  const float* bias;           // [A]
  float* logits;               // [B][A] for this step or null
  int32_t* out_cls;            // [B] this step's selected classes
  int32_t* cls_next;           // [B] next step's input classes
  const int32_t* next_inputs;  // teacher row for the next step or null
  int A, mode;
  uint32_t seed;
  int64_t stream_offset;
  int64_t t;
  // whole-call view (the persistent step kernel derives the per-step fields above)
  int32_t* out_base;           // [n_steps][B]
  float* logits_base;          // [n_logit_steps][B][A] or null
  int n_logit_steps;
  const int32_t* inputs;       // [n_inputs][B]
  int n_inputs, B;
};

// The per-step fields of step i of a call starting at absolute step t0.
__device__ __forceinline__ SelectArgs sel_step(const SelectArgs& s, int64_t t0, int i) {
  SelectArgs r = s;
  r.t = t0 + i;
  r.out_cls = s.out_base + (size_t)i * s.B;
  r.logits = (s.logits_base && i < s.n_logit_steps) ? s.logits_base + (size_t)i * s.B * s.A : nullptr;
  r.next_inputs = (i + 1 < s.n_inputs) ? s.inputs + (size_t)(i + 1) * s.B : nullptr;
  return r;
}

struct ChainArgs {
  int B, L;
  int n_steps;             // steps of this launch (the fused kernel runs them all)
  int64_t t0;              // absolute step index of the first one
  int32_t dil[kMaxChainLayers];    // dilations
  int32_t slot0[kMaxChainLayers];  // t0 mod dil[l]: the ring slot of layer l at step 0
  const int64_t* qoff;     // [L] byte offset of layer l's ring (slot 0, tile 0)
  int64_t slot_stride;     // bytes between ring slots (all tiles of one slot)
  uint8_t* queue;
  const uint8_t* w;
  const float* embed;  // [A][128]
  const float* dil_b;  // [L][256]
  const float* res_b;  // [L][128]
  const int32_t* cls;  // [B]
  uint8_t* zimg;
  int has_dil_bias, has_res_bias;
  long long* trace;  // [L][kTraceSlots] or null
  // fused skip role (zflag != null): blocks >= nchain accumulate the skip sum
  int nchain;
  uint32_t* zflag;         // [B/128] per tile pair: chain tiles x layers stashed so far
  int zring;               // layers in the z stash ring (slot = global layer index % zring)
  uint32_t* zfree;         // [B/128] per tile pair: z tiles read by the tail blocks, or null
  int ztail;               // tail blocks per pair (reads per z tile)
  uint32_t* cls_ready;     // [B/128] per tile pair: steps whose selection is written
  const uint8_t* wskip2;   // [S/SK][L][2 K-chunks][SK rows][128 B]
  const float* skip_bsum;  // [S]
  uint8_t* simg;           // head1's A images [B/128][S/64][16 KB]
  int S, SK;
  // fused heads (heads != 0): head1 by the pair's skip blocks (H / nsk columns each), head2
  // + selection by its first skip block; sflag / hflag count the blocks done with simg / himg
  int heads, H;
  int pair_mode;         // tail blocks in 2-CTA clusters exchanging through DSMEM
  int split;             // chain tiles over 2-CTA clusters, one dilated N-half per CTA
  int fold;              // folded chain: 128-row tiles over 2-CTA clusters (chain_fold.cuh)
  int zpub;              // z stash publications per tile pair per layer (2, or 4 when split)
  uint32_t* sflag;       // [B/128] (cumulative over the launch's steps)
  uint32_t* hflag;       // [B/128]
  const uint8_t* wh1b;   // [nsk][S/64][H/nsk rows][128 B]
  const uint8_t* wh2;    // [H/64][A rows][128 B]
  const float* h1_b;     // [H]
  uint8_t* himg;         // head2's A images [B/128][H/64][16 KB]
  SelectArgs sel;
};

__device__ __forceinline__ void trace_at(const ChainArgs& a, int l, int slot, long long v) {
  if (a.trace != nullptr && blockIdx.x == 0) a.trace[l * kTraceSlots + slot] = v;
}
// Step timeline in global time (ns): row L of the trace, written by chain block 0 and the
// first skip block (tools/trace_chain.py). Slots: 0 chain start, 1 chain last layer done,
// 2 skip: last z tile seen, 3 s published, 4 head1 done, 5 head2 accumulator, 6 selection done
__device__ __forceinline__ void trace_g(const ChainArgs& a, bool who, int slot) {
  if (a.trace != nullptr && who) a.trace[a.L * kTraceSlots + slot] = globaltimer_ns();
}
// Byte offset (tile 0) of the ring slot layer l reads and writes at step i of the launch.
__device__ __forceinline__ int64_t qbase_of(const ChainArgs& a, int i, int l) {
  const int d = a.dil[l];
  int s = a.slot0[l] + i;  // 32-bit: i < n_steps
  s = (d & (d - 1)) == 0 ? (s & (d - 1)) : s % d;
  return a.qoff[l] + (int64_t)s * a.slot_stride;
}

// Gumbel noise -log(-log u) of class cls; v + gumbel_noise(...) == v - log(-log u) exactly.
__device__ __forceinline__ float gumbel_noise(uint32_t prefix, int cls) {
  const float u = noise_uniform(prefix, (uint32_t)cls);
  return -__logf(-__logf(u));
}

// ReLU(v + bias[0..32)) -> 16 packed fp16 pairs (bias null: none). The bias (identical for
// every thread; global or shared memory, hence generic loads) comes in as 8 independent
// 16-byte loads: scalar loads next to 64 live accumulator values were serialised by the
// register budget (~2 us
// per 128-column epilogue).
__device__ __forceinline__ void relu_pack32(const float (&v)[32], const float* bias, uint32_t (&w)[16]) {
  const float4* b4 = reinterpret_cast<const float4*>(bias);
  float4 b[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) b[q] = bias ? b4[q] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    w[2 * q] = pack_h2(fmaxf(v[4 * q] + b[q].x, 0.f), fmaxf(v[4 * q + 1] + b[q].y, 0.f));
    w[2 * q + 1] = pack_h2(fmaxf(v[4 * q + 2] + b[q].z, 0.f), fmaxf(v[4 * q + 3] + b[q].w, 0.f));
  }
}

// ReLU(acc + bias) of TMEM columns [c0, c0 + ncols) of row r -> fp16 SW128 image chunks;
// column c0 + j is global column n0 + j, in chunk (n0 + j) / 64 of the tile's images at img.
__device__ __forceinline__ void epi_relu_image(uint32_t trow, int r, int c0, int ncols, int n0,
                                               const float* bias, uint8_t* img) {
#pragma unroll 1
  for (int cc = 0; cc < ncols / 32; ++cc) {
    float v[32];
    uint32_t w[16];
    tmem_ld32(trow + c0 + 32 * cc, v);
    const int n = n0 + 32 * cc;
    relu_pack32(v, bias + n, w);
    uint8_t* dst = img + (size_t)(n / 64) * kTile;
    const int p0 = (n & 63) / 8;
#pragma unroll
    for (int p = 0; p < 4; ++p)
      *reinterpret_cast<uint4*>(dst + swz(r, p0 + p)) =
          make_uint4(w[4 * p], w[4 * p + 1], w[4 * p + 2], w[4 * p + 3]);
  }
}

// Same, into a shared-memory copy of the images (chunk j of the thread's columns at
// sdst + j * 16 KB), bank-conflict free through the swizzle; the caller bulk-stores it.
__device__ __forceinline__ void epi_relu_image_smem(uint32_t trow, int r, int c0, int ncols,
                                                    int n0, const float* bias, uint32_t sdst) {
#pragma unroll 1
  for (int cc = 0; cc < ncols / 32; ++cc) {
    float v[32];
    uint32_t w[16];
    tmem_ld32(trow + c0 + 32 * cc, v);
    relu_pack32(v, bias + n0 + 32 * cc, w);
    const uint32_t dst = sdst + (uint32_t)(cc >> 1) * kTile;
    const int p0 = (cc & 1) * 4;
#pragma unroll
    for (int p = 0; p < 4; ++p)
      st_shared_v4(dst + swz(r, p0 + p), w[4 * p], w[4 * p + 1], w[4 * p + 2], w[4 * p + 3]);
  }
}

// head2 epilogue: the logits of row r (TMEM columns [0, A)) + bias, this thread's half h of
// the classes, then the selection rule; the 256 epilogue threads exchange per-row partials
// through xch ([4][2][128] words, bar.sync 1, 256).
// noise_col >= 0: the Gumbel noise of the row's classes was precomputed into TMEM columns
// noise_col + class (fused tail); otherwise it is hashed here. add_has_bias: those columns
// hold bias + noise (Gumbel) or the bias alone (other modes), so no bias loads are needed.
__device__ __forceinline__ void epi_select(uint32_t trow, int r, int h, int stream,
                                        const SelectArgs& g, float* xch, int noise_col = -1,
                                        bool add_has_bias = false, const ChainArgs* tra = nullptr,
                                        bool folded = false) {
  const int HALF = g.A / 2, A = g.A, mode = g.mode;
  const float* bias = g.bias;
  const uint32_t prefix = noise_prefix(g.seed, (uint32_t)(g.stream_offset + stream), (uint32_t)g.t);
  const int cbase = h * HALF;
  float* lrow = g.logits ? g.logits + (size_t)stream * A : nullptr;
  const bool tm_add = noise_col >= 0 && add_has_bias;
  const bool pre_noise = noise_col >= 0 && mode == FW_SAMPLE_GUMBEL;
  float best = -INFINITY, mx = -INFINITY;
  int bi = A;
  if (folded) {
    // head2 accumulated onto (bias + noise) in TMEM columns noise_col..: the scores are
    // there already (argmax / Gumbel steps without logits output)
#pragma unroll 1
    for (int cc = 0; cc < HALF / 64; ++cc) {
      float x[64];
      tmem_ld64(trow + noise_col + cbase + 64 * cc, x);
      float bv[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      int bj[4] = {0, 1, 2, 3};
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        if (x[i] > bv[i & 3]) {
          bv[i & 3] = x[i];
          bj[i & 3] = i;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int col = cbase + 64 * cc + bj[u];
        if (bv[u] > best || (bv[u] == best && col < bi)) {
          best = bv[u];
          bi = col;
        }
      }
    }
  } else if (tm_add) {
    // x = acc + (bias + noise): the score (Gumbel) or the logit (other modes), one pass with
    // no memory traffic. Four independent running maxima (a single compare-select chain is
    // latency-bound), merged lowest index first on ties; mx (inverse CDF) is the max logit.
#pragma unroll 1
    for (int cc = 0; cc < HALF / 32; ++cc) {
      float x[64];
      tmem_ld32x2(trow + cbase + 32 * cc, trow + noise_col + cbase + 32 * cc, x);
      float bv[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      int bj[4] = {0, 1, 2, 3};
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float sc = x[i] + x[32 + i];
        if (sc > bv[i & 3]) {
          bv[i & 3] = sc;
          bj[i & 3] = i;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        mx = fmaxf(mx, bv[u]);
        const int col = cbase + 32 * cc + bj[u];
        if (bv[u] > best || (bv[u] == best && col < bi)) {
          best = bv[u];
          bi = col;
        }
      }
      if (tra && cc < 3) {
        asm volatile("" ::"f"(best) : "memory");
        trace_g(*tra, true, 21 + cc);
      }
    }
    if (lrow) {  // logits out (acc + bias), a second pass
#pragma unroll 1
      for (int cc = 0; cc < HALF / 32; ++cc) {
        float v[32];
        tmem_ld32(trow + cbase + 32 * cc, v);
        const float4* b4 = reinterpret_cast<const float4*>(bias + cbase + 32 * cc);
        float4* d4 = reinterpret_cast<float4*>(lrow + cbase + 32 * cc);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 b = __ldg(b4 + q);
          d4[q] = make_float4(v[4 * q] + b.x, v[4 * q + 1] + b.y, v[4 * q + 2] + b.z, v[4 * q + 3] + b.w);
        }
      }
    }
  } else {
#pragma unroll 1
    for (int cc = 0; cc < HALF / 32; ++cc) {
      float vg[64];  // logits | noise
      float* v = vg;
      const float* gn = vg + 32;
      if (pre_noise)
        tmem_ld32x2(trow + cbase + 32 * cc, trow + noise_col + cbase + 32 * cc, vg);
      else
        tmem_ld32(trow + cbase + 32 * cc, *reinterpret_cast<float(*)[32]>(vg));
      const float4* b4 = reinterpret_cast<const float4*>(bias + cbase + 32 * cc);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 b = __ldg(b4 + q);
        v[4 * q] += b.x;
        v[4 * q + 1] += b.y;
        v[4 * q + 2] += b.z;
        v[4 * q + 3] += b.w;
      }
      // (separate loops: folded into one, the compiler evaluated the noise hash for every
      // element even when the noise came precomputed)
      if (pre_noise) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float sc = v[i] + gn[i];
          if (sc > best) {
            best = sc;
            bi = cbase + 32 * cc + i;
          }
        }
      } else if (mode == FW_SAMPLE_GUMBEL) {
#pragma unroll 4
        for (int i = 0; i < 32; ++i) {
          const int col = cbase + 32 * cc + i;
          const float sc = v[i] + gumbel_noise(prefix, col);
          if (sc > best) {
            best = sc;
            bi = col;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          mx = fmaxf(mx, v[i]);
          if (v[i] > best) {
            best = v[i];
            bi = cbase + 32 * cc + i;
          }
        }
      }
      if (lrow) {
        float4* d4 = reinterpret_cast<float4*>(lrow + cbase + 32 * cc);
#pragma unroll
        for (int i = 0; i < 8; ++i) d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
    }
  }
  if (tra) trace_g(*tra, true, 26);
  float* xb = xch;                              // best score  [2][128]
  int* xi = reinterpret_cast<int*>(xch + 256);  // best index [2][128]
  float* xm = xch + 512;                        // max [2][128]
  float* xs = xch + 768;                        // sum [2][128]
  xb[h * 128 + r] = best;
  xi[h * 128 + r] = bi;
  xm[h * 128 + r] = mx;
  named_bar_sync(1, 256);
  int choice;
  if (g.mode != FW_SAMPLE_INVCDF) {
    const float ob = xb[(h ^ 1) * 128 + r];
    const int oi = xi[(h ^ 1) * 128 + r];
    choice = (ob > best || (ob == best && oi < bi)) ? oi : bi;
  } else {
    const float m = fmaxf(mx, xm[(h ^ 1) * 128 + r]);
    float part = 0.f;
    for (int cc = 0; cc < HALF / 32; ++cc) {
      float v[32];
      tmem_ld32(trow + cbase + 32 * cc, v);
      tmem_wait_ld();
      for (int i = 0; i < 32; ++i) part += __expf(v[i] + bias[cbase + 32 * cc + i] - m);
    }
    xs[h * 128 + r] = part;
    named_bar_sync(1, 256);
    const float s0 = xs[r], total = s0 + xs[128 + r];
    const float thr = noise_uniform(prefix, kUniformClass) * total;
    float run = (h == 0) ? 0.f : s0;
    int found = g.A;
    // warp-uniform trip count: tcgen05.ld is .sync.aligned across the warp
    for (int cc = 0; cc < HALF / 32; ++cc) {
      float v[32];
      tmem_ld32(trow + cbase + 32 * cc, v);
      tmem_wait_ld();
      for (int i = 0; i < 32; ++i) {
        run += __expf(v[i] + bias[cbase + 32 * cc + i] - m);
        if (found == g.A && run > thr) found = cbase + 32 * cc + i;
      }
    }
    xi[h * 128 + r] = found;
    named_bar_sync(1, 256);
    const int f0 = xi[r], f1 = xi[128 + r];
    choice = f0 < g.A ? f0 : (f1 < g.A ? f1 : g.A - 1);
  }
  if (tra) trace_g(*tra, true, 27);
  if (h == 0) {
    g.out_cls[stream] = choice;
    g.cls_next[stream] = g.next_inputs ? g.next_inputs[stream] : choice;
  }
}

#include "chain_tc.cuh"

// ---- generic [128 x BN] tile GEMM over pre-swizzled A/B images ----------------------
struct GemmArgs {
  const uint8_t* a;  // [mtiles][kch][16 KB]: SW128 images, or a_plain: [8 K-pieces][128][16 B]
  const uint8_t* b;  // [ntiles][kch][BN * 128 B]
  int kch;
  int a_plain;
  const float* bias;  // [N]
  uint8_t* out_img;   // epi 0: [mtiles][N/64][16 KB]
  int n_total;
  SelectArgs sel;  // epi 1 (head2 + selection)
};

// Each pipeline stage holds kGemmGroup consecutive 64-K chunks of A and of B, each side
// fetched by ONE bulk copy (consecutive chunks are contiguous in the images) from its own
// producer warp: copy cost is per operation and a thread's copies run one at a time
// (tools/ring_bw.cu), so fewer, larger copies from two warps keep the tensor pipe fed.
constexpr int kGemmGroup = 2;
constexpr int kGemmThreads = 352;  // warp 0: A producer, 1: MMA, 2..9: epilogue, 10: B producer
template <int BN>
constexpr int gemm_stages() {
  return BN == 256 ? 2 : 3;
}
template <int BN>
constexpr uint32_t gemm_stage_bytes() {
  return kGemmGroup * (kTile + BN * 128);
}
template <int BN>
constexpr size_t gemm_smem() {
  return 1024 + gemm_stages<BN>() * gemm_stage_bytes<BN>() + 256 + 4 * 128 * 4 * 2;
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_kernel(GemmArgs g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr int S = gemm_stages<BN>();
  constexpr uint32_t SB = gemm_stage_bytes<BN>();
  constexpr uint32_t A_BYTES = kGemmGroup * kTile, B_BYTES = kGemmGroup * BN * 128;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * SB);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* acc_full = bars + 2 * S;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * S + 1);
  float* xch = reinterpret_cast<float*>(smem + S * SB + 256);  // [4][128][2] exchange
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x, nt = blockIdx.y;
  const int groups = g.kch / kGemmGroup;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 2);  // one expect_tx arrival per producer warp
      mbar_init(&empty[i], 1);
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0 || warp == 10) {
    if (lane == 0) {
      const bool is_a = warp == 0;
      const uint8_t* base = is_a ? g.a + (size_t)mt * g.kch * kTile
                                 : g.b + (size_t)nt * g.kch * (BN * 128);
      const uint32_t bytes = is_a ? A_BYTES : B_BYTES;
      for (int gi = 0; gi < groups; ++gi) {
        const int stage = gi % S;
        mbar_wait(&empty[stage], ((uint32_t)(gi / S) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[stage], bytes);
        bulk_g2s(smem + stage * SB + (is_a ? 0 : A_BYTES), base + (size_t)gi * bytes, bytes,
                 &full[stage]);
      }
    }
  } else if (warp == 1) {  // MMA issuer: the converged warp, MMAs under elect.sync
    const uint32_t id = idesc_f16(128, BN);
    const uint32_t s0 = smem_u32(smem);
    for (int gi = 0; gi < groups; ++gi) {
      const int stage = gi % S;
      mbar_wait(&full[stage], (uint32_t)(gi / S) & 1);
      tc_fence_after();
      const uint32_t sa = s0 + stage * SB, sb = sa + A_BYTES;
      if (elect_one()) {
#pragma unroll
        for (int c = 0; c < kGemmGroup; ++c)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_bf16(tmem,
                     g.a_plain ? sdesc_plain(sa + c * kTile + kk * 4096, 2048, 128)
                               : sdesc_sw128(sa + c * kTile + kk * 32),
                     sdesc_sw128(sb + c * (BN * 128) + kk * 32), id, (gi | c | kk) != 0);
        mma_commit(&empty[stage]);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(acc_full);
    __syncwarp();
  } else {
    const int sub = warp & 3, h = (warp - 2) >> 2;
    const int r = sub * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(sub * 32) << 16);
    mbar_wait(acc_full, 0);
    tc_fence_after();
    constexpr int HALF = BN / 2;  // columns per thread
    if (EPI == 0)
      epi_relu_image(trow, r, h * HALF, HALF, nt * BN + h * HALF, g.bias,
                     g.out_img + (size_t)mt * (g.n_total / 64) * kTile);
    else
      epi_select(trow, r, h, mt * 128 + r, g.sel, xch);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, BN);
}

// ---- host-side packing ---------------------------------------------------------------
// Operand images are fp16. The weights are the model's bf16 values: every bf16 value with
// |w| >= 2^-17 is exactly representable in fp16 (8 significand bits fit in 11), smaller
// ones round with an absolute error below 2^-25 -- the weights the tensor cores see are the
// bf16 weights. Activations are rounded to fp16 instead of bf16 at the same MMA rate: with
// bf16 activation operands the config-4 logits drift to ~2e-2 of the fp64 oracle, with
// fp16 to ~3e-3 ("Numerics of the tcgen05 path").
uint16_t f16_bits(float f) {
  __half b = __float2half_rn(__bfloat162float(__float2bfloat16_rn(f)));
  uint16_t u;
  std::memcpy(&u, &b, 2);
  return u;
}

uint16_t f16_bits_exact(double v) {
  __half b = __float2half_rn((float)v);
  uint16_t u;
  std::memcpy(&u, &b, 2);
  return u;
}

// Rows [0, nrows) of (row, k) -> fp16 bits, K slice [k0, k0+64), as a swizzled image.
template <typename F>
void pack_image_bits(uint8_t* dst, int nrows, int k0, F bits) {
  for (int r = 0; r < nrows; ++r)
    for (int k = 0; k < 64; ++k) {
      const size_t off = (size_t)(r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 3) ^ (r & 7))) << 4) + (k & 7) * 2;
      const uint16_t b = bits(r, k0 + k);
      std::memcpy(dst + off, &b, 2);
    }
}

// Rows [0, nrows) of the (row, k) -> value function, K slice [k0, k0+64), as a swizzled image.
template <typename F>
void pack_image(uint8_t* dst, int nrows, int k0, F val) {
  for (int r = 0; r < nrows; ++r)
    for (int k = 0; k < 64; ++k) {
      const size_t off = (size_t)(r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 3) ^ (r & 7))) << 4) + (k & 7) * 2;
      const uint16_t b = f16_bits(val(r, k0 + k));
      std::memcpy(dst + off, &b, 2);
    }
}

template <typename T>
int dev_alloc(T** p, size_t bytes) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
  if (e != cudaSuccess) {
    set_error(std::string("tcgen05 path allocation: ") + cudaGetErrorString(e));
    return FW_ERR_CUDA;
  }
  return FW_OK;
}

int upload_bytes(uint8_t** dst, const std::vector<uint8_t>& src) {
  int rc = dev_alloc(dst, src.size());
  if (rc) return rc;
  cudaError_t e = cudaMemcpy(*dst, src.data(), src.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    set_error(std::string("tcgen05 weight upload: ") + cudaGetErrorString(e));
    return FW_ERR_CUDA;
  }
  return FW_OK;
}

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}


}  // namespace

bool tc_supported(const CellDims& d, int batch, std::string* why) {
  auto no = [&](const char* m) {
    if (why) *why = m;
    return false;
  };
  if (d.dtype != FW_DTYPE_BF16) return no("needs bf16 weights");
  if (d.R != kR || d.D != kD) return no("needs residual = dilation = 128 channels");
  if (d.S % 128 || d.H % 128 || d.S > 2048 || d.H > 2048) return no("needs skip/head multiples of 128");
  if (d.A != 256) return no("needs 256 classes");
  if (d.L > kMaxChainLayers) return no("needs at most 128 layers");
  // the chain's pops are staged two layers ahead of their use; with fewer than 3 layers that
  // is the same layer of the next step, read before this step's push of it
  if (d.L < 3) return no("needs at least 3 layers");
  if (batch % 128) return no("needs a batch that is a multiple of 128 streams");
  return true;
}

int tc_create(Handle& h, const fw_cell_desc* desc) {
  const CellDims& d = h.dims;
  const int L = d.L, S = d.S, H = d.H, A = d.A;
  TcState* tc = new TcState();
  h.tc = tc;
  tc->ntile = h.batch / 128;
  auto any_nonzero = [](const float* p, size_t n) {
    for (size_t i = 0; i < n; ++i)
      if (p[i] != 0.f) return 1;
    return 0;
  };
  tc->has_dil_bias = any_nonzero(desc->dil_b, (size_t)L * 2 * kD);
  tc->has_res_bias = any_nonzero(desc->res_b, (size_t)L * kR);
  // chain weights, per layer in MMA issue order (10 chunks of [128 n][64 k]):
  //   dil N-half hh in {0,1}, K-chunks 2,3 (x_{t-d}); then per half K-chunks 0,1 (x_t);
  //   res K-chunks 0,1. N-half hh holds tanh rows 64hh..64hh+63 then sigmoid rows
  //   D+64hh..D+64hh+63, so one half's accumulator carries both gate inputs.
  {
    std::vector<uint8_t> img((size_t)L * kLayerBytes, 0);
    for (int l = 0; l < L; ++l) {
      uint8_t* base = img.data() + (size_t)l * kLayerBytes;
      const float* w0 = desc->dil_w + ((size_t)l * 2 + 0) * 2 * kD * kR;
      const float* w1 = desc->dil_w + ((size_t)l * 2 + 1) * 2 * kD * kR;
      const int order[8][2] = {{0, 2}, {0, 3}, {1, 2}, {1, 3}, {0, 0}, {0, 1}, {1, 0}, {1, 1}};
      for (int c = 0; c < 8; ++c) {
        const int hh = order[c][0], kc = order[c][1];
        pack_image(base + (size_t)c * kChunk, 128, kc * 64, [&](int n, int k) {
          const int row = n < 64 ? 64 * hh + n : kD + 64 * hh + (n - 64);
          return k < kR ? w0[(size_t)row * kR + k] : w1[(size_t)row * kR + (k - kR)];
        });
      }
      const float* wr = desc->res_w + (size_t)l * kR * kD;
      for (int c = 0; c < 2; ++c)
        pack_image(base + (size_t)(8 + c) * kChunk, 128, c * 64,
                   [&](int n, int k) { return wr[(size_t)n * kD + k]; });
    }
    if (int rc = upload_bytes(&tc->wchain, img)) return rc;
  }
  const int kskip = L * kD / 64;
  {
    std::vector<uint8_t> img((size_t)(S / 128) * kskip * kTile);
    for (int nb = 0; nb < S / 128; ++nb)
      for (int kc = 0; kc < kskip; ++kc)
        pack_image(img.data() + ((size_t)nb * kskip + kc) * kTile, 128, kc * 64, [&](int n, int k) {
          const int l = k / kD, j = k % kD;
          return desc->skip_w[((size_t)l * S + nb * 128 + n) * kD + j];
        });
    if (int rc = upload_bytes(&tc->wskip, img)) return rc;
  }
  // fused skip role: one block per (128-row tile pair, SK-column block of S) next to the
  // B/64 chain blocks, all co-resident (cooperative launch) when the SMs suffice
  {
    tc->SK = (S % 256 == 0) ? 256 : 128;
    tc->nchain = h.batch / kChainRows;
    tc->nskip = (h.batch / 128) * (S / tc->SK);
    int sms = 0, coop = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h.device);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, h.device);
    tc->fused = coop && (tc->nchain + tc->nskip <= sms);
    const int SK = tc->SK;
    std::vector<uint8_t> img((size_t)(S / SK) * L * 2 * SK * 128);
    for (int e = 0; e < S / SK; ++e)
      for (int l = 0; l < L; ++l)
        for (int c = 0; c < 2; ++c)
          pack_image(img.data() + (((size_t)e * L + l) * 2 + c) * SK * 128, SK, c * 64,
                     [&](int n, int k) { return desc->skip_w[((size_t)l * S + e * SK + n) * kD + k]; });
    if (int rc = upload_bytes(&tc->wskip2, img)) return rc;
    if (int rc = dev_alloc(&tc->zflag, sizeof(uint32_t) * 5 * (h.batch / 128))) return rc;
    // ring offsets: layer l's d_l slots follow the earlier layers', each slot holds every tile
    std::vector<int64_t> qoff(L);
    for (int l = 0, acc = 0; l < L; ++l) {
      qoff[l] = (int64_t)acc * (h.batch / kChainRows) * kSlotBytes;
      acc += h.dil[l];
    }
    if (int rc = dev_alloc(&tc->d_qoff, sizeof(int64_t) * L)) return rc;
    cudaMemcpy(tc->d_qoff, qoff.data(), sizeof(int64_t) * L, cudaMemcpyHostToDevice);
    // fused heads: head1's N split over the pair's nsk skip blocks, 128 or 256 columns each
    const int nsk = S / SK, n1 = H / nsk;
    // the fused step kernel runs all steps of a call in one launch, so it needs the heads
    // too; other shapes keep per-step launches with the skip / head GEMM kernels
    tc->heads = tc->fused && (H % nsk == 0) && (n1 == 128 || n1 == 256);
    tc->fused = tc->heads;
    // split chain: each 64-stream tile over a 2-CTA cluster, one dilated N-half per CTA
    // (needs the pair tail's cluster launch and room for twice the chain CTAs)
    const char* se = getenv("FW_CHAIN_SPLIT");
    tc->split = tc->heads && S == 512 && H == 512 && A == 256 && 2 * tc->nchain + tc->nskip <= sms &&
                !(se && atoi(se) == 0) && !getenv("FW_NO_CLUSTER");
    // folded chain (FW_CHAIN_FOLD=1; measured slower): one 128-row tile
    // per 2-CTA cluster -- the same B/64 chain CTAs as the unsplit kernel, every MMA at M = 128
    const char* fe = getenv("FW_CHAIN_FOLD");
    tc->fold = tc->heads && S == 512 && H == 512 && A == 256 && tc->nchain + tc->nskip <= sms &&
               fe && atoi(fe) != 0 && !getenv("FW_NO_CLUSTER");
    if (tc->fold) tc->split = 0;
    // 2-SM chain (FW_CHAIN_2SM=1): the unsplit grid, tile pairs as clusters issuing
    // cta_group::2 MMAs (chain_2sm.cuh)
    const char* ce = getenv("FW_CHAIN_2SM");
    tc->cg2 = !tc->fold && tc->heads && S == 512 && H == 512 && A == 256 &&
              tc->nchain + tc->nskip <= sms && ce && atoi(ce) != 0 && !getenv("FW_NO_CLUSTER");
    if (tc->cg2 && atoi(ce) == 2) tc->cg2 = 2;  // the folded 2-SM chain
    if (tc->cg2) tc->split = 0;
    if (tc->split) tc->nchain *= 2;
    if (tc->heads) {
      std::vector<uint8_t> w1((size_t)nsk * (S / 64) * n1 * 128);
      for (int e = 0; e < nsk; ++e)
        for (int c = 0; c < S / 64; ++c)
          pack_image(w1.data() + ((size_t)e * (S / 64) + c) * n1 * 128, n1, c * 64,
                     [&](int n, int k) { return desc->head1_w[(size_t)(e * n1 + n) * S + k]; });
      if (int rc = upload_bytes(&tc->wh1b, w1)) return rc;
    }
  }
  if (tc->cg2) {
    // per layer, per CTA r of a pair, 16 KB halves [64 n][128 k] (2 SW128 K-chunks each) in
    // MMA order: x_{t-d} taps of N-halves 0, 1, x_t taps of N-halves 0, 1, (folded: WF_l =
    // W0_l Wr_{l-1} of N-halves 0, 1,) residual. Dilated N-half h, CTA r: rows 0..31 tanh of
    // channels 64h + 32r + j, rows 32..63 their sigmoid; residual, CTA r: output channels
    // 64r .. 64r + 63
    const HostCell& c = h.host;
    const bool f2 = tc->cg2 == 2;
    const int nh = f2 ? c2::kLayerStagesF : c2::kLayerStages;
    const size_t lbytes = (size_t)2 * nh * c2::kHalfW;
    std::vector<uint8_t> img((size_t)L * lbytes, 0);
    std::vector<float> fb((size_t)L * 2 * kD);
    std::vector<double> wf((size_t)2 * kD * kD);
    for (int l = 0; l < L; ++l) {
      const float* w0 = c.dil_w.data() + ((size_t)l * 2 + 0) * 2 * kD * kR;
      const float* w1 = c.dil_w.data() + ((size_t)l * 2 + 1) * 2 * kD * kR;
      const float* wr = c.res_w.data() + (size_t)l * kR * kD;
      const float* wrp = l > 0 ? c.res_w.data() + (size_t)(l - 1) * kR * kD : nullptr;
      for (int row = 0; row < 2 * kD; ++row) {
        double b = c.dil_b[(size_t)l * 2 * kD + row];
        if (l > 0) {
          for (int j = 0; j < kR; ++j) b += (double)w0[(size_t)row * kR + j] * c.res_b[(size_t)(l - 1) * kR + j];
          if (f2)
            for (int k = 0; k < kD; ++k) {
              double acc = 0;
              for (int j = 0; j < kR; ++j) acc += (double)w0[(size_t)row * kR + j] * wrp[(size_t)j * kD + k];
              wf[(size_t)row * kD + k] = acc;
            }
        }
        fb[(size_t)l * 2 * kD + row] = (float)b;
      }
      for (int r = 0; r < 2; ++r) {
        uint8_t* base = img.data() + (size_t)l * lbytes + (size_t)r * nh * c2::kHalfW;
        auto row_of = [&](int hh, int n) { return n < 32 ? 64 * hh + 32 * r + n : kD + 64 * hh + 32 * r + (n - 32); };
        for (int s = 0; s < 4; ++s) {
          const int hh = s & 1;
          const float* wt = s < 2 ? w1 : w0;
          for (int kc = 0; kc < 2; ++kc)
            pack_image(base + (size_t)s * c2::kHalfW + (size_t)kc * 8192, 64, kc * 64,
                       [&](int n, int k) { return wt[(size_t)row_of(hh, n) * kR + k]; });
        }
        int sres = 4;
        if (f2) {
          for (int hh = 0; hh < 2 && l > 0; ++hh)
            for (int kc = 0; kc < 2; ++kc)
              pack_image_bits(base + (size_t)(4 + hh) * c2::kHalfW + (size_t)kc * 8192, 64, kc * 64,
                              [&](int n, int k) { return f16_bits_exact(wf[(size_t)row_of(hh, n) * kD + k]); });
          sres = 6;
        }
        // residual of this layer (unfolded) / of layer l - 1 (folded: x_l = x_{l-1} + Wr_{l-1} z)
        const float* wres = f2 ? wrp : wr;
        if (wres)
          for (int kc = 0; kc < 2; ++kc)
            pack_image(base + (size_t)sres * c2::kHalfW + (size_t)kc * 8192, 64, kc * 64,
                       [&](int n, int k) { return wres[(size_t)(64 * r + n) * kD + k]; });
      }
    }
    if (int rc = upload_bytes(&tc->w2sm, img)) return rc;
    if (f2) {
      for (float v : fb) tc->fold_has_bias |= (v != 0.f);
      if (int rc = dev_alloc(&tc->fold_b, sizeof(float) * fb.size())) return rc;
      cudaMemcpy(tc->fold_b, fb.data(), sizeof(float) * fb.size(), cudaMemcpyHostToDevice);
    }
  }
  if (tc->fold) {
    // per layer 14 chunks [128 n][64 k]: W1 / W0 / WF N-halves (tanh rows 64hh.. then sigmoid
    // rows D + 64hh..) x 2 K-chunks, then Wr_{l-1} x 2 K-chunks; WF_l = W0_l Wr_{l-1} and the
    // folded bias b_l + W0_l br_{l-1} in fp64 from the bf16-rounded weights
    const HostCell& c = h.host;
    const int D2 = 2 * kD;
    std::vector<uint8_t> img((size_t)L * fold::kLayerBytes, 0);
    std::vector<float> fb((size_t)L * D2);
    std::vector<double> wf((size_t)D2 * kD);
    for (int l = 0; l < L; ++l) {
      const float* w0 = c.dil_w.data() + ((size_t)l * 2 + 0) * D2 * kR;
      const float* w1 = c.dil_w.data() + ((size_t)l * 2 + 1) * D2 * kR;
      const float* wr = l > 0 ? c.res_w.data() + (size_t)(l - 1) * kR * kD : nullptr;
      const float* br = l > 0 ? c.res_b.data() + (size_t)(l - 1) * kR : nullptr;
      for (int row = 0; row < D2; ++row) {
        double b = c.dil_b[(size_t)l * D2 + row];
        if (l > 0) {
          for (int j = 0; j < kR; ++j) b += (double)w0[(size_t)row * kR + j] * br[j];
          for (int k = 0; k < kD; ++k) {
            double acc = 0;
            for (int j = 0; j < kR; ++j) acc += (double)w0[(size_t)row * kR + j] * wr[(size_t)j * kD + k];
            wf[(size_t)row * kD + k] = acc;
          }
        }
        fb[(size_t)l * D2 + row] = (float)b;
      }
      uint8_t* base = img.data() + (size_t)l * fold::kLayerBytes;
      auto row_of = [&](int hh, int n) { return n < 64 ? 64 * hh + n : kD + 64 * hh + (n - 64); };
      for (int hh = 0; hh < 2; ++hh)
        for (int kc = 0; kc < 2; ++kc) {
          pack_image(base + (size_t)(0 + 2 * hh + kc) * kChunk, 128, kc * 64,
                     [&](int n, int k) { return w1[(size_t)row_of(hh, n) * kR + k]; });
          pack_image(base + (size_t)(4 + 2 * hh + kc) * kChunk, 128, kc * 64,
                     [&](int n, int k) { return w0[(size_t)row_of(hh, n) * kR + k]; });
          if (l > 0)
            pack_image_bits(base + (size_t)(8 + 2 * hh + kc) * kChunk, 128, kc * 64, [&](int n, int k) {
              return f16_bits_exact(wf[(size_t)row_of(hh, n) * kD + k]);
            });
        }
      if (l > 0)
        for (int kc = 0; kc < 2; ++kc)
          pack_image(base + (size_t)(12 + kc) * kChunk, 128, kc * 64,
                     [&](int n, int k) { return wr[(size_t)n * kD + k]; });
    }
    if (int rc = upload_bytes(&tc->wfold, img)) return rc;
    for (float v : fb) tc->fold_has_bias |= (v != 0.f);
    if (int rc = dev_alloc(&tc->fold_b, sizeof(float) * fb.size())) return rc;
    cudaMemcpy(tc->fold_b, fb.data(), sizeof(float) * fb.size(), cudaMemcpyHostToDevice);
  }
  {
    std::vector<uint8_t> img((size_t)(H / 128) * (S / 64) * kTile);
    for (int nb = 0; nb < H / 128; ++nb)
      for (int kc = 0; kc < S / 64; ++kc)
        pack_image(img.data() + ((size_t)nb * (S / 64) + kc) * kTile, 128, kc * 64,
                   [&](int n, int k) { return desc->head1_w[(size_t)(nb * 128 + n) * S + k]; });
    if (int rc = upload_bytes(&tc->wh1, img)) return rc;
  }
  {
    std::vector<uint8_t> img((size_t)(H / 64) * A * 128);
    for (int kc = 0; kc < H / 64; ++kc)
      pack_image(img.data() + (size_t)kc * A * 128, A, kc * 64,
                 [&](int n, int k) { return desc->head2_w[(size_t)n * H + k]; });
    if (int rc = upload_bytes(&tc->wh2, img)) return rc;
  }
  {
    std::vector<float> bsum(S, 0.f);
    for (int l = 0; l < L; ++l)
      for (int n = 0; n < S; ++n) bsum[n] += __bfloat162float(__float2bfloat16_rn(desc->skip_b[(size_t)l * S + n]));
    if (int rc = dev_alloc(&tc->skip_bsum, sizeof(float) * S)) return rc;
    cudaMemcpy(tc->skip_bsum, bsum.data(), sizeof(float) * S, cudaMemcpyHostToDevice);
  }
  if (int rc = dev_alloc(&tc->zimg, (size_t)tc->ntile * kskip * kTile)) return rc;
  if (int rc = dev_alloc(&tc->simg, (size_t)tc->ntile * (S / 64) * kTile)) return rc;
  if (int rc = dev_alloc(&tc->himg, (size_t)tc->ntile * (H / 64) * kTile)) return rc;
  if (int rc = dev_alloc(&tc->cls, sizeof(int32_t) * h.batch)) return rc;
  cudaError_t e = set_smem(step_kernel, kChainSmem);
  if (e == cudaSuccess) e = set_smem(step_kernel_fold, kChainSmem);
  if (e == cudaSuccess) e = set_smem(step_kernel_2sm, kChainSmem);
  if (e == cudaSuccess) e = set_smem(step_kernel_2sf, kChainSmem);
  if (e == cudaSuccess) e = set_smem(gemm_kernel<128, 0>, gemm_smem<128>());
  if (e == cudaSuccess) e = set_smem(gemm_kernel<256, 1>, gemm_smem<256>());
  if (e != cudaSuccess) {
    set_error(std::string("tcgen05 kernel attributes: ") + cudaGetErrorString(e));
    return FW_ERR_CUDA;
  }
  return FW_OK;
}

void tc_destroy(Handle& h) {
  TcState* tc = h.tc;
  if (!tc) return;
  void* ptrs[] = {tc->w2sm, tc->wfold, tc->fold_b, tc->wchain, tc->wskip, tc->wskip2, tc->zflag, tc->d_qoff, tc->wh1b, tc->wh1, tc->wh2, tc->skip_bsum,
                  tc->zimg, tc->simg, tc->himg, tc->cls};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete tc;
  h.tc = nullptr;
}

cudaError_t launch_cell_tc(Handle& h, const CellRun& run, cudaStream_t st, int64_t* launches) {
  TcState* tc = h.tc;
  const CellDims& d = h.dims;
  const int B = h.batch, L = d.L, S = d.S, H = d.H;
  cudaError_t e = cudaMemcpyAsync(tc->cls, run.inputs, sizeof(int32_t) * B,
                                  cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  ChainArgs ca{};
  ca.B = B;
  ca.L = L;
  ca.queue = reinterpret_cast<uint8_t*>(h.d_queue);
  ca.fold = tc->fold;
  ca.w = tc->fold ? tc->wfold : tc->cg2 ? tc->w2sm : tc->wchain;
  ca.embed = h.w.embed;
  ca.dil_b = (tc->fold || tc->cg2 == 2) ? tc->fold_b : h.w.dil_b;
  ca.res_b = h.w.res_b;
  ca.cls = tc->cls;
  ca.zimg = tc->zimg;
  ca.has_dil_bias = (tc->fold || tc->cg2 == 2) ? tc->fold_has_bias : tc->has_dil_bias;
  ca.has_res_bias = tc->has_res_bias;
  ca.trace = tc->trace;
  const int npairs_all = B / 128;
  ca.nchain = tc->nchain;
  ca.split = tc->split;
  ca.zpub = tc->split ? 4 : 2;
  ca.zflag = tc->fused ? tc->zflag : nullptr;
  // z stash: a 16-layer ring per pair in the fused kernel (the unfused skip GEMM reads all L)
  ca.zring = tc->fused ? std::min(L, 16) : L;
  ca.zfree = tc->fused ? tc->zflag + 4 * npairs_all : nullptr;
  ca.ztail = tc->nskip / npairs_all;  // tail blocks per pair, each reads every z tile
  ca.wskip2 = tc->wskip2;
  ca.skip_bsum = tc->skip_bsum;
  ca.simg = tc->simg;
  ca.S = S;
  ca.SK = tc->SK;
  ca.heads = tc->heads;
  // pair mode: a 2-CTA cluster per tile pair (S = H = 512, A = 256, cluster launch)
  ca.pair_mode = tc->heads && S == 512 && H == 512 && d.A == 256 && !getenv("FW_NO_CLUSTER");
  ca.H = H;
  ca.sflag = tc->zflag + npairs_all;
  ca.hflag = tc->zflag + 2 * npairs_all;
  ca.wh1b = tc->wh1b;
  ca.wh2 = tc->wh2;
  ca.h1_b = h.w.h1_b;
  ca.himg = tc->himg;
  const int grid = tc->fused ? tc->nchain + tc->nskip : tc->nchain;
  void* kargs[] = {&ca};
  for (int l = 0; l < L; ++l) {
    ca.dil[l] = h.dil[l];
    ca.slot0[l] = (int32_t)(run.t0 % h.dil[l]);
  }
  ca.qoff = tc->d_qoff;
  ca.slot_stride = (int64_t)(B / kChainRows) * kSlotBytes;
  ca.cls_ready = tc->zflag + 3 * npairs_all;
  GemmArgs skip{};
  skip.a = tc->zimg;
  skip.b = tc->wskip;
  skip.kch = L * kD / 64;
  skip.a_plain = 1;  // the chain kernel's z stash: [tile][L][16 K-pieces][128 rows][16 B]
  skip.bias = tc->skip_bsum;
  skip.out_img = tc->simg;
  skip.n_total = S;
  GemmArgs h1{};
  h1.a = tc->simg;
  h1.b = tc->wh1;
  h1.kch = S / 64;
  h1.bias = h.w.h1_b;
  h1.out_img = tc->himg;
  h1.n_total = H;
  GemmArgs h2{};
  h2.a = tc->himg;
  h2.b = tc->wh2;
  h2.kch = H / 64;
  SelectArgs sel{};
  sel.bias = h.w.h2_b;
  sel.A = d.A;
  sel.mode = run.mode;
  sel.seed = run.seed;
  sel.stream_offset = run.stream_offset;
  sel.cls_next = tc->cls;
  sel.out_base = run.out;
  sel.logits_base = run.logits;
  sel.n_logit_steps = run.n_logit_steps;
  sel.inputs = run.inputs;
  sel.n_inputs = run.n_inputs;
  sel.B = B;
  if (tc->fused) {
    // ONE cooperative launch runs every step: the chain blocks of a tile pair start step i+1
    // as soon as the pair's selection of step i is written (counters, no host round trip)
    const int timed = h.timing ? timing_reserve(h, 1) : 0;
    if (timed) cudaEventRecord(h.tev[0], st);
    const int per_launch = getenv("FW_STEPS_PER_LAUNCH") ? atoi(getenv("FW_STEPS_PER_LAUNCH")) : 0;
    const int chunk = per_launch > 0 ? per_launch : run.n_steps;
    for (int i0 = 0; i0 < run.n_steps; i0 += chunk) {
      ca.n_steps = std::min(chunk, run.n_steps - i0);
      ca.t0 = run.t0 + i0;
      for (int l = 0; l < L; ++l) ca.slot0[l] = (int32_t)(ca.t0 % h.dil[l]);
      ca.sel = sel;
      ca.sel.out_base = run.out + (size_t)i0 * B;
      ca.sel.logits_base = run.logits ? run.logits + (size_t)i0 * B * d.A : nullptr;
      ca.sel.n_logit_steps = run.n_logit_steps - i0;
      ca.sel.inputs = run.inputs + (size_t)std::min(i0, run.n_inputs) * B;
      ca.sel.n_inputs = std::max(0, run.n_inputs - i0);
      ca.sel.t = ca.t0;
      ca.sel.out_cls = ca.sel.out_base;
      ca.sel.logits = (run.logits && i0 < run.n_logit_steps) ? ca.sel.logits_base : nullptr;
      ca.sel.next_inputs = (1 < ca.sel.n_inputs) ? ca.sel.inputs + B : nullptr;
      e = cudaMemsetAsync(tc->zflag, 0, sizeof(uint32_t) * 5 * npairs_all, st);
      if (e != cudaSuccess) return e;
      {
        // cooperative (all blocks co-resident: the tail blocks wait on the chain blocks) and
        // clustered in pairs (a tile pair's two tail blocks share distributed shared memory)
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kChainThreads);
        cfg.dynamicSmemBytes = kChainSmem;
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = 2;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.attrs = at;
        // the cluster dimension for the pair tail (and the split / folded chain, which need it)
        cfg.numAttrs = (ca.pair_mode || ca.fold || tc->cg2) ? 2 : 1;
        e = cudaLaunchKernelExC(&cfg, ca.fold ? (const void*)step_kernel_fold
                                      : tc->cg2 == 2 ? (const void*)step_kernel_2sf
                                      : tc->cg2 ? (const void*)step_kernel_2sm
                                                : (const void*)step_kernel, kargs);
      }
      if (e != cudaSuccess) return e;
    }
    if (timed) {
      cudaEventRecord(h.tev[1], st);
      cudaEventRecord(h.tev[2], st);
    }
    h.tev_used = timed;
    h.timed_steps = timed ? run.n_steps : 0;
    *launches = 1;
    return cudaGetLastError();
  }
  // per-step launches: the step kernel (chain only) + skip / head1 / head2 GEMMs
  const dim3 gskip(tc->ntile, S / 128), gh1(tc->ntile, H / 128), gh2(tc->ntile, 1);
  const int timed = h.timing ? timing_reserve(h, run.n_steps) : 0;
  ca.n_steps = 1;
  for (int i = 0; i < run.n_steps; ++i) {
    ca.t0 = run.t0 + i;
    for (int l = 0; l < L; ++l) ca.slot0[l] = (int32_t)((run.t0 + i) % h.dil[l]);
    sel.t = run.t0 + i;
    sel.logits = (run.logits && i < run.n_logit_steps) ? run.logits + (size_t)i * B * d.A : nullptr;
    sel.out_cls = run.out + (size_t)i * B;
    sel.next_inputs = (i + 1 < run.n_inputs) ? run.inputs + (size_t)(i + 1) * B : nullptr;
    h2.sel = sel;
    static const bool dbg = getenv("FW_DEBUG_SYNC") != nullptr;
    auto chk = [&](const char* what) {
      if (!dbg) return;
      cudaError_t ce = cudaStreamSynchronize(st);
      if (ce != cudaSuccess) fprintf(stderr, "fw debug: %s failed: %s\n", what, cudaGetErrorString(ce));
    };
    if (i < timed) cudaEventRecord(h.tev[3 * i], st);
    step_kernel<<<grid, kChainThreads, kChainSmem, st>>>(ca);
    chk("step_kernel");
    if (i < timed) cudaEventRecord(h.tev[3 * i + 1], st);
    gemm_kernel<128, 0><<<gskip, kGemmThreads, gemm_smem<128>(), st>>>(skip);
    chk("skip gemm");
    gemm_kernel<128, 0><<<gh1, kGemmThreads, gemm_smem<128>(), st>>>(h1);
    chk("head1 gemm");
    gemm_kernel<256, 1><<<gh2, kGemmThreads, gemm_smem<256>(), st>>>(h2);
    chk("head2 gemm");
    if (i < timed) cudaEventRecord(h.tev[3 * i + 2], st);
  }
  h.tev_used = timed;
  h.timed_steps = timed;
  *launches = 4 * (int64_t)run.n_steps;
  if (getenv("FW_DEBUG_SYNC")) {
    cudaError_t ce = cudaStreamSynchronize(st);
    fprintf(stderr, "fw debug: unfused %d steps done: %s\n", run.n_steps, cudaGetErrorString(ce));
  }
  return cudaGetLastError();
}

}  // namespace fw
