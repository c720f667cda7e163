// K1m: the fp32 configs' step kernel on warp-level tensor-core MMAs (BASELINE configs 3 and 5,
// R = D = 64, S = H = A = 256).
//
// A CTA owns BT = 8 NT streams for the whole generate call and runs every layer of every step
// on the device, like the weight-staged SIMT kernel (cell_simt.cu, K1s) -- same ring pops and
// pushes, bias prefetch, weight ring fed by a producer warp with bulk copies -- but each GEMM
// is a tile product on the tensor cores: output channels on the MMA's M (16 per tile),
// streams on N (8 per tile), input channels on K (16 per step). At 8-16 streams per CTA the
// GEMMs are far below a tcgen05 tile (M = 64/128 rows of streams, TMEM round trips, ~300
// cycles from issue to a visible commit); mma.sync m16n8k16 keeps the accumulators in
// registers, so the gate, the residual update and the skip sum are register epilogues
// (tools/hmma_rate.cu: 21 cycles dependent latency, 0.5 MMA/clk per SM).
//
// fp32 accuracy from fp16 tensor cores: every operand v is split into hi = fp16(v) and
// lo = fp16(v - hi) (22 significant bits), and each product is the three MMAs
// hi.hi + hi.lo + lo.hi accumulated in fp32 (the dropped lo.lo term is ~2^-22 relative);
// tolerance 1e-4 on the logits (north star). The running sums (residual stream, skip sum)
// are added in fp32 outside the MMAs: the tensor cores' fp32 accumulation is not IEEE-exact,
// and accumulating x through 96 layers inside it gave 1.5e-4 on cfg5's logits.
//
// Weights are packed on the host into per-lane fragment order: tile (K-step kt, M-tile mt)
// is 1 KB -- 32 lanes x 16 B of hi fragments, then of lo -- so a warp loads a fragment with
// one conflict-free 16-byte shared load per lane. A matrix streams through the ring in
// K-step slabs (all M-tiles of one kt); every compute warp walks every stage.
//   dilated: M = 2D, tile j rows 0..7 = tanh channels 8j.., rows 8..15 = sigmoid channels
//            8j.. -- a thread's accumulator holds both gate inputs of one channel, so
//            z = tanh(a) sigmoid(b) is computed in registers; K = 2R (x_t | x_{t-d})
//   cat:     M = R + S (residual rows, then skip rows), K = D; the accumulators start from
//            x_l + b_res / s + b_skip, so x_{l+1} and the running skip sum come out directly
//   heads:   M = H (K = S), then M = A (K = H)
// Activations feeding a GEMM (x_t | x_{t-d}, z, ReLU(s), h) are written in the B-fragment
// order (hi | lo per lane) by the producing epilogue.
#include <cuda_fp16.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.h"
#include "select.cuh"
#include "tc_ptx.cuh"

namespace fw {

struct HmmaPlan {
  uint32_t* w = nullptr;      // fragment images: per layer dil | cat, then head1 | head2
  int64_t layer_words = 0;    // per-layer stride (32-bit words)
  int64_t a_words = 0;        // phase-A image words within a layer (phase B follows)
  int64_t head_off = 0;       // word offset of the top layer's skip (head1, head2 follow)
  int64_t top_words = 0;
  int64_t h1_words = 0;
  float* bsum = nullptr;      // [S] sum over layers of the skip biases
};

namespace {

constexpr int kHmNT = 256;              // compute threads (8 warps)
constexpr int kHmThreads = kHmNT + 32;  // + the weight producer warp
constexpr int kHmBar = 1;               // named barrier of the compute warps
constexpr int kHmStages = 5;
constexpr int kHmStage = 32 * 1024;     // one weight stage (phase-A slab 32 KB; 16 KB slabs pair up)
constexpr int kTileBytes = 1024;        // one (kt, mt) fragment tile: hi | lo
constexpr int kBFragBytes = 512;        // one (kt, nt) activation fragment: 32 lanes x 16 B

template <int R_, int D_, int S_, int H_, int A_>
struct HmShape {
  static constexpr int R = R_, D = D_, S = S_, H = H_, A = A_;
};
using Cfg35 = HmShape<64, 64, 256, 256, 256>;

struct HmmaParams {
  int B, L;
  const int* dil;
  const int64_t* qoff;
  float* queue;
  const uint32_t* w;
  int64_t layer_words, a_words, head_off, top_words, h1_words;
  const float *embed, *dil_b, *res_b, *bsum, *h1_b, *h2_b;
  CellRun run;
  long long* trace;  // fw_debug_trace: [L + 2][8] clock64 stamps of CTA 0's thread 0, or null
};

struct HmLayout {
  int xb, zb, sb, hb, xf, lg, pops, bias, hbias, lcon, cls, bars, ring;
  size_t total;
};

template <int NT, class Sh>
HmLayout hm_layout(int L) {
  constexpr int BT = 8 * NT;
  HmLayout y{};
  int o = 0;
  auto take = [&](int bytes) {
    const int at = o;
    o += (bytes + 127) & ~127;
    return at;
  };
  y.xb = take(2 * (2 * Sh::R / 16) * NT * kBFragBytes);
  y.zb = take(2 * (Sh::D / 16) * NT * kBFragBytes);
  y.sb = take((Sh::S / 16) * NT * kBFragBytes);
  y.hb = take((Sh::H / 16) * NT * kBFragBytes);
  y.xf = take(4 * Sh::R * BT);
  y.lg = take(4 * BT * Sh::A);
  y.pops = take(4 * 4 * BT * Sh::R);
  y.bias = take(4 * 4 * (2 * Sh::D + Sh::R));
  y.hbias = take(4 * (Sh::H + Sh::A + Sh::S));
  y.lcon = take(8 * 2 * L);
  y.cls = take(4 * BT);
  y.bars = take(8 * 2 * kHmStages);
  y.ring = o;
  y.total = (size_t)o + (size_t)kHmStages * kHmStage;
  return y;
}

struct HmRing {
  uint64_t* full;
  uint64_t* empty;
  uint8_t* buf;
  int slot;
  uint32_t ph;
  __device__ __forceinline__ void advance() {
    if (++slot == kHmStages) {
      slot = 0;
      ph ^= 1u;
    }
  }
};

// Producer: a matrix of SLABS K-step slabs of SLAB bytes, as many whole slabs per stage as
// fit; each copy is split over 4 lanes (one thread's bulk copies run one after another).
template <int SLABS, int SLAB>
__device__ __forceinline__ void hm_produce(HmRing& rg, const uint32_t* W) {
  constexpr int per = kHmStage / SLAB;
  static_assert(per >= 1, "a K-step slab must fit a stage");
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int k0 = 0; k0 < SLABS; k0 += per) {
    const int n = min(per, SLABS - k0);
    const uint32_t bytes = (uint32_t)n * SLAB;
    if (lane == 0) {
      ptx::mbar_wait(&rg.empty[rg.slot], rg.ph ^ 1u);
      ptx::mbar_arrive_expect_tx(&rg.full[rg.slot], bytes);
    }
    __syncwarp();
    const uint32_t slice = (bytes + 63) / 64 * 16;  // 4 slices, 16-byte multiples
    const uint32_t off = (uint32_t)lane * slice;
    if (lane < 4 && off < bytes)
      ptx::bulk_g2s(rg.buf + (size_t)rg.slot * kHmStage + off,
                    reinterpret_cast<const uint8_t*>(W) + (size_t)k0 * SLAB + off,
                    min(slice, bytes - off), &rg.full[rg.slot]);
    rg.advance();
  }
}

__device__ __forceinline__ void hmma(float (&c)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// acc[j][nt][p] (+)= tile (warp + 8 j) of W . B, j < NTL (this warp's tile count, a
// compile-time constant: no per-step branches), over all K steps; the three split products
// p = hi.hi, hi.lo, lo.hi in separate accumulators (independent dependency chains). Every
// warp walks every stage of the matrix (its slabs hold all M-tiles); no CTA barrier.
template <int NTL, int MTW, int NT, int KT, int MT>
__device__ __forceinline__ void hm_gemm_n(HmRing& rg, const uint8_t* bfrag, float (&acc)[MTW][NT][3][4]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int per = kHmStage / (MT * kTileBytes);
#pragma unroll
  for (int k0 = 0; k0 < KT; k0 += per) {
    ptx::mbar_wait(&rg.full[rg.slot], rg.ph);
    const uint8_t* st = rg.buf + (size_t)rg.slot * kHmStage + (size_t)warp * kTileBytes + lane * 16;
#pragma unroll
    for (int kk = 0; kk < per && k0 + kk < KT; ++kk) {
      const int kt = k0 + kk;
      uint4 bf[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        bf[nt] = *reinterpret_cast<const uint4*>(bfrag + ((size_t)kt * NT + nt) * kBFragBytes + lane * 16);
#pragma unroll
      for (int j = 0; j < NTL; ++j) {
        const uint8_t* tp = st + ((size_t)kk * MT + 8 * j) * kTileBytes;
        const uint4 ah = *reinterpret_cast<const uint4*>(tp);
        const uint4 al = *reinterpret_cast<const uint4*>(tp + 512);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          hmma(acc[j][nt][0], ah, bf[nt].x, bf[nt].y);
          hmma(acc[j][nt][1], ah, bf[nt].z, bf[nt].w);
          hmma(acc[j][nt][2], al, bf[nt].x, bf[nt].y);
        }
      }
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&rg.empty[rg.slot]);
    rg.advance();
  }
}
// warps [0, MT - 8 (MTW - 1)) own MTW tiles, the others MTW - 1
template <int MTW, int NT, int KT, int MT>
__device__ __forceinline__ void hm_gemm(HmRing& rg, const uint8_t* bfrag, float (&acc)[MTW][NT][3][4]) {
  constexpr int full_warps = MT - 8 * (MTW - 1);
  if constexpr (full_warps >= 8) {
    hm_gemm_n<MTW, MTW, NT, KT, MT>(rg, bfrag, acc);
  } else {
    if ((int)(threadIdx.x >> 5) < full_warps) hm_gemm_n<MTW, MTW, NT, KT, MT>(rg, bfrag, acc);
    else hm_gemm_n<MTW - 1, MTW, NT, KT, MT>(rg, bfrag, acc);
  }
}

// v -> (hi, lo) fp16 halves at activation (k, n) of a B-fragment buffer: K-step k / 16,
// lane 4 (n % 8) + (k % 8) / 2, register (k % 16) / 8, half k % 2.
template <int NT>
__device__ __forceinline__ int b_off(int k, int n) {
  const int kt = k >> 4, kk = k & 15, nt = n >> 3, g = n & 7;
  const int lane = 4 * g + ((kk & 7) >> 1);
  return ((kt * NT + nt) * 32 + lane) * 16 + (kk >> 3) * 4 + (kk & 1) * 2;
}
__device__ __forceinline__ void put_hl(uint8_t* p, float v) {
  const __half hi = __float2half_rn(v);
  const __half lo = __float2half_rn(v - __half2float(hi));
  *reinterpret_cast<__half*>(p) = hi;
  *reinterpret_cast<__half*>(p + 8) = lo;
}
template <int NT>
__device__ __forceinline__ void put_b(uint8_t* buf, int k, int n, float v) {
  put_hl(buf + b_off<NT>(k, n), v);
}
// z = tanh(a) sigmoid(g) with MUFU exponentials and approximate reciprocals (ex2, rcp:
// ~1e-7 absolute; the accurate tanhf / expf / IEEE divisions were most of the gate's ~150
// instructions per value)
__device__ __forceinline__ float hm_gate(float a, float g) {
  const float th = 1.f - __fdividef(2.f, __expf(2.f * a) + 1.f);
  return th * __fdividef(1.f, 1.f + __expf(-g));
}

// accumulator element e (0..3) of tile row base m0 = 16 mt: row m0 + g + 8 (e >> 1), stream
// 8 nt + 2 t + (e & 1)
__device__ __forceinline__ float acc_sum(const float (&a)[3][4], int e) { return a[0][e] + (a[1][e] + a[2][e]); }

template <int NT, class Sh>
__global__ void __launch_bounds__(kHmThreads, 1) cell_hmma_kernel(HmmaParams p, HmLayout y) {
  constexpr int BT = 8 * NT;
  constexpr int R = Sh::R, D = Sh::D, S = Sh::S, H = Sh::H, A = Sh::A;
  constexpr int KT1 = 2 * R / 16, MT1 = 2 * D / 16, KT2 = D / 16, MTS = S / 16, MTR = R / 16;
  constexpr int MTH1 = H / 16, MTH2 = A / 16, MTWH = ((MTH1 > MTH2 ? MTH1 : MTH2) + 7) / 8;
  static_assert(MT1 == 8 && MTS == 16 && MTR <= 8 && KT1 == 2 * KT2, "cfg3 / cfg5 shapes");
  static_assert(2 * MT1 + MTS <= kHmStage / kTileBytes, "a phase-A slab fits a stage");
  constexpr int NB = 2 * D + R;  // per-layer biases: dil | res (the skip biases are summed)
  // (the shared window itself, not an aligned generic pointer into it: the compiler then emits
  // LDS / STS instead of generic loads and stores -- 128-byte alignment is all the bulk copies
  // and 16-byte fragment loads need)
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int XB = KT1 * NT * kBFragBytes, ZB = KT2 * NT * kBFragBytes;
  uint8_t* xb = sm + y.xb;  // [2][KT1][NT] fragments: x_t (k < R) | x_{t-d}
  uint8_t* zb = sm + y.zb;  // [2][KT2][NT]: z of layers gg & 1
  uint8_t* sbf = sm + y.sb;
  uint8_t* hbf = sm + y.hb;
  float* xf = reinterpret_cast<float*>(sm + y.xf);  // [R][BT] x_l, fp32
  float* lg = reinterpret_cast<float*>(sm + y.lg);  // [BT][A] logits
  float* pops = reinterpret_cast<float*>(sm + y.pops);  // [4][BT][R]
  float* bias = reinterpret_cast<float*>(sm + y.bias);  // [4][NB]
  float* hbias = reinterpret_cast<float*>(sm + y.hbias);  // h1 | h2 | sum of the skip biases
  const int L = p.L;
  // [2][L]: element offset of layer l's ring slot at steps t (row 0) and t + 1 (row 1)
  int64_t* qbo_s = reinterpret_cast<int64_t*>(sm + y.lcon);
  int* cls = reinterpret_cast<int*>(sm + y.cls);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + y.bars);
  HmRing rg{bars, bars + kHmStages, sm + y.ring, 0, 0u};

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int s0 = blockIdx.x * BT;
  const int nb = min(BT, p.B - s0);
  const CellRun& run = p.run;
  const int B = p.B;
  const int GL = run.n_steps * L;
  if (tid == 0) {
    for (int i = 0; i < kHmStages; ++i) {
      ptx::mbar_init(&rg.full[i], 1);
      ptx::mbar_init(&rg.empty[i], kHmNT / 32);
    }
    ptx::fence_mbar_init();
  }
  if (tid < BT) cls[tid] = (tid < nb) ? run.inputs[s0 + tid] : 0;
  constexpr int R4 = R / 4;
  const size_t slot_elems = (size_t)((B + 127) / 128) * 128 * R;
  for (int e = tid; e < 2 * L; e += blockDim.x) {
    const int l = e % L;
    qbo_s[e] = p.qoff[l] + (int64_t)((run.t0 + e / L) % p.dil[l]) * (int64_t)slot_elems;
  }
  for (int e = tid; e < H + A + S; e += blockDim.x)
    hbias[e] = e < H ? p.h1_b[e] : e < H + A ? p.h2_b[e - H] : p.bsum[e - H - A];
  // the z buffers start as zeros (layer 0's skip slot multiplies the "previous z" by zeros)
  for (int e = tid; e < 2 * ZB / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(zb)[e] = 0u;
  __syncthreads();

  if (warp == kHmNT / 32) {  // ---- weight producer: the step's matrices in consumption order
    for (int i = 0; i < run.n_steps; ++i) {
      for (int l = 0; l < L; ++l) {
        const uint32_t* wl = p.w + (size_t)l * p.layer_words;
        hm_produce<KT1 / 2, (2 * MT1 + MTS) * kTileBytes>(rg, wl);      // phase A
        hm_produce<1, KT2 * MTR * kTileBytes>(rg, wl + p.a_words);       // phase B
      }
      hm_produce<KT2, MTS * kTileBytes>(rg, p.w + p.head_off);           // top layer's skip
      hm_produce<S / 16, MTH1 * kTileBytes>(rg, p.w + p.head_off + p.top_words);
      hm_produce<H / 16, MTH2 * kTileBytes>(rg, p.w + p.head_off + p.top_words + p.h1_words);
    }
    return;
  }

  // ring layout [B/128][R/4][128 streams][4 channels] fp32 (the SIMT handles' queues); pops
  // by thread e <-> (stream b, 4-channel chunk c4), prefetched three layers ahead; pushes from
  // the epilogues that produce x
  auto ring_elem = [&](int64_t base, int st, int c) {
    return p.queue + base + ((size_t)((st >> 7) * R4 + (c >> 2)) * 128 + (st & 127)) * 4 + (c & 3);
  };
  // the ring pops, the bias prefetch and the conversion of the pops to B fragments run on the
  // warps the residual GEMM leaves idle (warps >= R / 16), during phase B
  constexpr int kPf = kHmNT - 32 * MTR;  // prefetcher threads
  const bool pf = warp >= MTR;
  const int pe = tid - 32 * MTR;
  // pops and biases of global layer gg = layer l of step row (0: this step, 1: the next)
  auto prefetch = [&](int gg, int l, int row) {
    if (gg < GL) {
      const int64_t base = qbo_s[row * L + l];
      for (int e = pe; e < nb * R4; e += kPf) {
        const int b = e / R4, c4 = e % R4;
        ptx::cp_async16(ptx::smem_u32(pops + ((gg % 4) * BT + b) * R + 4 * c4), ring_elem(base, s0 + b, 4 * c4));
      }
      float* bb = bias + (gg % 4) * NB;
      for (int e = pe; e < NB / 4; e += kPf) {
        const int o = 4 * e;
        const float* src = o < 2 * D ? p.dil_b + (size_t)l * 2 * D + o : p.res_b + (size_t)l * R + (o - 2 * D);
        ptx::cp_async16(ptx::smem_u32(bb + o), src);
      }
    }
    ptx::cp_async_commit();
  };
  // this thread's prefetched x_{t-d} chunks of layer gg -> B fragments (k = R + channel), in
  // the prefetch's thread <-> (stream, 4-channel chunk) map
  constexpr int CH = (BT * R4 + kPf - 1) / kPf;  // chunks per prefetcher thread
  int pop_bo[CH][4];
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = pe + c * kPf;
      pop_bo[c][q] = b_off<NT>(R + 4 * (e % R4) + q, e / R4);
    }
  auto take_pops = [&](int gg) {
    uint8_t* xd = xb + (size_t)(gg & 1) * XB;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int e = pe + c * kPf;
      if (e >= BT * R4) break;
      const int b = e / R4, c4 = e % R4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (b < nb) v = *reinterpret_cast<const float4*>(pops + ((gg % 4) * BT + b) * R + 4 * c4);
      put_hl(xd + pop_bo[c][0], v.x);
      put_hl(xd + pop_bo[c][1], v.y);
      put_hl(xd + pop_bo[c][2], v.z);
      put_hl(xd + pop_bo[c][3], v.w);
    }
  };
  if (pf)
    for (int k = 0; k < 3; ++k) prefetch(k, k % L, k / L);
  // per-thread constant offsets of the epilogues' elements (B fragments, ring slots)
  int gate_bo[NT][2];  // z of channel 8 warp + g, streams 8 nt + 2 t4 + e
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) gate_bo[nt][e] = b_off<NT>(8 * warp + g, 8 * nt + 2 * t4 + e);
  int res_bo[NT][4], res_ro[NT][4];  // warps < R / 16: the residual tile `warp`
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int m = 16 * warp + g + 8 * (e >> 1), n = 8 * nt + 2 * t4 + (e & 1), st = s0 + n;
      res_bo[nt][e] = b_off<NT>(m, n);
      res_ro[nt][e] = ((st >> 7) * R4 + (m >> 2)) * 512 + (st & 127) * 4 + (m & 3);
    }
  if (pf) {
    ptx::cp_async_wait<2>();
    take_pops(0);
  }
  const uint32_t lane16 = (uint32_t)lane * 16;

  for (int i = 0; i < run.n_steps; ++i) {
    const int64_t t = run.t0 + i;
    // layer 0's input: the embedding of each stream's class
    {
      uint8_t* x0 = xb + (size_t)((i * L) & 1) * XB;
      if (i > 0) {  // slot table: step t in row 0, t + 1 in row 1 (the prefetches of the
                    // previous step's last layers read row 1 before this barrier)
        for (int e = tid; e < L; e += kHmNT) {
          qbo_s[e] = qbo_s[L + e];
          qbo_s[L + e] = p.qoff[e] + (int64_t)((t + 1) % p.dil[e]) * (int64_t)slot_elems;
        }
        ptx::named_bar_sync(kHmBar, kHmNT);
      }
      for (int e = tid; e < BT * R; e += kHmNT) {
        const int b = e / R, r = e % R;
        const float v = __ldg(p.embed + (size_t)clamp_class(cls[b], A) * R + r);
        xf[r * BT + b] = v;
        put_b<NT>(x0, r, b, v);
        if (b < nb) *ring_elem(qbo_s[0], s0 + b, r) = v;  // push x_0[t] (its pop was read ahead)
      }
    }
    // running skip sum of this thread's tiles (warp, warp + 8) x streams, fp32 (added outside
    // the tensor cores' accumulation)
    float s_reg[2][NT][4] = {};
    ptx::named_bar_sync(kHmBar, kHmNT);
    for (int l = 0; l < L; ++l) {
      const int gg = i * L + l;
      long long* tr = (p.trace != nullptr && blockIdx.x == 0 && tid == 0) ? p.trace + (size_t)l * 8 : nullptr;
      if (tr) tr[0] = clock64();
      const uint8_t* xc = xb + (size_t)(gg & 1) * XB;
      uint8_t* xn = xb + (size_t)((gg + 1) & 1) * XB;
      uint8_t* zc = zb + (size_t)(gg & 1) * ZB;
      const uint8_t* zp = zb + (size_t)((gg + 1) & 1) * ZB;  // z of layer gg - 1
      const float* bl = bias + (gg % 4) * NB;
      // ---- phase A: dilated GEMM of layer l (tile `warp`: tanh and sigmoid rows of channels
      // 8 warp ..) interleaved with the skip GEMM of layer l - 1 (tiles warp, warp + 8), off
      // the dependent path; per stage two dilated K-steps and one skip K-step
      {
        float dacc[NT][3][4] = {};
        float sacc[2][NT][3][4] = {};
#pragma unroll
        for (int q = 0; q < KT1 / 2; ++q) {
          ptx::mbar_wait(&rg.full[rg.slot], rg.ph);
          const uint8_t* st = rg.buf + (size_t)rg.slot * kHmStage + lane16;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int kt = 2 * q + kk;
            const uint8_t* tp = st + (size_t)(kk * MT1 + warp) * kTileBytes;
            const uint4 ah = *reinterpret_cast<const uint4*>(tp);
            const uint4 al = *reinterpret_cast<const uint4*>(tp + 512);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const uint4 bf = *reinterpret_cast<const uint4*>(xc + (size_t)(kt * NT + nt) * kBFragBytes + lane16);
              hmma(dacc[nt][0], ah, bf.x, bf.y);
              hmma(dacc[nt][1], ah, bf.z, bf.w);
              hmma(dacc[nt][2], al, bf.x, bf.y);
            }
          }
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const uint8_t* tp = st + (size_t)(2 * MT1 + warp + 8 * j) * kTileBytes;
            const uint4 ah = *reinterpret_cast<const uint4*>(tp);
            const uint4 al = *reinterpret_cast<const uint4*>(tp + 512);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const uint4 bf = *reinterpret_cast<const uint4*>(zp + (size_t)(q * NT + nt) * kBFragBytes + lane16);
              hmma(sacc[j][nt][0], ah, bf.x, bf.y);
              hmma(sacc[j][nt][1], ah, bf.z, bf.w);
              hmma(sacc[j][nt][2], al, bf.x, bf.y);
            }
          }
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&rg.empty[rg.slot]);
          rg.advance();
        }
        if (tr) tr[1] = clock64();
        // gate: a thread holds tanh and sigmoid inputs of channel 8 warp + g for streams
        // 8 nt + 2 t4 + {0, 1}
        const int ch = 8 * warp + g;
        const float bt = bl[ch], bs = bl[D + ch];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float a = acc_sum(dacc[nt], e) + bt;
            const float s = acc_sum(dacc[nt], 2 + e) + bs;
            put_hl(zc + gate_bo[nt][e], hm_gate(a, s));
          }
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) s_reg[j][nt][e] += acc_sum(sacc[j][nt], e);
      }
      if (tr) tr[2] = clock64();
      // this thread's pops of layer gg + 1 have landed: the read of the slot the residual
      // epilogue pushes into (layer gg + 1's, after the barrier) is complete
      if (pf) ptx::cp_async_wait<1>();
      if (tr) tr[3] = clock64();
      ptx::named_bar_sync(kHmBar, kHmNT);
      if (tr) tr[4] = clock64();
      // ---- phase B: x_{l+1} = x_l + (W_res z_l + b_res) on warps < R / 16 (tile `warp`)
      {
        ptx::mbar_wait(&rg.full[rg.slot], rg.ph);
        if (warp < MTR) {
          const uint8_t* st = rg.buf + (size_t)rg.slot * kHmStage + lane16;
          float racc[NT][3][4] = {};
#pragma unroll
          for (int kt = 0; kt < KT2; ++kt) {
            const uint8_t* tp = st + (size_t)(kt * MTR + warp) * kTileBytes;
            const uint4 ah = *reinterpret_cast<const uint4*>(tp);
            const uint4 al = *reinterpret_cast<const uint4*>(tp + 512);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const uint4 bf = *reinterpret_cast<const uint4*>(zc + (size_t)(kt * NT + nt) * kBFragBytes + lane16);
              hmma(racc[nt][0], ah, bf.x, bf.y);
              hmma(racc[nt][1], ah, bf.z, bf.w);
              hmma(racc[nt][2], al, bf.x, bf.y);
            }
          }
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&rg.empty[rg.slot]);
          if (l + 1 < L) {  // (the top layer's residual output has no consumer)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int m = 16 * warp + g + 8 * (e >> 1), n = 8 * nt + 2 * t4 + (e & 1);
                const float xv = xf[m * BT + n] + (acc_sum(racc[nt], e) + bl[2 * D + m]);
                xf[m * BT + n] = xv;
                put_hl(xn + res_bo[nt][e], xv);
                if (n < nb) p.queue[qbo_s[l + 1] + res_ro[nt][e]] = xv;  // push x_{l+1}[t]
              }
          }
        } else {
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&rg.empty[rg.slot]);
          if (gg + 1 < GL) take_pops(gg + 1);
          prefetch(gg + 3, l + 3 < L ? l + 3 : l + 3 - L, l + 3 < L ? 0 : 1);
        }
        rg.advance();
      }
      if (tr) tr[5] = clock64();
      ptx::named_bar_sync(kHmBar, kHmNT);
      if (tr) tr[6] = clock64();
    }
    // the top layer's skip, then ReLU(s + sum of the skip biases) -> head1's B fragments
    {
      float acc[2][NT][3][4] = {};
      hm_gemm<2, NT, KT2, MTS>(rg, zb + (size_t)((i * L + L - 1) & 1) * ZB, acc);
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int m = 16 * (warp + 8 * j) + g + 8 * (e >> 1), n = 8 * nt + 2 * t4 + (e & 1);
            const float sv = (s_reg[j][nt][e] + acc_sum(acc[j][nt], e)) + hbias[H + A + m];
            put_b<NT>(sbf, m, n, fmaxf(sv, 0.f));
          }
    }
    ptx::named_bar_sync(kHmBar, kHmNT);
    // head: logits = W2 relu(W1 relu(s) + b1) + b2
#pragma unroll 1
    for (int hd = 0; hd < 2; ++hd) {
      const int MT = hd == 0 ? MTH1 : MTH2;
      float acc[MTWH][NT][3][4] = {};
      if (hd == 0) hm_gemm<MTWH, NT, S / 16, MTH1>(rg, sbf, acc);
      else hm_gemm<MTWH, NT, H / 16, MTH2>(rg, hbf, acc);
#pragma unroll
      for (int j = 0; j < MTWH; ++j) {
        const int mt = warp + 8 * j;
        if (mt >= MT) continue;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int m = 16 * mt + g + 8 * (e >> 1), n = 8 * nt + 2 * t4 + (e & 1);
            const float v = acc_sum(acc[j][nt], e) + hbias[(hd == 0 ? 0 : H) + m];
            if (hd == 0) put_b<NT>(hbf, m, n, fmaxf(v, 0.f));
            else lg[n * A + m] = v;
          }
      }
      ptx::named_bar_sync(kHmBar, kHmNT);
    }
    if (run.logits != nullptr && i < run.n_logit_steps) {
      float* dst = run.logits + ((size_t)i * B + s0) * A;
      for (int e = tid; e < nb * A; e += kHmNT) dst[e] = lg[e];
    }
    for (int b = warp; b < nb; b += kHmNT / 32) {
      const uint32_t gs = (uint32_t)(run.stream_offset + s0 + b);
      const uint32_t prefix = noise_prefix(run.seed, gs, (uint32_t)t);
      const int c = select_class(lg + b * A, A, run.mode, prefix);
      if (lane == 0) {
        run.out[(size_t)i * B + s0 + b] = c;
        cls[b] = (i + 1 < run.n_inputs) ? run.inputs[(size_t)(i + 1) * B + s0 + b] : c;
      }
    }
    ptx::named_bar_sync(kHmBar, kHmNT);
  }
  ptx::cp_async_wait<0>();
}

// ---- host: fragment images --------------------------------------------------------------
uint16_t h16(float v) {
  __half h = __float2half_rn(v);
  uint16_t u;
  std::memcpy(&u, &h, 2);
  return u;
}

// Tile (mt, kt) of W(m, k) -> 1 KB at dst: [hi: 32 lanes x 4 regs][lo: 32 x 4], register r
// of lane (g, t): row 16 mt + g + 8 (r & 1), columns 16 kt + 2 t + 8 (r >> 1) + {0, 1} (the
// m16n8k16 A fragment); hi = fp16(w), lo = fp16(w - hi).
template <typename F>
void pack_tile(uint32_t* dst, int mt, int kt, F W) {
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    for (int r = 0; r < 4; ++r) {
      const int m = 16 * mt + g + 8 * (r & 1), k = 16 * kt + 2 * t + 8 * (r >> 1);
      uint32_t hw = 0, lw = 0;
      for (int q = 0; q < 2; ++q) {
        const float v = W(m, k + q);
        const uint16_t hi = h16(v);
        __half hh;
        std::memcpy(&hh, &hi, 2);
        const uint16_t lo = h16(v - __half2float(hh));
        hw |= (uint32_t)hi << (16 * q);
        lw |= (uint32_t)lo << (16 * q);
      }
      dst[lane * 4 + r] = hw;
      dst[128 + lane * 4 + r] = lw;
    }
  }
}
// a whole matrix as [K/16][M/16] tiles (K-step slabs)
template <typename F>
void pack_frag(uint32_t* dst, int M, int K, F W) {
  for (int kt = 0; kt < K / 16; ++kt)
    for (int mt = 0; mt < M / 16; ++mt) pack_tile(dst + ((size_t)kt * (M / 16) + mt) * 256, mt, kt, W);
}

template <int NT, class Sh>
cudaError_t launch_hmma_t(Handle& h, const CellRun& run, cudaStream_t st) {
  const HmLayout y = hm_layout<NT, Sh>(h.dims.L);
  if (y.total > 227 * 1024) return cudaErrorNotSupported;
  cudaError_t e = cudaFuncSetAttribute(cell_hmma_kernel<NT, Sh>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)y.total);
  if (e != cudaSuccess) return e;
  HmmaParams p{};
  p.B = h.batch;
  p.L = h.dims.L;
  p.dil = h.d_dil;
  p.qoff = h.d_qoff;
  p.queue = h.d_queue;
  p.w = h.hmma->w;
  p.layer_words = h.hmma->layer_words;
  p.a_words = h.hmma->a_words;
  p.top_words = h.hmma->top_words;
  p.bsum = h.hmma->bsum;
  p.head_off = h.hmma->head_off;
  p.h1_words = h.hmma->h1_words;
  p.embed = h.w.embed;
  p.dil_b = h.w.dil_b;
  p.res_b = h.w.res_b;
  p.h1_b = h.w.h1_b;
  p.h2_b = h.w.h2_b;
  p.run = run;
  p.trace = h.lat_trace;
  const int grid = (h.batch + 8 * NT - 1) / (8 * NT);
  cell_hmma_kernel<NT, Sh><<<grid, kHmThreads, y.total, st>>>(p, y);
  return cudaGetLastError();
}

}  // namespace

bool hmma_supported(const CellDims& d) {
  return d.R == 64 && d.D == 64 && d.S == 256 && d.H == 256 && d.A == 256 && d.L >= 3 &&
         d.dtype == FW_DTYPE_F32;
}

int hmma_build(Handle& h) {
  if (h.hmma) return FW_OK;
  const CellDims& d = h.dims;
  const HostCell& c = h.host;
  const int L = d.L, R = d.R, D = d.D, S = d.S, H = d.H, A = d.A;
  const int MT1 = 2 * D / 16, MTS = S / 16, MTR = R / 16, KT1 = 2 * R / 16, KT2 = D / 16;
  // per layer l: phase A = KT1 / 2 slabs of [dil K-steps 2q, 2q+1 (MT1 tiles each) | skip of
  // layer l - 1, K-step q (MTS tiles)] (layer 0: zero skip weights); phase B = the residual
  // [KT2][MTR]; then the top layer's skip [KT2][MTS], head1, head2
  const int64_t a_words = (int64_t)(KT1 / 2) * (2 * MT1 + MTS) * 256;
  const int64_t b_words = (int64_t)KT2 * MTR * 256;
  const int64_t top_words = (int64_t)KT2 * MTS * 256;
  const int64_t h1_words = (int64_t)(S / 16) * (H / 16) * 256;
  const int64_t h2_words = (int64_t)(H / 16) * (A / 16) * 256;
  HmmaPlan* plan = new HmmaPlan();
  plan->layer_words = a_words + b_words;
  plan->a_words = a_words;
  plan->head_off = (int64_t)L * plan->layer_words;
  plan->top_words = top_words;
  plan->h1_words = h1_words;
  std::vector<uint32_t> img((size_t)(plan->head_off + top_words + h1_words + h2_words), 0u);
  auto skipW = [&](int l) {
    const float* ws = c.skip_w.data() + (size_t)l * S * D;
    return [ws, D](int m, int k) { return ws[(size_t)m * D + k]; };
  };
  for (int l = 0; l < L; ++l) {
    uint32_t* base = img.data() + (size_t)l * plan->layer_words;
    const float* w0 = c.dil_w.data() + ((size_t)l * 2 + 0) * 2 * D * R;
    const float* w1 = c.dil_w.data() + ((size_t)l * 2 + 1) * 2 * D * R;
    auto dilW = [&](int m, int k) {
      const int j = m >> 4, r = m & 15;
      const int row = r < 8 ? 8 * j + r : D + 8 * j + (r - 8);  // tanh / sigmoid channel
      return k < R ? w0[(size_t)row * R + k] : w1[(size_t)row * R + (k - R)];
    };
    for (int q = 0; q < KT1 / 2; ++q) {
      uint32_t* slab = base + (size_t)q * (2 * MT1 + MTS) * 256;
      for (int kk = 0; kk < 2; ++kk)
        for (int mt = 0; mt < MT1; ++mt) pack_tile(slab + (size_t)(kk * MT1 + mt) * 256, mt, 2 * q + kk, dilW);
      if (l > 0)
        for (int mt = 0; mt < MTS; ++mt) pack_tile(slab + (size_t)(2 * MT1 + mt) * 256, mt, q, skipW(l - 1));
    }
    const float* wr = c.res_w.data() + (size_t)l * R * D;
    pack_frag(base + a_words, R, D, [&](int m, int k) { return wr[(size_t)m * D + k]; });
  }
  uint32_t* hd = img.data() + plan->head_off;
  pack_frag(hd, S, D, skipW(L - 1));
  pack_frag(hd + top_words, H, S, [&](int m, int k) { return c.h1_w[(size_t)m * S + k]; });
  pack_frag(hd + top_words + h1_words, A, H, [&](int m, int k) { return c.h2_w[(size_t)m * H + k]; });
  std::vector<float> bsum(S, 0.f);
  for (int l = 0; l < L; ++l)
    for (int n = 0; n < S; ++n) bsum[n] += c.skip_b[(size_t)l * S + n];
  cudaError_t e = cudaMalloc(&plan->w, img.size() * 4);
  if (e == cudaSuccess) e = cudaMemcpy(plan->w, img.data(), img.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&plan->bsum, S * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpy(plan->bsum, bsum.data(), S * sizeof(float), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (plan->w) cudaFree(plan->w);
    if (plan->bsum) cudaFree(plan->bsum);
    delete plan;
    set_error(std::string("warp-MMA weight images: ") + cudaGetErrorString(e));
    return FW_ERR_CUDA;
  }
  h.hmma = plan;
  return FW_OK;
}

void hmma_destroy(Handle& h) {
  if (!h.hmma) return;
  if (h.hmma->w) cudaFree(h.hmma->w);
  if (h.hmma->bsum) cudaFree(h.hmma->bsum);
  delete h.hmma;
  h.hmma = nullptr;
}

// streams per CTA: 8 (NT = 1) up to 1,184 streams (148 CTAs), else 16; FW_HMMA_NT overrides
cudaError_t launch_cell_hmma(Handle& h, const CellRun& run, cudaStream_t st) {
  if (!hmma_supported(h.dims)) return cudaErrorNotSupported;
  if (hmma_build(h) != FW_OK) return cudaErrorMemoryAllocation;
  int nt = (h.batch + 7) / 8 <= 148 ? 1 : 2;
  if (const char* ev = getenv("FW_HMMA_NT")) nt = atoi(ev) == 2 ? 2 : 1;
  return nt == 1 ? launch_hmma_t<1, Cfg35>(h, run, st) : launch_hmma_t<2, Cfg35>(h, run, st);
}

}  // namespace fw
