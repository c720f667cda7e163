// Folded chain of the tcgen05 step kernel (included by cell_tc.cu after chain_tc.cuh): one
// 128-stream tile per 2-CTA cluster, CTA `half` computing dilated N-half `half` (64 tanh +
// 64 sigmoid columns, z channels 64 half .. +63), every MMA at M = 128.
//
// The residual update is folded into the next layer's dilated GEMM. With
//   a_l = W0_l x_l + W1_l x_l[t-d] + b_l,   x_l = x_{l-1} + Wr_{l-1} z_{l-1} + br_{l-1},
// layer l >= 1 computes
//   a_l = W1_l x_l[t-d] + W0_l x_{l-1} + (W0_l Wr_{l-1}) z_{l-1} + (b_l + W0_l br_{l-1}):
// the first two terms do not depend on z_{l-1} and are issued while layer l-1's gate runs,
// so the per-layer dependent path is z_{l-1} -> 8 MMAs (K = 128, the folded weight WF_l) ->
// gate -> z_l, instead of z -> res MMA -> x -> fp16 x -> x_t MMA -> gate. x_l itself is still
// accumulated (fp32, in TMEM) by the residual MMA, off the dependent path, for the ring push
// and the next layer's W0 term. WF_l = W0_l Wr_{l-1} is formed in fp64 from the (bf16)
// weights and rounded once to fp16 -- the same operand precision as every other weight.
//
//   TMEM (128 lanes = the tile's rows):  [0,256) acc[g & 1] (double-buffered dilated
//   accumulator, 128 columns each) | [256,384) x_l fp32 | [384,448) fp16 x operand (packed) |
//   [448,480) this half's fp16 z operand (packed).
//   SMEM: 6-stage ring of 16 KB weight K-chunks (SW128 [128 n][64 k]) | 2 x 32 KB popped ring
//   slots (x_{t-d}, no-swizzle K-major [16 K-pieces][128 rows][16 B], the slot's own layout:
//   one bulk copy per layer, used as the SS A operand) | 2 x 16 KB own z half | 2 x 16 KB the
//   peer's z half (same layout, 8 K-pieces) | barriers.
//
//   warp 0  lane 0  producer: weight chunks in MMA order + the ring pops (bulk copies)
//   warp 1          MMA issuer (converged warp, elect.sync)
//   warps 2..9      gate: quadrant q = warp % 4, column group cs = (warp - 2) / 4 -- z columns
//                   32 cs .. +31 of this half for rows 32q .. +31; z -> own image (SMEM) and,
//                   by st.async, into the peer's image
//   warps 10..13    x: the fp32 residual stream (TMEM) -> fp16 operand (TMEM) + this half's
//                   8 K-pieces of the ring push; the embedding gather at layer 0
//   warp 14 lane 0  publisher: own z half -> the z stash (one 16 KB bulk store), release
//
// Per layer g (l = g % L) the MMA issue order is xd(g) [W1 . x_{t-d}] -> W0(g) [W0 . x_{l-1}
// (l = 0: W0 . x_0, the embedding)] -> WF(g) own z half -> res(g) own half [x_l += Wr_{l-1}
// z_{l-1}] -> (the peer's half arrives) WF(g) peer half -> commit acc_full -> res(g) peer half
// -> commit x_full. The own halves' A operands are in TMEM, the peer's z in shared memory.
namespace fold {
constexpr uint32_t kWChunk = 16384;  // one [128 n][64 k] SW128 fp16 weight chunk
constexpr int kWStages = 6;
constexpr uint32_t kSlot = 32768;    // one tile's ring slot: [16 K-pieces][128 rows][16 B]
constexpr uint32_t kZHalf = 16384;   // one z half: [8 K-pieces][128 rows][16 B]
constexpr uint32_t kOffW = 0;
constexpr uint32_t kOffPop = kOffW + kWStages * kWChunk;  // 96 KB
constexpr uint32_t kOffZo = kOffPop + 2 * kSlot;           // 160 KB
constexpr uint32_t kOffZp = kOffZo + 2 * kZHalf;           // 192 KB
constexpr uint32_t kOffBar = kOffZp + 2 * kZHalf;          // 224 KB
constexpr size_t kSmem = 1024 + kOffBar + 512;
// global weight image per layer: 14 chunks, [W1 h0 | W1 h1 | W0 h0 | W0 h1 | WF h0 | WF h1 |
// Wr_{l-1}] x 2 K-chunks each
constexpr int kLayerChunks = 14;
constexpr uint32_t kLayerBytes = kLayerChunks * kWChunk;
constexpr uint32_t kTAcc = 0, kTX = 256, kTXt = 384, kTZ = 448;
}  // namespace fold

// mbarrier waits of the folded chain trap after ~4 s (2^33 cycles) instead of hanging the GPU
__device__ __forceinline__ void fwait(uint64_t* bar, uint32_t parity) {
  if (mbar_test(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_test(bar, parity))
    if (clock64() - t0 > (1ll << 33)) __trap();
}
__device__ __forceinline__ void fwait_cluster(uint64_t* bar, uint32_t parity) {
  const long long t0 = clock64();
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (!done && clock64() - t0 > (1ll << 33)) __trap();
  }
}

// Barriers whose phases a waiter could otherwise see two ahead of the one it waits for (a
// parity wait cannot tell phase k from k + 2) come in pairs indexed by the event's parity:
// event k completes phase k >> 1 of bar[k & 1], and the dependency structure keeps event k + 2
// behind every wait for event k.
__device__ __forceinline__ void wait_event(uint64_t* pair, int k) {
  if (k >= 0) fwait(pair + (k & 1), (uint32_t)(k >> 1) & 1);
}
// residual MMAs (layers with l >= 1) up to and including global layer g
__device__ __forceinline__ int res_layers_upto(int g, int L) { return g - g / L; }
// z halves sent to the peer before global layer g (every layer but each step's top one)
__device__ __forceinline__ int sends_before(int g, int L) { return g - g / L; }

// trace slots (CTA 0, clock64; tools/trace_fold.py): MMA 0 acc_free 1 pop 2 xt 3 zown 4 zpeer
// 5 acc_full committed 6 x_full committed; gate 8 acc_full seen 9 ld 10 math 11 own-image wait
// 12 zown arrive 13 send wait 14 sent; x 16 x_full seen 17 xt arrive; publisher 20 zown seen 21
// released; producer 24 layer start 25 after pop
#define FT(slot) trace_at(a, l, slot, clock64())
__device__ __forceinline__ void chain_fold_role(const ChainArgs& a, uint8_t* smem) {
  using namespace fold;
  const int tile = (int)blockIdx.x >> 1, half = (int)(blockIdx.x & 1);
  const uint32_t peer = (uint32_t)(half ^ 1);
  const int L = a.L, G = a.n_steps * L;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* wfull = bars;            // [6]
  uint64_t* wempty = bars + 6;       // [6]
  uint64_t* pop_full = bars + 12;    // [2] tx: ring slot of layer g in pop buffer g & 1
  uint64_t* pop_empty = bars + 14;   // [2] commit: xd(g) has read pop buffer g & 1
  uint64_t* acc_full = bars + 16;    // commit per layer
  uint64_t* acc_free = bars + 17;    // [2] 256 gate threads: acc[g & 1] of layer g read out
  uint64_t* x_full = bars + 19;      // [2] commit per residual MMA (event k = k-th residual)
  uint64_t* xt_ready = bars + 21;    // [2] 128 x threads: fp16 x operand of layer g written
  uint64_t* zown_ready = bars + 23;  // [2] 256 gate threads: own z half of layer g in zown[g & 1]
  uint64_t* zpeer_full = bars + 25;  // [2] tx: the peer's z half of send s in zpeer[s & 1]
  uint64_t* stage_free = bars + 27;  // [2] publisher: zown[b]'s stash store has read it
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 29);
  uint8_t* wring = smem + kOffW;
  uint8_t* popb = smem + kOffPop;
  uint8_t* zown = smem + kOffZo;
  uint8_t* zpeer = smem + kOffZp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 17; ++i) mbar_init(bars + i, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_free + b, 256);
      mbar_init(x_full + b, 1);
      mbar_init(xt_ready + b, 128);
      mbar_init(zown_ready + b, 256);
      mbar_init(zpeer_full + b, 1);
      mbar_init(stage_free + b, 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync();  // both CTAs' barriers exist before any z crosses
  const uint32_t tmem = *tmem_holder;
  // the tile's ring slot of layer l at step i (both halves' rows, all 16 K-pieces)
  auto slot_of = [&](int g) -> uint8_t* {
    return a.queue + qbase_of(a, g / L, g % L) + (size_t)tile * kSlot;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---- producer: weight chunks in MMA order; ring pops ----
      int wq = 0;
      auto put = [&](const uint8_t* src) {
        const int st = wq % fold::kWStages;
        fwait(wempty + st, ((uint32_t)(wq / fold::kWStages) & 1) ^ 1);
        mbar_arrive_expect_tx(wfull + st, kWChunk);
        bulk_g2s(wring + st * kWChunk, src, kWChunk, wfull + st);
        ++wq;
      };
      auto pop = [&](int g) {
        const int b = g & 1;
        if (g >= 2) fwait(pop_empty + b, (uint32_t)((g >> 1) - 1) & 1);
        // the slot's rows were pushed (generic-proxy stores) at least one step ago
        fence_proxy_async_all();
        mbar_arrive_expect_tx(pop_full + b, kSlot);
        bulk_g2s(popb + b * kSlot, slot_of(g), kSlot, pop_full + b);
      };
      pop(0);
      if (G > 1) pop(1);
      for (int g = 0; g < G; ++g) {
        const int l = g % L;
        const uint8_t* wl = a.w + (size_t)l * fold::kLayerBytes;
        FT(24);
        put(wl + (0 + 2 * half) * kWChunk);      // W1, K-chunk 0
        put(wl + (1 + 2 * half) * kWChunk);      // W1, K-chunk 1
        put(wl + (4 + 2 * half) * kWChunk);      // W0, K-chunk 0
        put(wl + (5 + 2 * half) * kWChunk);      // W0, K-chunk 1
        if (l > 0) {
          put(wl + (8 + 2 * half + half) * kWChunk);        // WF, own K-chunk
          put(wl + (12 + half) * kWChunk);                  // Wr_{l-1}, own K-chunk
          put(wl + (8 + 2 * half + (1 - half)) * kWChunk);  // WF, peer K-chunk
          put(wl + (12 + 1 - half) * kWChunk);              // Wr_{l-1}, peer K-chunk
        }
        if (g + 2 < G) pop(g + 2);
        FT(25);
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer ----
    const uint32_t id = idesc_f16(128, 128);
    const uint32_t sw = smem_u32(wring), sp = smem_u32(popb), szp = smem_u32(zpeer);
    int wq = 0;
    // one weight K-chunk (64 K = 4 MMAs), A from `amake(kk)`
    auto chunk = [&](uint32_t d, auto amake, bool first_init) {
      const int st = wq % fold::kWStages;
      fwait(wfull + st, (uint32_t)(wq / fold::kWStages) & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) amake(d, kk, sdesc_sw128(sw + st * kWChunk + kk * 32), id,
                                            (first_init && kk == 0) ? 0u : 1u);
        mma_commit(wempty + st);
      }
      __syncwarp();
      ++wq;
    };
    auto ss = [](uint32_t base) {
      return [base](uint32_t d, int kk, uint64_t b, uint32_t idd, uint32_t acc) {
        mma_bf16(d, sdesc_plain(base + (uint32_t)kk * 4096, 2048, 128), b, idd, acc);
      };
    };
    auto ts = [](uint32_t col) {
      return [col](uint32_t d, int kk, uint64_t b, uint32_t idd, uint32_t acc) {
        mma_bf16_ta(d, col + (uint32_t)kk * 8, b, idd, acc);
      };
    };
    for (int g = 0; g < G; ++g) {
      const int l = g % L;
      const uint32_t acc = tmem + kTAcc + 128u * (uint32_t)(g & 1);
      wait_event(acc_free, g - 2);  // gate(g-2) read acc[g & 1]
      if (lane == 0) FT(0);
      // x_{t-d} taps: A = the popped slot (K-pieces 0..7 | 8..15)
      fwait(pop_full + (g & 1), (uint32_t)(g >> 1) & 1);
      if (lane == 0) FT(1);
      tc_fence_after();
      const uint32_t pb = sp + (uint32_t)(g & 1) * kSlot;
      chunk(acc, ss(pb), true);
      chunk(acc, ss(pb + 8 * 2048), false);
      if (elect_one()) mma_commit(pop_empty + (g & 1));
      __syncwarp();
      // x_t taps on x_{l-1} (l = 0: on x_0 itself), A = the fp16 x operand in TMEM
      wait_event(xt_ready, l == 0 ? g : g - 1);
      if (lane == 0) FT(2);
      tc_fence_after();
      chunk(acc, ts(tmem + kTXt), false);
      chunk(acc, ts(tmem + kTXt + 32), false);
      if (l > 0) {
        const int gz = g - 1;  // z_{l-1}
        wait_event(zown_ready, gz);
        if (lane == 0) FT(3);
        tc_fence_after();
        chunk(acc, ts(tmem + kTZ), false);
        // x_l = x_{l-1} + Wr_{l-1} z_{l-1} (fp32, TMEM): own half now, peer half below
        chunk(tmem + kTX, ts(tmem + kTZ), false);
        const int s = sends_before(gz, L), zb = s & 1;
        if (elect_one()) mbar_arrive_expect_tx(zpeer_full + zb, kZHalf);
        __syncwarp();
        // cluster-scope acquire of the peer's st.async writes, then generic -> async proxy
        fwait_cluster(zpeer_full + zb, (uint32_t)(s >> 1) & 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (lane == 0) FT(4);
        tc_fence_after();
        const uint32_t zp = szp + (uint32_t)zb * kZHalf;
        chunk(acc, ss(zp), false);
        if (elect_one()) mma_commit(acc_full);
        __syncwarp();
        if (lane == 0) FT(5);
        chunk(tmem + kTX, ss(zp), false);
        if (elect_one()) mma_commit(x_full + ((res_layers_upto(g, L) - 1) & 1));
        __syncwarp();
        if (lane == 0) FT(6);
      } else {
        if (elect_one()) mma_commit(acc_full);
        __syncwarp();
      }
    }
  } else if (warp >= 2 && warp < 10) {  // ---- gate ----
    const int q = warp & 3, cs = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t szo = smem_u32(zown);
    for (int g = 0; g < G; ++g) {
      const int l = g % L;
      fwait(acc_full, (uint32_t)g & 1);
      const bool tr = warp == 2 && lane == 0;
      if (tr) FT(8);
      tc_fence_after();
      float v[64];  // tanh columns 32cs.. | sigmoid columns 64 + 32cs..
      const uint32_t acc = trow + kTAcc + 128u * (uint32_t)(g & 1);
      tmem_ld32x2(acc + 32 * cs, acc + 64 + 32 * cs, v);
      tc_fence_before();
      mbar_arrive(acc_free + (g & 1));
      if (tr) FT(9);
      if (a.has_dil_bias) {
        const float4* bt = reinterpret_cast<const float4*>(a.dil_b + (size_t)l * 256 + 64 * half + 32 * cs);
        const float4* bs = reinterpret_cast<const float4*>(a.dil_b + (size_t)l * 256 + 128 + 64 * half + 32 * cs);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 x = __ldg(bt + j), y = __ldg(bs + j);
          v[4 * j] += x.x; v[4 * j + 1] += x.y; v[4 * j + 2] += x.z; v[4 * j + 3] += x.w;
          v[32 + 4 * j] += y.x; v[33 + 4 * j] += y.y; v[34 + 4 * j] += y.z; v[35 + 4 * j] += y.w;
        }
      }
      uint32_t zw[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) zw[j] = gate2_h2(v[2 * j], v[2 * j + 1], v[32 + 2 * j], v[33 + 2 * j]);
      // own image reuse: layer g-2's z was read by the MMAs of layer g-1 (x_full of g-1) and
      // by its stash store; the peer's image of this send was read by the peer's layer g-1,
      // which only ran after this CTA's send of layer g-1 -- sent after x_full of g-1 here.
      // Waiting for x_full of layer g itself before the send orders this CTA's reads of the
      // peer's z_{l-1} (res of layer g) before the peer's next send into that buffer.
      if (tr) {
        asm volatile("" ::"r"(zw[0]), "r"(zw[15]) : "memory");
        FT(10);
      }
      if (g >= 2) fwait(stage_free + (g & 1), (uint32_t)(((g >> 1) - 1) & 1));
      if (g > 0) wait_event(x_full, res_layers_upto(g - 1, L) - 1);
      if (tr) FT(11);
      const uint32_t zdst = szo + (uint32_t)(g & 1) * kZHalf + (uint32_t)r * 16;
#pragma unroll
      for (int m = 0; m < 4; ++m)
        st_shared_v4(zdst + (uint32_t)(4 * cs + m) * 2048, zw[4 * m], zw[4 * m + 1], zw[4 * m + 2],
                     zw[4 * m + 3]);
      // the own half's MMA operand (TMEM; its readers of layer g-1 finished before acc_full)
      tmem_st16(trow + kTZ + 16 * cs, *reinterpret_cast<const float(*)[16]>(zw));
      fence_proxy_async();  // generic shared writes -> bulk-store reads
      tc_fence_before();
      mbar_arrive(zown_ready + (g & 1));
      if (tr) FT(12);
      if (l + 1 < L) {  // the peer's WF / res of layer g+1 read this half
        wait_event(x_full, res_layers_upto(g, L) - 1);
        if (tr) FT(13);
        const int s = sends_before(g, L), zb = s & 1;
        const uint32_t pbar = mapa(zpeer_full + zb, peer);
        const uint32_t pdst = mapa(zpeer + zb * kZHalf, peer) + (uint32_t)r * 16;
#pragma unroll
        for (int m = 0; m < 4; ++m)
          asm volatile(
              "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(
                  pdst + (uint32_t)(4 * cs + m) * 2048),
              "r"(zw[4 * m]), "r"(zw[4 * m + 1]), "r"(zw[4 * m + 2]), "r"(zw[4 * m + 3]), "r"(pbar)
              : "memory");
        if (tr) FT(14);
      }
    }
  } else if (warp >= 10 && warp < 14) {  // ---- x: residual stream -> fp16 operand + push ----
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    for (int g = 0; g < G; ++g) {
      const int i = g / L, l = g % L;
      const float4* src4 = nullptr;  // l = 0: the embedding row of the input class
      if (l == 0) {
        // the previous step's top-layer residual MMA is done with TMEM x
        if (g > 0) wait_event(x_full, res_layers_upto(g - 1, L) - 1);
        if (i > 0) wait_counter(a.cls_ready + tile, (uint32_t)i);
        const int c = clamp_class(a.cls[tile * 128 + r], 256);
        src4 = reinterpret_cast<const float4*>(a.embed + (size_t)c * kR);
      } else {
        wait_event(x_full, res_layers_upto(g, L) - 1);
        if (warp == 10 && lane == 0) FT(16);
        tc_fence_after();
      }
      // 64 channels at a time, the peer's half first: x (fp32, TMEM) -> fp16 operand columns
      // (TMEM); then, after the release, the push of this half's 8 K-pieces of row r (the
      // slot's pop for this step was read by xd(g), ahead of this layer's x_full)
      uint32_t w[32];
#pragma unroll 1
      for (int k = 0; k < 2; ++k) {
        const int hh = k == 0 ? 1 - half : half;
        float x[64];
        if (l == 0) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float4 e = __ldg(src4 + 16 * hh + j);
            x[4 * j] = e.x; x[4 * j + 1] = e.y; x[4 * j + 2] = e.z; x[4 * j + 3] = e.w;
          }
          tmem_st32(trow + kTX + 64 * hh, *reinterpret_cast<float(*)[32]>(x));
          tmem_st32(trow + kTX + 64 * hh + 32, *reinterpret_cast<float(*)[32]>(x + 32));
        } else {
          tmem_ld64(trow + kTX + 64 * hh, x);
          if (a.has_res_bias) {
            const float4* b4 = reinterpret_cast<const float4*>(a.res_b + (size_t)(l - 1) * kR + 64 * hh);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float4 b = __ldg(b4 + j);
              x[4 * j] += b.x; x[4 * j + 1] += b.y; x[4 * j + 2] += b.z; x[4 * j + 3] += b.w;
            }
            tmem_st32(trow + kTX + 64 * hh, *reinterpret_cast<float(*)[32]>(x));
            tmem_st32(trow + kTX + 64 * hh + 32, *reinterpret_cast<float(*)[32]>(x + 32));
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) w[j] = pack_h2(x[2 * j], x[2 * j + 1]);
        tmem_st32(trow + kTXt + 32 * hh, *reinterpret_cast<float(*)[32]>(w));
      }
      tc_fence_before();
      mbar_arrive(xt_ready + (g & 1));
      if (warp == 10 && lane == 0) FT(17);
      uint4* dst = reinterpret_cast<uint4*>(slot_of(g)) + r;
#pragma unroll
      for (int m = 0; m < 8; ++m)
        dst[(size_t)(8 * half + m) * 128] = make_uint4(w[4 * m], w[4 * m + 1], w[4 * m + 2], w[4 * m + 3]);
    }
  } else if (warp == 14) {  // ---- publisher: own z half -> the z stash -> the tail ----
    if (lane == 0) {
      for (int g = 0; g < G; ++g) {
        const int l = g % L;
        wait_event(zown_ready, g);
        FT(20);
        if (a.zfree != nullptr && g >= a.zring)
          wait_counter(a.zfree + tile, (uint32_t)a.ztail * (uint32_t)(g - a.zring + 1));
        uint8_t* dst = const_cast<uint8_t*>(zstash_tile(a, tile, g)) + half * kZHalf;
        bulk_s2g(dst, zown + (g & 1) * kZHalf, kZHalf);
        bulk_commit();
        bulk_wait0();             // in the stash (not just read out of SMEM)
        fence_proxy_async_all();  // async-proxy writes before the release
        red_release_gpu(a.zflag + tile, 1u);
        mbar_arrive(stage_free + (g & 1));
        FT(21);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync();  // no DSMEM traffic into a CTA that has exited
  if (warp == 1) tmem_dealloc(tmem, 512);
}
#undef FT
