// 2-SM chain of the tcgen05 step kernel (included by chain_tc.cuh): the two 64-stream tiles
// of a tile pair run as one 2-CTA cluster whose MMAs are 2-SM `tcgen05.mma.cta_group::2`
// (M = 128: 64 rows per CTA), issued by rank 0 for both. Each CTA holds the rows of its own
// tile and HALF of every weight operand (N split across the pair, read by the MMA from both
// CTAs' shared memory): per layer 80 KB of weight stages per CTA instead of 160 KB, and an
// M = 128, N = 128 K-step costs ~33 cycles against ~75 for the 1-SM M = 64 MMA of chain_tc.cuh
// (tools/cg2_probe.cu). Same per-layer structure as chain_tc.cuh (x_{t-d} and x_t taps ->
// gate -> residual), same ring, z stash and tail interface.
//
//   D layout (tools/cg2_probe.cu): CTA r's TMEM lane l < 64 holds its row l x the first N/2
//   columns, lane 64 + l the same row x the last N/2. The dilated weights are arranged so each
//   N = 128 half's lane groups pair gate inputs: lanes 0-63 get tanh | sigmoid of channels
//   64h + [0, 32), lanes 64-127 those of 64h + [32, 64) (CTA 0 holds the B rows of the
//   former, CTA 1 of the latter).
//   TMEM: [0,64) acc0 | [64,128) acc1 | [128,192) x (fp32 residual, channels 0-63 in lanes
//   0-63, 64-127 in lanes 64-127).
//   SMEM (A operands no-swizzle K-major [16 K-pieces][64 rows][16 B], B stages SW128):
//   4-stage ring of 32 KB weight stages (per layer: x_{t-d} taps | x_t taps | residual) |
//   2 x 16 KB pops | x_t operand 16 KB | 2 x 16 KB z
//   (the residual MMA's A operand and the z stash's source) | barriers.
//
//   warp 0 lane 0: producer (this CTA's halves, in MMA order); warp 15 lane 0 of rank 1:
//   relay (the stage's arrival -> rank 0's full barrier); warp 1 of rank 0: MMA issuer;
//   warps 2..9: gate (quadrant q, N-half (warp - 2) / 4); warps 10..13: x conversion, ring
//   push / pop, embedding; warp 14 lane 0: z stash publisher.
namespace c2 {
constexpr uint32_t kHalfW = 16384;   // one N-half of one weight matrix: [64 n][128 k] SW128
constexpr uint32_t kStage = 32768;   // per layer: x_{t-d} taps (2 halves) | x_t taps | residual
constexpr int kStages = 4;
constexpr int kLayerCopies = 3;
constexpr uint32_t kOp = 16384;      // one 64-row fp16 operand [16 pieces][64 rows][16 B]
constexpr uint32_t kOffW = 0;
constexpr uint32_t kOffPop = kOffW + kStages * kStage;  // 128 KB
constexpr uint32_t kOffXt = kOffPop + 2 * kOp;           // 160 KB
constexpr uint32_t kOffZ = kOffXt + kOp;                 // 176 KB
constexpr uint32_t kOffBar = kOffZ + 2 * kOp;            // 208 KB
constexpr size_t kSmem = 1024 + kOffBar + 512;
constexpr int kLayerStages = 5;  // image per CTA per layer: W1 h0 | W1 h1 | W0 h0 | W0 h1 | res
constexpr uint32_t kLayerBytes = 2 * kLayerStages * kHalfW;  // both CTAs' halves (160 KB)
constexpr uint32_t kTAcc0 = 0, kTAcc1 = 64, kTX = 128;
// folded variant: acc[2] at [0,128) | [128,256) (N-half h at + 64h), x at [256,320); image per
// layer per CTA: W1 h0 | W1 h1 | W0 h0 | W0 h1 | WF h0 | WF h1 | residual
constexpr uint32_t kTXF = 256;
constexpr int kLayerStagesF = 7;
constexpr uint32_t kLayerBytesF = 2 * kLayerStagesF * kHalfW;
}  // namespace c2

__device__ __forceinline__ void mma_cg2(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
// Remote arrive without a release fence: `.release.cluster` compiles to MEMBAR.ALL.GPU, which
// took ~0.9 us here (it waits for the thread's in-flight memory traffic). The data these
// arrivals cover (shared-memory operands, TMA-filled stages) is complete in the sender's
// shared memory before the arrive (CTA-scope barrier / complete_tx observed, proxy fence).
__device__ __forceinline__ void arrive_remote_relaxed(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr)
               : "memory");
}
// commit to the barrier at this smem offset in both CTAs of the pair
__device__ __forceinline__ void commit_cg2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// trace (pair 0, globaltimer ns, comparable across the two SMs): layer row slots 40 + 4 r + k,
// k = 0 x_full seen, 1 xt arrive, 2 z0 arrive, 3 acc0 seen
__device__ __forceinline__ void tr2(const ChainArgs& a, int l, int k) {
  if (a.trace != nullptr && blockIdx.x == 0) a.trace[l * kTraceSlots + 40 + k] = globaltimer_ns();
}
__device__ __forceinline__ void tr3(const ChainArgs& a, int l, int k) {  // either CTA of pair 0
  if (a.trace != nullptr && blockIdx.x < 2) a.trace[l * kTraceSlots + 32 + k] = globaltimer_ns();
}
__device__ __forceinline__ void chain_2sm_role(const ChainArgs& a, uint8_t* smem) {
  using namespace c2;
  // the pair's 2-SM MMAs need the cluster launch (a replay that dropped it, as ncu's, stops
  // here instead of issuing cta_group::2 instructions without a peer)
  if (cluster_size() != 2) __trap();
  const int tile = (int)blockIdx.x;
  const uint32_t rank = (uint32_t)(tile & 1);
  const bool leader = rank == 0;
  const int L = a.L, G = a.n_steps * L;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* wfull = bars;            // [8] leader: own tx + the relay's arrive; rank 1: own tx
  uint64_t* wempty = bars + 8;       // [8] MMA commit (both CTAs)
  uint64_t* acc0_full = bars + 16;   // MMA commit (both)
  uint64_t* acc1_full = bars + 17;
  uint64_t* x_full = bars + 18;      // MMA commit per layer (both)
  uint64_t* xd_ready = bars + 20;    // leader: 8 warp arrivals (4 local, 4 remote)
  uint64_t* xt_ready = bars + 21;    // leader: 8
  uint64_t* z_ready = bars + 22;     // [2] leader: 8 per N-half
  uint64_t* z_local = bars + 24;     // 8 local gate warps: this CTA's z of layer g written
  uint64_t* stage_free = bars + 25;  // [2] publisher: z buffer b's stash store has read it
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 27);
  uint8_t* wring = smem + kOffW;
  uint8_t* popb = smem + kOffPop;
  uint8_t* xtb = smem + kOffXt;
  uint8_t* zb = smem + kOffZ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(wfull + i, leader ? 2 : 1);
      mbar_init(wempty + i, 1);
    }
    for (int i = 16; i < 19; ++i) mbar_init(bars + i, 1);
    // (rank 1's queue warps arrive locally; its idle MMA warp forwards one remote arrive:
    // a remote release issued by the queue warps themselves waited for their in-flight pops)
    mbar_init(xd_ready, leader ? 5 : 4);
    mbar_init(xt_ready, leader ? 5 : 4);
    mbar_init(z_ready + 0, 8);
    mbar_init(z_ready + 1, 8);
    mbar_init(z_local, 8);
    mbar_init(stage_free + 0, 1);
    mbar_init(stage_free + 1, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' barriers and TMEM exist before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // a warp's "this operand is ready" arrival on the leader's barrier (local or remote)
  auto warp_arrive_leader = [&](uint64_t* bar) {
    __syncwarp();
    if (lane == 0) {
      if (leader) mbar_arrive(bar);
      else arrive_remote_relaxed(mapa(bar, 0));
    }
  };
  uint8_t* qtile = a.queue + (size_t)(tile >> 1) * 2 * kSlotBytes + (size_t)rank * 64 * 16;

  if (warp == 0) {
    if (lane == 0) {  // ---- producer: this CTA's weight halves, in MMA order ----
      int wq = 0;
      for (int g = 0; g < G; ++g) {
        const uint8_t* wl = a.w + (size_t)(g % L) * c2::kLayerBytes + (size_t)rank * c2::kLayerStages * c2::kHalfW;
        for (int s = 0; s < kLayerCopies; ++s, ++wq) {
          const int st = wq % kStages;
          const uint32_t bytes = s < 2 ? kStage : kHalfW;
          mbar_wait_cluster(wempty + st, ((uint32_t)(wq / c2::kStages) & 1) ^ 1);
          mbar_arrive_expect_tx(wfull + st, bytes);
          bulk_g2s(wring + st * kStage, wl + (size_t)s * kStage, bytes, wfull + st);
        }
      }
    }
  } else if (warp == 15) {
    if (lane == 0 && !leader) {  // ---- relay: rank 1's stage landed -> rank 0's full barrier
      const int nst = G * kLayerCopies;
      for (int wq = 0; wq < nst; ++wq) {
        const int st = wq % kStages;
        mbar_wait(wfull + st, (uint32_t)(wq / kStages) & 1);
        arrive_remote_relaxed(mapa(wfull + st, 0));
      }
    }
  } else if (warp == 1 && !leader) {
    // ---- rank 1's relay of its queue warps' operand-ready events to rank 0 ----
    if (lane == 0) {
      auto fwd = [&](uint64_t* bar, int k) {
        mbar_wait(bar, (uint32_t)k & 1);
        arrive_remote_relaxed(mapa(bar, 0));
      };
      fwd(xd_ready, 0);
      for (int g = 0; g < G; ++g) {
        mbar_wait(xt_ready, (uint32_t)g & 1);
        tr3(a, g % L, 0);
        fwd(xt_ready, g);
        tr3(a, g % L, 1);
        if (g + 1 < G) fwd(xd_ready, g + 1);
      }
    }
  } else if (warp == 1) {
    {  // ---- MMA issuer (rank 0; converged warp, elect.sync) ----
      const uint32_t id = idesc_f16(128, 128);
      const uint32_t sw = smem_u32(wring), sp = smem_u32(popb), sx = smem_u32(xtb), sz = smem_u32(zb);
      int wq = 0;
      auto stage_wait = [&]() -> uint32_t {
        const int st = wq % kStages;
        mbar_wait_cluster(wfull + st, (uint32_t)(wq / kStages) & 1);  // (+ rank 1's relay)
        tc_fence_after();
        return sw + (uint32_t)st * kStage;
      };
      auto stage_done = [&]() {
        if (elect_one()) commit_cg2(wempty + (wq % kStages));
        __syncwarp();
        ++wq;
      };
      // K-chunk c (64 K) of an A operand in the [16 pieces][64 rows][16 B] layout x one
      // weight stage (B: 2 K-chunks of SW128 [64 n][64 k]), 4 MMAs of K = 16
      auto kchunk = [&](uint32_t d, uint32_t aop, int c, uint32_t bst, bool init) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_cg2(d, sdesc_plain(aop + (uint32_t)(8 * c + 2 * kk) * 1024, 1024, 128),
                  sdesc_sw128(bst + (uint32_t)c * 8192 + kk * 32), id, (init && kk == 0) ? 0u : 1u);
      };
      for (int g = 0; g < G; ++g) {
        const int l = g % L;
        const uint32_t par = (uint32_t)g & 1;
        // x_{t-d} taps (initialise both accumulators); A = the popped slot
        mbar_wait_cluster(xd_ready, par);
        if (lane == 0) {
          trace_at(a, l, T_MMA_XD, clock64());
          tr2(a, l, 4);
        }
        tc_fence_after();
        const uint32_t pa = sp + par * kOp;
        {  // one stage: both N-halves' x_{t-d} taps; its release is also the pops' "free"
          const uint32_t bst = stage_wait();
          if (lane == 0) tr3(a, l, 3);
          if (elect_one()) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              kchunk(tmem + (h ? kTAcc1 : kTAcc0), pa, 0, bst + h * kHalfW, true);
              kchunk(tmem + (h ? kTAcc1 : kTAcc0), pa, 1, bst + h * kHalfW, false);
            }
          }
          __syncwarp();
          if (lane == 0) tr3(a, l, 4);
          stage_done();
        }
        if (lane == 0) tr3(a, l, 2);
        // x_t taps, N-half 0 then 1
        mbar_wait_cluster(xt_ready, par);
        if (lane == 0) {
          trace_at(a, l, T_MMA_XT, clock64());
          tr2(a, l, 5);
        }
        tc_fence_after();
        {
          const uint32_t bst = stage_wait();
          if (lane == 0) tr2(a, l, 6);
          if (elect_one()) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              kchunk(tmem + (h ? kTAcc1 : kTAcc0), sx, 0, bst + h * kHalfW, false);
              kchunk(tmem + (h ? kTAcc1 : kTAcc0), sx, 1, bst + h * kHalfW, false);
              commit_cg2(h ? acc1_full : acc0_full);
            }
          }
          __syncwarp();
          stage_done();
        }
        // residual: x += W_res z, K-chunk h once both CTAs' z of N-half h are written
        const uint32_t bst = stage_wait();
        const uint32_t za = sz + par * kOp;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          mbar_wait_cluster(z_ready + h, par);
          if (lane == 0) {
            trace_at(a, l, h ? T_MMA_Z1 : T_MMA_Z0, clock64());
            if (h == 0) tr2(a, l, 7);
          }
          tc_fence_after();
          if (l + 1 < L && elect_one()) kchunk(tmem + kTX, za, h, bst, false);
          __syncwarp();
        }
        stage_done();
        if (elect_one()) commit_cg2(x_full);  // (every layer: it also covers the x_t reads)
        __syncwarp();
        if (lane == 0) trace_at(a, l, T_MMA_XFULL, clock64());
      }
    }
  } else if (warp >= 2 && warp < 10) {  // ---- gate ----
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int rho = 32 * (q & 1) + lane, cb = q >> 1;  // row, channel block (32 channels)
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t szb = smem_u32(zb);
    const bool tr = warp == 2 && lane == 0;
    for (int g = 0; g < G; ++g) {
      const int l = g % L;
      const uint32_t par = (uint32_t)g & 1;
      // (the arrivals are the tensor core's commit: a CTA-scope wait, no L1 invalidation)
      mbar_wait(h ? acc1_full : acc0_full, par);
      tc_fence_after();
      if (tr) trace_at(a, l, h ? T_EPI_ACC1 : T_EPI_ACC0, clock64());
      if (warp == 2 && lane == 0) tr2(a, l, 3);
      float v[64];  // tanh inputs of channels 64h + 32cb + j | sigmoid inputs
      tmem_ld32x2(trow + (h ? kTAcc1 : kTAcc0), trow + (h ? kTAcc1 : kTAcc0) + 32, v);
      tc_fence_before();
      if (a.has_dil_bias) {
        const float* bd = a.dil_b + (size_t)l * 2 * kD + 64 * h + 32 * cb;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          v[j] += __ldg(bd + j);
          v[32 + j] += __ldg(bd + kD + j);
        }
      }
      uint32_t zw[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) zw[j] = gate2_h2(v[2 * j], v[2 * j + 1], v[32 + 2 * j], v[33 + 2 * j]);
      // z buffer `par` was last read by layer g - 2's residual and stash (the residual: before
      // this layer's acc commits; the stash: stage_free)
      if (g >= 2) mbar_wait(stage_free + par, (uint32_t)(((g >> 1) - 1) & 1));
      const uint32_t zrow = szb + par * kOp + (uint32_t)rho * 16;
#pragma unroll
      for (int m = 0; m < 4; ++m)
        st_shared_v4(zrow + (uint32_t)(8 * h + 4 * cb + m) * 1024, zw[4 * m], zw[4 * m + 1], zw[4 * m + 2],
                     zw[4 * m + 3]);
      fence_proxy_async();  // generic shared writes -> the MMA / bulk-store reads
      warp_arrive_leader(z_ready + h);
      if (lane == 0) mbar_arrive(z_local);
      if (tr) trace_at(a, l, h ? T_EPI_Z1 : T_EPI_Z0, clock64());
      if (warp == 2 && lane == 0) tr2(a, l, 2);
    }
  } else if (warp >= 10 && warp < 14) {  // ---- x: conversion, push, pops, embedding ----
    const int q = warp & 3;
    const int rho = 32 * (q & 1) + lane, cb = q >> 1;  // row, channel block (64 channels)
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t sxrow = smem_u32(xtb) + (uint32_t)rho * 16;
    auto qb = [&](int g) { return qbase_of(a, g / L, g % L); };
    // pops: this thread's 8 K-pieces (channels 64cb..) of its row of layer g's slot -> pop
    // buffer g & 1 (cp.async; the same thread pushed those bytes)
    auto load_slot = [&](int g) {
      const uint8_t* src = qtile + qb(g) + (size_t)rho * 16;
      const uint32_t dst = smem_u32(popb + (g & 1) * kOp) + (uint32_t)rho * 16;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int pc = 8 * cb + j;
        cp_async16(dst + (uint32_t)pc * 1024, src + (size_t)pc * kPairRows * 16);
      }
      cp_async_commit();
    };
    auto local_arrive = [&](uint64_t* bar) {
      __syncwarp();
      if (lane == 0) mbar_arrive(bar);
    };
    auto xd_signal = [&]() {
      fence_proxy_async();
      local_arrive(xd_ready);
    };
    load_slot(0);
    if (G > 1) load_slot(1);
    else cp_async_commit();
    cp_async_wait<1>();
    xd_signal();
    for (int g = 0; g < G; ++g) {
      const int i = g / L, l = g % L;
      const uint32_t par = (uint32_t)g & 1;
      // x_l of this thread's row and channel block: the embedding at l = 0, else the residual
      // stream (TMEM) + its pending bias; the previous layer's MMAs are done with x and x_t
      if (g > 0) mbar_wait(x_full, par ^ 1);
      if (warp == 10 && lane == 0) {
        trace_at(a, l, T_EPI_A, clock64());
        tr2(a, l, 0);
      }
      tc_fence_after();
      float x[64];
      if (l == 0) {
        if (i > 0) wait_counter(a.cls_ready + (tile >> 1), (uint32_t)i);
        const int c = clamp_class(a.cls[tile * 64 + rho], 256);
        const float4* e4 = reinterpret_cast<const float4*>(a.embed + (size_t)c * kR + 64 * cb);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float4 e = __ldg(e4 + j);
          x[4 * j] = e.x; x[4 * j + 1] = e.y; x[4 * j + 2] = e.z; x[4 * j + 3] = e.w;
        }
        tmem_st32(trow + kTX, *reinterpret_cast<float(*)[32]>(x));
        tmem_st32(trow + kTX + 32, *reinterpret_cast<float(*)[32]>(x + 32));
      } else {
        tmem_ld64(trow + kTX, x);
        if (a.has_res_bias) {
          const float* rb = a.res_b + (size_t)(l - 1) * kR + 64 * cb;
#pragma unroll
          for (int j = 0; j < 64; ++j) x[j] += __ldg(rb + j);
          tmem_st32(trow + kTX, *reinterpret_cast<float(*)[32]>(x));
          tmem_st32(trow + kTX + 32, *reinterpret_cast<float(*)[32]>(x + 32));
        }
      }
      tc_fence_before();
      uint32_t w[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) w[j] = pack_h2(x[2 * j], x[2 * j + 1]);
#pragma unroll
      for (int m = 0; m < 8; ++m)
        st_shared_v4(sxrow + (uint32_t)(8 * cb + m) * 1024, w[4 * m], w[4 * m + 1], w[4 * m + 2], w[4 * m + 3]);
      fence_proxy_async();
      local_arrive(xt_ready);
      if (warp == 10 && lane == 0) {
        trace_at(a, l, T_EPI_XT, clock64());
        tr2(a, l, 1);
      }
      // push x_l: this thread's 8 K-pieces of its row into ring slot t mod d_l (its pop was
      // read two layers ago by this thread)
      uint4* dst = reinterpret_cast<uint4*>(qtile + qb(g)) + rho;
#pragma unroll
      for (int m = 0; m < 8; ++m)
        dst[(size_t)(8 * cb + m) * kPairRows] = make_uint4(w[4 * m], w[4 * m + 1], w[4 * m + 2], w[4 * m + 3]);
      // the pop of layer g + 2 into the buffer layer g's x_{t-d} MMAs have finished with
      if (g + 1 < G) {
        // layer g's x_{t-d} MMAs are done with pop buffer g & 1: the release of its weight
        // stage (stage 3g of the ring)
        mbar_wait(wempty + (3 * g) % kStages, (uint32_t)((3 * g) / kStages) & 1);
        if (g + 2 < G) load_slot(g + 2);
        else cp_async_commit();
        cp_async_wait<1>();  // layer g + 1's pop
        xd_signal();
      }
    }
  } else if (warp == 14) {  // ---- publisher: this CTA's 64 rows of z_l -> the stash ----
    if (lane == 0) {
      for (int g = 0; g < G; ++g) {
        mbar_wait(z_local, (uint32_t)g & 1);
        if (a.zfree != nullptr && g >= a.zring)
          wait_counter(a.zfree + (tile >> 1), (uint32_t)a.ztail * (uint32_t)(g - a.zring + 1));
        uint8_t* dst = reinterpret_cast<uint8_t*>(zstash_rows(a.zimg, tile, a.zring, g % a.zring));
        const uint8_t* src = zb + (g & 1) * kOp;
        for (int j = 0; j < 16; ++j) bulk_s2g(dst + j * 2048, src + j * 1024, 1024);
        bulk_commit();
        bulk_wait0();             // in the stash
        fence_proxy_async_all();  // async-proxy writes before the release
        red_release_gpu(a.zflag + (tile >> 1), 1u);
        mbar_arrive(stage_free + (g & 1));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no DSMEM traffic or 2-SM MMA into a CTA that has exited
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// The 2-SM chain with the residual folded into the next layer's taps (FW_CHAIN_2SM=2):
// a_l = W1 x_l[t-d] + W0 x_{l-1} + (W0_l Wr_{l-1}) z_{l-1} + b', so the dependent path per
// layer is z -> 16 MMAs (WF) -> gate; x_{l-1} (the residual MMA + conversion) comes a layer
// early. Per layer and CTA 4 weight stages: x_{t-d} taps | x_t taps | WF | residual.
__device__ __forceinline__ void chain_2sf_role(const ChainArgs& a, uint8_t* smem) {
  using namespace c2;
  // the pair's 2-SM MMAs need the cluster launch (a replay that dropped it, as ncu's, stops
  // here instead of issuing cta_group::2 instructions without a peer)
  if (cluster_size() != 2) __trap();
  const int tile = (int)blockIdx.x;
  const uint32_t rank = (uint32_t)(tile & 1);
  const bool leader = rank == 0;
  const int L = a.L, G = a.n_steps * L;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* wfull = bars;            // [8] leader: own tx + the relay's arrive; rank 1: own tx
  uint64_t* wempty = bars + 8;       // [8] MMA commit (both CTAs)
  uint64_t* acc0_full = bars + 16;   // MMA commit (both)
  uint64_t* acc1_full = bars + 17;
  uint64_t* x_full = bars + 18;      // MMA commit per layer (both)
  uint64_t* xd_ready = bars + 20;    // leader: 8 warp arrivals (4 local, 4 remote)
  uint64_t* xt_ready = bars + 28;    // [2] by production parity: leader 5, rank 1 4
  uint64_t* z_ready = bars + 22;     // [2] leader: 8 per N-half
  uint64_t* z_local = bars + 24;     // 8 local gate warps: this CTA's z of layer g written
  uint64_t* stage_free = bars + 25;  // [2] publisher: z buffer b's stash store has read it
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 27);
  constexpr int kCopies = 4;  // per layer: W1 | W0 | WF (32 KB each) | residual (16 KB)
  uint8_t* wring = smem + kOffW;
  uint8_t* popb = smem + kOffPop;
  uint8_t* xtb = smem + kOffXt;
  uint8_t* zb = smem + kOffZ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(wfull + i, leader ? 2 : 1);
      mbar_init(wempty + i, 1);
    }
    for (int i = 16; i < 19; ++i) mbar_init(bars + i, 1);
    // (rank 1's queue warps arrive locally; its idle MMA warp forwards one remote arrive:
    // a remote release issued by the queue warps themselves waited for their in-flight pops)
    mbar_init(xd_ready, leader ? 5 : 4);
    mbar_init(xt_ready + 0, leader ? 5 : 4);
    mbar_init(xt_ready + 1, leader ? 5 : 4);
    mbar_init(z_ready + 0, 8);
    mbar_init(z_ready + 1, 8);
    mbar_init(z_local, 8);
    mbar_init(stage_free + 0, 1);
    mbar_init(stage_free + 1, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' barriers and TMEM exist before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // a warp's "this operand is ready" arrival on the leader's barrier (local or remote)
  auto warp_arrive_leader = [&](uint64_t* bar) {
    __syncwarp();
    if (lane == 0) {
      if (leader) mbar_arrive(bar);
      else arrive_remote_relaxed(mapa(bar, 0));
    }
  };
  uint8_t* qtile = a.queue + (size_t)(tile >> 1) * 2 * kSlotBytes + (size_t)rank * 64 * 16;

  if (warp == 0) {
    if (lane == 0) {  // ---- producer: this CTA's weight halves, in MMA order ----
      int wq = 0;
      for (int g = 0; g < G; ++g) {
        const uint8_t* wl = a.w + (size_t)(g % L) * c2::kLayerBytesF + (size_t)rank * c2::kLayerStagesF * c2::kHalfW;
        for (int s = 0; s < kCopies; ++s, ++wq) {
          const int st = wq % kStages;
          const uint32_t bytes = s < 3 ? kStage : kHalfW;
          mbar_wait_cluster(wempty + st, ((uint32_t)(wq / c2::kStages) & 1) ^ 1);
          mbar_arrive_expect_tx(wfull + st, bytes);
          bulk_g2s(wring + st * kStage, wl + (size_t)s * kStage, bytes, wfull + st);
        }
      }
    }
  } else if (warp == 15) {
    if (lane == 0 && !leader) {  // ---- relay: rank 1's stage landed -> rank 0's full barrier
      const int nst = G * kCopies;
      for (int wq = 0; wq < nst; ++wq) {
        const int st = wq % kStages;
        mbar_wait(wfull + st, (uint32_t)(wq / kStages) & 1);
        arrive_remote_relaxed(mapa(wfull + st, 0));
      }
    }
  } else if (warp == 1 && !leader) {
    // ---- rank 1's relay of its queue warps' operand-ready events to rank 0 ----
    if (lane == 0) {
      auto fwd = [&](uint64_t* bar, int k) {
        mbar_wait(bar, (uint32_t)k & 1);
        arrive_remote_relaxed(mapa(bar, 0));
      };
      fwd(xd_ready, 0);
      for (int g = 0; g < G; ++g) {
        mbar_wait(xt_ready + (g & 1), (uint32_t)(g >> 1) & 1);
        arrive_remote_relaxed(mapa(xt_ready + (g & 1), 0));
        if (g + 1 < G) fwd(xd_ready, g + 1);
      }
    }
  } else if (warp == 1) {
    {  // ---- MMA issuer (rank 0; converged warp, elect.sync) ----
      const uint32_t id = idesc_f16(128, 128);
      const uint32_t sw = smem_u32(wring), sp = smem_u32(popb), sx = smem_u32(xtb), sz = smem_u32(zb);
      int wq = 0;
      auto stage_wait = [&]() -> uint32_t {
        const int st = wq % kStages;
        mbar_wait_cluster(wfull + st, (uint32_t)(wq / kStages) & 1);  // (+ rank 1's relay)
        tc_fence_after();
        return sw + (uint32_t)st * kStage;
      };
      auto stage_done = [&]() {
        if (elect_one()) commit_cg2(wempty + (wq % kStages));
        __syncwarp();
        ++wq;
      };
      // K-chunk c (64 K) of an A operand in the [16 pieces][64 rows][16 B] layout x one
      // weight stage (B: 2 K-chunks of SW128 [64 n][64 k]), 4 MMAs of K = 16
      auto kchunk = [&](uint32_t d, uint32_t aop, int c, uint32_t bst, bool init) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_cg2(d, sdesc_plain(aop + (uint32_t)(8 * c + 2 * kk) * 1024, 1024, 128),
                  sdesc_sw128(bst + (uint32_t)c * 8192 + kk * 32), id, (init && kk == 0) ? 0u : 1u);
      };
      for (int g = 0; g < G; ++g) {
        const int l = g % L;
        const uint32_t par = (uint32_t)g & 1;
        const uint32_t accb = tmem + 128u * par;  // acc[g & 1]: N-half h at + 64 h
        // x_{t-d} taps (initialise acc[g & 1], last read by the gate of layer g - 2, whose
        // z the WF MMAs of layer g - 1 waited for); A = the popped slot
        mbar_wait_cluster(xd_ready, par);
        tc_fence_after();
        const uint32_t pa = sp + par * kOp;
        {
          const uint32_t bst = stage_wait();
          if (elect_one()) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              kchunk(accb + 64 * h, pa, 0, bst + h * kHalfW, true);
              kchunk(accb + 64 * h, pa, 1, bst + h * kHalfW, false);
            }
          }
          __syncwarp();
          stage_done();
        }
        // x_t taps on x_{l-1} (l = 0: on x_0, the embedding): production l == 0 ? g : g - 1
        {
          const int pr = l == 0 ? g : g - 1;
          mbar_wait_cluster(xt_ready + (pr & 1), (uint32_t)(pr >> 1) & 1);
          tc_fence_after();
          const uint32_t bst = stage_wait();
          if (elect_one()) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              kchunk(accb + 64 * h, sx, 0, bst + h * kHalfW, false);
              kchunk(accb + 64 * h, sx, 1, bst + h * kHalfW, false);
            }
          }
          __syncwarp();
          stage_done();
        }
        // z_{l-1} (both CTAs; layer 0: the previous step's top z, consumed unused)
        const uint32_t za = sz + (par ^ 1u) * kOp;
        {
          const uint32_t bst = stage_wait();  // WF
          if (g > 0) {
            mbar_wait_cluster(z_ready + 0, par ^ 1u);
            tc_fence_after();
            if (l > 0 && elect_one()) {
              kchunk(accb, za, 0, bst, false);
              kchunk(accb + 64, za, 0, bst + kHalfW, false);
            }
            __syncwarp();
            mbar_wait_cluster(z_ready + 1, par ^ 1u);
            tc_fence_after();
            if (l > 0 && elect_one()) {
              kchunk(accb, za, 1, bst, false);
              kchunk(accb + 64, za, 1, bst + kHalfW, false);
            }
            __syncwarp();
          }
          if (elect_one()) commit_cg2(acc0_full);
          __syncwarp();
          stage_done();
        }
        {  // x_l = x_{l-1} + Wr_{l-1} z_{l-1} (l >= 1), off the dependent path
          const uint32_t bst = stage_wait();
          if (l > 0 && elect_one()) {
            kchunk(tmem + kTXF, za, 0, bst, false);
            kchunk(tmem + kTXF, za, 1, bst, false);
          }
          __syncwarp();
          stage_done();
          if (elect_one()) commit_cg2(x_full);
          __syncwarp();
        }
      }
    }
  } else if (warp >= 2 && warp < 10) {  // ---- gate ----
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int rho = 32 * (q & 1) + lane, cb = q >> 1;  // row, channel block (32 channels)
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t szb = smem_u32(zb);
    const bool tr = warp == 2 && lane == 0;
    for (int g = 0; g < G; ++g) {
      const int l = g % L;
      const uint32_t par = (uint32_t)g & 1;
      // (the arrivals are the tensor core's commit: a CTA-scope wait, no L1 invalidation)
      mbar_wait(acc0_full, par);
      tc_fence_after();
      if (tr) trace_at(a, l, h ? T_EPI_ACC1 : T_EPI_ACC0, clock64());
      if (warp == 2 && lane == 0) (void)0, tr2(a, l, 3);
      float v[64];  // tanh inputs of channels 64h + 32cb + j | sigmoid inputs
      const uint32_t acch = trow + 128u * par + 64u * h;
      tmem_ld32x2(acch, acch + 32, v);
      tc_fence_before();
      if (a.has_dil_bias) {
        const float* bd = a.dil_b + (size_t)l * 2 * kD + 64 * h + 32 * cb;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          v[j] += __ldg(bd + j);
          v[32 + j] += __ldg(bd + kD + j);
        }
      }
      uint32_t zw[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) zw[j] = gate2_h2(v[2 * j], v[2 * j + 1], v[32 + 2 * j], v[33 + 2 * j]);
      // z buffer `par` was last read by layer g - 1's WF and residual MMAs (before this
      // layer's acc commit) and by layer g - 2's stash store (stage_free)
      if (g >= 2) mbar_wait(stage_free + par, (uint32_t)(((g >> 1) - 1) & 1));
      const uint32_t zrow = szb + par * kOp + (uint32_t)rho * 16;
#pragma unroll
      for (int m = 0; m < 4; ++m)
        st_shared_v4(zrow + (uint32_t)(8 * h + 4 * cb + m) * 1024, zw[4 * m], zw[4 * m + 1], zw[4 * m + 2],
                     zw[4 * m + 3]);
      fence_proxy_async();  // generic shared writes -> the MMA / bulk-store reads
      warp_arrive_leader(z_ready + h);
      if (lane == 0) mbar_arrive(z_local);
      if (tr) trace_at(a, l, h ? T_EPI_Z1 : T_EPI_Z0, clock64());
      if (warp == 2 && lane == 0) (void)0, tr2(a, l, 2);
    }
  } else if (warp >= 10 && warp < 14) {  // ---- x: conversion, push, pops, embedding ----
    const int q = warp & 3;
    const int rho = 32 * (q & 1) + lane, cb = q >> 1;  // row, channel block (64 channels)
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t sxrow = smem_u32(xtb) + (uint32_t)rho * 16;
    auto qb = [&](int g) { return qbase_of(a, g / L, g % L); };
    // pops: this thread's 8 K-pieces (channels 64cb..) of its row of layer g's slot -> pop
    // buffer g & 1 (cp.async; the same thread pushed those bytes)
    auto load_slot = [&](int g) {
      const uint8_t* src = qtile + qb(g) + (size_t)rho * 16;
      const uint32_t dst = smem_u32(popb + (g & 1) * kOp) + (uint32_t)rho * 16;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int pc = 8 * cb + j;
        cp_async16(dst + (uint32_t)pc * 1024, src + (size_t)pc * kPairRows * 16);
      }
      cp_async_commit();
    };
    auto local_arrive = [&](uint64_t* bar) {
      __syncwarp();
      if (lane == 0) mbar_arrive(bar);
    };
    auto xd_signal = [&]() {
      fence_proxy_async();
      local_arrive(xd_ready);
    };
    load_slot(0);
    if (G > 1) load_slot(1);
    else cp_async_commit();
    cp_async_wait<1>();
    xd_signal();
    int xf_seen = 0;
    for (int g = 0; g < G; ++g) {
      const int i = g / L, l = g % L;
      const uint32_t par = (uint32_t)g & 1;
      // x_l of this thread's row and channel block: the embedding at l = 0, else the residual
      // stream (TMEM) + its pending bias; the previous layer's MMAs are done with x and x_t
      // l >= 1: x_l = the residual MMA of this layer (x_full of g); l = 0: the embedding, once
      // the previous layer's MMAs are done with TMEM x and the x_t operand (x_full of g - 1)
      // (every phase in order: a parity wait that skipped the l = 0 phase could pass on the
      // phase before it)
      while (xf_seen < (l > 0 ? g + 1 : g)) {
        mbar_wait(x_full, (uint32_t)xf_seen & 1);
        ++xf_seen;
      }
      if (warp == 10 && lane == 0) {
        trace_at(a, l, T_EPI_A, clock64());
        (void)0, tr2(a, l, 0);
      }
      tc_fence_after();
      float x[64];
      if (l == 0) {
        if (i > 0) wait_counter(a.cls_ready + (tile >> 1), (uint32_t)i);
        const int c = clamp_class(a.cls[tile * 64 + rho], 256);
        const float4* e4 = reinterpret_cast<const float4*>(a.embed + (size_t)c * kR + 64 * cb);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float4 e = __ldg(e4 + j);
          x[4 * j] = e.x; x[4 * j + 1] = e.y; x[4 * j + 2] = e.z; x[4 * j + 3] = e.w;
        }
        tmem_st32(trow + kTXF, *reinterpret_cast<float(*)[32]>(x));
        tmem_st32(trow + kTXF + 32, *reinterpret_cast<float(*)[32]>(x + 32));
      } else {
        tmem_ld64(trow + kTXF, x);
        if (a.has_res_bias) {
          const float* rb = a.res_b + (size_t)(l - 1) * kR + 64 * cb;
#pragma unroll
          for (int j = 0; j < 64; ++j) x[j] += __ldg(rb + j);
          tmem_st32(trow + kTXF, *reinterpret_cast<float(*)[32]>(x));
          tmem_st32(trow + kTXF + 32, *reinterpret_cast<float(*)[32]>(x + 32));
        }
      }
      tc_fence_before();
      uint32_t w[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) w[j] = pack_h2(x[2 * j], x[2 * j + 1]);
#pragma unroll
      for (int m = 0; m < 8; ++m)
        st_shared_v4(sxrow + (uint32_t)(8 * cb + m) * 1024, w[4 * m], w[4 * m + 1], w[4 * m + 2], w[4 * m + 3]);
      fence_proxy_async();
      local_arrive(xt_ready + par);
      if (warp == 10 && lane == 0) {
        trace_at(a, l, T_EPI_XT, clock64());
        (void)0, tr2(a, l, 1);
      }
      // push x_l: this thread's 8 K-pieces of its row into ring slot t mod d_l (its pop was
      // read two layers ago by this thread)
      uint4* dst = reinterpret_cast<uint4*>(qtile + qb(g)) + rho;
#pragma unroll
      for (int m = 0; m < 8; ++m)
        dst[(size_t)(8 * cb + m) * kPairRows] = make_uint4(w[4 * m], w[4 * m + 1], w[4 * m + 2], w[4 * m + 3]);
      // the pop of layer g + 2 into the buffer layer g's x_{t-d} MMAs have finished with
      if (g + 1 < G) {
        // layer g's x_{t-d} MMAs are done with pop buffer g & 1: the release of its weight
        // stage (stage 3g of the ring)
        mbar_wait(wempty + (kCopies * g) % kStages, (uint32_t)((kCopies * g) / kStages) & 1);
        if (g + 2 < G) load_slot(g + 2);
        else cp_async_commit();
        cp_async_wait<1>();  // layer g + 1's pop
        xd_signal();
      }
    }
  } else if (warp == 14) {  // ---- publisher: this CTA's 64 rows of z_l -> the stash ----
    if (lane == 0) {
      for (int g = 0; g < G; ++g) {
        mbar_wait(z_local, (uint32_t)g & 1);
        if (a.zfree != nullptr && g >= a.zring)
          wait_counter(a.zfree + (tile >> 1), (uint32_t)a.ztail * (uint32_t)(g - a.zring + 1));
        uint8_t* dst = reinterpret_cast<uint8_t*>(zstash_rows(a.zimg, tile, a.zring, g % a.zring));
        const uint8_t* src = zb + (g & 1) * kOp;
        for (int j = 0; j < 16; ++j) bulk_s2g(dst + j * 2048, src + j * 1024, 1024);
        bulk_commit();
        bulk_wait0();             // in the stash
        fence_proxy_async_all();  // async-proxy writes before the release
        red_release_gpu(a.zflag + (tile >> 1), 1u);
        mbar_arrive(stage_free + (g & 1));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no DSMEM traffic or 2-SM MMA into a CTA that has exited
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
