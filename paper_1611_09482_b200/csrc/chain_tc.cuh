// Chain kernel of the tcgen05 path (included by cell_tc.cu): one 64-stream tile per CTA,
// the dependent chain of all L dilated layers of one generation step.
//
// Per layer l (a = W0 x_l[t] + W1 x_l[t-d] + b, z = tanh(a[:D]) * sigmoid(a[D:]),
// x_{l+1} = x_l + W_res z + b_res; the skip/head work is deferred to big-K GEMMs).
//
// Why 64 streams per CTA: the chain is a serial dependency per layer (x -> MMA -> gate ->
// res MMA -> x), and every MMA instruction costs ~72 cycles at N = 128 whether M is 64 or 128
// (tools/mma_rate.cu). What scales with the rows is the gate (2 MUFU ops per z, 16 per clock
// per SM: 1024 cycles per layer for 128 rows) and the activation traffic. 64-row tiles halve
// those per SM and put twice as many SMs on the chain for the same MMA latency.
//
//   TMEM, M = 64: row m of the tile lives in lane (m % 16) + 32 * (m / 16) of plane P0 and the
//   lane 16 above it in plane P1 (tools/m64_probe.cu). An MMA's TMEM A operand must sit in the
//   plane of its accumulator, so the dilated GEMM lives in P0 and the residual GEMM in P1:
//     P0 [0,128)    acc0  dil N-half 0: tanh rows 0..63 | sigmoid rows 0..63
//     P0 [128,256)  acc1  dil N-half 1: tanh rows 64..127 | sigmoid rows 64..127
//     P0 [256,320)  xt    fp16 x_l[t] operand (A from TMEM, packed pairs)
//     P0 [320,384)  xd    fp16 x_l[t-d] operand
//     P1 [0,128)    x     residual stream x_l, fp32; the res MMA accumulates onto it
//     P1 [128,192)  z     fp16 z operand of the res MMA
//   Gate and conversion use 16-lane (16x64b) accesses that touch one plane; the queue warps'
//   32x32b accesses touch both, and the columns of the other plane under their regions are
//   scratch. Every MMA takes A from TMEM (the operands are produced there; an SMEM A operand
//   is no faster inside this kernel, tools/mma_rate.cu). SMEM holds the weight stages A0 / A1 (32 KB each:
//   the x_{t-d} K-chunks of N-half 0 / 1), B (64 KB: the x_t K-chunks of both halves) and C
//   (32 KB: res), one bulk copy each per layer (~500 cycles per copy, tools/ring_bw.cu).
//
//   Queue slots hold x_l in fp16 (the precision the MMA consumes), 16 KB per tile laid out
//   [16 K-pieces][64 rows][8 fp16]: a warp's 16-byte accesses to one K-piece of 16
//   consecutive rows are 256 contiguous bytes. The z stash for the skip GEMM is laid out
//   [tile pair][L][16 K-pieces][128 rows][16 B] -- per 128-row GEMM tile the no-swizzle
//   K-major UMMA layout (sdesc_plain); tile 2p fills rows 0..63, tile 2p+1 rows 64..127.
//
//   warp 0  lane 0  weight producer (stages A0, A1, B, C in consumption order)
//   warp 14 lane 0  publisher (z stash release); warp 15: MMA completion watcher (trace only)
//   warp 1          MMA issuer: the converged warp issues under elect.sync (tools/mma_rate.cu)
//   warps 2..9      gate warps, quadrant q = warp % 4 (rows 16q..16q+15), half h = (warp-2)/4,
//                   all accesses 16x64b -- every lane busy: lane t holds row (t>>2) + 8(t&1),
//                   columns of parity (t>>1)&1; fp16 pairs are completed with one shuffle.
//                   x_l (P1) -> xt (P0) for channels 64h..64h+63, then per N-half the gate of
//                   16 z columns per lane (P0 acc -> P1 z)
//   warps 10..13    queue warps (lanes 0..15 = rows of quadrant q): push x_l (xt -> ring
//                   slot), x_{t-d} of layer l+1 (registers, loaded a layer ahead) -> xd once
//                   layer l's x_{t-d} MMAs are done, z stash (z -> HBM); L2 prefetch of the
//                   slot two layers ahead
//
// MMA issue order per layer: x_{t-d} halves 0 and 1 (normally issued during the previous
// layer) -> [xt_ready] x_t N-half 0 -> acc0_full -> x_t N-half 1 -> acc1_full -> [z0_ready]
// res K-chunk 0, next layer's x_{t-d} N-half 0 -> [z1_ready] res K-chunk 1 -> [x_pushed]
// x_full -> next layer's x_{t-d} N-half 1.

constexpr int kChainRows = 64;
// split chain: the z half crosses to the peer by bulk copies (async proxy end to end) when
// set, by st.async stores otherwise
#ifndef FW_SPLIT_BULK
#define FW_SPLIT_BULK 1
#endif
constexpr bool kSplitBulk = FW_SPLIT_BULK != 0;

constexpr int kChainThreads = 512;  // 16 warps; 128 registers per thread (4 warps per SMSP)
constexpr int kQueueWarp0 = 10;
constexpr uint32_t kP1 = 16u << 16;  // lane offset of plane P1
constexpr uint32_t kColXt = 256, kColXd = 320;  // P0
constexpr uint32_t kColX = 0, kColZ = 128;      // P1
constexpr uint32_t kSlotBytes = 16384;  // one tile's share of a ring slot (64 rows x 128 fp16)
// Ring slots are laid out per tile pair, [16 K-pieces][128 rows][8 fp16] (32 KB): the no-swizzle
// K-major operand layout of an M = 128 MMA; tile 2p holds rows 0..63, tile 2p+1 rows 64..127.
constexpr uint32_t kPairRows = 128;
constexpr uint32_t kStageA = 32768, kStageB = 65536, kStageC = 32768;
constexpr uint32_t kOffA0 = 0, kOffA1 = kOffA0 + kStageA, kOffB = kOffA1 + kStageA,
                   kOffC = kOffB + kStageB, kOffBars = kOffC + kStageC;
// skip role: a 2-stage ring of (z tile 32 KB | W_skip block SK x 128 x 2 B, <= 64 KB), later
// reused by the fused heads as a 4-stage ring of (A chunk 16 KB | B chunk <= 256 x 128 B);
// then barriers and the selection exchange buffer (4 KB)
constexpr uint32_t kSkipStage = 2 * kTile + 65536;
constexpr uint32_t kSkipBars = 2 * kSkipStage;
constexpr uint32_t kImgBytes = 8 * kTile;  // pair mode: the resident s / h image (128 KB)
constexpr uint32_t kWStage = 32768;        // pair mode: one head weight K-chunk (256 rows)
constexpr int kWStages = 3;                // pair mode: head weight ring depth
constexpr uint32_t kPairBars = kImgBytes + kWStages * kWStage;  // 224 KB
// pair mode, after the barriers: the bias of h (this block's 256 columns), staged once per
// launch (the bias of s initialises the skip accumulator instead)
constexpr uint32_t kPairBias = kPairBars + 256;
constexpr uint32_t kTailStage = 2 * (kTile + 32768);  // 2 K-chunks of A | 2 of B (N <= 256)
constexpr int kTailStages = 2;
// chain role: after its barriers, two 16 KB staging buffers for popped ring slots
constexpr uint32_t kOffXq = kOffBars + 1024;
// chain role: after the pop staging, two 16 KB staging images of the layer's z tile
// ([16 K-pieces][64 rows][16 B]) that the publisher bulk-stores into the z stash
constexpr uint32_t kOffZs = kOffXq + 2 * kSlotBytes;
constexpr size_t kSmemMax3(size_t a, size_t b, size_t c) { return a > b ? (a > c ? a : c) : (b > c ? b : c); }
constexpr size_t kChainSmem =
    1024 + kSmemMax3(kOffZs + 2 * kSlotBytes, kSkipBars + 8448, kPairBias + 1024);

// z stash row base of (tile, ring slot): [tile pair][zring][16 pieces][128 rows][16 B]. The
// fused kernel keeps a ring of zring (< L) layers per pair -- small enough to stay in L2,
// where the whole-step stash (42 MB for cfg4) was written back to DRAM; the unfused path's
// skip GEMM needs all L layers (zring = L, slot = layer).
__device__ __forceinline__ uint4* zstash_rows(uint8_t* zimg, int tile, int zring, int slot) {
  return reinterpret_cast<uint4*>(zimg + ((size_t)(tile >> 1) * zring + slot) * 2 * kTile) +
         (tile & 1) * kChainRows;
}
__device__ __forceinline__ const uint8_t* zstash_tile(const ChainArgs& a, int p, int g) {
  return a.zimg + ((size_t)p * a.zring + g % a.zring) * 2 * kTile;
}
// A tail producer has its stage of layer g back, so layer g-2's z has been read: count it
// (the chain waits for it before reusing that ring slot)
__device__ __forceinline__ void zring_consumed(const ChainArgs& a, int p, int g) {
  if (a.zfree != nullptr && g >= 2)
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(a.zfree + p) : "memory");
}

// ---- skip role: s = ReLU(sum_l W_skip_l z_l + sum_l b_skip_l) for one 128-row tile pair and
// one SK-column block of S, accumulated in TMEM layer by layer as the chain CTAs stash z_l
// (a per-pair counter in global memory, +1 per chain tile per layer). Runs on SMs the chain
// leaves idle, so the skip GEMM costs no time after the chain ends.
// With fused heads the pair's blocks then run head1 (H / nsk columns each, once every block
// of the pair has published its part of s) and block 0 head2 + the selection rule.
__device__ __forceinline__ void skip_role(const ChainArgs& a, uint8_t* smem, int k) {
  const int SK = a.SK, nsk = a.S / SK;
  const int p = k / nsk, e = k % nsk;
  const int L = a.L;
  const uint32_t bbytes = (uint32_t)SK * 256;  // 2 K-chunks of [SK rows][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSkipBars);
  uint64_t* full = bars;       // [2]
  uint64_t* empty = bars + 2;  // [2]
  uint64_t* acc_full = bars + 4;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 5);
  uint64_t* tfull = bars + 6;    // [4] fused heads ring
  uint64_t* tempty = bars + 10;  // [4]
  uint64_t* tacc = bars + 14;    // head1 (phase 0) / head2 (phase 1) accumulator complete
  uint64_t* tfree = bars + 15;   // 256: epilogue done reading TMEM (phase 0 s, 1 h)
  uint64_t* noise_ready = bars + 16;  // 128: Gumbel noise in TMEM [256,512)
  float* xch = reinterpret_cast<float*>(smem + kSkipBars + 256);
  // biases of this block's epilogues, staged while the chain runs: skip [0,SK), head1 [SK, SK+n1)
  float* sbias = reinterpret_cast<float*>(smem + kSkipBars + 256 + 4096);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.S, H = a.H, n1 = a.H / nsk;
  const bool heads = a.heads != 0, sel_block = heads && e == 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 15; ++i) mbar_init(bars + i, (i >= 6 && i < 10) ? 2 : 1);  // tfull: 2 producers
    mbar_init(tfree, 256);
    mbar_init(noise_ready, 128);
    fence_mbar_init();
  }
  // TMEM: accumulator (s, then h, then the logits) at [0,256); the selecting block keeps the
  // step's Gumbel noise of its 128 streams x 256 classes at [256,512), computed by warps
  // 10..13 while the chain runs
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int k1 = S / 64, k2 = H / 64;  // K-chunks of head1 / head2
  // fused heads' operand stream: 2 K-chunks per stage; A (the s / h images) by warp 0, B (the
  // W1 / W2 chunks) by warp 11 -- the copy engine's cost is per operation and a thread's
  // copies run one after another (tools/ring_bw.cu)
  const int it1 = k1 / 2, it2 = sel_block ? k2 / 2 : 0, nit = it1 + it2;
  auto tail_loads = [&](bool is_b, int step) {
    const uint32_t b1 = (uint32_t)n1 * 128, b2 = (uint32_t)a.sel.A * 128;
    for (int it = 0; it < nit; ++it) {
      const int T = step * nit + it, st = T % kTailStages;
      mbar_wait(tempty + st, ((uint32_t)(T / kTailStages) & 1) ^ 1);
      if (it == 0) {
        wait_counter(a.sflag + p, (uint32_t)(nsk * (step + 1)));
        fence_proxy_async_all();
      }
      if (it == it1) {
        wait_counter(a.hflag + p, (uint32_t)(nsk * (step + 1)));
        fence_proxy_async_all();
      }
      const bool two = it >= it1;
      const int c = two ? 2 * (it - it1) : 2 * it;
      const uint32_t bb = two ? b2 : b1;
      uint8_t* stage = smem + st * kTailStage;
      if (!is_b) {
        mbar_arrive_expect_tx(tfull + st, 2 * kTile);
        const uint8_t* src = two ? a.himg + ((size_t)p * k2 + c) * kTile
                                 : a.simg + ((size_t)p * k1 + c) * kTile;
        bulk_g2s(stage, src, 2 * kTile, tfull + st);
      } else {
        const uint8_t* src = two ? a.wh2 + (size_t)c * b2 : a.wh1b + ((size_t)e * k1 + c) * b1;
        mbar_arrive_expect_tx(tfull + st, 2 * bb);
        bulk_g2s(stage + 2 * kTile, src, 2 * bb, tfull + st);
      }
    }
  };
  if (warp == 0) {
    if (lane == 0) {  // producer: z tile of (p, l) once both chain tiles stashed it
      for (int i = 0; i < a.n_steps; ++i) {
        for (int l = 0; l < L; ++l) {
          const int g = i * L + l, st = g & 1;
          mbar_wait(empty + st, ((uint32_t)(g >> 1) & 1) ^ 1);
          zring_consumed(a, p, g);
          wait_counter(a.zflag + p, (uint32_t)a.zpub * (uint32_t)(g + 1));
          if (l == L - 1) trace_g(a, k == 0, 2);
          fence_proxy_async_all();
          uint8_t* stage = smem + st * kSkipStage;
          mbar_arrive_expect_tx(full + st, 2 * kTile + bbytes);
          bulk_g2s(stage, zstash_tile(a, p, g), 2 * kTile, full + st);
          bulk_g2s(stage + 2 * kTile, a.wskip2 + ((size_t)e * L + l) * bbytes, bbytes, full + st);
        }
        if (heads) tail_loads(false, i);
      }
    }
  } else if (warp == 1) {
    const uint32_t s0 = smem_u32(smem);
    const int ntacc = sel_block ? 2 : 1;
    for (int i = 0; i < a.n_steps; ++i) {
      const uint32_t id = idesc_f16(128, SK);
      for (int l = 0; l < L; ++l) {
        const int gl = i * L + l, st = gl & 1;
        mbar_wait(full + st, (uint32_t)(gl >> 1) & 1);
        tc_fence_after();
        const uint32_t sa = s0 + st * kSkipStage, sb = sa + 2 * kTile;
        if (elect_one()) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(tmem, sdesc_plain(sa + c * kTile + kk * 4096, 2048, 128),
                       sdesc_sw128(sb + c * (uint32_t)SK * 128 + kk * 32), id, (l | c | kk) != 0);
          mma_commit(empty + st);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(acc_full);
      __syncwarp();
      trace_g(a, k == 0 && lane == 0, 7);
      if (!heads) continue;
      for (int g = 0; g < ntacc; ++g) {
        const int nb = g == 0 ? n1 : a.sel.A;
        const uint32_t idh = idesc_f16(128, nb);
        // the epilogue has read the previous accumulator (2 tfree phases per step)
        mbar_wait(tfree, (uint32_t)(2 * i + g) & 1);
        tc_fence_after();
        trace_g(a, k == 0 && lane == 0, 8 + 3 * g);
        const int i0 = g == 0 ? 0 : it1, ni = g == 0 ? it1 : k2 / 2;
        for (int it = i0; it < i0 + ni; ++it) {
          const int T = i * nit + it, st = T % kTailStages;
          mbar_wait(tfull + st, (uint32_t)(T / kTailStages) & 1);
          tc_fence_after();
          const uint32_t sa = s0 + st * kTailStage, sb = sa + 2 * kTile;
          if (it == i0) trace_g(a, k == 0 && lane == 0, 9 + 3 * g);
          if (elect_one()) {
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_bf16(tmem, sdesc_sw128(sa + c * kTile + kk * 32),
                         sdesc_sw128(sb + c * (uint32_t)nb * 128 + kk * 32), idh,
                         (it > i0 || c || kk) ? 1u : 0u);
            mma_commit(tempty + st);
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit(tacc);
        __syncwarp();
        trace_g(a, k == 0 && lane == 0, 10 + 3 * g);
      }
    }
  } else if (warp >= 2 && warp < 10) {
    // epilogue: row r, columns [h*cols/2, (h+1)*cols/2) of the accumulator
    const int sub = warp & 3, h = (warp - 2) >> 2;
    const int r = sub * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(sub * 32) << 16);
    for (int i = threadIdx.x - 64; i < SK + (heads ? n1 : 0); i += 256)
      sbias[i] = i < SK ? a.skip_bsum[e * SK + i] : a.h1_b[e * n1 + (i - SK)];
    named_bar_sync(1, 256);
    const uint32_t stg = smem_u32(smem);
    for (int i = 0; i < a.n_steps; ++i) {
      mbar_wait(acc_full, (uint32_t)i & 1);
      tc_fence_after();
      trace_g(a, k == 0 && warp == 2 && lane == 0, 14);
      // ReLU(s + bias) -> this block's SK/64 chunks of the pair's s images: staged in shared
      // memory (the rings are idle now) and written with one bulk store -- per-thread
      // 16-byte stores of swizzled rows would touch 32 lines per warp instruction
      epi_relu_image_smem(trow, r, h * (SK / 2), SK / 2, h * (SK / 2), sbias, stg + h * (SK / 128) * kTile);
      fence_proxy_async();
      tc_fence_before();
      if (heads) mbar_arrive(tfree);  // s read out of TMEM
      named_bar_sync(1, 256);
      if (warp == 2 && lane == 0) {
        bulk_s2g(a.simg + ((size_t)p * (S / 64) + e * SK / 64) * kTile, smem, (uint32_t)SK * 256);
        bulk_commit();
        bulk_wait0();
        fence_proxy_async_all();
        if (heads) red_release_gpu(a.sflag + p, 1u);
        trace_g(a, k == 0, 3);
      }
      if (!heads) continue;
      // head1 part: h columns [e*n1, (e+1)*n1) -> the pair's h images
      mbar_wait(tacc, (uint32_t)(i * (sel_block ? 2 : 1)) & 1);
      tc_fence_after();
      trace_g(a, k == 0 && warp == 2 && lane == 0, 15);
      // the tail ring holds no live operands once head1's accumulator is complete
      named_bar_sync(1, 256);
      epi_relu_image_smem(trow, r, h * (n1 / 2), n1 / 2, h * (n1 / 2), sbias + SK,
                          stg + h * (n1 / 128) * kTile);
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(tfree);
      named_bar_sync(1, 256);
      if (warp == 2 && lane == 0) {
        bulk_s2g(a.himg + ((size_t)p * (H / 64) + e * n1 / 64) * kTile, smem, (uint32_t)n1 * 256);
        bulk_commit();
        bulk_wait0();
        fence_proxy_async_all();
        red_release_gpu(a.hflag + p, 1u);
        trace_g(a, k == 0, 4);
      }
      if (sel_block) {  // head2 logits + the selection rule for the pair's 128 streams
        mbar_wait(tacc, (uint32_t)(2 * i + 1) & 1);
        if (a.sel.mode == FW_SAMPLE_GUMBEL) mbar_wait(noise_ready, (uint32_t)i & 1);
        tc_fence_after();
        trace_g(a, k == 0 && warp == 2 && lane == 0, 5);
        const SelectArgs sel = sel_step(a.sel, a.t0, i);
        epi_select(trow, r, h, p * 128 + r, sel, xch, 256);
        // every selection of the pair is written: the chain blocks may start step i+1
        tc_fence_before();
        named_bar_sync(1, 256);
        if (warp == 2 && lane == 0) {
          red_release_gpu(a.cls_ready + p, 1u);
          trace_g(a, k == 0, 6);
          if (i == a.n_steps - 2) trace_g(a, k == 0, 17);
        }
      }
    }
  } else if (warp >= 10 && warp < 14) {
    // per step: the Gumbel noise (selecting block), then warp 11's half of the head operands
    const bool noise = sel_block && a.sel.mode == FW_SAMPLE_GUMBEL;
    const int sub = warp & 3;
    const int r = sub * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(sub * 32) << 16);
    for (int i = 0; i < a.n_steps; ++i) {
      if (noise) {
        // step i's noise of row r (stream p*128 + r), 256 classes -> TMEM [256,512), once
        // the previous step's selection has read the previous noise
        const uint32_t prefix = noise_prefix(a.sel.seed, (uint32_t)(a.sel.stream_offset + p * 128 + r),
                                             (uint32_t)(a.t0 + i));
        if (i > 0) wait_counter(a.cls_ready + p, (uint32_t)i);
#pragma unroll 1
        for (int cc = 0; cc < 8; ++cc) {
          float gn[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) gn[j] = gumbel_noise(prefix, 32 * cc + j);
          tmem_st32(trow + 256 + 32 * cc, gn);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(noise_ready);
      }
      if (warp == 11 && lane == 0 && heads) tail_loads(true, i);
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ---- tail role, pair mode (S = H = 512, the two blocks of a tile pair form a 2-CTA
// cluster): as skip_role, but the pair exchanges its halves of s and h through distributed
// shared memory instead of global memory + flags. Each block writes its half of s into its
// own A image and bulk-copies it into the peer's; both run head1 (256 columns of h each)
// with A resident and only W1 streamed; block 1 sends its half of h into block 0's image
// once block 0's head1 has released it; block 0 runs head2 and the selection rule.
// Step i's head2 accumulates onto the selection's bias (+ noise) columns: every step that
// writes no logits, except under the inverse-CDF rule (it needs the logits themselves).
__device__ __forceinline__ bool pair_folds(const ChainArgs& a, int i) {
  return a.sel.mode != FW_SAMPLE_INVCDF && !(a.sel.logits_base != nullptr && i < a.sel.n_logit_steps);
}
__device__ __forceinline__ void tail_pair_role(const ChainArgs& a, uint8_t* smem, int k) {
  const int p = k >> 1, e = k & 1;  // e == cluster rank
  const int L = a.L, S = a.S, H = a.H;
  const int ks = S / 64, kh = H / 64;
  const uint32_t peer = (uint32_t)(e ^ 1);
  // smem: skip ring [0,192K) while the chain runs; then the s / h image [0,128K) and the
  // head weight ring [128K,224K); barriers and biases after. The selection's exchange buffer
  // aliases ring stage 0 (idle once head2's MMAs are complete).
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kPairBars);
  uint64_t* full = bars;           // [2] skip ring
  uint64_t* empty = bars + 2;      // [2]
  uint64_t* acc_full = bars + 4;   // skip sum complete (once per step)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 5);
  uint64_t* wfull = bars + 6;      // [3] head weight ring: one 32 KB K-chunk per stage
  uint64_t* wempty = bars + 9;     // [3]
  uint64_t* tacc = bars + 12;      // head accumulator complete (block 0: 2 per step, 1: 1)
  uint64_t* own_ready = bars + 13; // 256: own half of the image written (+ TMEM read out)
  uint64_t* peer_full = bars + 14; // tx: the peer's half arrived (block 0: s, h; 1: s)
  uint64_t* a_free = bars + 15;    // block 1: block 0's image may take h (remote arrive)
  uint64_t* noise_ready = bars + 16;  // 128: Gumbel noise in TMEM [256,512)
  uint64_t* acc_init = bars + 17;     // 256: TMEM [0,256) holds the bias of s (next skip sum)
  // block 0: block 1 has consumed block 0's s half (its head1 is complete), so block 0 may
  // overwrite that half of its image -- the source of its outgoing s copy -- with h
  uint64_t* s_free = bars + 18;
  uint8_t* img = smem;                 // [8 K-chunks][16 KB]: s, then (block 0) h
  uint8_t* wring = smem + kImgBytes;   // kWStages x 32 KB
  float* xch = reinterpret_cast<float*>(wring);
  float* hbias = reinterpret_cast<float*>(smem + kPairBias);
  for (int c = threadIdx.x; c < 256; c += blockDim.x) hbias[c] = a.h1_b[e * 256 + c];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool sel_block = e == 0;
  const uint32_t half_bytes = 4 * kTile;  // 256 columns x 128 rows fp16
  if (threadIdx.x == 0) {
    for (int i = 0; i < 13; ++i) mbar_init(bars + i, 1);
    mbar_init(own_ready, 256);
    mbar_init(peer_full, 1);
    mbar_init(a_free, 1);
    mbar_init(noise_ready, 128);
    mbar_init(acc_init, 256);
    mbar_init(s_free, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(peer_full, half_bytes);  // armed before the peer can send
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync();  // both blocks' barriers exist and are armed before any exchange
  const uint32_t tmem = *tmem_holder;
  const int nw = ks + (sel_block ? kh : 0);  // head weight chunks per step
  // head weight stream: K-chunk sequence of a step, own half of the image first (head1: W1
  // rows [256e, 256e+256) chunks 4e.., 4e+1.., head2: W2 chunks 0..7), one 32 KB chunk per
  // ring stage; stage st is owned by producer thread st (warps 0, 11, 12), so three copies
  // are in flight
  auto chunk_of = [&](int j) { return j < ks ? (4 * e + j) % ks : j - ks; };
  auto head_loads = [&](int step, int owner) {
    mbar_wait(acc_full, (uint32_t)step & 1);  // the skip ring (same smem) is idle
    for (int j = 0; j < nw; ++j) {
      const int J = step * nw + j, st = J % kWStages;
      if (st != owner) continue;
      mbar_wait(wempty + st, ((uint32_t)(J / kWStages) & 1) ^ 1);
      const int c = chunk_of(j);
      const uint8_t* src = j < ks ? a.wh1b + ((size_t)e * ks + c) * kWStage
                                  : a.wh2 + (size_t)c * kWStage;
      mbar_arrive_expect_tx(wfull + st, kWStage);
      bulk_g2s(wring + st * kWStage, src, kWStage, wfull + st);
    }
  };
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < a.n_steps; ++i) {
        for (int l = 0; l < L; ++l) {
          const int g = i * L + l, st = g & 1;
          mbar_wait(empty + st, ((uint32_t)(g >> 1) & 1) ^ 1);
          zring_consumed(a, p, g);
          // the layer's skip weights do not depend on the chain: in flight before z is --
          // except in layers 0 and 1, whose stages overlap the previous step's s / h image
          // and head weight ring until the chain's z (behind that step's selection) says
          // the heads are done with them
          uint8_t* stage = smem + st * kSkipStage;
          const uint8_t* wsrc = a.wskip2 + ((size_t)e * L + l) * 65536;
          mbar_arrive_expect_tx(full + st, 2 * kTile + 65536);
          if (l >= 2) bulk_g2s(stage + 2 * kTile, wsrc, 65536, full + st);
          wait_counter(a.zflag + p, (uint32_t)a.zpub * (uint32_t)(g + 1));
          if (l == L - 1) trace_g(a, k == 0, 2);
          if (l < 2) bulk_g2s(stage + 2 * kTile, wsrc, 65536, full + st);
          fence_proxy_async_all();
          bulk_g2s(stage, zstash_tile(a, p, g), 2 * kTile, full + st);
        }
        // the step's last acquire in this SM is behind: the logits bias stays in L1 until
        // the selection reads it
        if (sel_block)
          for (int c = 0; c < 1024; c += 128) prefetch_l1(reinterpret_cast<const uint8_t*>(a.sel.bias) + c);
        head_loads(i, 0);
      }
    }
  } else if (warp == 1) {
    const uint32_t s0 = smem_u32(smem), si = smem_u32(img), sw = smem_u32(wring);
    const uint32_t id = idesc_f16(128, 256);
    int pf_phase = 0;  // phases of peer_full consumed
    for (int i = 0; i < a.n_steps; ++i) {
      for (int l = 0; l < L; ++l) {
        const int gl = i * L + l, st = gl & 1;
        if (l == 0) mbar_wait(acc_init, (uint32_t)i & 1);  // accumulator = bias of s
        mbar_wait(full + st, (uint32_t)(gl >> 1) & 1);
        tc_fence_after();
        const uint32_t sa = s0 + st * kSkipStage, sb = sa + 2 * kTile;
        if (elect_one()) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(tmem, sdesc_plain(sa + c * kTile + kk * 4096, 2048, 128),
                       sdesc_sw128(sb + c * 256 * 128 + kk * 32), id, 1u);
          mma_commit(empty + st);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(acc_full);
      __syncwarp();
      trace_g(a, k == 0 && lane == 0, 7);
      for (int g = 0; g < (sel_block ? 2 : 1); ++g) {
        // K order: own half of the image first (its chunks are written here), the peer's
        // half (arriving through DSMEM) second -- the MMAs start before the exchange ends.
        // head2 of a step without logits output accumulates onto the bias (+ Gumbel noise)
        // the noise warps left in TMEM [256,512): the selection reads finished scores.
        const bool fold = g == 1 && pair_folds(a, i);
        const uint32_t dacc = fold ? tmem + 256 : tmem;
        const int j0 = g == 0 ? 0 : ks, nj = g == 0 ? ks : kh;
        for (int j = j0; j < j0 + nj; ++j) {
          const int J = i * nw + j, st = J % kWStages;
          const int c = chunk_of(j), jj = j - j0;
          if (jj == 0) {
            mbar_wait(own_ready, (uint32_t)(2 * i + g) & 1);  // (+ previous accumulator read)
            if (fold) mbar_wait(noise_ready, (uint32_t)i & 1);
            tc_fence_after();
            trace_g(a, k == 0 && lane == 0, 8 + 3 * g);
          }
          if (jj == nj / 2) {
            mbar_wait(peer_full, (uint32_t)pf_phase & 1);
            ++pf_phase;
            if (lane == 0) mbar_arrive_expect_tx(peer_full, half_bytes);  // re-arm
            __syncwarp();
            tc_fence_after();
          }
          mbar_wait(wfull + st, (uint32_t)(J / kWStages) & 1);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16(dacc, sdesc_sw128(si + c * kTile + kk * 32),
                       sdesc_sw128(sw + st * kWStage + kk * 32), id, (fold || jj || kk) ? 1u : 0u);
            mma_commit(wempty + st);
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit(tacc);
        __syncwarp();
        trace_g(a, k == 0 && lane == 0, 10 + 3 * g);
      }
    }
  } else if (warp >= 2 && warp < 10) {
    const int sub = warp & 3, hf = (warp - 2) >> 2;
    const int r = sub * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(sub * 32) << 16);
    const uint32_t si = smem_u32(img);
    // the bias of s into this thread's accumulator row / columns: the next skip sum starts
    // from it (once the accumulator's previous contents have been read)
    auto init_acc = [&]() {
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {
        const float4* b4 = reinterpret_cast<const float4*>(a.skip_bsum + e * 256 + hf * 128 + 32 * cc);
        float v[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 b = __ldg(b4 + q);
          v[4 * q] = b.x;
          v[4 * q + 1] = b.y;
          v[4 * q + 2] = b.z;
          v[4 * q + 3] = b.w;
        }
        tmem_st32(trow + hf * 128 + 32 * cc, v);
      }
      tc_fence_before();
      mbar_arrive(acc_init);
    };
    init_acc();
    // own half of an image: TMEM accumulator columns [0,256) + bias -> ReLU -> fp16 chunks
    // 4e .. 4e+3; then (sender) one bulk copy of those 64 KB into the peer's image
    const bool t2 = k == 0 && warp == 2 && lane == 0;
    auto own_half = [&](const float* bias) {
      epi_relu_image_smem(trow, r, hf * 128, 128, hf * 128, bias, si + (4 * e + 2 * hf) * kTile);
      trace_g(a, t2, 21);
      fence_proxy_async();  // generic smem writes -> MMA / bulk-copy reads
      tc_fence_before();
      mbar_arrive(own_ready);
      trace_g(a, t2, 22);
    };
    auto send_half = [&]() {
      named_bar_sync(1, 256);
      trace_g(a, t2, 23);
      if (warp == 2 && lane == 0)
        bulk_s2peer(mapa(img + 4 * e * kTile, peer), img + 4 * e * kTile, half_bytes,
                    mapa(peer_full, peer));
    };
    for (int i = 0; i < a.n_steps; ++i) {
      mbar_wait(acc_full, (uint32_t)i & 1);
      tc_fence_after();
      trace_g(a, k == 0 && warp == 2 && lane == 0, 14);
      own_half(nullptr);  // s (its bias came with the accumulator)
      send_half();
      trace_g(a, k == 0 && warp == 2 && lane == 0, 3);
      // head1 complete: own half of h (this block's s and the peer's s half are dead)
      mbar_wait(tacc, (uint32_t)(i * (sel_block ? 2 : 1)) & 1);
      tc_fence_after();
      trace_g(a, k == 0 && warp == 2 && lane == 0, 15);
      if (sel_block) {
        // block 1 may now overwrite chunks 4..7 of this image with its half of h
        if (warp == 2 && lane == 0) mbar_arrive_remote(mapa(a_free, peer));
        // the outgoing copy of this block's s half (chunks 0..3, about to take h) has landed
        // in block 1 and been consumed by its head1 (a DSMEM bulk copy's source read is only
        // known complete through the receiver)
        mbar_wait_cluster(s_free, (uint32_t)i & 1);
        own_half(hbias);
        trace_g(a, k == 0 && warp == 2 && lane == 0, 4);
        mbar_wait(tacc, 1);  // head2 (2i+1 & 1)
        mbar_wait(noise_ready, (uint32_t)i & 1);
        tc_fence_after();
        trace_g(a, k == 0 && warp == 2 && lane == 0, 5);
        const SelectArgs sel = sel_step(a.sel, a.t0, i);
        trace_g(a, t2, 28);
        epi_select(trow, r, hf, p * 128 + r, sel, xch, 256, true, t2 ? &a : nullptr,
                   pair_folds(a, i));
        trace_g(a, t2, 24);
        tc_fence_before();
        named_bar_sync(1, 256);
        // hand the classes to the chain first: the next step's skip accumulator (init_acc,
        // global bias loads + TMEM stores) is not needed before its layer 0 publishes z
        if (warp == 2 && lane == 0) {
          red_release_gpu(a.cls_ready + p, 1u);
          trace_g(a, k == 0, 6);
          if (i == a.n_steps - 2) trace_g(a, k == 0, 17);
        }
        if (i + 1 < a.n_steps) init_acc();
        trace_g(a, t2, 25);
      } else {
        // block 0's head1 is complete, so this block's outgoing s copy (chunks 4..7, about
        // to take h) has landed there; and this block's head1 has consumed block 0's s half
        if (warp == 2 && lane == 0) mbar_arrive_remote(mapa(s_free, peer));
        mbar_wait_cluster(a_free, (uint32_t)i & 1);
        own_half(hbias);  // h columns 256..511 into this image's chunks 4..7
        send_half();  // (before init_acc: block 0's head2 waits for this half of h)
        if (i + 1 < a.n_steps) init_acc();
      }
    }
  } else if (warp >= 10 && warp < 14) {
    // block 0: TMEM [256,512) of row r <- the logits bias (+ the step's Gumbel noise), added
    // to the logits by the selection
    const bool gumbel = a.sel.mode == FW_SAMPLE_GUMBEL;
    const int sub = warp & 3;
    const int r = sub * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(sub * 32) << 16);
    for (int i = 0; i < a.n_steps; ++i) {
      if (sel_block) {
        const uint32_t prefix = noise_prefix(a.sel.seed, (uint32_t)(a.sel.stream_offset + p * 128 + r),
                                             (uint32_t)(a.t0 + i));
        if (i > 0) wait_counter(a.cls_ready + p, (uint32_t)i);
#pragma unroll 1
        for (int cc = 0; cc < 8; ++cc) {
          float gn[32];
          const float4* b4 = reinterpret_cast<const float4*>(a.sel.bias + 32 * cc);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 b = __ldg(b4 + q);
            gn[4 * q] = b.x;
            gn[4 * q + 1] = b.y;
            gn[4 * q + 2] = b.z;
            gn[4 * q + 3] = b.w;
          }
          if (gumbel) {
#pragma unroll
            for (int j = 0; j < 32; ++j) gn[j] += gumbel_noise(prefix, 32 * cc + j);
          }
          tmem_st32(trow + 256 + 32 * cc, gn);
        }
        tc_fence_before();
        mbar_arrive(noise_ready);
      }
      if ((warp == 11 || warp == 12) && lane == 0) head_loads(i, warp - 10);
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync();  // no DSMEM traffic into a block that has exited
  if (warp == 1) tmem_dealloc(tmem, 512);
}

#include "chain_fold.cuh"
static_assert(fold::kSmem <= kChainSmem, "folded chain shared memory");
#include "chain_2sm.cuh"
static_assert(c2::kSmem <= kChainSmem, "2-SM chain shared memory");

// One launch per step: blocks [0, nchain) run the chain of one 64-stream tile each, blocks
// [nchain, nchain + nskip) the skip role (when fused; launched cooperatively so that all
// blocks are co-resident -- the skip blocks wait on the chain blocks).
__global__ void __launch_bounds__(kChainThreads, 1) step_kernel(ChainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  if ((int)blockIdx.x >= a.nchain) {
    // pair mode needs the 2-CTA cluster launch; a launch that lost its cluster attribute
    // (seen under the profiler's kernel replay) runs the global-memory tail instead
    if (a.pair_mode && cluster_size() == 2)
      tail_pair_role(a, smem, (int)blockIdx.x - a.nchain);
    else
      skip_role(a, smem, (int)blockIdx.x - a.nchain);
    return;
  }
  uint8_t* stA0 = smem + kOffA0;
  uint8_t* stA1 = smem + kOffA1;
  uint8_t* stB = smem + kOffB;
  uint8_t* stC = smem + kOffC;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBars);
  uint64_t* fullA0 = bars + 0;
  uint64_t* fullA1 = bars + 1;
  uint64_t* fullB = bars + 2;
  uint64_t* fullC = bars + 3;
  uint64_t* emptyA0 = bars + 4;
  uint64_t* emptyA1 = bars + 5;
  uint64_t* emptyB = bars + 6;
  uint64_t* emptyC = bars + 7;
  uint64_t* acc0_full = bars + 8;
  uint64_t* acc1_full = bars + 9;
  uint64_t* x_full = bars + 10;
  uint64_t* xd_ready = bars + 11;  // 128: queue warps (TMEM xd holds layer l's x_{t-d})
  uint64_t* x_pushed = bars + 12;  // 128: queue warps read xt (layer l's push issued)
  uint64_t* z_read = bars + 13;    // 128: queue warps read z (stash issued)
  uint64_t* xt_ready = bars + 14;  // 256: gate warps
  uint64_t* z0_ready = bars + 15;  // 256
  uint64_t* z1_ready = bars + 16;  // 256
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 17);
  uint64_t* xd_free = bars + 18;   // commit: this layer's x_{t-d} MMAs are done with TMEM xd
  uint64_t* z_stashed = bars + 21;  // 128: queue warps' z of this layer staged (or stored)
  uint64_t* stage_free = bars + 19;  // [2] publisher: the z staging image's bulk store is done
  uint64_t* probe = bars + 24;      // [6] trace only: commits after MMA groups (warp 14 stamps)
  const bool tracing = a.trace != nullptr && blockIdx.x == 0;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // split mode: the two CTAs of a cluster share one 64-stream tile, CTA `half` computing the
  // dilated N-half `half` (its z columns 64 half .. +63); both keep the full residual stream
  const bool split = a.split != 0;
  const int tile = split ? (int)blockIdx.x >> 1 : (int)blockIdx.x;
  const int half = split ? (int)(blockIdx.x & 1) : 0;
  const int L = a.L;
  const int G = a.n_steps * L;  // layers of all steps of this launch, in order
  // split: the peer's z half lands here (2 layer-parity buffers of [8 K-pieces][64 rows][16 B]
  // in the unused A1 stage), completing zpeer[parity]'s transaction count
  uint8_t* zpeer_buf = smem + kOffA1;
  uint64_t* zpeer = bars + 30;  // [2]

  if (threadIdx.x == 0) {
    for (int i = 0; i < 11; ++i) mbar_init(bars + i, 1);
    mbar_init(xd_ready, 128);
    mbar_init(x_pushed, 128);
    mbar_init(z_read, 128);
    mbar_init(xt_ready, 256);
    mbar_init(z0_ready, 256);
    mbar_init(z1_ready, 256);
    mbar_init(xd_free, 1);
    mbar_init(z_stashed, 128);
    for (int i = 0; i < 6; ++i) mbar_init(probe + i, 1);
    mbar_init(zpeer + 0, 1);
    mbar_init(zpeer + 1, 1);
    mbar_init(stage_free + 0, 1);
    mbar_init(stage_free + 1, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (split) cluster_sync();  // both halves' barriers exist before any z crosses
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0 && split) {  // ---- weight producer, split: A_half | B_half | C ----
      int gc = 0;
      for (int g = 0; g < G; ++g) {
        const int l = g % L;
        const uint8_t* wl = a.w + (size_t)l * kLayerBytes;
        const uint32_t ph = ((uint32_t)g & 1) ^ 1;
        mbar_wait(emptyA0, ph);
        mbar_arrive_expect_tx(fullA0, kStageA);
        bulk_g2s(stA0, wl + half * kStageA, kStageA, fullA0);
        mbar_wait(emptyB, ph);
        mbar_arrive_expect_tx(fullB, kStageB / 2);
        bulk_g2s(stB, wl + 2 * kStageA + half * (kStageB / 2), kStageB / 2, fullB);
        if (l + 1 < L) {
          mbar_wait(emptyC, ((uint32_t)gc & 1) ^ 1);
          mbar_arrive_expect_tx(fullC, kStageC);
          bulk_g2s(stC, wl + 2 * kStageA + kStageB, kStageC, fullC);
          ++gc;
        }
      }
    } else if (lane == 0) {  // ---- weight producer ----
      int gc = 0;  // res stages loaded (all but each step's top layer)
      for (int g = 0; g < G; ++g) {
        const int l = g % L;
        const uint8_t* wl = a.w + (size_t)l * kLayerBytes;  // A0 | A1 | B | C
        const uint32_t ph = ((uint32_t)g & 1) ^ 1;
        mbar_wait(emptyA0, ph);
        trace_at(a, l, T_PROD_A0, clock64());
        mbar_arrive_expect_tx(fullA0, kStageA);
        bulk_g2s(stA0, wl, kStageA, fullA0);
        mbar_wait(emptyA1, ph);
        trace_at(a, l, T_PROD_A1, clock64());
        mbar_arrive_expect_tx(fullA1, kStageA);
        bulk_g2s(stA1, wl + kStageA, kStageA, fullA1);
        mbar_wait(emptyB, ph);
        trace_at(a, l, T_PROD_B, clock64());
        mbar_arrive_expect_tx(fullB, kStageB);
        bulk_g2s(stB, wl + 2 * kStageA, kStageB, fullB);
        if (l + 1 < L) {
          mbar_wait(emptyC, ((uint32_t)gc & 1) ^ 1);
          trace_at(a, l, T_PROD_C, clock64());
          mbar_arrive_expect_tx(fullC, kStageC);
          bulk_g2s(stC, wl + 2 * kStageA + kStageB, kStageC, fullC);
          ++gc;
        }
      }
    }
  } else if (warp == 1 && split) {  // ---- MMA issuer, split mode: one N-half ----
    const uint32_t id = idesc_f16(kChainRows, 128);
    const uint32_t sa0 = smem_u32(stA0), sb = smem_u32(stB), sc = smem_u32(stC),
                   zp = smem_u32(zpeer_buf);
    auto mma_tmem_a = [&](uint32_t d, uint32_t a_col, uint32_t b_saddr) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_bf16_ta(d, a_col + kk * 8, sdesc_sw128(b_saddr + kk * 32), id, 1u);
    };
    // x_{t-d} taps of this half: initialise acc0 (stage A0), then free the operand
    auto xd_mma = [&]() {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16_ta(tmem, tmem + kColXd + 32 * c + 8 * kk, sdesc_sw128(sa0 + c * kChunk + kk * 32),
                      id, (c | kk) ? 1u : 0u);
      mma_commit(emptyA0);
      mma_commit(xd_free);
    };
    bool early = false;
    int gc = 0;
    for (int g = 0; g < G; ++g) {
      const int l = g % L;
      const uint32_t par = (uint32_t)g & 1;
      const bool nx = l + 1 < L, nxg = g + 1 < G;
      if (!early) {
        mbar_wait(xd_ready, par);
        tc_fence_after();
        mbar_wait(fullA0, par);
        tc_fence_after();
        if (elect_one()) xd_mma();
        __syncwarp();
      }
      early = false;
      mbar_wait(xt_ready, par);
      tc_fence_after();
      mbar_wait(fullB, par);
      tc_fence_after();
      if (elect_one()) {
        mma_tmem_a(tmem, tmem + kColXt + 0, sb + 0 * kChunk);
        mma_tmem_a(tmem, tmem + kColXt + 32, sb + 1 * kChunk);
      }
      __syncwarp();
      if (g > 0) mbar_wait(z_read, par ^ 1);  // the previous layer's stash has read z
      if (elect_one()) {
        mma_commit(acc0_full);
        mma_commit(emptyB);
      }
      __syncwarp();
      // own z half (TMEM) -> residual K-chunk `half`
      mbar_wait(z0_ready, par);
      tc_fence_after();
      if (nx) {
        mbar_wait(fullC, (uint32_t)gc & 1);
        tc_fence_after();
        if (elect_one()) mma_tmem_a(tmem + kP1 + kColX, tmem + kP1 + kColZ + 32 * half, sc + half * kChunk);
        __syncwarp();
      }
      // acc0 was read by the gate: the next layer's x_{t-d} (the next step's layer 0 too)
      if (nxg) {
        mbar_wait(xd_ready, par ^ 1);
        tc_fence_after();
        mbar_wait(fullA0, par ^ 1);
        tc_fence_after();
        if (elect_one()) xd_mma();
        __syncwarp();
        early = true;
      }
      // the peer's z half (SMEM, bulk-copied through DSMEM) -> residual K-chunk 1 - half
      const int zb = g & 1;
      if (elect_one()) mbar_arrive_expect_tx(zpeer + zb, 8192);
      __syncwarp();
      // cluster-scope acquire: the peer's st.async writes complete on this barrier with
      // cluster-scope release; then the proxy fence orders them (generic proxy) before this
      // thread's MMA reads (async proxy)
      mbar_wait_cluster(zpeer + zb, (uint32_t)(g >> 1) & 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_after();
      if (nx) {
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // K = 16 (2 pieces) per MMA, half h = kk / 2
            mma_bf16(tmem + kP1 + kColX,
                     sdesc_plain(zp + zb * 8192 + (kk >> 1) * 4096 + (kk & 1) * 256, 128, 512),
                     sdesc_sw128(sc + (1 - half) * kChunk + kk * 32), id, 1u);
          mma_commit(emptyC);
        }
        __syncwarp();
        mbar_wait(x_pushed, par);
        if (elect_one()) mma_commit(x_full);
        __syncwarp();
        ++gc;
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer (whole warp; MMAs under elect.sync) ----
    const uint32_t id = idesc_f16(kChainRows, 128);
    const uint32_t sa0 = smem_u32(stA0), sa1 = smem_u32(stA1), sb = smem_u32(stB),
                   sc = smem_u32(stC);
    long long wwait = 0;
    auto wait_w = [&](uint64_t* bar, uint32_t par) {
      const long long w0 = clock64();
      mbar_wait(bar, par);
      wwait += clock64() - w0;
      tc_fence_after();
    };
    // one 64-K chunk: A from TMEM columns a_col.. (K 16 per 8 packed columns), B image
    auto mma_tmem_a = [&](uint32_t d, uint32_t a_col, uint32_t b_saddr) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_bf16_ta(d, a_col + kk * 8, sdesc_sw128(b_saddr + kk * 32), id, 1u);
    };
    // x_{t-d} half hh (initialises acc hh): A = TMEM xd, B = stage A_hh chunks
    auto xd_half = [&](int hh) {
      const uint32_t acc = tmem + 128 * hh, sa = hh ? sa1 : sa0;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16_ta(acc, tmem + kColXd + 32 * c + 8 * kk, sdesc_sw128(sa + c * kChunk + kk * 32),
                      id, (c | kk) ? 1u : 0u);
      mma_commit(hh ? emptyA1 : emptyA0);
    };
    bool early[2] = {false, false};
    int gc = 0;  // res layers issued (parity of fullC)
    for (int g = 0; g < G; ++g) {
      const int l = g % L;
      const uint32_t par = (uint32_t)g & 1;
      const bool nx = l + 1 < L, nxg = g + 1 < G;
      if (lane == 0) trace_at(a, l, T_H0_EARLY, (early[0] ? 1 : 0) + (early[1] ? 2 : 0));
      if (!early[0] || !early[1]) {
        mbar_wait(xd_ready, par);
        tc_fence_after();
      }
      if (!early[0]) {
        wait_w(fullA0, par);
        if (elect_one()) xd_half(0);
        __syncwarp();
      }
      if (lane == 0) trace_at(a, l, T_MMA_XD, clock64());
      // x_t half 0: stage B chunks 0, 1
      mbar_wait(xt_ready, par);
      if (lane == 0) trace_at(a, l, T_MMA_XT, clock64());
      tc_fence_after();
      wait_w(fullB, par);
      if (elect_one()) {
        mma_tmem_a(tmem + 0, tmem + kColXt + 0, sb + 0 * kChunk);
        mma_tmem_a(tmem + 0, tmem + kColXt + 32, sb + 1 * kChunk);
      }
      __syncwarp();
      // the gate warps rewrite z after acc0_full: the previous layer's stash has read it
      if (g > 0) mbar_wait(z_read, par ^ 1);
      if (elect_one()) {
        mma_commit(acc0_full);
        if (tracing) mma_commit(probe + 0);
      }
      __syncwarp();
      if (lane == 0) trace_at(a, l, T_MMA_ACC0, clock64());
      if (!early[1]) {
        wait_w(fullA1, par);
        if (elect_one()) {
          xd_half(1);
          mma_commit(xd_free);
        }
        __syncwarp();
      }
      if (tracing && elect_one()) mma_commit(probe + 1);
      __syncwarp();
      early[0] = early[1] = false;
      if (elect_one()) {
        mma_tmem_a(tmem + 128, tmem + kColXt + 0, sb + 2 * kChunk);
        mma_tmem_a(tmem + 128, tmem + kColXt + 32, sb + 3 * kChunk);
        mma_commit(acc1_full);
        mma_commit(emptyB);
        if (tracing) mma_commit(probe + 2);
      }
      __syncwarp();
      if (lane == 0) trace_at(a, l, T_MMA_ACC1, clock64());
      // z halves: res MMA (all but the top layer), A = z and D = x in plane P1
      mbar_wait(z0_ready, par);
      if (lane == 0) trace_at(a, l, T_MMA_Z0, clock64());
      tc_fence_after();
      if (nx) {
        wait_w(fullC, (uint32_t)gc & 1);
        if (elect_one()) mma_tmem_a(tmem + kP1 + kColX, tmem + kP1 + kColZ + 0, sc + 0 * kChunk);
        __syncwarp();
      }
      if (tracing && elect_one()) mma_commit(probe + 3);
      __syncwarp();
      if (nxg) {
        // acc0 is free (gate half 0 done): the next layer's x_{t-d} N-half 0 (the next
        // step's layer 0 included -- it needs no input class). Its operand follows this
        // layer's x_{t-d} MMAs (xd_free) within a few hundred cycles and its weights loaded a
        // layer ago, so waiting here costs little; issued after x_full instead it would sit
        // in front of the next layer's x_t MMAs.
        mbar_wait(xd_ready, par ^ 1);
        tc_fence_after();
        wait_w(fullA0, par ^ 1);
        if (elect_one()) xd_half(0);
        __syncwarp();
        early[0] = true;
      }
      if (tracing && elect_one()) mma_commit(probe + 4);
      __syncwarp();
      mbar_wait(z1_ready, par);
      if (lane == 0) trace_at(a, l, T_MMA_Z1, clock64());
      tc_fence_after();
      if (nx) {
        if (elect_one()) {
          mma_tmem_a(tmem + kP1 + kColX, tmem + kP1 + kColZ + 32, sc + 1 * kChunk);
          mma_commit(emptyC);
        }
        __syncwarp();
        if (tracing && elect_one()) mma_commit(probe + 5);
        __syncwarp();
        // the gate warps rewrite xt after x_full: this layer's push has read it
        mbar_wait(x_pushed, par);
        if (elect_one()) mma_commit(x_full);
        __syncwarp();
        ++gc;
        if (lane == 0) trace_at(a, l, T_MMA_XFULL, clock64());
        // (x_{t-d} half 1 stays in the layer: issued here it would hold the tensor pipe
        // and this warp when the next layer's x_t MMAs become ready)
      } else {
        if (tracing && elect_one()) mma_commit(probe + 5);
        __syncwarp();
      }
      if (lane == 0) trace_at(a, l, T_MMA_WWAIT, wwait);
    }
  } else if (warp >= kQueueWarp0 && warp < kQueueWarp0 + 4) {
    // ---- queue warps: lanes 0..15 own rows 16q..16q+15 (32x32b accesses; lanes 16..31
    // see plane P1) ----
    const int q = warp & 3;
    const int r = q * 16 + (lane & 15);
    const bool act = lane < 16;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const bool pf = warp == kQueueWarp0 && lane == 0;
    const bool tq = pf;
    const uint8_t* qtile = a.queue + (size_t)(tile >> 1) * 2 * kSlotBytes + (tile & 1) * kChainRows * 16;
    auto qb = [&](int g) { return qbase_of(a, g / L, g % L); };
    // pops: each thread copies its own row of layer g's slot into staging buffer Xq[g & 1]
    // (16 x 16 B, cp.async) two layers ahead -- no registers held across layers, and the
    // same thread wrote that row with its push, so plain program order covers the reuse of
    // ring slots within a launch (the copy of layer g+2 is issued before the push of layer
    // g: with L >= 3, tc_supported, those are different layers). K-piece j (K 8j..8j+7) of row r is the 16 bytes at
    // (j * 64 + r) * 16: packed words 4j .. 4j+3 of the operand row.
    uint8_t* xq = smem + kOffXq;
    auto load_slot = [&](int g) {
      if (act) {
        const uint8_t* src = qtile + qb(g) + (size_t)r * 16;
        const uint32_t dst = smem_u32(xq + (g & 1) * kSlotBytes) + (uint32_t)r * 16;
#pragma unroll
        for (int j = 0; j < 16; ++j) cp_async16(dst + (uint32_t)j * kChainRows * 16, src + (size_t)j * kPairRows * 16);
      }
      cp_async_commit();
    };
    // row r of layer g's x_{t-d} -> TMEM xd (lanes 16..31 store zeros into P1's scratch
    // columns), then the copy of layer g+2 into the freed buffer
    auto store_xd = [&](int g) {
      cp_async_wait<1>();  // layer g's copies done (g+1's may be in flight)
      const uint32_t src = smem_u32(xq + (g & 1) * kSlotBytes) + (uint32_t)r * 16;
      uint32_t xd[64];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        uint32_t v0 = 0, v1 = 0, v2 = 0, v3 = 0;
        if (act)
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                       : "r"(src + (uint32_t)j * kChainRows * 16));
        xd[4 * j] = v0;
        xd[4 * j + 1] = v1;
        xd[4 * j + 2] = v2;
        xd[4 * j + 3] = v3;
      }
      tmem_st32(trow + kColXd, *reinterpret_cast<float(*)[32]>(xd));
      tmem_st32(trow + kColXd + 32, *reinterpret_cast<float(*)[32]>(xd + 32));
      tc_fence_before();
      mbar_arrive(xd_ready);
      if (g + 2 < G) load_slot(g + 2);
      else cp_async_commit();  // keep one group per layer for the wait count
    };
    // 64 TMEM columns of packed fp16 pairs (32x32b: lanes 0..15 read P0, 16..31 read P1)
    // -> 16 K-pieces at dst (+ j * stride rows) from the lanes with `mine`
    // (split: only the 16-column groups c of this CTA's half; the peer does the others)
    const int c_lo = split ? 2 * half : 0, c_hi = split ? 2 * half + 2 : 4;
    auto tmem_to_pieces = [&](uint32_t col, uint4* dst, int stride, bool mine) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c < c_lo || c >= c_hi) continue;
        float v[16];
        tmem_ld16(trow + col + 16 * c, v);
        tmem_wait_ld();
        if (mine) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            dst[(4 * c + j) * stride] =
                make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                           __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
        }
      }
    };
    uint32_t zseen = 0;  // tail reads of the z ring observed (lane 0)
    load_slot(0);
    if (G > 1) load_slot(1);
    else cp_async_commit();
    store_xd(0);
    for (int g = 0; g < G; ++g) {
      const int l = g % L;
      const uint32_t par = (uint32_t)g & 1;
      // the tail's z-ring read count, loaded now and looked at before the stash below
      uint32_t zpeek = 0;
      if (a.zfree != nullptr && lane == 0 && g >= a.zring) zpeek = ld_relaxed_gpu(a.zfree + (tile >> 1));
      // push x_l (P0 xt columns, lanes 0..15) into ring slot (t mod d_l); this thread's pop
      // of its row of that slot completed before store_xd of this layer
      mbar_wait(xt_ready, par);
      tc_fence_after();
      tmem_to_pieces(kColXt, reinterpret_cast<uint4*>(const_cast<uint8_t*>(qtile) + qb(g)) + r,
                     kPairRows, act);
      tc_fence_before();
      mbar_arrive(x_pushed);
      if (tq) trace_at(a, l, T_Q_LOAD, clock64());
      // x_{t-d} of the next layer -> TMEM xd once this layer's x_{t-d} MMAs are done
      if (g + 1 < G) {
        mbar_wait(xd_free, par);
        if (tq) trace_at(a, (g + 1) % L, T_G0_STS, clock64());
        tc_fence_after();
        store_xd(g + 1);
        if (tq) trace_at(a, (g + 1) % L, T_Q_XD, clock64());
      }
      // z stash of layer g (P1 z columns: lanes 16..31 of the quadrant hold the rows) into
      // ring slot g % zring, once the tail blocks have read layer g - zring from it (the
      // count observed last usually covers several layers ahead)
      if (a.zfree != nullptr && g >= a.zring) {
        const uint32_t need = (uint32_t)a.ztail * (uint32_t)(g - a.zring + 1);
        if (lane == 0) {
          zseen = max(zseen, zpeek);  // the count read at the top of this layer
          if (zseen < need) zseen = wait_counter_val(a.zfree + (tile >> 1), need);
        }
        __syncwarp();
      }
      mbar_wait(split ? z0_ready : z1_ready, par);
      tc_fence_after();
      if (a.zflag != nullptr) {
        // fused: z into a shared-memory staging image; the publisher bulk-stores it into the
        // stash, waits for the store's completion and only then releases the counter the
        // tail blocks acquire (per-thread global stores published by another warp's release
        // were seen stale by the tail now and then: the release covers only its own warp)
        if (g >= 2) mbar_wait(stage_free + (g & 1), (uint32_t)(((g >> 1) - 1) & 1));
        tmem_to_pieces(kColZ, reinterpret_cast<uint4*>(smem + kOffZs + (g & 1) * kSlotBytes) + r,
                       kChainRows, !act);
        fence_proxy_async();  // generic shared writes -> the bulk store (async proxy)
      } else {
        tmem_to_pieces(kColZ, zstash_rows(a.zimg, tile, a.zring, g % a.zring) + r, 2 * kChainRows, !act);
      }
      tc_fence_before();
      mbar_arrive(z_read);
      mbar_arrive(z_stashed);
      if (tq) trace_at(a, l, T_SP2, clock64());
      if (tq) trace_at(a, l, T_SP1, clock64());
      if (tq) trace_at(a, l, T_SP3, clock64());
    }
  } else if (warp == 14) {
    // ---- publisher: z_l of this tile -> the tail blocks (release of the stash stores) ----
    if (a.zflag != nullptr) {
      // one K-piece (1 KB) per lane: a thread's bulk copies run one after another, several
      // threads' overlap
      const int j0 = split ? 8 * half : 0, j1 = split ? 8 * half + 8 : 16;  // K-pieces
      const int j = j0 + lane;
      for (int g = 0; g < G; ++g) {
        mbar_wait(z_stashed, (uint32_t)g & 1);
        if (j < j1) {
          const uint8_t* src = smem + kOffZs + (g & 1) * kSlotBytes;
          uint8_t* dst = reinterpret_cast<uint8_t*>(zstash_rows(a.zimg, tile, a.zring, g % a.zring));
          bulk_s2g(dst + j * 2048, src + j * 1024, 1024);
          bulk_commit();
          bulk_wait0();             // this piece is in the stash
          fence_proxy_async_all();  // async-proxy writes before the release below
        }
        __syncwarp();
        if (lane == 0) {
          red_release_gpu(a.zflag + (tile >> 1), 1u);
          mbar_arrive(stage_free + (g & 1));
        }
        __syncwarp();
      }
    }
  } else if (warp == 15) {
    if (lane == 0 && tracing && !split) {  // (the split MMA issuer commits no probes)
      // trace: completion times of the MMA groups (probe commits, in pipe order)
      for (int g = 0; g < G; ++g)
        for (int k = 0; k < 6; ++k) {
          mbar_wait(probe + k, (uint32_t)g & 1);
          trace_at(a, g % L, 32 + k, clock64());
        }
    }
  } else if (warp >= 2 && warp < 10) {
    // ---- gate warps: quadrant q, half h; 16x64b accesses: lane t holds row
    // 16q + (t>>2) + 8(t&1), columns of parity (t>>1)&1 ----
    const int q = warp & 3, h = (warp - 2) >> 2;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const int pc = (lane >> 1) & 1;
    const int row = q * 16 + (lane >> 2) + 8 * (lane & 1);
    const bool tr = (warp == 2 && lane == 0);
    // pack own fp16 pairs (v[2i], v[2i+1]) -- columns 4i+pc, 4i+2+pc -- and complete the
    // operand pairs with the partner lane (t ^ 2): parity 0 keeps the low halves (packed
    // column 2i), parity 1 the high halves (packed column 2i+1)
    auto pair_up = [&](uint32_t w) {
      const uint32_t o = __shfl_xor_sync(0xffffffffu, w, 2);
      return pc == 0 ? __byte_perm(w, o, 0x5410) : __byte_perm(o, w, 0x7632);
    };
    int gx = 0;  // x_full phases seen
    for (int g = 0; g < G; ++g) {
      const int i = g / L, l = g % L;
      const uint32_t par = (uint32_t)g & 1;
      if (l == 0) trace_g(a, tr, 0);
      if (tr) trace_at(a, l, T_EPI_A, clock64());
      // x_l channels 64h + 2j + pc (j < 32): the embedding at l = 0, else the P1 residual
      // stream (+ the pending bias)
      uint32_t xv[32];
      if (l == 0) {
        // step i's input class: written by the pair's selection of step i-1
        if (i > 0) wait_counter(a.cls_ready + (tile >> 1), (uint32_t)i);
        trace_g(a, tr, 16);
        const int c = clamp_class(a.cls[tile * kChainRows + row], 256);  // tc_supported: A = 256
        if (tr) {
          asm volatile("" ::"r"(c) : "memory");
          trace_g(a, true, 19);
        }
        // the row's 64 channels 64h.. as 8 float4 loads per lane pair (t, t^2): pair lane pc
        // loads floats 8q + 4pc .. +3 (one 32-byte sector per pair and load), then each lane
        // trades the two values of the partner's parity
        const float4* e4 = reinterpret_cast<const float4*>(a.embed + (size_t)c * kR + 64 * h) + pc;
        float4 ev[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) ev[q] = __ldg(e4 + 2 * q);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float s0 = pc ? ev[q].x : ev[q].y, s1 = pc ? ev[q].z : ev[q].w;
          const float r0 = __shfl_xor_sync(0xffffffffu, s0, 2), r1 = __shfl_xor_sync(0xffffffffu, s1, 2);
          xv[4 * q] = __float_as_uint(pc ? r0 : ev[q].x);
          xv[4 * q + 1] = __float_as_uint(pc ? r1 : ev[q].z);
          xv[4 * q + 2] = __float_as_uint(pc ? ev[q].y : r0);
          xv[4 * q + 3] = __float_as_uint(pc ? ev[q].w : r1);
        }
        if (tr) {
          asm volatile("" ::"r"(xv[0]), "r"(xv[31]) : "memory");
          trace_g(a, true, 20);
        }
        tmem_st_16x64b_x32(trow + kP1 + kColX + 64 * h, xv);
      } else {
        mbar_wait(x_full, (uint32_t)gx & 1);
        ++gx;
        if (tr) trace_at(a, l, T_EPI_XFULL, clock64());
        tc_fence_after();
        tmem_ld_16x64b_x32(trow + kP1 + kColX + 64 * h, xv);
        tmem_wait_ld();
        if (a.has_res_bias) {
          const float* rb = a.res_b + (size_t)(l - 1) * kR + 64 * h + pc;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            xv[j] = __float_as_uint(__uint_as_float(xv[j]) + __ldg(rb + 2 * j));
          tmem_st_16x64b_x32(trow + kP1 + kColX + 64 * h, xv);
        }
      }
      {
        uint32_t xp[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          xp[i] = pair_up(pack_h2(__uint_as_float(xv[2 * i]), __uint_as_float(xv[2 * i + 1])));
        tmem_st_16x64b_x16(trow + kColXt + 32 * h, xp);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(xt_ready);
      if (tr) trace_at(a, l, T_EPI_XT, clock64());
      if (l == 0) trace_g(a, tr, 18);
      // gate of N-half hh: this lane's 16 z columns 64hh + 32h + 2j + pc, j < 16 (split: the
      // CTA's one half, accumulated in acc0)
      const float* bd = a.dil_b + (size_t)l * 2 * kD;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if (split && hh > 0) break;
        const int zh = split ? half : hh;  // the z columns' half
        mbar_wait(hh == 0 ? acc0_full : acc1_full, par);
        if (tr) trace_at(a, l, hh == 0 ? T_EPI_ACC0 : T_EPI_ACC1, clock64());
        tc_fence_after();
        uint32_t ts[32];  // tanh columns | sigmoid columns
        tmem_ld_16x64b_x16_2(trow + 128 * hh + 32 * h, trow + 128 * hh + 64 + 32 * h, ts);
        if (tr) trace_at(a, l, hh == 0 ? T_G0_LD : T_G1_LD, clock64());
        float at[16], as[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          at[j] = __uint_as_float(ts[j]);
          as[j] = __uint_as_float(ts[16 + j]);
        }
        if (a.has_dil_bias) {
          const int j0 = 64 * zh + 32 * h + pc;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            at[j] += __ldg(bd + j0 + 2 * j);
            as[j] += __ldg(bd + kD + j0 + 2 * j);
          }
        }
        // z = tanh(a) * sigmoid(b) with sigmoid(b) = 0.5 + 0.5 tanh(b / 2), evaluated for
        // an element pair in packed fp16 (z's operand precision)
        uint32_t zw[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          zw[i] = pair_up(gate2_h2(at[2 * i], at[2 * i + 1], as[2 * i], as[2 * i + 1]));
        if (tr) {
          asm volatile("" ::"r"(zw[0]), "r"(zw[7]) : "memory");
          trace_at(a, l, hh == 0 ? T_G0_MATH : T_G1_MATH, clock64());
        }
        tmem_st_16x64b_x8(trow + kP1 + kColZ + 32 * zh + 16 * h, zw);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(hh == 0 ? z0_ready : z1_ready);
        if (split) {
          // this half's z -> the peer's residual K-chunk: 16-byte K-pieces (8 z columns of
          // one row) stored straight into the peer's operand image [h][8-row group][4 pieces]
          // [8 rows][16 B] (K-adjacent core matrices 128 B apart, 8-row groups 512 B apart)
          // by st.async, each completing 16 bytes of the peer's zpeer transaction count -- no
          // staging, no barrier across the gate warps, no bulk-copy queue. Piece m of this
          // lane group (z columns 32h + 8m .. +7) = packed columns 4m .. 4m+3, held
          // alternately by this lane (parity pc) and its partner t ^ 2.
          uint32_t pw[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) pw[i] = __shfl_xor_sync(0xffffffffu, zw[i], 2);
          const int zb = g & 1;
          const int rg = row >> 3, r8 = row & 7;  // 8-row group, row inside it
          const uint32_t zbar = mapa(zpeer + zb, (uint32_t)(half ^ 1));
          uint8_t* stage = smem + kOffB + 32768 + zb * 8192;  // (stage B's unused half)
#pragma unroll
          for (int mm = 0; mm < 2; ++mm) {
            const int m = 2 * pc + mm;
            const uint32_t lo0 = pc == 0 ? zw[2 * m] : pw[2 * m], hi0 = pc == 0 ? pw[2 * m] : zw[2 * m];
            const uint32_t lo1 = pc == 0 ? zw[2 * m + 1] : pw[2 * m + 1],
                           hi1 = pc == 0 ? pw[2 * m + 1] : zw[2 * m + 1];
            const uint32_t off = (uint32_t)(h * 4096 + rg * 512 + m * 128 + r8 * 16);
            if (kSplitBulk) {
              st_shared_v4(smem_u32(stage + off), lo0, hi0, lo1, hi1);
            } else {
              asm volatile(
                  "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(
                      mapa(zpeer_buf + zb * 8192 + off, (uint32_t)(half ^ 1))),
                  "r"(lo0), "r"(hi0), "r"(lo1), "r"(hi1), "r"(zbar)
                  : "memory");
            }
          }
          if (kSplitBulk) {  // the warp's 16 rows x 4 pieces: one contiguous 1 KB block
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              const uint32_t off = (uint32_t)(h * 4096 + q * 1024);
              bulk_s2peer(mapa(zpeer_buf + zb * 8192 + off, (uint32_t)(half ^ 1)), stage + off, 1024, zbar);
            }
          }
        }
      }
      if (l == L - 1) trace_g(a, tr, 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (split) cluster_sync();  // no DSMEM copy into a CTA that has exited
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// The folded chain (FW_CHAIN_FOLD=1, chain_fold.cuh) as its own kernel, so the default step
// kernel's code and register allocation are those the race checks ran on.
__global__ void __launch_bounds__(kChainThreads, 1) step_kernel_fold(ChainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  if ((int)blockIdx.x >= a.nchain) {
    if (a.pair_mode && cluster_size() == 2)
      tail_pair_role(a, smem, (int)blockIdx.x - a.nchain);
    else
      skip_role(a, smem, (int)blockIdx.x - a.nchain);
    return;
  }
  chain_fold_role(a, smem);
}

// The 2-SM chain (chain_2sm.cuh) with the same tail roles.
__global__ void __launch_bounds__(kChainThreads, 1) step_kernel_2sm(ChainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  if ((int)blockIdx.x >= a.nchain) {
    if (a.pair_mode && cluster_size() == 2)
      tail_pair_role(a, smem, (int)blockIdx.x - a.nchain);
    else
      skip_role(a, smem, (int)blockIdx.x - a.nchain);
    return;
  }
  chain_2sm_role(a, smem);
}

// The folded 2-SM chain (FW_CHAIN_2SM=2, chain_2sm.cuh chain_2sf_role) with the same tails.
__global__ void __launch_bounds__(kChainThreads, 1) step_kernel_2sf(ChainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  if ((int)blockIdx.x >= a.nchain) {
    if (a.pair_mode && cluster_size() == 2)
      tail_pair_role(a, smem, (int)blockIdx.x - a.nchain);
    else
      skip_role(a, smem, (int)blockIdx.x - a.nchain);
    return;
  }
  chain_2sf_role(a, smem);
}

