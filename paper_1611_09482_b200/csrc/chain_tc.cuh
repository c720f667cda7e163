// Chain kernel of the tcgen05 path (included by cell_tc.cu): one 128-stream tile per
// CTA, the dependent chain of all L dilated layers of one generation step.
//
// Per layer l (a = W0 x_l[t] + W1 x_l[t-d] + b, z = tanh(a[:D]) * sigmoid(a[D:]),
// x_{l+1} = x_l + W_res z + b_res; the skip/head work is deferred to big-K GEMMs):
//
//   TMEM (512 columns x 128 lanes, lane = stream row):
//     [0,128)    acc0  dil N-half 0: tanh rows 0..63 | sigmoid rows 0..63
//     [128,256)  acc1  dil N-half 1: tanh rows 64..127 | sigmoid rows 64..127
//     [256,384)  x     residual stream x_l, fp32; the res MMA accumulates onto it
//     [384,448)  xt/z  fp16 x_l[t] operand of the dilated MMAs, then (once those are done)
//                      the fp16 z operand of the res MMA -- packed pairs
//     [448,512)  xd    fp16 x_l[t-d] operand
//   Every MMA takes its A operand from TMEM: an A operand in shared memory costs the
//   tensor pipe ~107 instead of ~72 cycles per 128x128x16 MMA (tools/mma_latency.cu), and
//   shared-memory bandwidth is what the weight stream needs. SMEM holds only the weight
//   stages A0 / A1 (32 KB each: the x_{t-d} K-chunks of N-half 0 / 1), B (64 KB: the x_t
//   K-chunks of both halves) and C (32 KB: res), one bulk copy each per layer (the copy
//   engine costs ~500 cycles per operation almost regardless of size, tools/ring_bw.cu).
//
//   Queue slots hold x_l in fp16 (the precision the MMA consumes), 32 KB per tile laid out
//   [16 K-pieces][128 rows][8 fp16] so that a warp's 16-byte accesses to one K-piece of 32
//   consecutive rows are 512 contiguous bytes. The z stash for the skip GEMM uses the same
//   layout per (tile, layer) -- the no-swizzle K-major UMMA layout (sdesc_plain).
//
//   warp 0  lane 0  weight producer (stages A0, A1, B, C in consumption order)
//   warp 1          MMA issuer: the converged warp issues under elect.sync (tools/mma_rate.cu)
//   warps 2..9      gate warps (row r = 32*(warp%4)+lane, column half h = (warp-2)/4):
//                   x_l -> xt, then per N-half the gate of 32 z columns of row r
//   warps 10..13    queue warps (one stream row each), all HBM traffic of the activations:
//                   push x_l (TMEM xt -> ring slot), x_{t-d} of layer l+1 (registers, loaded
//                   a layer ahead) -> TMEM xd once layer l's x_{t-d} MMAs are done, z stash
//                   (TMEM z -> HBM); L2 prefetch of the slot two layers ahead
//
// MMA issue order per layer: [xd_ready] x_{t-d} N-half 0 (normally issued during the
// previous layer) -> [xt_ready] x_t N-half 0 -> acc0_full -> x_{t-d} N-half 1 -> x_t
// N-half 1 -> acc1_full -> [z0_ready] res K-chunk 0, next layer's x_{t-d} N-half 0 if its
// operands are in -> [z1_ready] res K-chunk 1 -> [z_read] x_full.

constexpr int kChainThreads = 448;
constexpr int kQueueWarp0 = 10;
constexpr uint32_t kColX = 256, kColXt = 384, kColZ = 384, kColXd = 448;
constexpr uint32_t kSlotBytes = 32768;  // one tile's ring slot: [16 K-pieces][128 rows][8 fp16]
constexpr uint32_t kStageA = 32768, kStageB = 65536, kStageC = 32768;
constexpr uint32_t kOffA0 = 0, kOffA1 = kOffA0 + kStageA,
                   kOffB = kOffA1 + kStageA, kOffC = kOffB + kStageB,
                   kOffBars = kOffC + kStageC;
constexpr size_t kChainSmem = 1024 + kOffBars + 256;

__global__ void __launch_bounds__(kChainThreads, 1) chain_kernel(ChainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
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
  uint64_t* z_read = bars + 13;    // 128: queue warps read the z columns (stash issued)
  uint64_t* xt_ready = bars + 14;  // 256: gate warps
  uint64_t* z0_ready = bars + 15;  // 256
  uint64_t* z1_ready = bars + 16;  // 256
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 17);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int L = a.L;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 11; ++i) mbar_init(bars + i, 1);
    mbar_init(xd_ready, 128);
    mbar_init(x_pushed, 128);
    mbar_init(z_read, 128);
    mbar_init(xt_ready, 256);
    mbar_init(z0_ready, 256);
    mbar_init(z1_ready, 256);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ---- weight producer ----
      for (int l = 0; l < L; ++l) {
        const uint8_t* wl = a.w + (size_t)l * kLayerBytes;  // A0 | A1 | B | C
        const uint32_t ph = ((uint32_t)l & 1) ^ 1;
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
          mbar_wait(emptyC, ph);
          trace_at(a, l, T_PROD_C, clock64());
          mbar_arrive_expect_tx(fullC, kStageC);
          bulk_g2s(stC, wl + 2 * kStageA + kStageB, kStageC, fullC);
        }
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer (whole warp; MMAs under elect.sync) ----
    const uint32_t id = idesc_f16(128, 128);
    const uint32_t sa0 = smem_u32(stA0), sa1 = smem_u32(stA1),
                   sb = smem_u32(stB), sc = smem_u32(stC);
    long long wwait = 0;
    auto wait_w = [&](uint64_t* bar, uint32_t par) {
      const long long w0 = clock64();
      mbar_wait(bar, par);
      wwait += clock64() - w0;
      tc_fence_after();
    };
    // one 64-K chunk: A from TMEM columns a_col.., B image at b_saddr
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
    // warp-uniform non-blocking probe of layer lx's x_{t-d} operand and stage A0
    auto xd_h0_ready = [&](int lx) {
      const uint32_t pn = (uint32_t)lx & 1;
      int ok = lane == 0 ? (mbar_test(xd_ready, pn) && mbar_test(fullA0, pn)) : 0;
      return __shfl_sync(0xffffffffu, ok, 0) != 0;
    };
    bool h0_early = false;
    for (int l = 0; l < L; ++l) {
      const uint32_t par = (uint32_t)l & 1;
      const bool nx = l + 1 < L;
      if (lane == 0) trace_at(a, l, T_H0_EARLY, h0_early ? 1 : 0);
      if (!h0_early) {
        mbar_wait(xd_ready, par);
        tc_fence_after();
        wait_w(fullA0, par);
        if (elect_one()) xd_half(0);
        __syncwarp();
      }
      if (lane == 0) trace_at(a, l, T_MMA_XD, clock64());
      h0_early = false;
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
      if (elect_one()) mma_commit(acc0_full);
      __syncwarp();
      if (lane == 0) trace_at(a, l, T_MMA_ACC0, clock64());
      // x_{t-d} half 1 + x_t half 1
      wait_w(fullA1, par);
      if (elect_one()) {
        xd_half(1);
        mma_tmem_a(tmem + 128, tmem + kColXt + 0, sb + 2 * kChunk);
        mma_tmem_a(tmem + 128, tmem + kColXt + 32, sb + 3 * kChunk);
        mma_commit(acc1_full);
        mma_commit(emptyB);
      }
      __syncwarp();
      if (lane == 0) trace_at(a, l, T_MMA_ACC1, clock64());
      // z halves: res MMA (all but the top layer), A = z columns in TMEM
      mbar_wait(z0_ready, par);
      if (lane == 0) trace_at(a, l, T_MMA_Z0, clock64());
      tc_fence_after();
      if (nx) {
        wait_w(fullC, par);
        if (elect_one()) mma_tmem_a(tmem + kColX, tmem + kColZ + 0, sc + 0 * kChunk);
        __syncwarp();
        // acc0 is free (gate half 0 done): start layer l+1's x_{t-d} N-half 0 now if its
        // operand and weights are already in place -- never wait for them here
        if (xd_h0_ready(l + 1)) {
          tc_fence_after();
          if (elect_one()) xd_half(0);
          __syncwarp();
          h0_early = true;
        }
      }
      mbar_wait(z1_ready, par);
      if (lane == 0) trace_at(a, l, T_MMA_Z1, clock64());
      tc_fence_after();
      if (nx) {
        if (elect_one()) {
          mma_tmem_a(tmem + kColX, tmem + kColZ + 32, sc + 1 * kChunk);
          mma_commit(emptyC);
        }
        __syncwarp();
        // the gate warps rewrite the xt/z columns after x_full: the z stash has read them
        mbar_wait(z_read, par);
        if (elect_one()) mma_commit(x_full);
        __syncwarp();
        if (lane == 0) trace_at(a, l, T_MMA_XFULL, clock64());
        if (!h0_early && xd_h0_ready(l + 1)) {
          tc_fence_after();
          if (elect_one()) xd_half(0);
          __syncwarp();
          h0_early = true;
        }
      }
      if (lane == 0) trace_at(a, l, T_MMA_WWAIT, wwait);
    }
    // the last layer's stash loads of the z columns precede the TMEM dealloc (final barrier)
  } else if (warp >= kQueueWarp0 && warp < kQueueWarp0 + 4) {
    // ---- queue warps: one stream row per thread ----
    const int sub = warp & 3;
    const int r = sub * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(sub * 32) << 16);
    const bool pf = warp == kQueueWarp0 && lane == 0;
    const bool tq = pf;
    const uint8_t* qtile = a.queue + (size_t)tile * kSlotBytes;
    if (pf)
      for (int l = 0; l < 2 && l < L; ++l) bulk_prefetch_l2(qtile + a.qbase[l], kSlotBytes);
    // K-piece j (K 8j..8j+7) of row r is the 16 bytes at (j * 128 + r) * 16: packed words
    // 4j .. 4j+3 of the operand row
    uint32_t xd[64];
    auto load_slot = [&](int l) {
      const uint4* src = reinterpret_cast<const uint4*>(qtile + a.qbase[l]) + r;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint4 v = src[j * 128];
        xd[4 * j] = v.x;
        xd[4 * j + 1] = v.y;
        xd[4 * j + 2] = v.z;
        xd[4 * j + 3] = v.w;
      }
    };
    auto store_xd = [&]() {
      tmem_st32(trow + kColXd, *reinterpret_cast<float(*)[32]>(xd));
      tmem_st32(trow + kColXd + 32, *reinterpret_cast<float(*)[32]>(xd + 32));
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(xd_ready);
    };
    // 64 TMEM columns of packed fp16 pairs (row r) -> 16 K-pieces at dst (+ j * 2 KB)
    auto tmem_to_pieces = [&](uint32_t col, uint4* dst) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float v[16];
        tmem_ld16(trow + col + 16 * c, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dst[(4 * c + j) * 128] =
              make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                         __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
      }
    };
    load_slot(0);
    store_xd();
    if (L > 1) load_slot(1);
    for (int l = 0; l < L; ++l) {
      const uint32_t par = (uint32_t)l & 1;
      if (pf && l + 2 < L) bulk_prefetch_l2(qtile + a.qbase[l + 2], kSlotBytes);
      // push x_l (the xt operand columns) into ring slot (t mod d_l); this thread's own
      // loads of that slot completed before store_xd of this layer
      mbar_wait(xt_ready, par);
      tc_fence_after();
      tmem_to_pieces(kColXt, reinterpret_cast<uint4*>(const_cast<uint8_t*>(qtile) + a.qbase[l]) + r);
      tc_fence_before();
      mbar_arrive(x_pushed);
      if (tq) trace_at(a, l, T_Q_LOAD, clock64());
      // x_{t-d} of layer l+1 -> TMEM xd once layer l's x_{t-d} MMAs are done (acc1_full)
      if (l + 1 < L) {
        mbar_wait(acc1_full, par);
        tc_fence_after();
        store_xd();
        if (tq) trace_at(a, l + 1, T_Q_XD, clock64());
        if (l + 2 < L) load_slot(l + 2);  // in flight during layer l+1
      }
      // z stash of layer l for the skip GEMM: [tile][L][16 K-pieces][128 rows][16 B]
      mbar_wait(z1_ready, par);
      tc_fence_after();
      tmem_to_pieces(kColZ, reinterpret_cast<uint4*>(a.zimg + ((size_t)tile * L + l) * 2 * kTile) + r);
      tc_fence_before();
      mbar_arrive(z_read);
      if (tq) trace_at(a, l, T_SP1, clock64());
    }
  } else if (warp >= 2 && warp < 10) {
    // ---- gate warps: (row r, column half h) ----
    const int sub = warp & 3, h = (warp - 2) >> 2;
    const int r = sub * 32 + lane;
    const int stream = tile * 128 + r;
    const uint32_t trow = tmem + ((uint32_t)(sub * 32) << 16);
    const int c = a.cls[stream];
    const bool tr = (warp == 2 && lane == 0);
    for (int l = 0; l < L; ++l) {
      const uint32_t par = (uint32_t)l & 1;
      if (tr) trace_at(a, l, T_EPI_A, clock64());
      // x_l: the embedding at l = 0, else the TMEM residual stream (+ the pending bias)
      float x[64];
      if (l == 0) {
        ld64(x, a.embed + (size_t)c * kR + 64 * h);
        tmem_st32(trow + kColX + 64 * h, *reinterpret_cast<float(*)[32]>(x));
        tmem_st32(trow + kColX + 64 * h + 32, *reinterpret_cast<float(*)[32]>(x + 32));
      } else {
        mbar_wait(x_full, par ^ 1);
        if (tr) trace_at(a, l, T_EPI_XFULL, clock64());
        tc_fence_after();
        tmem_ld32(trow + kColX + 64 * h, *reinterpret_cast<float(*)[32]>(x));
        tmem_ld32(trow + kColX + 64 * h + 32, *reinterpret_cast<float(*)[32]>(x + 32));
        tmem_wait_ld();
        if (a.has_res_bias) {
          const float4* rb = reinterpret_cast<const float4*>(a.res_b + (size_t)(l - 1) * kR + 64 * h);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float4 b = __ldg(rb + i);
            x[4 * i] += b.x;
            x[4 * i + 1] += b.y;
            x[4 * i + 2] += b.z;
            x[4 * i + 3] += b.w;
          }
          tmem_st32(trow + kColX + 64 * h, *reinterpret_cast<float(*)[32]>(x));
          tmem_st32(trow + kColX + 64 * h + 32, *reinterpret_cast<float(*)[32]>(x + 32));
        }
      }
      {
        float xp[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) xp[i] = __uint_as_float(pack_h2(x[2 * i], x[2 * i + 1]));
        tmem_st32(trow + kColXt + 32 * h, xp);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(xt_ready);
      if (tr) trace_at(a, l, T_EPI_XT, clock64());
      // gate of N-half hh -> z columns 64*hh + [32h, 32h+32) -> TMEM z columns
      // kColZ + 32*hh + 16*h .. +16 (packed pairs; z shares the columns of xt)
      const float* bd = a.dil_b + (size_t)l * 2 * kD;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        mbar_wait(hh == 0 ? acc0_full : acc1_full, par);
        if (tr) trace_at(a, l, hh == 0 ? T_EPI_ACC0 : T_EPI_ACC1, clock64());
        tc_fence_after();
        float at[32], as[32];
        tmem_ld32(trow + 128 * hh + 32 * h, at);
        tmem_ld32(trow + 128 * hh + 64 + 32 * h, as);
        tmem_wait_ld();
        if (tr) trace_at(a, l, hh == 0 ? T_G0_LD : T_G1_LD, clock64());
        if (a.has_dil_bias) {
          const int j0 = 64 * hh + 32 * h;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            at[i] += __ldg(bd + j0 + i);
            as[i] += __ldg(bd + kD + j0 + i);
          }
        }
        float pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2)
          // z = tanh(a) * sigmoid(b) with sigmoid(b) = 0.5 + 0.5 tanh(b / 2), evaluated for
          // an element pair in packed fp16 (z's operand precision)
          pk[i >> 1] = __uint_as_float(gate2_h2(at[i], at[i + 1], as[i], as[i + 1]));
        if (tr) {
          asm volatile("" ::"f"(pk[0]), "f"(pk[15]) : "memory");
          trace_at(a, l, hh == 0 ? T_G0_MATH : T_G1_MATH, clock64());
        }
        if (hh == 0) {
          // z half 0 overwrites the xt operand: the x_t MMAs of N-half 1 (acc1_full) and the
          // queue push have read it
          mbar_wait(acc1_full, par);
          mbar_wait(x_pushed, par);
          tc_fence_after();
        }
        tmem_st16(trow + kColZ + 32 * hh + 16 * h, pk);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(hh == 0 ? z0_ready : z1_ready);
        if (tr) trace_at(a, l, hh == 0 ? T_EPI_Z0 : T_EPI_Z1, clock64());
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}
