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
//     [384,448)  xt    fp16 x_l[t] operand (A from TMEM, packed pairs)
//     [448,512)  xd    fp16 x_l[t-d] operand
//   SMEM: Z (fp16 z operand, 2 x 16 KB images) | Sq (32 KB fp32 pop staging) |
//         weight stages A (64 KB: dil K-chunks of x_{t-d}), B (64 KB: dil K-chunks of
//         x_t), C (32 KB: res) -- each filled by ONE bulk copy per layer: the copy engine
//         costs ~500 cycles per operation almost regardless of size (tools/ring_bw.cu),
//         so the chain moves its 160 KB of weights per layer in 3 operations.
//
//   warp 0  lane 0  weight producer (stages A, B, C in consumption order)
//   warp 1  lane 0  MMA issuer
//   warps 2..9      gate warps (row r = 32*(warp%4)+lane, column half h = (warp-2)/4)
//   warps 10..13    queue warps (one stream row each): pop x_{t-d} (Sq -> fp16 -> TMEM xd),
//                   push x_l (TMEM -> HBM ring slot, 512-byte coalesced stores)
//   warp 14 lane 0  pop issuer: the tile's 64 KB ring slot as two 32 KB bulk copies
//
// MMA issue order per layer: [xd_ready] stage A (x_{t-d} half, both N-halves) ->
// [xt_ready] stage B: N-half 0 -> acc0_full, N-half 1 -> acc1_full ->
// [z0_ready, x_read] res K-chunk 0 (stage C) -> [z1_ready] z stash store, res K-chunk 1
// -> x_full. The x_{t-d} half of each layer's GEMM so runs before x_l is known.

constexpr int kChainThreads = 480;
constexpr int kQueueWarp0 = 10;
constexpr int kPopWarp = 14;
constexpr uint32_t kColXt = 384, kColXd = 448;
constexpr uint32_t kSqBytes = 32768;  // half a tile slot: channels 64h..64h+63 of 128 rows
constexpr uint32_t kStageA = 65536, kStageB = 65536, kStageC = 32768;
constexpr uint32_t kOffZ = 0, kOffSq = 2 * kTile, kOffA = kOffSq + kSqBytes,
                   kOffB = kOffA + kStageA, kOffC = kOffB + kStageB,
                   kOffBars = kOffC + kStageC;
constexpr size_t kChainSmem = 1024 + kOffBars + 256;

__global__ void __launch_bounds__(kChainThreads, 1) chain_kernel(ChainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* Z = smem + kOffZ;
  uint8_t* Sq = smem + kOffSq;
  uint8_t* stA = smem + kOffA;
  uint8_t* stB = smem + kOffB;
  uint8_t* stC = smem + kOffC;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBars);
  uint64_t* fullA = bars + 0;
  uint64_t* fullB = bars + 1;
  uint64_t* fullC = bars + 2;
  uint64_t* emptyA = bars + 3;
  uint64_t* emptyB = bars + 4;
  uint64_t* emptyC = bars + 5;
  uint64_t* xd_ready = bars + 6;   // 128: queue warps
  uint64_t* xt_ready = bars + 7;   // 256: gate warps
  uint64_t* z0_ready = bars + 8;   // 256
  uint64_t* z1_ready = bars + 9;   // 256
  uint64_t* x_read = bars + 10;    // 128: queue warps read x_l for the push
  uint64_t* sq_free = bars + 11;   // 128: queue warps consumed Sq
  uint64_t* acc0_full = bars + 12;
  uint64_t* acc1_full = bars + 13;
  uint64_t* x_full = bars + 14;
  uint64_t* s_full = bars + 15;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int L = a.L;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 6; ++i) mbar_init(bars + i, 1);
    mbar_init(xd_ready, 128);
    mbar_init(xt_ready, 256);
    mbar_init(z0_ready, 256);
    mbar_init(z1_ready, 256);
    mbar_init(x_read, 128);
    mbar_init(sq_free, 128);
    for (int i = 12; i < 16; ++i) mbar_init(bars + i, 1);
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
        const uint8_t* wl = a.w + (size_t)l * kLayerBytes;  // chunks 0-3 | 4-7 | 8-9
        const uint32_t ph = ((uint32_t)l & 1) ^ 1;
        mbar_wait(emptyA, ph);
        trace_at(a, l, T_PROD_A, clock64());
        mbar_arrive_expect_tx(fullA, kStageA);
        bulk_g2s(stA, wl, kStageA, fullA);
        mbar_wait(emptyB, ph);
        trace_at(a, l, T_PROD_B, clock64());
        mbar_arrive_expect_tx(fullB, kStageB);
        bulk_g2s(stB, wl + 4 * kChunk, kStageB, fullB);
        if (l + 1 < L) {
          mbar_wait(emptyC, ph);
          trace_at(a, l, T_PROD_C, clock64());
          mbar_arrive_expect_tx(fullC, kStageC);
          bulk_g2s(stC, wl + 8 * kChunk, kStageC, fullC);
        }
      }
    }
  } else if (warp == kPopWarp) {
    if (lane == 0) {  // ---- pop issuer: slot layout [B/128][R/4][128][4], half h = 32 KB ----
      for (int k = 0; k < 2 * L; ++k) {
        const int l = k >> 1, h = k & 1;
        if (k > 0) mbar_wait(sq_free, (uint32_t)(k - 1) & 1);
        trace_at(a, l, h ? T_POP1 : T_POP0, clock64());
        mbar_arrive_expect_tx(s_full, kSqBytes);
        bulk_g2s(Sq, a.queue + a.qbase[l] + ((size_t)tile * (kR / 4) + 16 * h) * 512, kSqBytes,
                 s_full);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      const uint32_t id = idesc_f16(128, 128);
      const uint32_t zs = smem_u32(Z), sa = smem_u32(stA), sb = smem_u32(stB), sc = smem_u32(stC);
      long long wwait = 0;
      auto wait_w = [&](uint64_t* bar, uint32_t par) {
        const long long w0 = clock64();
        mbar_wait(bar, par);
        wwait += clock64() - w0;
        tc_fence_after();
      };
      // one 64-K chunk: B image at b_saddr, A from TMEM column a_col or smem image a_saddr
      auto mma_tmem_a = [&](uint32_t d, uint32_t a_col, uint32_t b_saddr, bool first) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16_ta(d, a_col + kk * 8, sdesc_sw128(b_saddr + kk * 32), id,
                      (first && kk == 0) ? 0u : 1u);
      };
      auto mma_smem_a = [&](uint32_t d, uint32_t a_saddr, uint32_t b_saddr) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16(d, sdesc_sw128(a_saddr + kk * 32), sdesc_sw128(b_saddr + kk * 32), id, 1u);
      };
      // x_{t-d} half, stage A chunks [h0 kc2, h0 kc3 | h1 kc2, h1 kc3]. N-half 0 initialises
      // acc0 and is issued as early as its operands allow (during the previous layer's
      // second gate half, when the tensor pipe idles); N-half 1 follows the critical acc0.
      auto xd_h0 = [&](int l) {
        mma_tmem_a(tmem + 0, tmem + kColXd + 0, sa + 0 * kChunk, true);
        mma_tmem_a(tmem + 0, tmem + kColXd + 32, sa + 1 * kChunk, false);
      };
      auto xd_h1 = [&]() {
        mma_tmem_a(tmem + 128, tmem + kColXd + 0, sa + 2 * kChunk, true);
        mma_tmem_a(tmem + 128, tmem + kColXd + 32, sa + 3 * kChunk, false);
        mma_commit(emptyA);
      };
      bool h0_early = false;
      for (int l = 0; l < L; ++l) {
        const uint32_t par = (uint32_t)l & 1;
        if (!h0_early) {
          mbar_wait(xd_ready, par);
          tc_fence_after();
          wait_w(fullA, par);
          xd_h0(l);
        }
        trace_at(a, l, T_MMA_XD, clock64());
        h0_early = false;
        // x_t half: stage B chunks [h0 kc0, h0 kc1, h1 kc0, h1 kc1]
        mbar_wait(xt_ready, par);
        trace_at(a, l, T_MMA_XT, clock64());
        tc_fence_after();
        wait_w(fullB, par);
        mma_tmem_a(tmem + 0, tmem + kColXt + 0, sb + 0 * kChunk, false);
        mma_tmem_a(tmem + 0, tmem + kColXt + 32, sb + 1 * kChunk, false);
        bulk_wait_read0();  // Z is rewritten once acc0_full is seen: stash copy done reading
        mma_commit(acc0_full);
        trace_at(a, l, T_MMA_ACC0, clock64());
        xd_h1();
        mma_tmem_a(tmem + 128, tmem + kColXt + 0, sb + 2 * kChunk, false);
        mma_tmem_a(tmem + 128, tmem + kColXt + 32, sb + 3 * kChunk, false);
        mma_commit(acc1_full);
        mma_commit(emptyB);
        trace_at(a, l, T_MMA_ACC1, clock64());
        // z halves: res MMA (all but the top layer) + one bulk store of the z stash
        mbar_wait(z0_ready, par);
        trace_at(a, l, T_MMA_Z0, clock64());
        tc_fence_after();
        if (l + 1 < L) {
          mbar_wait(x_read, par);  // queue warps have read x_l before the MMA updates it
          tc_fence_after();
          wait_w(fullC, par);
          mma_smem_a(tmem + 256, zs + 0 * kTile, sc + 0 * kChunk);
          // acc0 is free (gate half 0 done): start layer l+1's x_{t-d} N-half 0 now if its
          // operand and weights are already in place -- never wait for them here
          const uint32_t pn = (uint32_t)(l + 1) & 1;
          if (mbar_test(xd_ready, pn) && mbar_test(fullA, pn)) {
            tc_fence_after();
            xd_h0(l + 1);
            h0_early = true;
          }
        }
        mbar_wait(z1_ready, par);
        trace_at(a, l, T_MMA_Z1, clock64());
        tc_fence_after();
        bulk_s2g(a.zimg + ((size_t)tile * L * 2 + 2 * l) * kTile, Z, 2 * kTile);
        bulk_commit();
        if (l + 1 < L) {
          mma_smem_a(tmem + 256, zs + 1 * kTile, sc + 1 * kChunk);
          mma_commit(emptyC);
          mma_commit(x_full);
          trace_at(a, l, T_MMA_XFULL, clock64());
        }
        trace_at(a, l, T_MMA_WWAIT, wwait);
      }
      bulk_wait0();  // the last layer's stash is globally visible before the kernel ends
    }
    __syncwarp();
  } else if (warp >= kQueueWarp0 && warp < kQueueWarp0 + 4) {
    // ---- queue warps: one stream row per thread ----
    const int sub = warp & 3;
    const int r = sub * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(sub * 32) << 16);
    const float* sq = reinterpret_cast<const float*>(Sq) + (size_t)r * 4;
    for (int l = 0; l < L; ++l) {
      // pop: x_l[t-d] from Sq (two halves) -> packed fp16 in registers, releasing Sq as soon
      // as a half is consumed so the next half's copy starts at once; then, once layer l-1's
      // dil MMAs are done with the xd columns, -> TMEM xd
      uint32_t pk[2][32];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = 2 * l + h;
        mbar_wait(s_full, (uint32_t)k & 1);
        const float* src = sq;  // Sq is [16][128][4]: chunk j of row r at (j * 128 + r) * 16 B
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float4 f = *reinterpret_cast<const float4*>(src + (size_t)j * 512);
          pk[h][2 * j] = pack_h2(f.x, f.y);
          pk[h][2 * j + 1] = pack_h2(f.z, f.w);
        }
        // every shared load must have returned before Sq is released (the next pop
        // overwrites it through the async proxy): make the arrive depend on all of them
        asm volatile("" ::"r"(pk[h][0] ^ pk[h][1] ^ pk[h][2] ^ pk[h][3] ^ pk[h][4] ^ pk[h][5] ^
                               pk[h][6] ^ pk[h][7] ^ pk[h][8] ^ pk[h][9] ^ pk[h][10] ^ pk[h][11] ^
                               pk[h][12] ^ pk[h][13] ^ pk[h][14] ^ pk[h][15] ^ pk[h][16] ^
                               pk[h][17] ^ pk[h][18] ^ pk[h][19] ^ pk[h][20] ^ pk[h][21] ^
                               pk[h][22] ^ pk[h][23] ^ pk[h][24] ^ pk[h][25] ^ pk[h][26] ^
                               pk[h][27] ^ pk[h][28] ^ pk[h][29] ^ pk[h][30] ^ pk[h][31])
                     : "memory");
        // generic-proxy reads of Sq must be ordered before the async-proxy (TMA) overwrite
        fence_proxy_async();
        mbar_arrive(sq_free);
      }
      if (l > 0) mbar_wait(acc1_full, (uint32_t)(l - 1) & 1);
      tmem_st32(trow + kColXd, *reinterpret_cast<float(*)[32]>(pk[0]));
      tmem_st32(trow + kColXd + 32, *reinterpret_cast<float(*)[32]>(pk[1]));
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(xd_ready);
      if (warp == kQueueWarp0 && lane == 0) trace_at(a, l, T_Q_XD, clock64());
      // push: x_l (after the pending bias) -> ring slot t mod d_l, 512 B per warp store
      mbar_wait(xt_ready, (uint32_t)l & 1);
      tc_fence_after();
      float* dst = a.queue + a.qbase[l] + ((size_t)tile * (kR / 4) * 128 + r) * 4;
#pragma unroll 1
      for (int q4 = 0; q4 < 4; ++q4) {
        float x[32];
        tmem_ld32(trow + 256 + 32 * q4, x);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<float4*>(dst + (size_t)(8 * q4 + j) * 512) =
              make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
      }
      tc_fence_before();
      mbar_arrive(x_read);
      if (warp == kQueueWarp0 && lane == 0) trace_at(a, l, T_Q_PUSHED, clock64());
    }
  } else if (warp >= 2 && warp < 10) {
    // ---- gate warps: (row r, column half h) ----
    const int sub = warp & 3, h = (warp - 2) >> 2;
    const int r = sub * 32 + lane;
    const int stream = tile * 128 + r;
    const uint32_t trow = tmem + ((uint32_t)(sub * 32) << 16);
    const uint32_t zs = smem_u32(Z);
    const int c = a.cls[stream];
    const bool tr = (warp == 2 && lane == 0);
    for (int l = 0; l < L; ++l) {
      const uint32_t par = (uint32_t)l & 1;
      if (tr) trace_at(a, l, T_EPI_A, clock64());
      // x_l: the embedding at l = 0, else the TMEM residual stream (+ the pending bias)
      float x[64];
      if (l == 0) {
        ld64(x, a.embed + (size_t)c * kR + 64 * h);
        tmem_st32(trow + 256 + 64 * h, *reinterpret_cast<float(*)[32]>(x));
        tmem_st32(trow + 256 + 64 * h + 32, *reinterpret_cast<float(*)[32]>(x + 32));
      } else {
        mbar_wait(x_full, par ^ 1);
        if (tr) trace_at(a, l, T_EPI_XFULL, clock64());
        tc_fence_after();
        tmem_ld32(trow + 256 + 64 * h, *reinterpret_cast<float(*)[32]>(x));
        tmem_ld32(trow + 256 + 64 * h + 32, *reinterpret_cast<float(*)[32]>(x + 32));
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
          tmem_st32(trow + 256 + 64 * h, *reinterpret_cast<float(*)[32]>(x));
          tmem_st32(trow + 256 + 64 * h + 32, *reinterpret_cast<float(*)[32]>(x + 32));
        }
      }
      {
        float pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = __uint_as_float(pack_h2(x[2 * i], x[2 * i + 1]));
        tmem_st32(trow + kColXt + 32 * h, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(xt_ready);
      if (tr) trace_at(a, l, T_EPI_XT, clock64());
      // gate of N-half hh -> z columns 64*hh + [32h, 32h+32)
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
        if (a.has_dil_bias) {
          const int j0 = 64 * hh + 32 * h;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            at[i] += __ldg(bd + j0 + i);
            as[i] += __ldg(bd + kD + j0 + i);
          }
        }
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2)
          // z = tanh(a) * sigmoid(b) with sigmoid(b) = 0.5 + 0.5 tanh(b / 2), evaluated for
          // an element pair in packed fp16 (z's operand precision): 2 MUFU + 2 HFMA2 per pair
          pk[i >> 1] = gate2_h2(at[i], at[i + 1], as[i], as[i + 1]);
#pragma unroll
        for (int p = 0; p < 4; ++p)
          st_shared_v4(zs + hh * kTile + swz(r, 4 * h + p), pk[4 * p], pk[4 * p + 1], pk[4 * p + 2],
                       pk[4 * p + 3]);
        fence_proxy_async();
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
