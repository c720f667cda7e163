// K1c: the small-batch (latency-bound) step kernel -- one stream per thread-block cluster.
//
// At one stream a generation step is a chain of L dependent layers of small GEMVs
// (the weight roofline is < 1 us, the chain is the bound).
// The C CTAs of a cluster split every GEMV's outputs, so per layer the critical path is
// one slice GEMV, the gate, one exchange of z through distributed shared memory and ONE
// cluster barrier:
//
//   phase l:  a_l = W0_l x_{l-1} + (W0_l W_res,l-1) z_{l-1} + W1_l x_l[t-d_l] + c_l
//             (the residual update folded into the dilated taps: x_l = x_{l-1} + W_res z
//             + b is linear, so with W'_l = W0_l W_res,l-1 and c_l = b_l + W0_l b_res,l-1
//             the layer reads x_{l-1} and z_{l-1}, both all-gathered at the previous
//             barrier, and never waits for x_l),
//             z_l = tanh(a_l[:D]) * sigmoid(a_l[D:])        -> this CTA's D/C columns
//             x_l = x_{l-1} + W_res,l-1 z_{l-1} + b_res      -> this CTA's R/C channels,
//                   pushed into ring l (fast.py:192: the layer input is cached)
//             s  += W_skip,l-1 z_{l-1} + b_skip             -> this CTA's S/C columns
//             z_l and x_l slices -> every CTA (st.shared::cluster), barrier.cluster
//   then s += W_skip,L-1 z_{L-1}, ReLU(s) / h / logits all-gathered (3 barriers), every CTA
//   selects the class redundantly (deterministic).
//
// Folding changes only the fp32 rounding order (the oracle's fp64 reference is the same
// math); W' is computed in fp64 from the (bf16-rounded, where applicable) weights.
//
// Weights: per CTA, per phase, one contiguous block of its slices (dil rows interleaved
// tanh/sigmoid so a z column's two outputs land in one warp; rows padded so a warp's
// lanes hit distinct banks). When every block of a step fits in shared memory they stay
// resident for the whole launch (cfg1); otherwise a producer streams them through a
// two-slot ring with 1-D bulk copies one phase ahead (cfg2). GEMVs: LPO lanes per output
// (k = sub + LPO*i), fixed-order shuffle reduction.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.h"
#include "select.cuh"
#include "tc_ptx.cuh"

namespace fw {

namespace {

constexpr int kLatNT = 256;  // 8 warps
constexpr int kLatPad = 64;  // zero floats after every input vector (padded GEMV rows)

// Per-C packed weights and their layout (host-computed, uploaded once per handle and C).
struct LatLayout {
  int C = 0;
  int Dc, Rc, Sc, Hc, Ac;
  int Kd, Kpd, lpo_d;    // dil: K = 2R + D, padded row, lanes per output
  int Kprs, lpo_rs;      // res | skip rows over z (K = D)
  int Kph1, lpo_h1;      // head1 over ReLU(s) (K = S)
  int Kph2, lpo_h2;      // head2 over h (K = H)
  // float offsets inside a phase block
  int64_t o_dil, o_bd, o_rs, o_br, o_bs, phase_floats;
  int64_t post_floats;   // block L: skip rows + bias
  int64_t h1_floats, h2_floats;
  int64_t step_floats;      // all blocks of a step (per rank)
  int64_t max_block;
  int resident;
  float* d_w = nullptr;     // [C][step_floats]
};

}  // namespace

struct LatPlan {
  LatLayout lay;
};

namespace {

struct LatParams {
  CellDims d;
  int B;
  const int* dil;
  const int64_t* qoff;
  float* queue;
  const float* embed;
  const float* w;  // this launch's packed weights [C][step_floats]
  LatLayout lay;
  CellRun run;
};

__device__ __forceinline__ uint32_t lat_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void lat_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t lat_mapa(const float* p, uint32_t q) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(a)
               : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(q));
  return a;
}
__device__ __forceinline__ void lat_st_remote(uint32_t a, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
// v -> the same float of every CTA of the cluster
template <int C>
__device__ __forceinline__ void lat_bcast(const float* p, float v) {
#pragma unroll
  for (int q = 0; q < C; ++q) lat_st_remote(lat_mapa(p, (uint32_t)q), v);
}

// out[o] = sum_k W[o * Kp + k] * in[k] for o < n (LPO lanes per output, k = sub + LPO i,
// two accumulators, fixed-order shuffle reduction); epi(o, v) on the output's lane sub 0.
// Also returns v to every lane of the output group (for the gate's pair exchange).
template <typename Epi>
__device__ __forceinline__ void lat_gemv(const float* W, int Kp, int K, int n, int lpo,
                                         const float* in, Epi epi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int opw = 32 / lpo, sub = lane & (lpo - 1);
  for (int o0 = warp * opw; o0 < n; o0 += (kLatNT / 32) * opw) {
    const int o = o0 + lane / lpo;
    float a0 = 0.f, a1 = 0.f;
    if (o < n) {
      const float* w = W + (int64_t)o * Kp;
      int k = sub;
      for (; k + lpo < K; k += 2 * lpo) {
        a0 = fmaf(w[k], in[k], a0);
        a1 = fmaf(w[k + lpo], in[k + lpo], a1);
      }
      if (k < K) a0 = fmaf(w[k], in[k], a0);
    }
    float v = a0 + a1;
    for (int off = lpo >> 1; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    epi(o, v, sub, lpo);
  }
}

template <int C>
__global__ void __launch_bounds__(kLatNT) cell_lat_kernel(LatParams p) {
  extern __shared__ __align__(16) float smem[];
  const CellDims d = p.d;
  const LatLayout& Y = p.lay;
  const int R = d.R, D = d.D, S = d.S, H = d.H, A = d.A, L = d.L;
  const int Dc = Y.Dc, Rc = Y.Rc, Sc = Y.Sc, Hc = Y.Hc, Ac = Y.Ac;
  const uint32_t rank = lat_rank();
  const int stream = blockIdx.x / C;
  const int tid = threadIdx.x;
  const int j0 = (int)rank * Dc, r0 = (int)rank * Rc, k0 = (int)rank * Sc;
  // shared memory: weights | inbuf[2][2R + D + pad] | xall[L][R] | s[Sc] | sf[S + pad] |
  // hf[H + pad] | lg[A] | cls
  float* wsm = smem;
  const int64_t wfl = Y.resident ? Y.step_floats : 2 * Y.max_block;
  const int in_len = 2 * R + D + kLatPad;
  uint64_t* full = reinterpret_cast<uint64_t*>(wsm + wfl);  // [2] ring slots (16-byte aligned)
  float* inbuf = wsm + wfl + 4;
  float* xall = inbuf + 2 * in_len;
  float* s_s = xall + L * R;
  float* sf = s_s + ((Sc + 3) & ~3);
  float* hf = sf + S + kLatPad;
  float* lg = hf + H + kLatPad;
  int* cls = reinterpret_cast<int*>(lg + A);
  const float* wg = p.w + (int64_t)rank * Y.step_floats;  // this rank's blocks in global
  const int nblk = L + 3;
  auto block_off = [&](int b) -> int64_t {  // float offset of block b inside a step
    return b <= L ? (int64_t)b * Y.phase_floats
                  : (int64_t)L * Y.phase_floats + Y.post_floats + (b == L + 2 ? Y.h1_floats : 0);
  };
  auto block_len = [&](int b) -> int64_t {
    return b < L ? Y.phase_floats : (b == L ? Y.post_floats : (b == L + 1 ? Y.h1_floats : Y.h2_floats));
  };
  const CellRun& run = p.run;
  const int B = p.B;
  const int Rp = (R + 3) & ~3;
  const size_t slot_elems = (size_t)((B + 127) / 128) * 128 * Rp;
  auto ring_ptr = [&](int l, int64_t t, int r) {
    return p.queue + p.qoff[l] + (size_t)(t % p.dil[l]) * slot_elems +
           ((size_t)((stream >> 7) * (Rp / 4) + (r >> 2)) * 128 + (stream & 127)) * 4 + (r & 3);
  };

  // zero the padded tails of the input vectors (the padded weight columns are zero, so the
  // pads must be finite), load resident weights, init the ring barriers
  for (int e = tid; e < 2 * in_len; e += kLatNT) inbuf[e] = 0.f;
  for (int e = tid; e < S + kLatPad; e += kLatNT) sf[e] = 0.f;
  for (int e = tid; e < H + kLatPad; e += kLatNT) hf[e] = 0.f;
  if (tid == 0) {
    ptx::mbar_init(&full[0], 1);
    ptx::mbar_init(&full[1], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  int64_t g = 0;  // blocks consumed (ring mode)
  auto issue = [&](int64_t gi) {  // ring: block gi of the launch into slot gi & 1
    const int b = (int)(gi % nblk);
    const uint32_t bytes = (uint32_t)(block_len(b) * 4);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::mbar_arrive_expect_tx(&full[gi & 1], bytes);
    ptx::bulk_g2s(wsm + (gi & 1) * Y.max_block, wg + block_off(b), bytes, &full[gi & 1]);
  };
  if (Y.resident) {
    if (tid == 0) {
      const uint32_t bytes = (uint32_t)(Y.step_floats * 4);
      ptx::mbar_arrive_expect_tx(&full[0], bytes);
      ptx::bulk_g2s(wsm, wg, bytes, &full[0]);
    }
  } else if (tid == 0) {
    issue(0);
  }
  // block b of the current step, waited for
  auto take = [&](int b) -> const float* {
    if (Y.resident) return wsm + block_off(b);
    ptx::mbar_wait(&full[g & 1], (uint32_t)((g >> 1) & 1));
    const float* w = wsm + (g & 1) * Y.max_block;
    if (tid == 0 && g + 1 < (int64_t)run.n_steps * nblk) issue(g + 1);
    ++g;
    return w;
  };
  if (Y.resident) ptx::mbar_wait(&full[0], 0);
  // pops of the first step (each CTA keeps every layer's x_{t-d}; later steps' pops are
  // loaded during the previous step's heads, after its last push)
  for (int e = tid; e < L * R; e += kLatNT) xall[e] = __ldcg(ring_ptr(e / R, run.t0, e % R));
  if (tid == 0) cls[0] = run.inputs[stream];
  __syncthreads();

  for (int i = 0; i < run.n_steps; ++i) {
    const int64_t t = run.t0 + i;
    // phase 0 input: x_0 = E[c_t] (z part: any finite value, its weights are zero), x_0[t-d]
    {
      const float* e = p.embed + (size_t)clamp_class(cls[0], A) * R;
      for (int r = tid; r < R; r += kLatNT) {
        inbuf[r] = __ldg(e + r);
        inbuf[R + r] = xall[r];
      }
      for (int k = tid; k < Sc; k += kLatNT) s_s[k] = 0.f;
    }
    __syncthreads();
    for (int l = 0; l < L; ++l) {
      const float* wb = take(l);
      const float* in = inbuf + (l & 1) * in_len;
      float* nxt = inbuf + ((l + 1) & 1) * in_len;
      // dilated taps (+ folded residual) of this CTA's z columns; rows 2j / 2j+1 = the
      // tanh / sigmoid pre-activation of column j0 + j
      const float* bd = wb + Y.o_bd;
      lat_gemv(wb + Y.o_dil, Y.Kpd, Y.Kd, 2 * Dc, Y.lpo_d, in, [&](int o, float v, int sub, int lpo) {
        const float pv = __shfl_down_sync(0xffffffffu, v, lpo);  // the sigmoid row's sum
        if (o < 2 * Dc && sub == 0 && (o & 1) == 0) {
          const float z = tanhf(v + bd[o]) * sigmoidf_(pv + bd[o + 1]);
          lat_bcast<C>(nxt + 2 * R + j0 + (o >> 1), z);
        }
      });
      // x_l slice (residual of the previous layer; x_0 itself at l = 0) -> ring l and every
      // CTA; s slice += skip of the previous layer
      const float* br = wb + Y.o_br;
      const float* bs = wb + Y.o_bs;
      lat_gemv(wb + Y.o_rs, Y.Kprs, D, Rc + Sc, Y.lpo_rs, in + 2 * R, [&](int o, float v, int sub, int) {
        if (o < Rc + Sc && sub == 0) {
          if (o < Rc) {
            const float x = in[r0 + o] + v + br[o];
            lat_bcast<C>(nxt + r0 + o, x);
            *ring_ptr(l, t, r0 + o) = x;  // push x_l[t] (its pop was read before this step)
          } else if (l > 0) {
            s_s[o - Rc] += v + bs[o - Rc];
          }
        }
      });
      // the next phase's x_{l+1}[t-d]
      if (l + 1 < L)
        for (int r = tid; r < R; r += kLatNT) nxt[R + r] = xall[(l + 1) * R + r];
      lat_cluster_sync();
    }
    // the top layer's skip: s += W_skip,L-1 z_{L-1} + b
    {
      const float* wb = take(L);
      const float* in = inbuf + (L & 1) * in_len;
      lat_gemv(wb, Y.Kprs, D, Sc, Y.lpo_rs, in + 2 * R, [&](int o, float v, int sub, int) {
        if (o < Sc && sub == 0) {
          const float s = s_s[o] + v + wb[(int64_t)Sc * Y.Kprs + o];
          lat_bcast<C>(sf + k0 + o, fmaxf(s, 0.f));
        }
      });
    }
    // every push of this step is done (barrier L-1): the next step's pops
    if (i + 1 < run.n_steps)
      for (int e = tid; e < L * R; e += kLatNT) xall[e] = __ldcg(ring_ptr(e / R, t + 1, e % R));
    lat_cluster_sync();
    {
      const float* wb = take(L + 1);
      const int h0 = (int)rank * Hc;
      lat_gemv(wb, Y.Kph1, S, Hc, Y.lpo_h1, sf, [&](int o, float v, int sub, int) {
        if (o < Hc && sub == 0) lat_bcast<C>(hf + h0 + o, fmaxf(v + wb[(int64_t)Hc * Y.Kph1 + o], 0.f));
      });
    }
    lat_cluster_sync();
    {
      const float* wb = take(L + 2);
      const int a0 = (int)rank * Ac;
      float* dst = (run.logits != nullptr && i < run.n_logit_steps)
                       ? run.logits + ((size_t)i * B + stream) * A + a0 : nullptr;
      lat_gemv(wb, Y.Kph2, H, Ac, Y.lpo_h2, hf, [&](int o, float v, int sub, int) {
        if (o < Ac && sub == 0) {
          const float x = v + wb[(int64_t)Ac * Y.Kph2 + o];
          lat_bcast<C>(lg + a0 + o, x);
          if (dst) dst[o] = x;
        }
      });
    }
    lat_cluster_sync();
    if (tid < 32) {
      const uint32_t prefix = noise_prefix(run.seed, (uint32_t)(run.stream_offset + stream), (uint32_t)t);
      const int c = select_class(lg, A, run.mode, prefix);
      if (tid == 0) {
        if (rank == 0) run.out[(size_t)i * B + stream] = c;
        cls[0] = (i + 1 < run.n_inputs) ? run.inputs[(size_t)(i + 1) * B + stream] : c;
      }
    }
    __syncthreads();
  }
  lat_cluster_sync();  // no DSMEM writes into a CTA that has exited
}

int pow2_floor(int v) {
  int p = 1;
  while (p * 2 <= v) p *= 2;
  return p;
}
// lanes per output so that the n outputs fill the CTA's 8 warps (at least 2 outputs per warp
// when pairs must share a warp)
int lpo_for(int n, int max_lpo) {
  int lpo = pow2_floor(std::max(1, kLatNT / std::max(n, 1)));
  return std::max(1, std::min(lpo, max_lpo));
}
// row stride: K rounded to a multiple of the lanes per output, then to lpo (mod 32) so the
// 32 / lpo rows a warp reads start in distinct banks
int kpad(int K, int lpo) {
  const int k32 = (K + 31) / 32 * 32;
  return lpo >= 32 ? k32 : k32 + lpo;
}
int64_t up4(int64_t v) { return (v + 3) & ~(int64_t)3; }  // 16-byte granules

}  // namespace

bool lat_supported(const CellDims& d, int C) {
  return C >= 2 && d.D % C == 0 && d.R % C == 0 && d.S % C == 0 && d.H % C == 0 &&
         d.A % C == 0 && (int64_t)d.L * d.R <= 16384 && d.R <= 1024 && d.D <= 1024;
}

void lat_destroy(Handle& h) {
  if (!h.lat) return;
  if (h.lat->lay.d_w) cudaFree(h.lat->lay.d_w);
  delete h.lat;
  h.lat = nullptr;
}

// Packs (once per handle and cluster size) every rank's per-phase weight blocks from the
// host copy of the model: dil rows [W0 | W1 | W0 W_res(prev)] interleaved tanh/sigmoid,
// folded bias, res | skip rows of the previous layer and their biases; the top layer's skip
// block; head1 / head2 slices with biases.
static int lat_prepare(Handle& h, int C, std::string* err) {
  if (h.lat && h.lat->lay.C == C) return FW_OK;
  lat_destroy(h);
  const CellDims& d = h.dims;
  const int L = d.L, R = d.R, D = d.D, S = d.S, H = d.H, A = d.A;
  const HostCell& w = h.host;
  LatLayout Y;
  Y.C = C;
  Y.Dc = D / C;
  Y.Rc = R / C;
  Y.Sc = S / C;
  Y.Hc = H / C;
  Y.Ac = A / C;
  Y.Kd = 2 * R + D;
  Y.lpo_d = lpo_for(2 * Y.Dc, 16);  // a z column's two rows in one warp
  Y.Kpd = kpad(Y.Kd, Y.lpo_d);
  Y.lpo_rs = lpo_for(Y.Rc + Y.Sc, 32);
  Y.Kprs = kpad(D, Y.lpo_rs);
  Y.lpo_h1 = lpo_for(Y.Hc, 32);
  Y.Kph1 = kpad(S, Y.lpo_h1);
  Y.lpo_h2 = lpo_for(Y.Ac, 32);
  Y.Kph2 = kpad(H, Y.lpo_h2);
  Y.o_dil = 0;
  Y.o_bd = up4((int64_t)2 * Y.Dc * Y.Kpd);
  Y.o_rs = Y.o_bd + up4(2 * Y.Dc);
  Y.o_br = Y.o_rs + up4((int64_t)(Y.Rc + Y.Sc) * Y.Kprs);
  Y.o_bs = Y.o_br + up4(Y.Rc);
  Y.phase_floats = Y.o_bs + up4(Y.Sc);
  Y.post_floats = up4((int64_t)Y.Sc * Y.Kprs) + up4(Y.Sc);
  Y.h1_floats = up4((int64_t)Y.Hc * Y.Kph1) + up4(Y.Hc);
  Y.h2_floats = up4((int64_t)Y.Ac * Y.Kph2) + up4(Y.Ac);
  Y.step_floats = (int64_t)L * Y.phase_floats + Y.post_floats + Y.h1_floats + Y.h2_floats;
  Y.max_block = std::max(std::max(Y.phase_floats, Y.post_floats), std::max(Y.h1_floats, Y.h2_floats));
  // activations + barriers beside the weights; resident when a step's blocks fit
  const int64_t act_floats = 2 * (2 * R + D + kLatPad) + (int64_t)L * R + up4(Y.Sc) + S + kLatPad +
                             H + kLatPad + A + 4 + 8;
  const int64_t budget = 220 * 1024 / 4;
  Y.resident = (Y.step_floats + act_floats <= budget && Y.step_floats * 4 < (1u << 20)) ? 1 : 0;
  if (!Y.resident && 2 * Y.max_block + act_floats > budget) {
    *err = "small-batch cluster kernel: a phase's weight slices exceed shared memory";
    return FW_ERR_UNSUPPORTED;
  }
  std::vector<float> img((size_t)C * Y.step_floats, 0.f);
  // [l][o][k] accessors of the host model (reference layouts)
  auto W0 = [&](int l, int o, int k) { return (double)w.dil_w[(((size_t)l * 2 + 0) * 2 * D + o) * R + k]; };
  auto W1 = [&](int l, int o, int k) { return (double)w.dil_w[(((size_t)l * 2 + 1) * 2 * D + o) * R + k]; };
  auto Wr = [&](int l, int r, int k) { return (double)w.res_w[((size_t)l * R + r) * D + k]; };
  auto Ws = [&](int l, int s, int k) { return (double)w.skip_w[((size_t)l * S + s) * D + k]; };
  for (int q = 0; q < C; ++q) {
    float* base = img.data() + (size_t)q * Y.step_floats;
    for (int l = 0; l < L; ++l) {
      float* blk = base + (size_t)l * Y.phase_floats;
      for (int j = 0; j < Y.Dc; ++j)
        for (int half = 0; half < 2; ++half) {
          const int o = half * D + q * Y.Dc + j;  // tanh column (half 0) / sigmoid column
          float* row = blk + Y.o_dil + (int64_t)(2 * j + half) * Y.Kpd;
          double bias = w.dil_b[(size_t)l * 2 * D + o];
          for (int k = 0; k < R; ++k) {
            row[k] = (float)W0(l, o, k);
            row[R + k] = (float)W1(l, o, k);
          }
          if (l > 0) {
            for (int c = 0; c < D; ++c) {
              double acc = 0.0;
              for (int k = 0; k < R; ++k) acc += W0(l, o, k) * Wr(l - 1, k, c);
              row[2 * R + c] = (float)acc;
            }
            for (int k = 0; k < R; ++k) bias += W0(l, o, k) * (double)w.res_b[(size_t)(l - 1) * R + k];
          }
          blk[Y.o_bd + 2 * j + half] = (float)bias;
        }
      if (l > 0) {
        for (int r = 0; r < Y.Rc; ++r) {
          for (int k = 0; k < D; ++k) blk[Y.o_rs + (int64_t)r * Y.Kprs + k] = (float)Wr(l - 1, q * Y.Rc + r, k);
          blk[Y.o_br + r] = w.res_b[(size_t)(l - 1) * R + q * Y.Rc + r];
        }
        for (int s = 0; s < Y.Sc; ++s) {
          for (int k = 0; k < D; ++k)
            blk[Y.o_rs + (int64_t)(Y.Rc + s) * Y.Kprs + k] = (float)Ws(l - 1, q * Y.Sc + s, k);
          blk[Y.o_bs + s] = w.skip_b[(size_t)(l - 1) * S + q * Y.Sc + s];
        }
      }
    }
    float* post = base + (size_t)L * Y.phase_floats;
    for (int s = 0; s < Y.Sc; ++s) {
      for (int k = 0; k < D; ++k) post[(int64_t)s * Y.Kprs + k] = (float)Ws(L - 1, q * Y.Sc + s, k);
      post[(int64_t)Y.Sc * Y.Kprs + s] = w.skip_b[(size_t)(L - 1) * S + q * Y.Sc + s];
    }
    float* h1 = post + Y.post_floats;
    for (int o = 0; o < Y.Hc; ++o) {
      for (int k = 0; k < S; ++k) h1[(int64_t)o * Y.Kph1 + k] = w.h1_w[(size_t)(q * Y.Hc + o) * S + k];
      h1[(int64_t)Y.Hc * Y.Kph1 + o] = w.h1_b[q * Y.Hc + o];
    }
    float* h2 = h1 + Y.h1_floats;
    for (int o = 0; o < Y.Ac; ++o) {
      for (int k = 0; k < H; ++k) h2[(int64_t)o * Y.Kph2 + k] = w.h2_w[(size_t)(q * Y.Ac + o) * H + k];
      h2[(int64_t)Y.Ac * Y.Kph2 + o] = w.h2_b[q * Y.Ac + o];
    }
  }
  cudaError_t e = cudaMalloc(&Y.d_w, sizeof(float) * img.size());
  if (e == cudaSuccess) e = cudaMemcpy(Y.d_w, img.data(), sizeof(float) * img.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (Y.d_w) cudaFree(Y.d_w);
    *err = std::string("small-batch cluster kernel weights: ") + cudaGetErrorString(e);
    return FW_ERR_CUDA;
  }
  h.lat = new LatPlan{Y};
  return FW_OK;
}

static size_t lat_smem_bytes(const CellDims& d, const LatLayout& Y) {
  const int64_t wfl = Y.resident ? Y.step_floats : 2 * Y.max_block;
  const int64_t act = 2 * (2 * d.R + d.D + kLatPad) + (int64_t)d.L * d.R + ((Y.Sc + 3) & ~3) +
                      d.S + kLatPad + d.H + kLatPad + d.A + 4 + 4;  // + 2 mbarriers, + cls
  return sizeof(float) * (size_t)(wfl + act) + 16;
}

template <int C>
static cudaError_t lat_launch(const LatParams& p, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(cell_lat_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  if (C > 8) {
    e = cudaFuncSetAttribute(cell_lat_kernel<C>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.B * C);
  cfg.blockDim = dim3(kLatNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  void* args[] = {const_cast<LatParams*>(&p)};
  return cudaLaunchKernelExC(&cfg, (const void*)cell_lat_kernel<C>, args);
}

// Launches the small-batch kernel with clusters of C CTAs; returns cudaErrorNotSupported
// (nothing launched) when the shape does not fit it.
cudaError_t launch_cell_lat(Handle& h, const CellRun& run, int C, cudaStream_t st) {
  if (!lat_supported(h.dims, C)) return cudaErrorNotSupported;
  std::string err;
  const int rc = lat_prepare(h, C, &err);
  if (rc == FW_ERR_UNSUPPORTED) return cudaErrorNotSupported;
  if (rc != FW_OK) {
    set_error(err);
    return cudaErrorMemoryAllocation;
  }
  LatParams p;
  p.d = h.dims;
  p.B = h.batch;
  p.dil = h.d_dil;
  p.qoff = h.d_qoff;
  p.queue = h.d_queue;
  p.embed = h.w.embed;
  p.w = h.lat->lay.d_w;
  p.lay = h.lat->lay;
  p.run = run;
  const size_t smem = lat_smem_bytes(h.dims, p.lay);
  switch (C) {
    case 2: return lat_launch<2>(p, smem, st);
    case 4: return lat_launch<4>(p, smem, st);
    case 8: return lat_launch<8>(p, smem, st);
    case 16: return lat_launch<16>(p, smem, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace fw
