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

constexpr int kLatNT = 512;   // 16 warps: the phases are latency-bound, more lanes per GEMV
constexpr int kLatPad = 128;  // zero floats after every input vector (padded GEMV rows)

constexpr int lat_pow2_floor(int v) {
  int p = 1;
  while (p * 2 <= v) p *= 2;
  return p;
}
constexpr int lat_max(int a, int b) { return a > b ? a : b; }
constexpr int lat_min(int a, int b) { return a < b ? a : b; }
constexpr int64_t lat_max64(int64_t a, int64_t b) { return a > b ? a : b; }
// lanes per output so that the n outputs fill `threads` (at most max_lpo)
constexpr int lpo_for(int n, int max_lpo, int threads) {
  return lat_max(1, lat_min(lat_pow2_floor(lat_max(1, threads / lat_max(n, 1))), max_lpo));
}
// row stride (floats): K rounded up to whole chunks of every lane of an output group
// (4 lpo floats, at least 32), then offset so the 16-byte chunks a quarter-warp loads -- 8 / lpo
// rows, lpo consecutive chunks each -- land in distinct bank groups
constexpr int kpad(int K, int lpo) {
  return lpo < 8 ? (K + lat_max(32, 4 * lpo) - 1) / lat_max(32, 4 * lpo) * lat_max(32, 4 * lpo) + 4 * lpo
                 : (K + lat_max(32, 4 * lpo) - 1) / lat_max(32, 4 * lpo) * lat_max(32, 4 * lpo);
}
constexpr int64_t up4(int64_t v) { return (v + 3) & ~(int64_t)3; }  // 16-byte granules
constexpr int lat_lg2(int v) {
  int r = 0;
  while ((1 << r) < v) ++r;
  return r;
}

// Geometry of one rank's weight blocks for a shape (R, D, S, H, A) and cluster size C --
// independent of L. Computed at compile time for the BASELINE shapes the kernel is
// specialised for (the loops of the phases then unroll), at run time otherwise.
struct LatGeom {
  int Dc, Rc, Sc, Hc, Ac;
  int Kd, Kpd, lpo_d;    // dil: K = 2R + D, padded row, lanes per output
  int Kprs, lpo_rs;      // res | skip rows over z (K = D)
  int Kph1, lpo_h1;      // head1 over ReLU(s) (K = S)
  int Kph2, lpo_h2;      // head2 over h (K = H)
  int lg_d, lg_rs, lg_h1, lg_h2;  // log2 of the lanes per output
  // float offsets inside a phase block
  int64_t o_dil, o_bd, o_rs, o_br, o_bs, phase_floats;
  int64_t post_floats;   // block L: skip rows + bias
  int64_t h1_floats, h2_floats;  // one head block: rows (h1r / h2r of the slice) + biases
  int h1p, h2p, h1r, h2r;          // head slices split into parts of at most h1r / h2r rows
  int64_t max_block;
};

constexpr LatGeom lat_geom(int R, int D, int S, int H, int A, int C) {
  LatGeom g{};
  g.Dc = D / C;
  g.Rc = R / C;
  g.Sc = S / C;
  g.Hc = H / C;
  g.Ac = A / C;
  g.Kd = 2 * R + D;
  g.lpo_d = lpo_for(2 * g.Dc, 16, kLatNT / 2);  // a z column's two rows in one warp
  g.Kpd = kpad(g.Kd, g.lpo_d);
  g.lpo_rs = lpo_for(g.Rc + g.Sc, 32, kLatNT / 2);
  g.Kprs = kpad(D, g.lpo_rs);
  g.lpo_h1 = lpo_for(g.Hc, 32, kLatNT);
  g.Kph1 = kpad(S, g.lpo_h1);
  g.lpo_h2 = lpo_for(g.Ac, 32, kLatNT);
  g.Kph2 = kpad(H, g.lpo_h2);
  g.lg_d = lat_lg2(g.lpo_d);
  g.lg_rs = lat_lg2(g.lpo_rs);
  g.lg_h1 = lat_lg2(g.lpo_h1);
  g.lg_h2 = lat_lg2(g.lpo_h2);
  g.o_dil = 0;
  g.o_bd = up4((int64_t)2 * g.Dc * g.Kpd);
  g.o_rs = g.o_bd + up4(2 * g.Dc);
  g.o_br = g.o_rs + up4((int64_t)(g.Rc + g.Sc) * g.Kprs);
  g.o_bs = g.o_br + up4(g.Rc);
  g.phase_floats = g.o_bs + up4(g.Sc);
  g.post_floats = up4((int64_t)g.Sc * g.Kprs) + up4(g.Sc);
  // head slices in parts no larger than a phase block (the ring's slot size), so a config
  // with wide heads and narrow layers (cfg3) still streams through two slots
  const int64_t cap = lat_max64(g.phase_floats, g.post_floats);
  g.h1r = g.Hc;
  g.h1p = 1;
  while (g.h1r > 1 && up4((int64_t)g.h1r * g.Kph1) + up4(g.h1r) > cap) g.h1r = (g.Hc + ++g.h1p - 1) / g.h1p;
  g.h1p = (g.Hc + g.h1r - 1) / g.h1r;
  g.h1_floats = up4((int64_t)g.h1r * g.Kph1) + up4(g.h1r);
  g.h2r = g.Ac;
  g.h2p = 1;
  while (g.h2r > 1 && up4((int64_t)g.h2r * g.Kph2) + up4(g.h2r) > cap) g.h2r = (g.Ac + ++g.h2p - 1) / g.h2p;
  g.h2p = (g.Ac + g.h2r - 1) / g.h2r;
  g.h2_floats = up4((int64_t)g.h2r * g.Kph2) + up4(g.h2r);
  g.max_block = lat_max64(lat_max64(g.phase_floats, g.post_floats), lat_max64(g.h1_floats, g.h2_floats));
  return g;
}

// Per-C packed weights and their layout (host-computed, uploaded once per handle and C).
struct LatLayout {
  int C = 0;
  LatGeom g{};
  int64_t step_floats;      // all blocks of a step (per rank)
  int resident;
  float* d_w = nullptr;     // [C][step_floats]
};

// Compile-time shapes the kernel is specialised for (0: the generic kernel, shape at run
// time): BASELINE configs 1, 2 and 3 at their cluster sizes.
template <int R_, int D_, int S_, int H_, int A_, int C_>
struct LatShape {
  static constexpr bool kFixed = true;
  static constexpr int R = R_, D = D_, S = S_, H = H_, A = A_;
  static constexpr LatGeom G = lat_geom(R_, D_, S_, H_, A_, C_);
};
struct LatAnyShape {
  static constexpr bool kFixed = false;
  static constexpr int R = 0, D = 0, S = 0, H = 0, A = 0;
  static constexpr LatGeom G{};
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
  long long* trace;  // diagnostics: [phase][8] globaltimer stamps of CTA 0 in step 1, or null
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
// out[o] = sum_k W[o * Kp + k] * in[k] for o < n: LPO lanes per output, lane `sub` takes the
// 16-byte chunks k = 4 (sub + LPO i) .. +3 (LDS.128 of weights and inputs; rows padded so
// a warp's chunks fall in distinct banks, inputs padded with zeros past K), two
// accumulators, fixed-order shuffle reduction; epi(o, v, sub, lpo) on every lane.
// The warps [w0, w0 + nw) of the CTA compute it (the layer phases run the dilated GEMV and
// the residual/skip GEMV side by side on the two halves of the CTA).
template <typename Epi>
__device__ __forceinline__ void lat_gemv(const float* W, int Kp, int K, int n, int lg_lpo,
                                         const float* in, Epi epi, int w0 = 0, int nw = kLatNT / 32) {
  const int warp = (threadIdx.x >> 5) - w0, lane = threadIdx.x & 31;
  if (warp < 0 || warp >= nw) return;
  const int lpo = 1 << lg_lpo, opw = 32 >> lg_lpo, sub = lane & (lpo - 1);
  const float4* in4 = reinterpret_cast<const float4*>(in);
  for (int o0 = warp * opw; o0 < n; o0 += nw * opw) {
    const int o = o0 + (lane >> lg_lpo);
    float a0 = 0.f, a1 = 0.f;
    if (o < n) {
      const float4* w4 = reinterpret_cast<const float4*>(W + (int64_t)o * Kp);
      int c = sub;  // 16-byte chunk index
      const int nc = (K + 3) >> 2;
      for (; c + lpo < nc; c += 2 * lpo) {
        const float4 w0 = w4[c], x0 = in4[c], w1 = w4[c + lpo], x1 = in4[c + lpo];
        a0 = fmaf(w0.x, x0.x, a0);
        a1 = fmaf(w1.x, x1.x, a1);
        a0 = fmaf(w0.y, x0.y, a0);
        a1 = fmaf(w1.y, x1.y, a1);
        a0 = fmaf(w0.z, x0.z, a0);
        a1 = fmaf(w1.z, x1.z, a1);
        a0 = fmaf(w0.w, x0.w, a0);
        a1 = fmaf(w1.w, x1.w, a1);
      }
      if (c < nc) {
        const float4 w0 = w4[c], x0 = in4[c];
        a0 = fmaf(w0.x, x0.x, a0);
        a0 = fmaf(w0.y, x0.y, a0);
        a0 = fmaf(w0.z, x0.z, a0);
        a0 = fmaf(w0.w, x0.w, a0);
      }
    }
    float v = a0 + a1;
    for (int off = lpo >> 1; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    epi(o, v, sub, lpo);
  }
}

// fp32 gate, MUFU-based: tanh(a) = 1 - 2 / (e^{2a} + 1), sigmoid(g) = 1 / (1 + e^{-g});
// absolute error ~1e-7 (the SIMT configs' logits tolerance is 1e-4)
__device__ __forceinline__ float lat_gate(float a, float g) {
  const float th = 1.f - 2.f * __frcp_rn(__expf(2.f * a) + 1.f);
  return th * __frcp_rn(1.f + __expf(-g));
}

// Asynchronous remote store: v -> shared::cluster address `addr`, completing `bytes` of the
// transaction count of the receiver's mbarrier `mbar` (also a shared::cluster address).
__device__ __forceinline__ void lat_st_async(uint32_t addr, float v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr),
               "r"(__float_as_uint(v)), "r"(mbar)
               : "memory");
}
// Wait for a phase of a local mbarrier completed by other CTAs' st.async transactions: the
// data is shared memory of this CTA, so a CTA-scope acquire suffices (a cluster-scope one
// would also invalidate L1 -- CCTL.IVALL -- on every exchange).
__device__ __forceinline__ void lat_wait(uint64_t* bar, uint32_t parity) { ptx::mbar_wait(bar, parity); }
__device__ __forceinline__ long long lat_now() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One exchange: this CTA's staged slices -> the same floats of every CTA of the cluster,
// signalling each receiver's mbarrier `bar`. Up to three segments (src, dst, n) flattened
// into one index space so every thread issues at most a few remote stores (a st.async is
// not free to issue: ~ the DSMEM round trip).
struct LatSeg {
  const float* src;
  float* dst;
  int n;
};
__device__ __forceinline__ void lat_st_async4(uint32_t addr, float4 v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(addr),
               "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
               "r"(__float_as_uint(v.w)), "r"(mbar)
               : "memory");
}
// items (16-byte chunks when the segment allows it, else single floats) of one segment
__device__ __forceinline__ int lat_items(const LatSeg& s) {
  const bool v4 = (s.n & 3) == 0 && ((reinterpret_cast<uintptr_t>(s.dst) | reinterpret_cast<uintptr_t>(s.src)) & 15) == 0;
  return v4 ? s.n >> 2 : s.n;
}
template <int C>
__device__ __forceinline__ void lat_send1(const LatSeg& s, int f, uint32_t bar_local) {
  const int k = f / C;
  const uint32_t q = (uint32_t)(f - k * C);
  const uint32_t mbar = lat_mapa(reinterpret_cast<const float*>(__cvta_shared_to_generic(bar_local)), q);
  if (lat_items(s) != s.n)
    lat_st_async4(lat_mapa(s.dst + 4 * k, q), reinterpret_cast<const float4*>(s.src)[k], mbar);
  else
    lat_st_async(lat_mapa(s.dst + k, q), s.src[k], mbar);
}
template <int C>
__device__ __forceinline__ void lat_send(LatSeg a, LatSeg b, LatSeg c, uint64_t* bar) {
  const int na = lat_items(a) * C, nb = lat_items(b) * C, nall = na + nb + lat_items(c) * C;
  const uint32_t bl = ptx::smem_u32(bar);
  for (int e = threadIdx.x; e < nall; e += kLatNT) {
    if (e < na)
      lat_send1<C>(a, e, bl);
    else if (e < na + nb)
      lat_send1<C>(b, e - na, bl);
    else
      lat_send1<C>(c, e - na - nb, bl);
  }
}

template <int C, class Sh>
__global__ void __launch_bounds__(kLatNT) cell_lat_kernel(LatParams p) {
  extern __shared__ __align__(16) float smem[];
  const CellDims d = p.d;
  const LatLayout& Yr = p.lay;
  // the geometry: compile-time constants for a specialised shape (the phases' loops unroll)
  const LatGeom Y = Sh::kFixed ? Sh::G : Yr.g;
  const int R = Sh::kFixed ? Sh::R : d.R, D = Sh::kFixed ? Sh::D : d.D,
            S = Sh::kFixed ? Sh::S : d.S, H = Sh::kFixed ? Sh::H : d.H,
            A = Sh::kFixed ? Sh::A : d.A, L = d.L;
  const int Dc = Y.Dc, Rc = Y.Rc, Sc = Y.Sc, Hc = Y.Hc, Ac = Y.Ac;
  const uint32_t rank = lat_rank();
  const int stream = blockIdx.x / C;
  const int tid = threadIdx.x;
  const int j0 = (int)rank * Dc, r0 = (int)rank * Rc, k0 = (int)rank * Sc;
  const int h0 = (int)rank * Hc, a0 = (int)rank * Ac;
  // shared memory: weights | barriers (ring [2], exchange [2]) | inbuf[2][2R + D + pad] |
  // staged slices (z, x, x_{t-d}, ReLU(s), h, logits) | s[Sc] | sf[S + pad] | hf[H + pad] |
  // lg[A] | cls
  float* wsm = smem;
  const int64_t wfl = Yr.resident ? Yr.step_floats : 2 * Y.max_block;
  const int in_len = (2 * R + D + kLatPad + 3) & ~3;
  uint64_t* full = reinterpret_cast<uint64_t*>(wsm + wfl);  // [2] weight ring slots
  uint64_t* xbar = full + 2;                                  // [2] exchanges (alternating)
  float* inbuf = wsm + wfl + 8;
  // staged outputs of this CTA (<= Dc + 2 Rc or Sc + Rc, Hc, Ac), double-buffered by
  // exchange parity: a thread still sending exchange e reads them while the fastest thread
  // can already be writing exchange e + 1's (it cannot reach e + 2 before every thread of
  // this CTA has sent e + 1)
  float* stg2 = inbuf + 2 * in_len;
  const int stg_len = (max(max(Dc + 2 * Rc, Sc + Rc), max(Hc, Ac)) + 3) & ~3;
  float* s_s = stg2 + 2 * stg_len;
  float* sf = s_s + ((Sc + 3) & ~3);
  float* hf = sf + ((S + kLatPad + 3) & ~3);
  float* lg = hf + ((H + kLatPad + 3) & ~3);
  int* cls = reinterpret_cast<int*>(lg + A);
  // this step's ring slot base (element offset) of every layer, + layer 0's of the next step
  int64_t* rslot = reinterpret_cast<int64_t*>((reinterpret_cast<uintptr_t>(cls + 4) + 7) & ~(uintptr_t)7);
  const float* wg = p.w + (int64_t)rank * Yr.step_floats;  // this rank's blocks in global
  // blocks of a step: L phases, the top skip, h1p parts of head1, h2p parts of head2
  const int nblk = L + 1 + Y.h1p + Y.h2p;
  auto block_off = [&](int b) -> int64_t {  // float offset of block b inside a step
    if (b <= L) return (int64_t)b * Y.phase_floats;
    const int64_t hb = (int64_t)L * Y.phase_floats + Y.post_floats;
    const int p = b - L - 1;
    return p < Y.h1p ? hb + p * Y.h1_floats : hb + Y.h1p * Y.h1_floats + (p - Y.h1p) * Y.h2_floats;
  };
  auto block_len = [&](int b) -> int64_t {
    return b < L ? Y.phase_floats : (b == L ? Y.post_floats : (b - L - 1 < Y.h1p ? Y.h1_floats : Y.h2_floats));
  };
  const CellRun& run = p.run;
  const int B = p.B;
  const int Rp = (R + 3) & ~3;
  const size_t slot_elems = (size_t)((B + 127) / 128) * 128 * Rp;
  const int64_t soff = (int64_t)(stream >> 7) * (Rp / 4) * 512 + (stream & 127) * 4;
  auto ring_at = [&](int64_t base, int r) {  // channel r of this stream in the slot at `base`
    return p.queue + base + soff + (int64_t)(r >> 2) * 512 + (r & 3);
  };
  auto slot_base = [&](int l, int64_t t) { return p.qoff[l] + (t % p.dil[l]) * (int64_t)slot_elems; };
  // control duties (weight-ring copies, exchange arming, trace stamps) sit on the last
  // thread, which owns no ring channel and (for up to kLatNT - 1 items) sends nothing
  const int ctl = kLatNT - 1;
  const bool tracer = p.trace != nullptr && blockIdx.x == 0 && tid == ctl;
  auto stamp = [&](int i, int ph, int k) {
    if (tracer && i == 1) p.trace[ph * 8 + k] = lat_now();
  };

  // zero the padded tails of the input vectors (the padded weight columns are zero, so the
  // pads must be finite); barriers; resident weights
  for (int e = tid; e < 2 * in_len; e += kLatNT) inbuf[e] = 0.f;
  for (int e = tid; e < S + kLatPad; e += kLatNT) sf[e] = 0.f;
  for (int e = tid; e < H + kLatPad; e += kLatNT) hf[e] = 0.f;
  if (tid == ctl) {
    for (int k = 0; k < 4; ++k) ptx::mbar_init(&full[k], 1);
    ptx::fence_mbar_init();
  }
  // every CTA's exchange barriers exist before any remote store targets them
  lat_cluster_sync();
  int64_t g = 0;  // weight blocks consumed (ring mode)
  auto issue = [&](int64_t gi) {  // ring: block gi of the launch into slot gi & 1
    const int b = (int)(gi % nblk);
    const uint32_t bytes = (uint32_t)(block_len(b) * 4);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::mbar_arrive_expect_tx(&full[gi & 1], bytes);
    ptx::bulk_g2s(wsm + (gi & 1) * Y.max_block, wg + block_off(b), bytes, &full[gi & 1]);
  };
  if (tid == ctl) {
    if (Yr.resident) {
      const uint32_t bytes = (uint32_t)(Yr.step_floats * 4);
      ptx::mbar_arrive_expect_tx(&full[0], bytes);
      ptx::bulk_g2s(wsm, wg, bytes, &full[0]);
    } else {
      issue(0);
    }
  }
  // block b of the current step, waited for; the next block's copy goes into the slot the
  // previous phase released (every phase ends with a CTA barrier before its sends)
  auto take = [&](int b) -> const float* {
    if (Yr.resident) return wsm + block_off(b);
    ptx::mbar_wait(&full[g & 1], (uint32_t)((g >> 1) & 1));
    const float* w = wsm + (g & 1) * Y.max_block;
    if (tid == ctl && g + 1 < (int64_t)run.n_steps * nblk) issue(g + 1);
    ++g;
    return w;
  };
  if (Yr.resident) ptx::mbar_wait(&full[0], 0);
  // exchange e of the launch completes on xbar[e & 1]; this CTA arms it with the bytes it
  // will receive (transactions that arrive first drive the count negative until then)
  int64_t ex = 0;
  auto arm = [&](int64_t e, int floats) {
    if (tid == ctl)  // relaxed: orders nothing this thread did before (it sent nothing)
      asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                       ptx::smem_u32(&xbar[e & 1])), "r"((uint32_t)(floats * 4))
                   : "memory");
  };
  auto wait_ex = [&](int64_t e) { lat_wait(&xbar[e & 1], (uint32_t)((e >> 1) & 1)); };
  // the first step's x_0[t-d] (later steps': exchanged with ReLU(s) of the step before)
  for (int r = tid; r < R; r += kLatNT) inbuf[R + r] = __ldcg(ring_at(slot_base(0, run.t0), r));
  if (tid == 0) cls[0] = run.inputs[stream];
  __syncthreads();

  for (int i = 0; i < run.n_steps; ++i) {
    const int64_t t = run.t0 + i;
    const bool more = i + 1 < run.n_steps;
    // phase 0 input: x_0 = E[c_t] (z part: any finite value, its weights are zero); the
    // step's ring slots (one modulo per layer per step)
    {
      const float* e = p.embed + (size_t)clamp_class(cls[0], A) * R;
      for (int r = tid; r < R; r += kLatNT) inbuf[r] = __ldg(e + r);
      for (int k = tid; k < Sc; k += kLatNT) s_s[k] = 0.f;
      for (int l = tid; l <= L; l += kLatNT) rslot[l] = l < L ? slot_base(l, t) : slot_base(0, t + 1);
    }
    __syncthreads();
    for (int l = 0; l < L; ++l) {
      // ring pops and pushes of channel r0 + tid are this thread's alone (tid < Rc): it reads
      // back only its own earlier stores (program order, no cross-CTA fence); the pop of
      // the next layer's slot is issued first, its value is needed at the end of the phase
      const bool pop = l + 1 < L;
      float popv = 0.f;
      if (pop && tid < Rc) popv = __ldcg(ring_at(rslot[l + 1], r0 + tid));
      stamp(i, l, 0);
      if (l > 0) wait_ex(ex - 1);  // x_{l-1}, z_{l-1}, x_l[t-d_l] from every CTA
      stamp(i, l, 1);
      const float* wb = take(l);
      const float* in = inbuf + (l & 1) * in_len;
      float* nxt = inbuf + ((l + 1) & 1) * in_len;
      float* stg = stg2 + (ex & 1) * stg_len;
      // data of the next phase (or the top layer's z for the skip): armed before this CTA
      // sends its own part of it
      arm(ex, D + R + (pop ? R : 0));
      // dilated taps (+ folded residual) of this CTA's z columns; rows 2j / 2j+1 = the
      // tanh / sigmoid pre-activation of column j0 + j
      const float* bd = wb + Y.o_bd;
      constexpr int kHalf = kLatNT / 64;  // warps per GEMV of a layer phase
      lat_gemv(wb + Y.o_dil, Y.Kpd, Y.Kd, 2 * Dc, Y.lg_d, in, [&](int o, float v, int sub, int lpo) {
        const float pv = __shfl_down_sync(0xffffffffu, v, lpo);  // the sigmoid row's sum
        if (o < 2 * Dc && sub == 0 && (o & 1) == 0)
          stg[o >> 1] = lat_gate(v + bd[o], pv + bd[o + 1]);
      }, 0, kHalf);
      stamp(i, l, 2);
      // x_l slice (residual of the previous layer; x_0 itself at l = 0); s slice += skip of
      // the previous layer
      const float* br = wb + Y.o_br;
      const float* bs = wb + Y.o_bs;
      lat_gemv(wb + Y.o_rs, Y.Kprs, D, Rc + Sc, Y.lg_rs, in + 2 * R, [&](int o, float v, int sub, int) {
        if (o < Rc + Sc && sub == 0) {
          if (o < Rc)
            stg[Dc + o] = in[r0 + o] + v + br[o];
          else if (l > 0)
            s_s[o - Rc] += v + bs[o - Rc];
        }
      }, kHalf, kHalf);
      stamp(i, l, 3);
      if (pop && tid < Rc) stg[Dc + Rc + tid] = popv;
      stamp(i, l, 4);
      __syncthreads();  // every warp is done with `in` and the staged slices are complete
      stamp(i, l, 5);
      lat_send<C>(LatSeg{stg, nxt + 2 * R + j0, Dc}, LatSeg{stg + Dc, nxt + r0, Rc},
                  LatSeg{stg + Dc + Rc, nxt + R + r0, pop ? Rc : 0}, &xbar[ex & 1]);
      stamp(i, l, 6);
      if (tid < Rc) *ring_at(rslot[l], r0 + tid) = stg[Dc + tid];  // push x_l[t]
      stamp(i, l, 7);
      ++ex;
    }
    // the top layer's skip: s += W_skip,L-1 z_{L-1} + b; ReLU(s) (+ the next step's
    // x_0[t+1-d_0] slice, popped by the thread that pushed it) to every CTA
    {
      float popv = 0.f;
      if (more && tid < Rc) popv = __ldcg(ring_at(rslot[L], r0 + tid));
      stamp(i, L, 0);
      wait_ex(ex - 1);
      stamp(i, L, 1);
      const float* wb = take(L);
      const float* in = inbuf + (L & 1) * in_len;
      float* stg = stg2 + (ex & 1) * stg_len;
      arm(ex, S + (more ? R : 0));
      lat_gemv(wb, Y.Kprs, D, Sc, Y.lg_rs, in + 2 * R, [&](int o, float v, int sub, int) {
        if (o < Sc && sub == 0) stg[o] = fmaxf(s_s[o] + v + wb[(int64_t)Sc * Y.Kprs + o], 0.f);
      });
      stamp(i, L, 2);
      if (more && tid < Rc) stg[Sc + tid] = popv;
      stamp(i, L, 4);
      __syncthreads();
      stamp(i, L, 5);
      lat_send<C>(LatSeg{stg, sf + k0, Sc}, LatSeg{stg + Sc, inbuf + R + r0, more ? Rc : 0},
                  LatSeg{stg, stg, 0}, &xbar[ex & 1]);
      stamp(i, L, 6);
      ++ex;
    }
    stamp(i, L + 1, 0);
    wait_ex(ex - 1);
    stamp(i, L + 1, 1);
    {
      float* stg = stg2 + (ex & 1) * stg_len;
      arm(ex, H);
      for (int part = 0; part < Y.h1p; ++part) {  // rows [part * h1r, ...) of the slice
        const float* wb = take(L + 1 + part);
        const int o0 = part * Y.h1r, n = min(Y.h1r, Hc - o0);
        lat_gemv(wb, Y.Kph1, S, n, Y.lg_h1, sf, [&](int o, float v, int sub, int) {
          if (o < n && sub == 0) stg[o0 + o] = fmaxf(v + wb[(int64_t)Y.h1r * Y.Kph1 + o], 0.f);
        });
        if (part + 1 < Y.h1p) __syncthreads();  // the ring slot is reused two parts on
      }
      __syncthreads();
      lat_send<C>(LatSeg{stg, hf + h0, Hc}, LatSeg{stg, stg, 0}, LatSeg{stg, stg, 0}, &xbar[ex & 1]);
      ++ex;
    }
    stamp(i, L + 2, 0);
    wait_ex(ex - 1);
    stamp(i, L + 2, 1);
    {
      float* stg = stg2 + (ex & 1) * stg_len;
      arm(ex, A);
      float* dst = (run.logits != nullptr && i < run.n_logit_steps)
                       ? run.logits + ((size_t)i * B + stream) * A + a0 : nullptr;
      for (int part = 0; part < Y.h2p; ++part) {
        const float* wb = take(L + 1 + Y.h1p + part);
        const int o0 = part * Y.h2r, n = min(Y.h2r, Ac - o0);
        lat_gemv(wb, Y.Kph2, H, n, Y.lg_h2, hf, [&](int o, float v, int sub, int) {
          if (o < n && sub == 0) {
            const float x = v + wb[(int64_t)Y.h2r * Y.Kph2 + o];
            stg[o0 + o] = x;
            if (dst) dst[o0 + o] = x;
          }
        });
        if (part + 1 < Y.h2p) __syncthreads();
      }
      __syncthreads();
      lat_send<C>(LatSeg{stg, lg + a0, Ac}, LatSeg{stg, stg, 0}, LatSeg{stg, stg, 0}, &xbar[ex & 1]);
      ++ex;
    }
    stamp(i, L + 3, 0);
    wait_ex(ex - 1);
    stamp(i, L + 3, 1);
    if (tid < 32) {
      const uint32_t prefix = noise_prefix(run.seed, (uint32_t)(run.stream_offset + stream), (uint32_t)t);
      const int c = select_class(lg, A, run.mode, prefix);
      if (tid == 0) {
        if (rank == 0) run.out[(size_t)i * B + stream] = c;
        cls[0] = more && i + 1 < run.n_inputs ? run.inputs[(size_t)(i + 1) * B + stream] : c;
      }
    }
    __syncthreads();
    stamp(i, L + 3, 2);
  }
  lat_cluster_sync();  // no remote stores into a CTA that has exited
}

// shared memory beside the weights (floats): barriers, inbuf, staged slices, s, sf, hf,
// lg, cls -- the kernel's carve-up
int64_t lat_act_floats(const CellDims& d, const LatGeom& Y) {
  const int64_t stg = up4(std::max(std::max(Y.Dc + 2 * Y.Rc, Y.Sc + Y.Rc), std::max(Y.Hc, Y.Ac)));
  return 8 + 2 * up4(2 * d.R + d.D + kLatPad) + 2 * stg + up4(Y.Sc) + up4(d.S + kLatPad) + up4(d.H + kLatPad) +
         d.A + 4 + 2 * (d.L + 1) + 2;
}

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
  LatLayout Yl;
  Yl.C = C;
  Yl.g = lat_geom(R, D, S, H, A, C);
  const LatGeom& Y = Yl.g;
  Yl.step_floats = (int64_t)L * Y.phase_floats + Y.post_floats + Y.h1p * Y.h1_floats + Y.h2p * Y.h2_floats;
  // activations + barriers beside the weights; resident when a step's blocks fit
  const int64_t act_floats = lat_act_floats(d, Y);
  const int64_t budget = 220 * 1024 / 4;
  Yl.resident = (Yl.step_floats + act_floats <= budget && Yl.step_floats * 4 < (1u << 20)) ? 1 : 0;
  if (!Yl.resident && 2 * Y.max_block + act_floats > budget) {
    *err = "small-batch cluster kernel: a phase's weight slices exceed shared memory";
    return FW_ERR_UNSUPPORTED;
  }
  std::vector<float> img((size_t)C * Yl.step_floats, 0.f);
  // [l][o][k] accessors of the host model (reference layouts)
  auto W0 = [&](int l, int o, int k) { return (double)w.dil_w[(((size_t)l * 2 + 0) * 2 * D + o) * R + k]; };
  auto W1 = [&](int l, int o, int k) { return (double)w.dil_w[(((size_t)l * 2 + 1) * 2 * D + o) * R + k]; };
  auto Wr = [&](int l, int r, int k) { return (double)w.res_w[((size_t)l * R + r) * D + k]; };
  auto Ws = [&](int l, int s, int k) { return (double)w.skip_w[((size_t)l * S + s) * D + k]; };
  for (int q = 0; q < C; ++q) {
    float* base = img.data() + (size_t)q * Yl.step_floats;
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
      float* part = h1 + (o / Y.h1r) * Y.h1_floats;
      const int ro = o % Y.h1r;
      for (int k = 0; k < S; ++k) part[(int64_t)ro * Y.Kph1 + k] = w.h1_w[(size_t)(q * Y.Hc + o) * S + k];
      part[(int64_t)Y.h1r * Y.Kph1 + ro] = w.h1_b[q * Y.Hc + o];
    }
    float* h2 = h1 + Y.h1p * Y.h1_floats;
    for (int o = 0; o < Y.Ac; ++o) {
      float* part = h2 + (o / Y.h2r) * Y.h2_floats;
      const int ro = o % Y.h2r;
      for (int k = 0; k < H; ++k) part[(int64_t)ro * Y.Kph2 + k] = w.h2_w[(size_t)(q * Y.Ac + o) * H + k];
      part[(int64_t)Y.h2r * Y.Kph2 + ro] = w.h2_b[q * Y.Ac + o];
    }
  }
  cudaError_t e = cudaMalloc(&Yl.d_w, sizeof(float) * img.size());
  if (e == cudaSuccess) e = cudaMemcpy(Yl.d_w, img.data(), sizeof(float) * img.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (Yl.d_w) cudaFree(Yl.d_w);
    *err = std::string("small-batch cluster kernel weights: ") + cudaGetErrorString(e);
    return FW_ERR_CUDA;
  }
  h.lat = new LatPlan{Yl};
  return FW_OK;
}

static size_t lat_smem_bytes(const CellDims& d, const LatLayout& Y) {
  const int64_t wfl = Y.resident ? Y.step_floats : 2 * Y.g.max_block;
  return sizeof(float) * (size_t)(wfl + lat_act_floats(d, Y.g)) + 16;
}

template <int C, class Sh>
static cudaError_t lat_launch(const LatParams& p, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(cell_lat_kernel<C, Sh>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  if (C > 8) {
    e = cudaFuncSetAttribute(cell_lat_kernel<C, Sh>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
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
  return cudaLaunchKernelExC(&cfg, (const void*)cell_lat_kernel<C, Sh>, args);
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
  p.trace = h.lat_trace;
  const size_t smem = lat_smem_bytes(h.dims, p.lay);
  // BASELINE configs 1, 2 (every L) and 3 at their cluster sizes run a kernel specialised
  // for the shape (FW_LAT_GENERIC=1 forces the generic one)
  static const bool generic = getenv("FW_LAT_GENERIC") != nullptr;
  const CellDims& d = h.dims;
  auto is = [&](int R, int D, int S, int H, int A) {
    return !generic && d.R == R && d.D == D && d.S == S && d.H == H && d.A == A;
  };
  switch (C) {
    case 2:
      if (is(64, 64, 256, 256, 256)) return lat_launch<2, LatShape<64, 64, 256, 256, 256, 2>>(p, smem, st);
      return lat_launch<2, LatAnyShape>(p, smem, st);
    case 4: return lat_launch<4, LatAnyShape>(p, smem, st);
    case 8: return lat_launch<8, LatAnyShape>(p, smem, st);
    case 16:
      if (is(32, 32, 128, 128, 256)) return lat_launch<16, LatShape<32, 32, 128, 128, 256, 16>>(p, smem, st);
      if (is(128, 128, 256, 256, 256)) return lat_launch<16, LatShape<128, 128, 256, 256, 256, 16>>(p, smem, st);
      return lat_launch<16, LatAnyShape>(p, smem, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace fw
