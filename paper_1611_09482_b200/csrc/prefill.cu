// Full-sequence (time-parallel) forward of the gated cell over given inputs: SURVEY §8(f)
// rank 1, the GPU analogue of the reference's forward_full / causal_dilated_conv
// (oracle.py:84-123) applied to the cell, used to prefill the ring queues from a long
// primer (the reference steps primers one sample at a time, fast.py:244-245).
//
// fw_cell_prefill(h, inputs [T][B], T, logits?) leaves the handle exactly where T
// teacher-forced steps of fw_cell_generate would: every layer's ring holds the last d_l
// values of its input x_l, the step counter advances by T, and (if requested) the logits of
// all T steps are written. Instead of T dependent steps, time is processed in chunks of Tc
// steps, and within a chunk every layer runs once over all Tc*B (time, stream) rows:
//
//   Xcat = [x_l[t] | x_l[t-d_l]]      (x_l[t-d] from the chunk, or from the ring before it)
//   a    = Xcat W_dil + b_dil         (GEMM, fp32 accumulation)
//   z    = tanh(a[:D]) * sigmoid(a[D:])
//   ring slot (t mod d_l) <- x_l[t]   (the chunk's last min(d_l, Tc) steps)
//   x_{l+1} = x_l + z W_res + b_res   (GEMM accumulating onto x)
//   s   += z W_skip                   (GEMM accumulating onto s; only when logits are wanted)
//   logits = W2 ReLU(W1 ReLU(s + sum b_skip) + b1) + b2
//
// Every kernel here is hand-written (no library GEMM): the contractions run on
// gemm_rows<T>, a register-tiled 128 x 128 CUDA-core GEMM with fp32 accumulation and
// operands of type T -- fp32 for SIMT handles (the fp32 configs' exact arithmetic, no TF32),
// fp16 for tcgen05 handles (the precision their step kernel feeds the tensor cores: fp16
// x_t / x_{t-d} / z / ReLU(s) / h, bf16 weights, whose products are exact in fp32). Every
// channel count is allowed (no multiple-of-8 requirement): the elementwise kernels move one
// channel per thread and the GEMM predicates its edges. The ring is read and written in the
// handle's own slot layout.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "internal.h"
#include "select.cuh"

namespace fw {
namespace {

// ---- ring slot addressing (the handle's layout) -------------------------------------------
struct Ring {
  uint8_t* base;      // h.d_queue
  const int64_t* off; // [L] element offset (SIMT, floats) or byte offset (tcgen05) of layer l
  int64_t slot;       // slot stride: elements (SIMT) or bytes (tcgen05)
  int Rp;             // SIMT: channels padded to 4
  int fp16;           // tcgen05 layout
};
// SIMT: [B/128][Rp/4][128 streams][4 channels] fp32; tcgen05: [B/128][R/8][128 rows][8] fp16
__device__ __forceinline__ float ring_ld(const Ring& q, int l, int64_t s, int b, int r) {
  if (q.fp16)
    return __half2float(*reinterpret_cast<const __half*>(
        q.base + q.off[l] + s * q.slot + (int64_t)(b >> 7) * 32768 + (r >> 3) * 2048 + (b & 127) * 16 +
        (r & 7) * 2));
  const float* base = reinterpret_cast<const float*>(q.base) + q.off[l] + s * q.slot;
  return base[((int64_t)((b >> 7) * (q.Rp / 4) + (r >> 2)) * 128 + (b & 127)) * 4 + (r & 3)];
}
__device__ __forceinline__ void ring_st(const Ring& q, int l, int64_t s, int b, int r, float x) {
  if (q.fp16) {
    *reinterpret_cast<__half*>(q.base + q.off[l] + s * q.slot + (int64_t)(b >> 7) * 32768 +
                               (r >> 3) * 2048 + (b & 127) * 16 + (r & 7) * 2) = __float2half_rn(x);
    return;
  }
  float* base = reinterpret_cast<float*>(q.base) + q.off[l] + s * q.slot;
  base[((int64_t)((b >> 7) * (q.Rp / 4) + (r >> 2)) * 128 + (b & 127)) * 4 + (r & 3)] = x;
}

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__half x) { return __half2float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __half from_f<__half>(float x) { return __float2half_rn(x); }

// ---- elementwise kernels: one (row, channel) per thread, rows are (step, stream) ----------
// X[row][:] = embed[cls[row]][:], row = tt * B + b
__global__ void embed_rows(const int32_t* __restrict__ cls, const float* __restrict__ embed,
                           float* __restrict__ X, int64_t n, int R, int A) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * R) return;
  const int64_t row = e / R;
  const int r = (int)(e - row * R);
  X[e] = __ldg(embed + (int64_t)clamp_class(cls[row], A) * R + r);
}

// x_l = X + the previous layer's residual bias (add_bias writes it into X afterwards);
// Xcat[row] = [x_l[t] | x_l[t-d]] in the operand type; x_l[t-d] from this chunk's rows or,
// before the chunk, from ring slot (t mod d) (= (t-d) mod d, not yet overwritten). Rows
// with t-d inside the chunk read X of an earlier row -- the bias is added there too.
template <typename T>
__global__ void gather_taps(const float* __restrict__ X, const float* __restrict__ rbias,
                            T* __restrict__ Xcat, Ring q, int l, int d, int64_t t_abs0, int Tc,
                            int B, int R) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)Tc * B;
  if (e >= n * R) return;
  const int64_t row = e / R;
  const int r = (int)(e - row * R);
  const int tt = (int)(row / B), b = (int)(row - (int64_t)tt * B);
  const float bias = rbias ? __ldg(rbias + r) : 0.f;
  const float x = X[e] + bias;
  const float xd = tt - d >= 0 ? X[((int64_t)(tt - d) * B + b) * R + r] + bias
                               : ring_ld(q, l, (t_abs0 + tt) % d, b, r);
  Xcat[row * 2 * R + r] = from_f<T>(x);
  Xcat[row * 2 * R + R + r] = from_f<T>(xd);
}

// Y[row][c] += bias[c]
__global__ void add_bias(float* __restrict__ Y, const float* __restrict__ bias, int64_t n, int C) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * C) return;
  Y[e] += __ldg(bias + (int)(e % C));
}

// ring slot (t mod d) <- x_l[t] for the chunk's last min(d, Tc) steps
__global__ void push_taps(const float* __restrict__ X, Ring q, int l, int d, int64_t t_abs0, int Tc,
                          int B, int R) {
  const int first = Tc > d ? Tc - d : 0;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)(Tc - first) * B;
  if (e >= n * R) return;
  const int64_t row = e / R + (int64_t)first * B;
  const int r = (int)(e % R);
  const int tt = (int)(row / B), b = (int)(row - (int64_t)tt * B);
  ring_st(q, l, (t_abs0 + tt) % d, b, r, X[row * R + r]);
}

// z = tanh(a[:D] + b[:D]) * sigmoid(a[D:] + b[D:]) in the operand type
template <typename T>
__global__ void gate_rows(const float* __restrict__ Adil, const float* __restrict__ bias,
                          T* __restrict__ Z, int64_t n, int D) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * D) return;
  const int64_t row = e / D;
  const int c = (int)(e - row * D);
  const float a = Adil[row * 2 * D + c] + __ldg(bias + c);
  const float g = Adil[row * 2 * D + D + c] + __ldg(bias + D + c);
  Z[e] = from_f<T>(tanhf(a) * (1.f / (1.f + expf(-g))));
}

// out = ReLU(Y + bias) in the operand type
template <typename T>
__global__ void relu_rows(const float* __restrict__ Y, const float* __restrict__ bias, T* __restrict__ out,
                          int64_t n, int C) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * C) return;
  out[e] = from_f<T>(fmaxf(Y[e] + __ldg(bias + (int)(e % C)), 0.f));
}

__global__ void f32_to_f16(const float* __restrict__ src, __half* __restrict__ dst, int64_t n) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[e] = __float2half_rn(src[e]);
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }

// fw_cell_select: row i of logits [n][A] is stream i % B at step t0 + i / B; one warp per row
__global__ void select_rows(const float* __restrict__ logits, int64_t n, int B, int A, int mode,
                            uint32_t seed, int64_t stream_offset, int64_t t0, int32_t* __restrict__ out) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  const int b = (int)(row % B);
  const uint32_t prefix = noise_prefix(seed, (uint32_t)(stream_offset + b), (uint32_t)(t0 + row / B));
  const int c = select_class(logits + row * A, A, mode, prefix);
  if ((threadIdx.x & 31) == 0) out[row] = c;
}

// ---- GEMM: C[n][N] (+)= A[n][K] W[K][N], row-major, fp32 accumulation -------------------------
// 128 x 128 output tile per 256-thread CTA, K in slices of 16 staged through shared memory
// (A transposed to k-major so a thread's 8 rows are two float4 reads), 8 x 8 outputs per
// thread (rows ty*4 + {0..3, 64..67}, columns tx*4 + {0..3, 64..67}: conflict-free float4
// reads), double-buffered slices with the next slice's global loads in registers while the
// current one is multiplied. Edges are predicated (any n, K, N).
constexpr int kBM = 128, kBN = 128, kBK = 16, kGemmNT = 256;

template <typename T>
__global__ void __launch_bounds__(kGemmNT, 2) gemm_rows(const T* __restrict__ A, const T* __restrict__ W,
                                                     float* __restrict__ C, int64_t n, int K, int N,
                                                     int accumulate) {
  __shared__ __align__(16) float As[2][kBK][kBM];
  __shared__ __align__(16) float Ws[2][kBK][kBN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * kBM;
  const int n0 = blockIdx.x * kBN;
  // loader mapping: A slice = 128 rows x 16 k (8 elements per thread: row tid/2, k 8*(tid&1)..),
  // W slice = 16 k x 128 columns (8 per thread: k tid/16, columns 8*(tid&15)..)
  const int ar = tid >> 1, ak = (tid & 1) * 8;
  const int wk = tid >> 4, wc = (tid & 15) * 8;
  float ra[8], rw[8];
  auto load = [&](int k0) {
    const int64_t row = m0 + ar;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = k0 + ak + j;
      ra[j] = (row < n && k < K) ? to_f(A[row * K + k]) : 0.f;
    }
    const int k = k0 + wk;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = n0 + wc + j;
      rw[j] = (k < K && c < N) ? to_f(W[(int64_t)k * N + c]) : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 8; ++j) As[buf][ak + j][ar] = ra[j];
#pragma unroll
    for (int j = 0; j < 8; ++j) Ws[buf][wk][wc + j] = rw[j];
  };
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  const int nk = (K + kBK - 1) / kBK;
  load(0);
  store(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load((kt + 1) * kBK);
#pragma unroll
    for (int k = 0; k < kBK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + ty * 4]);
      const float4 w0 = *reinterpret_cast<const float4*>(&Ws[buf][k][tx * 4]);
      const float4 w1 = *reinterpret_cast<const float4*>(&Ws[buf][k][64 + tx * 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], wv[j], acc[i][j]);
    }
    if (kt + 1 < nk) {
      store(buf ^ 1);
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (row >= n) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (c >= N) continue;
      float* p = C + row * N + c;
      *p = accumulate ? *p + acc[i][j] : acc[i][j];
    }
  }
}

template <typename T>
cudaError_t gemm(const T* A, const T* W, float* C, int64_t n, int K, int N, bool accumulate,
                 cudaStream_t st) {
  const dim3 grid((unsigned)((N + kBN - 1) / kBN), (unsigned)((n + kBM - 1) / kBM));
  gemm_rows<T><<<grid, kGemmNT, 0, st>>>(A, W, C, n, K, N, accumulate ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace

// Per-handle prefill state: fp16 weight copies (tcgen05 handles), ring offsets, scratch.
struct PrefillState {
  __half *dil16 = nullptr, *res16 = nullptr, *skip16 = nullptr, *h116 = nullptr, *h216 = nullptr;
  float* bsum = nullptr;  // [S] sum of the skip biases
  int64_t* off = nullptr; // [L] ring offsets in the handle's units
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
};

void prefill_destroy(Handle& h) {
  PrefillState* p = h.prefill;
  if (!p) return;
  void* ptrs[] = {p->dil16, p->res16, p->skip16, p->h116, p->h216, p->bsum, p->off, p->scratch};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  delete p;
  h.prefill = nullptr;
}

namespace {

int pf_fail(const std::string& msg) {
  set_error(msg);
  return FW_ERR_CUDA;
}

#define PF_CUDA(call)                                                     \
  do {                                                                    \
    cudaError_t _e = (call);                                              \
    if (_e != cudaSuccess) return pf_fail(std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

int to_half_copy(__half** dst, const float* src, int64_t n) {
  PF_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), sizeof(__half) * (size_t)n));
  f32_to_f16<<<nblk(n), 256>>>(src, *dst, n);
  PF_CUDA(cudaGetLastError());
  return FW_OK;
}

int prefill_init(Handle& h) {
  if (h.prefill) return FW_OK;
  auto* p = new (std::nothrow) PrefillState();
  if (!p) return pf_fail("out of host memory");
  h.prefill = p;
  const CellDims& d = h.dims;
  const int L = d.L, R = d.R, D = d.D, S = d.S, H = d.H, A = d.A;
  const bool f16 = h.kernel == FW_KERNEL_TCGEN05;
  if (f16) {
    if (int rc = to_half_copy(&p->dil16, h.w.dilT, (int64_t)L * 2 * R * 2 * D)) return rc;
    if (int rc = to_half_copy(&p->res16, h.w.resT, (int64_t)L * D * R)) return rc;
    if (int rc = to_half_copy(&p->skip16, h.w.skipT, (int64_t)L * D * S)) return rc;
    if (int rc = to_half_copy(&p->h116, h.w.h1T, (int64_t)S * H)) return rc;
    if (int rc = to_half_copy(&p->h216, h.w.h2T, (int64_t)H * A)) return rc;
  }
  // sum of the skip biases (host side, from the device copy)
  std::vector<float> sb((size_t)L * S), bs(S, 0.f);
  PF_CUDA(cudaMemcpy(sb.data(), h.w.skip_b, sizeof(float) * sb.size(), cudaMemcpyDeviceToHost));
  for (int l = 0; l < L; ++l)
    for (int c = 0; c < S; ++c) bs[c] += sb[(size_t)l * S + c];
  PF_CUDA(cudaMalloc(&p->bsum, sizeof(float) * S));
  PF_CUDA(cudaMemcpy(p->bsum, bs.data(), sizeof(float) * S, cudaMemcpyHostToDevice));
  // ring offsets in the handle's units (capi.cu fw_cell_create / cell_tc.cu tc_create)
  std::vector<int64_t> off(L);
  const int Rp = (R + 3) & ~3;
  const int64_t Bp = ((int64_t)h.batch + 127) / 128 * 128;
  int64_t acc = 0;
  for (int l = 0; l < L; ++l) {
    off[l] = f16 ? acc * (h.batch / 64) * 16384 : acc * Bp * Rp;
    acc += h.dil[l];
  }
  PF_CUDA(cudaMalloc(&p->off, sizeof(int64_t) * L));
  PF_CUDA(cudaMemcpy(p->off, off.data(), sizeof(int64_t) * L, cudaMemcpyHostToDevice));
  PF_CUDA(cudaDeviceSynchronize());
  return FW_OK;
}

// The layer loop of one chunk, operand type T (float: SIMT handles, __half: tcgen05 handles).
template <typename T>
int prefill_chunk(Handle& h, PrefillState& p, const int32_t* cls, int tc, int64_t t_abs0, Ring q,
                  float* X, T* Xcat, float* Adil, T* Z, float* Sacc, T* Hin, float* H1, T* H1op,
                  float* logits, cudaStream_t st) {
  const CellDims& d = h.dims;
  const int L = d.L, R = d.R, D = d.D, S = d.S, H = d.H, A = d.A, B = h.batch;
  const bool f16 = sizeof(T) == 2;
  const bool heads = logits != nullptr;
  const int64_t n = (int64_t)tc * B;
  auto wsel = [&](const __half* w16, const float* w32) -> const T* {
    return f16 ? reinterpret_cast<const T*>(w16) : reinterpret_cast<const T*>(w32);
  };
  embed_rows<<<nblk(n * R), 256, 0, st>>>(cls, h.w.embed, X, n, R, A);
  for (int l = 0; l < L; ++l) {
    const int dl = h.dil[l];
    // x_l = X + b_res(l-1): the taps see it, X takes it right after
    const float* rb = l > 0 ? h.w.res_b + (size_t)(l - 1) * R : nullptr;
    gather_taps<T><<<nblk(n * R), 256, 0, st>>>(X, rb, Xcat, q, l, dl, t_abs0, tc, B, R);
    if (rb) add_bias<<<nblk(n * R), 256, 0, st>>>(X, rb, n, R);
    PF_CUDA(cudaGetLastError());
    const T* Wd = wsel(p.dil16 + (size_t)l * 2 * R * 2 * D, h.w.dilT + (size_t)l * 2 * R * 2 * D);
    PF_CUDA(gemm<T>(Xcat, Wd, Adil, n, 2 * R, 2 * D, false, st));
    gate_rows<T><<<nblk(n * D), 256, 0, st>>>(Adil, h.w.dil_b + (size_t)l * 2 * D, Z, n, D);
    // the ring takes x_l after this layer's taps were gathered
    push_taps<<<nblk((int64_t)std::min(tc, dl) * B * R), 256, 0, st>>>(X, q, l, dl, t_abs0, tc, B, R);
    PF_CUDA(cudaGetLastError());
    if (heads)
      PF_CUDA(gemm<T>(Z, wsel(p.skip16 + (size_t)l * D * S, h.w.skipT + (size_t)l * D * S), Sacc, n,
                      D, S, l > 0, st));
    if (l + 1 < L)
      PF_CUDA(gemm<T>(Z, wsel(p.res16 + (size_t)l * D * R, h.w.resT + (size_t)l * D * R), X, n, D,
                      R, true, st));
  }
  if (heads) {
    relu_rows<T><<<nblk(n * S), 256, 0, st>>>(Sacc, p.bsum, Hin, n, S);
    PF_CUDA(gemm<T>(Hin, wsel(p.h116, h.w.h1T), H1, n, S, H, false, st));
    relu_rows<T><<<nblk(n * H), 256, 0, st>>>(H1, h.w.h1_b, H1op, n, H);
    PF_CUDA(gemm<T>(H1op, wsel(p.h216, h.w.h2T), logits, n, H, A, false, st));
    add_bias<<<nblk(n * A), 256, 0, st>>>(logits, h.w.h2_b, n, A);
    PF_CUDA(cudaGetLastError());
  }
  return FW_OK;
}

}  // namespace

cudaError_t launch_cell_select(const Handle& h, const float* d_logits, int64_t n_rows, int64_t t0,
                               int mode, uint32_t seed, int64_t stream_offset, int32_t* d_out,
                               cudaStream_t st) {
  select_rows<<<(unsigned)((n_rows + 7) / 8), 256, 0, st>>>(d_logits, n_rows, h.user_batch, h.dims.A,
                                                          mode, seed, stream_offset, t0, d_out);
  return cudaGetLastError();
}

int cell_prefill(Handle& h, const int32_t* d_inputs, int T, float* d_logits, cudaStream_t st) {
  if (int rc = prefill_init(h)) return rc;
  PrefillState& p = *h.prefill;
  const CellDims& d = h.dims;
  const int R = d.R, D = d.D, S = d.S, H = d.H, A = d.A, B = h.batch;
  const bool f16 = h.kernel == FW_KERNEL_TCGEN05;
  const bool heads = d_logits != nullptr;
  const size_t ob = f16 ? 2 : 4;  // operand bytes
  // chunk: ~64K rows (FW_PREFILL_CHUNK overrides the steps per chunk, for tests)
  int Tc = (int)std::max<int64_t>(1, std::min<int64_t>(T, 65536 / B));
  if (const char* e = getenv("FW_PREFILL_CHUNK")) Tc = std::max(1, std::min(T, atoi(e)));
  const int64_t rows = (int64_t)Tc * B;
  // scratch: X fp32 [R], Xcat op [2R], Adil fp32 [2D], Z op [D], Sacc fp32 [S], Hin op [S],
  // H1 fp32 [H], H1op op [H]
  const size_t per_row = 4 * R + ob * 2 * R + 4 * 2 * D + ob * D +
                         (heads ? 4 * S + ob * S + 4 * H + ob * H : 0);
  const size_t need = per_row * (size_t)rows + 256 * 8;
  if (need > p.scratch_bytes) {
    if (p.scratch) cudaFree(p.scratch);
    p.scratch = nullptr;
    p.scratch_bytes = 0;
    PF_CUDA(cudaMalloc(&p.scratch, need));
    p.scratch_bytes = need;
  }
  uint8_t* sp = static_cast<uint8_t*>(p.scratch);
  auto carve = [&](size_t bytes) {
    void* r = sp;
    sp += (bytes + 255) & ~(size_t)255;
    return r;
  };
  float* X = static_cast<float*>(carve(4 * R * rows));
  void* Xcat = carve(ob * 2 * R * rows);
  float* Adil = static_cast<float*>(carve(4 * 2 * D * rows));
  void* Z = carve(ob * D * rows);
  float* Sacc = heads ? static_cast<float*>(carve(4 * S * rows)) : nullptr;
  void* Hin = heads ? carve(ob * S * rows) : nullptr;
  float* H1 = heads ? static_cast<float*>(carve(4 * H * rows)) : nullptr;
  void* H1op = heads ? carve(ob * H * rows) : nullptr;

  Ring q{reinterpret_cast<uint8_t*>(h.d_queue), p.off,
         f16 ? (int64_t)(B / 64) * 16384 : ((int64_t)B + 127) / 128 * 128 * ((R + 3) & ~3),
         (R + 3) & ~3, f16 ? 1 : 0};
  for (int c0 = 0; c0 < T; c0 += Tc) {
    const int tc = std::min(Tc, T - c0);
    const int32_t* cls = d_inputs + (int64_t)c0 * B;
    float* lg = heads ? d_logits + (int64_t)c0 * B * A : nullptr;
    int rc;
    if (f16)
      rc = prefill_chunk<__half>(h, p, cls, tc, h.t + c0, q, X, static_cast<__half*>(Xcat), Adil,
                                 static_cast<__half*>(Z), Sacc, static_cast<__half*>(Hin), H1,
                                 static_cast<__half*>(H1op), lg, st);
    else
      rc = prefill_chunk<float>(h, p, cls, tc, h.t + c0, q, X, static_cast<float*>(Xcat), Adil,
                                static_cast<float*>(Z), Sacc, static_cast<float*>(Hin), H1,
                                static_cast<float*>(H1op), lg, st);
    if (rc) return rc;
  }
  h.t += T;
  return FW_OK;
}

}  // namespace fw
