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
// The GEMMs are plain library GEMMs (cuBLAS, loaded at run time from the process or the
// toolkit -- no link-time dependency): operands fp16 for tcgen05 handles (the precision
// their step kernel feeds the tensor cores: fp16 x_t / x_{t-d} / z / ReLU(s) / h, bf16
// weights), fp32 with no TF32 for SIMT handles. The elementwise parts are the kernels
// below. The ring is read and written in the handle's own slot layout.
#include <cuda_fp16.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "internal.h"

namespace fw {
namespace {

// ---- cuBLAS, resolved at run time ------------------------------------------------------
// (the handful of entry points used; enum values from cublas_api.h / library_types.h)
typedef int (*cublasCreate_t)(void**);
typedef int (*cublasDestroy_t)(void*);
typedef int (*cublasSetStream_t)(void*, cudaStream_t);
typedef int (*cublasSetMathMode_t)(void*, int);
typedef int (*cublasGemmEx_t)(void*, int, int, int, int, int, const void*, const void*, int, int,
                              const void*, int, int, const void*, void*, int, int, int, int);
constexpr int kOpN = 0;
constexpr int kR16F = 2, kR32F = 0;          // CUDA_R_16F, CUDA_R_32F
constexpr int kCompute32F = 68;              // CUBLAS_COMPUTE_32F
constexpr int kCompute32FPedantic = 69;      // CUBLAS_COMPUTE_32F_PEDANTIC
constexpr int kGemmDefault = -1;             // CUBLAS_GEMM_DEFAULT
constexpr int kPedanticMath = 2;             // CUBLAS_PEDANTIC_MATH

struct Blas {
  void* lib = nullptr;
  cublasCreate_t create = nullptr;
  cublasDestroy_t destroy = nullptr;
  cublasSetStream_t set_stream = nullptr;
  cublasSetMathMode_t set_math = nullptr;
  cublasGemmEx_t gemm = nullptr;
};

bool load_blas(Blas& b, std::string* why) {
  if (b.gemm) return true;
  // the copy the process already has (e.g. PyTorch's), else the toolkit's
  const char* names[] = {"libcublas.so.12", "/usr/local/cuda/lib64/libcublas.so.12",
                         "libcublas.so"};
  for (const char* n : names) {
    b.lib = dlopen(n, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (b.lib) break;
  }
  if (!b.lib)
    for (const char* n : names) {
      b.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (b.lib) break;
    }
  if (!b.lib) {
    *why = "cuBLAS (libcublas.so.12) not found";
    return false;
  }
  b.create = (cublasCreate_t)dlsym(b.lib, "cublasCreate_v2");
  b.destroy = (cublasDestroy_t)dlsym(b.lib, "cublasDestroy_v2");
  b.set_stream = (cublasSetStream_t)dlsym(b.lib, "cublasSetStream_v2");
  b.set_math = (cublasSetMathMode_t)dlsym(b.lib, "cublasSetMathMode");
  b.gemm = (cublasGemmEx_t)dlsym(b.lib, "cublasGemmEx");
  if (!b.create || !b.destroy || !b.set_stream || !b.set_math || !b.gemm) {
    *why = "cuBLAS entry points missing";
    b.gemm = nullptr;
    return false;
  }
  return true;
}

// ---- ring slot addressing (the handle's layout) -------------------------------------------
struct Ring {
  uint8_t* base;      // h.d_queue
  const int64_t* off; // [L] element offset (SIMT, floats) or byte offset (tcgen05) of layer l
  int64_t slot;       // slot stride: elements (SIMT) or bytes (tcgen05)
  int Rp;             // SIMT: channels padded to 4
  int fp16;           // tcgen05 layout
};
// ---- 8-channel vectors: every elementwise kernel moves 8 consecutive channels per thread
// (16-byte fp16 / 2 x 16-byte fp32 accesses; all channel counts are multiples of 8)
struct V8 {
  float v[8];
};
__device__ __forceinline__ V8 ld8(const float* p) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  return V8{{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}};
}
__device__ __forceinline__ void st8(float* p, const V8& x) {
  reinterpret_cast<float4*>(p)[0] = make_float4(x.v[0], x.v[1], x.v[2], x.v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(x.v[4], x.v[5], x.v[6], x.v[7]);
}
__device__ __forceinline__ V8 ld8(const __half* p) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __half2* h = reinterpret_cast<const __half2*>(&u);
  V8 x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __half22float2(h[i]);
    x.v[2 * i] = f.x;
    x.v[2 * i + 1] = f.y;
  }
  return x;
}
__device__ __forceinline__ void st8(__half* p, const V8& x) {
  uint4 u;
  __half2* h = reinterpret_cast<__half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(x.v[2 * i], x.v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
// ring slot element group (stream b, channels r..r+7), r % 8 == 0
__device__ __forceinline__ V8 ring_ld8(const Ring& q, int l, int s, int b, int r) {
  if (q.fp16)
    return ld8(reinterpret_cast<const __half*>(q.base + q.off[l] + (int64_t)s * q.slot +
                                               (int64_t)(b >> 7) * 32768 + (r >> 3) * 2048 +
                                               (b & 127) * 16));
  const float* base = reinterpret_cast<const float*>(q.base) + q.off[l] + (int64_t)s * q.slot;
  const float* p0 = base + ((int64_t)((b >> 7) * (q.Rp / 4) + (r >> 2)) * 128 + (b & 127)) * 4;
  const float4 a = *reinterpret_cast<const float4*>(p0), c = *reinterpret_cast<const float4*>(p0 + 512);
  return V8{{a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w}};
}
__device__ __forceinline__ void ring_st8(const Ring& q, int l, int s, int b, int r, const V8& x) {
  if (q.fp16) {
    st8(reinterpret_cast<__half*>(q.base + q.off[l] + (int64_t)s * q.slot + (int64_t)(b >> 7) * 32768 +
                                  (r >> 3) * 2048 + (b & 127) * 16),
        x);
    return;
  }
  float* base = reinterpret_cast<float*>(q.base) + q.off[l] + (int64_t)s * q.slot;
  float* p0 = base + ((int64_t)((b >> 7) * (q.Rp / 4) + (r >> 2)) * 128 + (b & 127)) * 4;
  *reinterpret_cast<float4*>(p0) = make_float4(x.v[0], x.v[1], x.v[2], x.v[3]);
  *reinterpret_cast<float4*>(p0 + 512) = make_float4(x.v[4], x.v[5], x.v[6], x.v[7]);
}

// X[row][:] = embed[cls[row]][:], row = tt * B + b
__global__ void embed_rows(const int32_t* __restrict__ cls, const float* __restrict__ embed,
                           float* __restrict__ X, int64_t n, int R) {
  const int g8 = R / 8;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * g8) return;
  const int64_t row = e / g8;
  const int r = (int)(e - row * g8) * 8;
  st8(X + row * R + r, ld8(embed + (int64_t)cls[row] * R + r));
}

// x_l = X + the previous layer's residual bias (add_bias8 writes it into X afterwards);
// Xcat[row] = [x_l[t] | x_l[t-d]] in the operand type; x_l[t-d] from this chunk's rows or,
// before the chunk, from ring slot (t mod d) (= (t-d) mod d, not yet overwritten). Rows
// with t-d inside the chunk read X of an earlier row -- the bias is added there too.
template <typename T>
__global__ void gather_taps(float* __restrict__ X, const float* __restrict__ rbias, T* __restrict__ Xcat,
                            Ring q, int l, int d, int64_t t_abs0, int Tc, int B, int R) {
  const int g8 = R / 8;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)Tc * B;
  if (e >= n * g8) return;
  const int64_t row = e / g8;
  const int r = (int)(e - row * g8) * 8;
  const int tt = (int)(row / B), b = (int)(row - (int64_t)tt * B);
  V8 bias{};
  if (rbias) bias = ld8(rbias + r);
  V8 x = ld8(X + row * R + r);
  V8 xd;
  if (tt - d >= 0) {
    xd = ld8(X + ((int64_t)(tt - d) * B + b) * R + r);
#pragma unroll
    for (int i = 0; i < 8; ++i) xd.v[i] += bias.v[i];
  } else {
    xd = ring_ld8(q, l, (int)((t_abs0 + tt) % d), b, r);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) x.v[i] += bias.v[i];
  st8(Xcat + row * 2 * R + r, x);
  st8(Xcat + row * 2 * R + R + r, xd);
}

// X += bias (the residual bias of this layer's input, once every row's taps are gathered)
__global__ void add_bias8(float* __restrict__ Y, const float* __restrict__ bias, int64_t n, int C) {
  const int g8 = C / 8;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * g8) return;
  const int64_t row = e / g8;
  const int c = (int)(e - row * g8) * 8;
  V8 y = ld8(Y + row * C + c);
  const V8 bb = ld8(bias + c);
#pragma unroll
  for (int i = 0; i < 8; ++i) y.v[i] += bb.v[i];
  st8(Y + row * C + c, y);
}

// ring slot (t mod d) <- x_l[t] for the chunk's last min(d, Tc) steps
__global__ void push_taps(const float* __restrict__ X, Ring q, int l, int d, int64_t t_abs0, int Tc,
                          int B, int R) {
  const int g8 = R / 8;
  const int first = Tc > d ? Tc - d : 0;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)(Tc - first) * B;
  if (e >= n * g8) return;
  const int64_t row = e / g8 + (int64_t)first * B;
  const int r = (int)(e % g8) * 8;
  const int tt = (int)(row / B), b = (int)(row - (int64_t)tt * B);
  ring_st8(q, l, (int)((t_abs0 + tt) % d), b, r, ld8(X + row * R + r));
}

// z = tanh(a[:D] + b[:D]) * sigmoid(a[D:] + b[D:]) in the operand type
template <typename T>
__global__ void gate_rows(const float* __restrict__ Adil, const float* __restrict__ bias,
                          T* __restrict__ Z, int64_t n, int D) {
  const int g8 = D / 8;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * g8) return;
  const int64_t row = e / g8;
  const int c = (int)(e - row * g8) * 8;
  const V8 a = ld8(Adil + row * 2 * D + c), g = ld8(Adil + row * 2 * D + D + c);
  const V8 ba = ld8(bias + c), bg = ld8(bias + D + c);
  V8 z;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    z.v[i] = tanhf(a.v[i] + ba.v[i]) * (1.f / (1.f + expf(-(g.v[i] + bg.v[i]))));
  st8(Z + row * D + c, z);
}

// out = ReLU(Y + bias) in the operand type
template <typename T>
__global__ void relu_rows(const float* __restrict__ Y, const float* __restrict__ bias, T* __restrict__ out,
                          int64_t n, int C) {
  const int g8 = C / 8;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * g8) return;
  const int64_t row = e / g8;
  const int c = (int)(e - row * g8) * 8;
  V8 y = ld8(Y + row * C + c);
  const V8 bb = ld8(bias + c);
#pragma unroll
  for (int i = 0; i < 8; ++i) y.v[i] = fmaxf(y.v[i] + bb.v[i], 0.f);
  st8(out + row * C + c, y);
}

__global__ void f32_to_f16(const float* __restrict__ src, __half* __restrict__ dst, int64_t n) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[e] = __float2half_rn(src[e]);
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

// Per-handle prefill state: cuBLAS handle, fp16 weight copies (tcgen05 handles), scratch.
struct PrefillState {
  Blas blas;
  void* cublas = nullptr;
  __half *dil16 = nullptr, *res16 = nullptr, *skip16 = nullptr, *h116 = nullptr, *h216 = nullptr;
  float* bsum = nullptr;  // [S] sum of the skip biases
  int64_t* off = nullptr; // [L] ring offsets in the handle's units
  int64_t rows_cap = 0;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
};

void prefill_destroy(Handle& h) {
  PrefillState* p = h.prefill;
  if (!p) return;
  void* ptrs[] = {p->dil16, p->res16, p->skip16, p->h116, p->h216, p->bsum, p->off, p->scratch};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  if (p->cublas && p->blas.destroy) p->blas.destroy(p->cublas);
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
  std::string why;
  if (!load_blas(p->blas, &why)) return pf_fail(why);
  if (p->blas.create(&p->cublas) != 0) return pf_fail("cublasCreate failed");
  const CellDims& d = h.dims;
  const int L = d.L, R = d.R, D = d.D, S = d.S, H = d.H, A = d.A;
  const bool f16 = h.kernel == FW_KERNEL_TCGEN05;
  if (!f16) p->blas.set_math(p->cublas, kPedanticMath);  // fp32 configs: no TF32
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

}  // namespace

int cell_prefill(Handle& h, const int32_t* d_inputs, int T, float* d_logits, cudaStream_t st) {
  if (int rc = prefill_init(h)) return rc;
  PrefillState& p = *h.prefill;
  const CellDims& d = h.dims;
  const int L = d.L, R = d.R, D = d.D, S = d.S, H = d.H, A = d.A, B = h.batch;
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
  if (p.blas.set_stream(p.cublas, st) != 0) return pf_fail("cublasSetStream failed");
  const int dt = f16 ? kR16F : kR32F;
  const int ct = f16 ? kCompute32F : kCompute32FPedantic;
  // row-major C[n][out] (+)= A[n][in] W[in][out]  ==  column-major C^T = W^T A^T
  auto gemm = [&](const void* Aop, const void* W, void* C, int64_t n, int in, int out, int c_type,
                  float beta) {
    const float one = 1.f;
    return p.blas.gemm(p.cublas, kOpN, kOpN, out, (int)n, in, &one, W, dt, out, Aop, dt, in, &beta,
                       C, c_type, out, ct, kGemmDefault);
  };
  for (int c0 = 0; c0 < T; c0 += Tc) {
    const int tc = std::min(Tc, T - c0);
    const int64_t n = (int64_t)tc * B;
    const int64_t t_abs0 = h.t + c0;
    embed_rows<<<nblk(n * R / 8), 256, 0, st>>>(d_inputs + (int64_t)c0 * B, h.w.embed, X, n, R);
    for (int l = 0; l < L; ++l) {
      const int dl = h.dil[l];
      // x_l = X + b_res(l-1): the taps see it, X takes it right after
      const float* rb = l > 0 ? h.w.res_b + (size_t)(l - 1) * R : nullptr;
      if (f16)
        gather_taps<__half><<<nblk(n * R / 8), 256, 0, st>>>(X, rb, static_cast<__half*>(Xcat), q, l, dl, t_abs0, tc, B, R);
      else
        gather_taps<float><<<nblk(n * R / 8), 256, 0, st>>>(X, rb, static_cast<float*>(Xcat), q, l, dl, t_abs0, tc, B, R);
      if (rb) add_bias8<<<nblk(n * R / 8), 256, 0, st>>>(X, rb, n, R);
      PF_CUDA(cudaGetLastError());
      const void* Wd = f16 ? (const void*)(p.dil16 + (size_t)l * 2 * R * 2 * D)
                           : (const void*)(h.w.dilT + (size_t)l * 2 * R * 2 * D);
      if (gemm(Xcat, Wd, Adil, n, 2 * R, 2 * D, kR32F, 0.f)) return pf_fail("cublasGemmEx (dilated) failed");
      if (f16)
        gate_rows<__half><<<nblk(n * D / 8), 256, 0, st>>>(Adil, h.w.dil_b + (size_t)l * 2 * D, static_cast<__half*>(Z), n, D);
      else
        gate_rows<float><<<nblk(n * D / 8), 256, 0, st>>>(Adil, h.w.dil_b + (size_t)l * 2 * D, static_cast<float*>(Z), n, D);
      // the ring takes x_l after this layer's taps were gathered
      push_taps<<<nblk((int64_t)std::min(tc, dl) * B * R / 8), 256, 0, st>>>(X, q, l, dl, t_abs0, tc, B, R);
      PF_CUDA(cudaGetLastError());
      if (heads) {
        const void* Ws = f16 ? (const void*)(p.skip16 + (size_t)l * D * S) : (const void*)(h.w.skipT + (size_t)l * D * S);
        if (gemm(Z, Ws, Sacc, n, D, S, kR32F, l == 0 ? 0.f : 1.f)) return pf_fail("cublasGemmEx (skip) failed");
      }
      if (l + 1 < L) {
        const void* Wr = f16 ? (const void*)(p.res16 + (size_t)l * D * R) : (const void*)(h.w.resT + (size_t)l * D * R);
        if (gemm(Z, Wr, X, n, D, R, kR32F, 1.f)) return pf_fail("cublasGemmEx (residual) failed");
      }
    }
    if (heads) {
      float* out = d_logits + (int64_t)c0 * B * A;
      if (f16) {
        relu_rows<__half><<<nblk(n * S / 8), 256, 0, st>>>(Sacc, p.bsum, static_cast<__half*>(Hin), n, S);
        if (gemm(Hin, p.h116, H1, n, S, H, kR32F, 0.f)) return pf_fail("cublasGemmEx (head1) failed");
        relu_rows<__half><<<nblk(n * H / 8), 256, 0, st>>>(H1, h.w.h1_b, static_cast<__half*>(H1op), n, H);
        if (gemm(H1op, p.h216, out, n, H, A, kR32F, 0.f)) return pf_fail("cublasGemmEx (head2) failed");
      } else {
        relu_rows<float><<<nblk(n * S / 8), 256, 0, st>>>(Sacc, p.bsum, static_cast<float*>(Hin), n, S);
        if (gemm(Hin, h.w.h1T, H1, n, S, H, kR32F, 0.f)) return pf_fail("cublasGemmEx (head1) failed");
        relu_rows<float><<<nblk(n * H / 8), 256, 0, st>>>(H1, h.w.h1_b, static_cast<float*>(H1op), n, H);
        if (gemm(H1op, h.w.h2T, out, n, H, A, kR32F, 0.f)) return pf_fail("cublasGemmEx (head2) failed");
      }
      add_bias8<<<nblk(n * A / 8), 256, 0, st>>>(out, h.w.h2_b, n, A);
      PF_CUDA(cudaGetLastError());
    }
  }
  h.t += T;
  return FW_OK;
}

}  // namespace fw
