// C ABI of libfastwavenet.so (include/fastwavenet.h): handle lifetime,
// weight repacking, queue allocation, argument validation and dispatch.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "internal.h"

namespace fw {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

namespace {

int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return FW_ERR_CUDA;
}

#define FW_CUDA(call)                                 \
  do {                                                \
    cudaError_t _e = (call);                          \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

int invalid(const std::string& msg) {
  set_error(msg);
  return FW_ERR_INVALID;
}

float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

template <typename T>
int upload(T** dst, const T* src, size_t n) {
  FW_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), sizeof(T) * (n ? n : 1)));
  if (n) FW_CUDA(cudaMemcpy(*dst, src, sizeof(T) * n, cudaMemcpyHostToDevice));
  return FW_OK;
}

// [rows][cols] -> [cols][rows]
std::vector<float> transpose(const float* src, int rows, int cols, bool bf16) {
  std::vector<float> out((size_t)rows * cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      float v = src[(size_t)r * cols + c];
      out[(size_t)c * rows + r] = bf16 ? bf16_round(v) : v;
    }
  return out;
}

std::vector<float> maybe_round(const float* src, size_t n, bool bf16) {
  std::vector<float> out(src, src + n);
  if (bf16)
    for (auto& v : out) v = bf16_round(v);
  return out;
}

void free_cell(Handle& h) {
  float** ptrs[] = {&h.w.embed, &h.w.dilT, &h.w.dil_b, &h.w.resT, &h.w.res_b, &h.w.skipT,
                    &h.w.catT, &h.w.skip_b, &h.w.h1T, &h.w.h1_b, &h.w.h2T, &h.w.h2_b, &h.d_queue};
  for (float** p : ptrs) {
    if (*p) cudaFree(*p);
    *p = nullptr;
  }
  if (h.d_dil) cudaFree(h.d_dil);
  if (h.d_qoff) cudaFree(h.d_qoff);
  h.d_dil = nullptr;
  h.d_qoff = nullptr;
  if (h.tc) tc_destroy(h);
  prefill_destroy(h);
  lat_destroy(h);
  hmma_destroy(h);
  if (h.d_pad) cudaFree(h.d_pad);
  if (h.d_pad_lg) cudaFree(h.d_pad_lg);
  h.d_pad = nullptr;
  h.d_pad_lg = nullptr;
}

void free_plain(Handle& h) {
  void* ptrs[] = {h.p.dil, h.p.cin, h.p.cout, h.p.woff, h.p.boff, h.p.qoff,
                  h.p.roff, h.p.soff, h.p.taps, h.p.bias, h.p.queue,
                  h.naive.count, h.naive.goff, h.naive.gather, h.naive.gsrc, h.naive.voff,
                  h.naive.vals};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  h.p = PlainDev{};
  h.naive = NaivePlan{};
}

// The demand plan (reference naive.py:27-110): the top layer at offset 0, layer l-1
// wherever layer l's taps read it (o + k d_l); nodes in ascending offset order.
int build_naive_plan(Handle& h) {
  NaivePlan& pl = h.naive;
  if (pl.built) return FW_OK;
  const int n = (int)h.pdil.size(), w = h.p.w;
  std::vector<std::vector<int64_t>> dem(n);
  dem[n - 1] = {0};
  for (int l = n - 1; l > 0; --l) {
    std::vector<int64_t> v;
    for (int64_t o : dem[l])
      for (int k = 0; k < w; ++k) v.push_back(o + (int64_t)k * h.pdil[l]);
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    dem[l - 1] = v;
  }
  std::vector<int> count(n), gather, gsrc;
  std::vector<int64_t> goff(n), voff(n);
  int64_t vtot = 0;
  for (int l = 0; l < n; ++l) {
    count[l] = (int)dem[l].size();
    goff[l] = (int64_t)gather.size();
    voff[l] = vtot;
    const int cout = l + 1 < n ? h.pcin[l + 1] : 1;
    vtot += (int64_t)count[l] * cout;
    for (int64_t o : dem[l])
      for (int k = 0; k < w; ++k) {
        const int64_t src = o + (int64_t)k * h.pdil[l];
        gsrc.push_back((int)src);
        if (l == 0) {
          gather.push_back((int)src);
        } else {
          auto it = std::lower_bound(dem[l - 1].begin(), dem[l - 1].end(), src);
          gather.push_back((int)(it - dem[l - 1].begin()));
        }
      }
  }
  int rc;
  if ((rc = upload(&pl.count, count.data(), count.size()))) return rc;
  if ((rc = upload(&pl.goff, goff.data(), goff.size()))) return rc;
  if ((rc = upload(&pl.gather, gather.data(), gather.size()))) return rc;
  if ((rc = upload(&pl.gsrc, gsrc.data(), gsrc.size()))) return rc;
  if ((rc = upload(&pl.voff, voff.data(), voff.size()))) return rc;
  pl.vals_per_stream = vtot;
  FW_CUDA(cudaMalloc(&pl.vals, sizeof(double) * (size_t)vtot * h.batch));
  pl.built = 1;
  return FW_OK;
}

int check_handle(const fw_handle* h, bool want_plain) {
  if (!h) return invalid("null handle");
  if (h->h.is_plain != (want_plain ? 1 : 0))
    return invalid(want_plain ? "handle is not a plain-mode handle" : "handle is not a cell handle");
  return FW_OK;
}

int validate_cell(const fw_cell_desc* d) {
  if (!d) return invalid("null descriptor");
  if (d->n_layers < 1) return invalid("n_layers must be a positive integer");
  if (!d->dilations) return invalid("dilations must not be null");
  for (int l = 0; l < d->n_layers; ++l)
    if (d->dilations[l] < 1) return invalid("dilations must be positive integers");
  if (d->residual_channels < 1 || d->dilation_channels < 1 || d->skip_channels < 1 ||
      d->head_channels < 1 || d->classes < 1)
    return invalid("channel counts must be positive integers");
  if (d->residual_channels > 1024 || d->dilation_channels > 1024 || d->skip_channels > 4096 ||
      d->head_channels > 4096 || d->classes > 4096)
    return invalid("channel counts exceed the supported maximum");
  if (d->weight_dtype != FW_DTYPE_F32 && d->weight_dtype != FW_DTYPE_BF16)
    return invalid("weight_dtype must be FW_DTYPE_F32 or FW_DTYPE_BF16");
  const void* ptrs[] = {d->embed, d->dil_w, d->dil_b, d->res_w, d->res_b, d->skip_w,
                        d->skip_b, d->head1_w, d->head1_b, d->head2_w, d->head2_b};
  for (const void* p : ptrs)
    if (!p) return invalid("weight pointers must not be null");
  return FW_OK;
}

int validate_sampler(const fw_sampler* s) {
  if (!s) return invalid("null sampler");
  if (s->mode < FW_SAMPLE_ARGMAX || s->mode > FW_SAMPLE_GUMBEL) return invalid("unknown sampler mode");
  if (s->stream_offset < 0) return invalid("stream_offset must be non-negative");
  return FW_OK;
}

int run_cell_dev(Handle& h, const CellRun& run, cudaStream_t st);

template <typename T>
int grow(T** p, int64_t* have, int64_t need) {
  if (need <= *have) return FW_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  FW_CUDA(cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (size_t)need));
  *have = need;
  return FW_OK;
}

// The caller's buffers hold user_batch streams per step; a padded handle (tcgen05 with a
// batch that is not a multiple of 128) runs batch >= user_batch streams on the device, the
// extra ones fed class 0 and discarded. Stage inputs, outputs and logits through [n][batch]
// buffers with strided copies.
int run_cell(Handle& h, const CellRun& run, cudaStream_t st) {
  if (h.user_batch == h.batch) return run_cell_dev(h, run, st);
  const int64_t B = h.user_batch, Bp = h.batch, A = h.dims.A;
  if (int rc = grow(&h.d_pad, &h.d_pad_elems, ((int64_t)run.n_inputs + run.n_steps) * Bp)) return rc;
  if (run.logits && run.n_logit_steps)
    if (int rc = grow(&h.d_pad_lg, &h.d_pad_lg_elems, (int64_t)run.n_logit_steps * Bp * A)) return rc;
  int32_t* in = h.d_pad;
  int32_t* out = h.d_pad + (int64_t)run.n_inputs * Bp;
  FW_CUDA(cudaMemsetAsync(in, 0, sizeof(int32_t) * (size_t)run.n_inputs * Bp, st));
  FW_CUDA(cudaMemcpy2DAsync(in, sizeof(int32_t) * Bp, run.inputs, sizeof(int32_t) * B,
                            sizeof(int32_t) * B, run.n_inputs, cudaMemcpyDeviceToDevice, st));
  CellRun r = run;
  r.inputs = in;
  r.out = out;
  r.logits = (run.logits && run.n_logit_steps) ? h.d_pad_lg : nullptr;
  if (int rc = run_cell_dev(h, r, st)) return rc;
  FW_CUDA(cudaMemcpy2DAsync(run.out, sizeof(int32_t) * B, out, sizeof(int32_t) * Bp,
                            sizeof(int32_t) * B, run.n_steps, cudaMemcpyDeviceToDevice, st));
  if (r.logits)
    FW_CUDA(cudaMemcpy2DAsync(run.logits, sizeof(float) * B * A, h.d_pad_lg, sizeof(float) * Bp * A,
                              sizeof(float) * B * A, run.n_logit_steps, cudaMemcpyDeviceToDevice, st));
  return FW_OK;
}

int run_cell_dev(Handle& h, const CellRun& run, cudaStream_t st) {
  cudaError_t e;
  int64_t launches = 0;
  if (h.kernel == FW_KERNEL_TCGEN05) {
    e = launch_cell_tc(h, run, st, &launches);  // sets tev_used / timed_steps
  } else {
    // one persistent launch covers every step: time it as a whole
    const int timed = h.timing ? timing_reserve(h, 1) : 0;
    if (timed) cudaEventRecord(h.tev[0], st);
    e = launch_cell_simt(h, run, st, &launches);
    if (timed) {
      cudaEventRecord(h.tev[1], st);
      cudaEventRecord(h.tev[2], st);
    }
    h.tev_used = timed;
    h.timed_steps = timed ? run.n_steps : 0;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cell kernel launch");
  h.last_launches = launches;
  h.t += run.n_steps;
  return FW_OK;
}

}  // namespace
}  // namespace fw

using namespace fw;

extern "C" {

int32_t fw_version(void) { return 100; }

const char* fw_last_error(void) { return g_err.c_str(); }

int fw_cell_create(const fw_cell_desc* desc, int32_t batch, int32_t device, int32_t kernel,
                   fw_handle** out) {
  if (!out) return invalid("null output handle pointer");
  *out = nullptr;
  int rc = validate_cell(desc);
  if (rc) return rc;
  if (batch < 1) return invalid("batch must be a positive integer");
  if (kernel != FW_KERNEL_AUTO && kernel != FW_KERNEL_SIMT && kernel != FW_KERNEL_TCGEN05)
    return invalid("unknown kernel selector");
  int ndev = 0;
  FW_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return invalid("device index out of range");
  FW_CUDA(cudaSetDevice(device));

  auto* fh = new (std::nothrow) fw_handle();
  if (!fh) return invalid("out of host memory");
  Handle& h = fh->h;
  h.device = device;
  h.batch = batch;
  h.user_batch = batch;
  const int L = desc->n_layers, R = desc->residual_channels, D = desc->dilation_channels;
  const int S = desc->skip_channels, H = desc->head_channels, A = desc->classes;
  h.dims = CellDims{L, R, D, S, H, A, desc->weight_dtype};
  h.dil.assign(desc->dilations, desc->dilations + L);

  // tcgen05 tiles hold 128 streams: other batches of >= 128 run padded to the next multiple
  const int padded = batch >= 128 ? (batch + 127) / 128 * 128 : batch;
  std::string why;
  const bool tc_ok = tc_supported(h.dims, padded, &why);
  if (kernel == FW_KERNEL_TCGEN05 && !tc_ok) {
    delete fh;
    return invalid("tcgen05 kernel unsupported for this shape: " + why);
  }
  h.kernel = (kernel == FW_KERNEL_TCGEN05 || (kernel == FW_KERNEL_AUTO && tc_ok))
                 ? FW_KERNEL_TCGEN05
                 : FW_KERNEL_SIMT;
  if (h.kernel == FW_KERNEL_TCGEN05) h.batch = padded;

  auto fail = [&](int code) {
    free_cell(h);
    delete fh;
    return code;
  };
  const bool bf = desc->weight_dtype == FW_DTYPE_BF16;
  // queues: layer l holds d_l slots. SIMT: each slot [ceil(B/128)][R/4][128][4] fp32 (R
  // padded to a multiple of 4, streams to a multiple of 128). tcgen05: each slot
  // [B/128][16][128][8] fp16 -- per 128-stream tile pair 16 K-pieces of 8 channels (chain_tc.cuh).
  // Either way a 128-stream tile's slot is contiguous.
  const int Rp = (R + 3) & ~3;
  const int64_t Bp = ((int64_t)batch + 127) / 128 * 128;
  std::vector<int64_t> qoff(L);
  int64_t total = 0;
  for (int l = 0; l < L; ++l) {
    qoff[l] = total;
    total += (int64_t)h.dil[l] * Bp * Rp;
  }
  h.queue_bytes = h.kernel == FW_KERNEL_TCGEN05 ? total * 2 : total * 4;
  if ((rc = upload(&h.d_dil, h.dil.data(), L))) return fail(rc);
  if ((rc = upload(&h.d_qoff, qoff.data(), L))) return fail(rc);
  cudaError_t e = cudaMalloc(&h.d_queue, (size_t)h.queue_bytes);
  if (e != cudaSuccess) return fail(cuda_fail(e, "queue allocation"));
  e = cudaMemset(h.d_queue, 0, (size_t)h.queue_bytes);
  if (e != cudaSuccess) return fail(cuda_fail(e, "queue zero-fill"));

  // host copy (reference layouts, bf16-rounded where applicable) for lazily built images
  {
    HostCell& c = h.host;
    c.dil_w = maybe_round(desc->dil_w, (size_t)L * 2 * 2 * D * R, bf);
    c.dil_b = maybe_round(desc->dil_b, (size_t)L * 2 * D, bf);
    c.res_w = maybe_round(desc->res_w, (size_t)L * R * D, bf);
    c.res_b = maybe_round(desc->res_b, (size_t)L * R, bf);
    c.skip_w = maybe_round(desc->skip_w, (size_t)L * S * D, bf);
    c.skip_b = maybe_round(desc->skip_b, (size_t)L * S, bf);
    c.h1_w = maybe_round(desc->head1_w, (size_t)H * S, bf);
    c.h1_b = maybe_round(desc->head1_b, H, bf);
    c.h2_w = maybe_round(desc->head2_w, (size_t)A * H, bf);
    c.h2_b = maybe_round(desc->head2_b, A, bf);
  }
  // SIMT weights (also used by the tcgen05 path for nothing but kept small)
  {
    std::vector<float> embed = maybe_round(desc->embed, (size_t)A * R, bf);
    std::vector<float> dilT((size_t)L * 2 * R * 2 * D);
    std::vector<float> resT((size_t)L * D * R), skipT((size_t)L * D * S);
    for (int l = 0; l < L; ++l) {
      for (int k = 0; k < 2; ++k) {
        // dil_w[l][k] is (2D, R) -> rows k*R + c of [2R][2D]
        const float* src = desc->dil_w + ((size_t)l * 2 + k) * 2 * D * R;
        std::vector<float> tt = transpose(src, 2 * D, R, bf);
        std::memcpy(dilT.data() + (size_t)l * 2 * R * 2 * D + (size_t)k * R * 2 * D, tt.data(),
                    sizeof(float) * tt.size());
      }
      std::vector<float> rt = transpose(desc->res_w + (size_t)l * R * D, R, D, bf);
      std::memcpy(resT.data() + (size_t)l * D * R, rt.data(), sizeof(float) * rt.size());
      std::vector<float> st = transpose(desc->skip_w + (size_t)l * S * D, S, D, bf);
      std::memcpy(skipT.data() + (size_t)l * D * S, st.data(), sizeof(float) * st.size());
    }
    std::vector<float> h1T = transpose(desc->head1_w, H, S, bf);
    std::vector<float> h2T = transpose(desc->head2_w, A, H, bf);
    std::vector<float> dil_b = maybe_round(desc->dil_b, (size_t)L * 2 * D, bf);
    std::vector<float> res_b = maybe_round(desc->res_b, (size_t)L * R, bf);
    std::vector<float> skip_b = maybe_round(desc->skip_b, (size_t)L * S, bf);
    std::vector<float> h1_b = maybe_round(desc->head1_b, H, bf);
    std::vector<float> h2_b = maybe_round(desc->head2_b, A, bf);
    if ((rc = upload(&h.w.embed, embed.data(), embed.size()))) return fail(rc);
    if ((rc = upload(&h.w.dilT, dilT.data(), dilT.size()))) return fail(rc);
    if ((rc = upload(&h.w.dil_b, dil_b.data(), dil_b.size()))) return fail(rc);
    if ((rc = upload(&h.w.resT, resT.data(), resT.size()))) return fail(rc);
    if ((rc = upload(&h.w.res_b, res_b.data(), res_b.size()))) return fail(rc);
    if ((rc = upload(&h.w.skipT, skipT.data(), skipT.size()))) return fail(rc);
    {
      std::vector<float> catT((size_t)L * D * (S + R));
      for (size_t row = 0; row < (size_t)L * D; ++row) {
        std::memcpy(catT.data() + row * (S + R), skipT.data() + row * S, sizeof(float) * S);
        std::memcpy(catT.data() + row * (S + R) + S, resT.data() + row * R, sizeof(float) * R);
      }
      if ((rc = upload(&h.w.catT, catT.data(), catT.size()))) return fail(rc);
    }
    if ((rc = upload(&h.w.skip_b, skip_b.data(), skip_b.size()))) return fail(rc);
    if ((rc = upload(&h.w.h1T, h1T.data(), h1T.size()))) return fail(rc);
    if ((rc = upload(&h.w.h1_b, h1_b.data(), h1_b.size()))) return fail(rc);
    if ((rc = upload(&h.w.h2T, h2T.data(), h2T.size()))) return fail(rc);
    if ((rc = upload(&h.w.h2_b, h2_b.data(), h2_b.size()))) return fail(rc);
  }
  if (h.kernel == FW_KERNEL_TCGEN05) {
    if ((rc = tc_create(h, desc))) return fail(rc);
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(cuda_fail(e, "create synchronize"));
  *out = fh;
  return FW_OK;
}

int fw_cell_step(fw_handle* fh, const int32_t* d_in, int32_t* d_out, float* d_logits,
                 const fw_sampler* sampler, void* stream) {
  int rc = check_handle(fh, false);
  if (rc) return rc;
  if ((rc = validate_sampler(sampler))) return rc;
  if (!d_in || !d_out) return invalid("d_in and d_out must not be null");
  Handle& h = fh->h;
  FW_CUDA(cudaSetDevice(h.device));
  CellRun run{d_in, 1, 1, d_out, d_logits, d_logits ? 1 : 0, h.t, sampler->mode, sampler->seed,
              sampler->stream_offset};
  return run_cell(h, run, static_cast<cudaStream_t>(stream));
}

int fw_cell_generate(fw_handle* fh, const int32_t* d_inputs, int32_t n_inputs, int32_t n_steps,
                     int32_t* d_out, float* d_logits, int32_t n_logit_steps,
                     const fw_sampler* sampler, void* stream) {
  int rc = check_handle(fh, false);
  if (rc) return rc;
  if ((rc = validate_sampler(sampler))) return rc;
  if (n_steps < 0) return invalid("steps must be non-negative");
  if (n_steps == 0) return FW_OK;
  if (n_inputs < 1 || !d_inputs) return invalid("at least one input step is required");
  if (!d_out) return invalid("d_out must not be null");
  if (n_logit_steps < 0 || n_logit_steps > n_steps) return invalid("n_logit_steps out of range");
  Handle& h = fh->h;
  FW_CUDA(cudaSetDevice(h.device));
  CellRun run{d_inputs, n_inputs, n_steps, d_out, d_logits, d_logits ? n_logit_steps : 0, h.t,
              sampler->mode, sampler->seed, sampler->stream_offset};
  return run_cell(h, run, static_cast<cudaStream_t>(stream));
}

int fw_cell_generate_host(fw_handle* fh, const int32_t* h_inputs, int32_t n_inputs,
                          int32_t n_steps, int32_t* h_out, const fw_sampler* sampler,
                          void* stream) {
  int rc = check_handle(fh, false);
  if (rc) return rc;
  if ((rc = validate_sampler(sampler))) return rc;
  if (n_steps < 0) return invalid("steps must be non-negative");
  if (n_steps == 0) return FW_OK;
  if (n_inputs < 1 || !h_inputs || !h_out) return invalid("null host buffer or no inputs");
  Handle& h = fh->h;
  for (int64_t i = 0, n = (int64_t)n_inputs * h.user_batch; i < n; ++i)
    if (h_inputs[i] < 0 || h_inputs[i] >= h.dims.A) return invalid("input class ids out of range");
  FW_CUDA(cudaSetDevice(h.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t need = ((int64_t)n_inputs + n_steps) * h.user_batch;
  if (need > h.d_io_elems) {
    if (h.d_io) cudaFree(h.d_io);
    h.d_io = nullptr;
    h.d_io_elems = 0;
    FW_CUDA(cudaMalloc(&h.d_io, sizeof(int32_t) * (size_t)need));
    h.d_io_elems = need;
  }
  int32_t* d_in = h.d_io;
  int32_t* d_out = h.d_io + (int64_t)n_inputs * h.user_batch;
  FW_CUDA(cudaMemcpyAsync(d_in, h_inputs, sizeof(int32_t) * (size_t)n_inputs * h.user_batch,
                          cudaMemcpyHostToDevice, st));
  CellRun run{d_in, n_inputs, n_steps, d_out, nullptr, 0, h.t,
              sampler->mode, sampler->seed, sampler->stream_offset};
  if ((rc = run_cell(h, run, st))) return rc;
  FW_CUDA(cudaMemcpyAsync(h_out, d_out, sizeof(int32_t) * (size_t)n_steps * h.user_batch,
                          cudaMemcpyDeviceToHost, st));
  FW_CUDA(cudaStreamSynchronize(st));
  return FW_OK;
}

int fw_cell_select(fw_handle* fh, const float* d_logits, int64_t n_rows, int64_t step,
                   const fw_sampler* sampler, int32_t* d_out, void* stream) {
  int rc = check_handle(fh, false);
  if (rc) return rc;
  if ((rc = validate_sampler(sampler))) return rc;
  if (n_rows < 0) return invalid("n_rows must be non-negative");
  if (n_rows == 0) return FW_OK;
  if (!d_logits || !d_out) return invalid("d_logits and d_out must not be null");
  Handle& h = fh->h;
  FW_CUDA(cudaSetDevice(h.device));
  FW_CUDA(launch_cell_select(h, d_logits, n_rows, step, sampler->mode, sampler->seed,
                             sampler->stream_offset, d_out, static_cast<cudaStream_t>(stream)));
  h.last_launches = 1;
  return FW_OK;
}

int fw_cell_prefill(fw_handle* fh, const int32_t* d_inputs, int32_t T, float* d_logits,
                    void* stream) {
  int rc = check_handle(fh, false);
  if (rc) return rc;
  if (T < 0) return invalid("T must be non-negative");
  if (T == 0) return FW_OK;
  if (!d_inputs) return invalid("d_inputs must not be null");
  Handle& h = fh->h;
  FW_CUDA(cudaSetDevice(h.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // Two ways to the same end state. Time-parallel GEMMs (prefill.cu) move every layer's
  // fp32 intermediates through HBM, ~54 ns per (step, stream) for a cfg4-sized model; the
  // tcgen05 step kernel keeps them on chip and costs ~110 us per step for any batch up to
  // 4,096 streams. Below ~2,048 streams (and always on the SIMT path, whose steps are
  // latency-bound) the GEMMs win; above, teacher-forced steps do.
  // FW_PREFILL_MODE=gemm|steps forces one.
  const char* mode = getenv("FW_PREFILL_MODE");
  bool steps = h.kernel == FW_KERNEL_TCGEN05 && h.batch >= 2048;
  if (mode) steps = std::string(mode) == "steps";
  if (!steps && h.user_batch == h.batch) return cell_prefill(h, d_inputs, T, d_logits, st);
  if (!steps) {
    // padded handle: inputs to [T][batch] (pad streams class 0), logits back to [T][user]
    const int64_t B = h.user_batch, Bp = h.batch, A = h.dims.A;
    if (int rc2 = grow(&h.d_pad, &h.d_pad_elems, (int64_t)T * Bp)) return rc2;
    if (d_logits)
      if (int rc2 = grow(&h.d_pad_lg, &h.d_pad_lg_elems, (int64_t)T * Bp * A)) return rc2;
    FW_CUDA(cudaMemsetAsync(h.d_pad, 0, sizeof(int32_t) * (size_t)T * Bp, st));
    FW_CUDA(cudaMemcpy2DAsync(h.d_pad, sizeof(int32_t) * Bp, d_inputs, sizeof(int32_t) * B,
                              sizeof(int32_t) * B, T, cudaMemcpyDeviceToDevice, st));
    if (int rc2 = cell_prefill(h, h.d_pad, T, d_logits ? h.d_pad_lg : nullptr, st)) return rc2;
    if (d_logits)
      FW_CUDA(cudaMemcpy2DAsync(d_logits, sizeof(float) * B * A, h.d_pad_lg, sizeof(float) * Bp * A,
                                sizeof(float) * B * A, T, cudaMemcpyDeviceToDevice, st));
    return FW_OK;
  }
  const int64_t need = (int64_t)T * h.user_batch;
  if (need > h.d_io_elems) {
    if (h.d_io) cudaFree(h.d_io);
    h.d_io = nullptr;
    h.d_io_elems = 0;
    FW_CUDA(cudaMalloc(&h.d_io, sizeof(int32_t) * (size_t)need));
    h.d_io_elems = need;
  }
  CellRun run{d_inputs, T, T, h.d_io, d_logits, d_logits ? T : 0, h.t, FW_SAMPLE_ARGMAX, 0u, 0};
  return run_cell(h, run, st);
}

int fw_plain_create(const fw_plain_desc* d, int32_t batch, int32_t device, fw_handle** out) {
  if (!out) return invalid("null output handle pointer");
  *out = nullptr;
  if (!d) return invalid("null descriptor");
  if (d->blocks < 1) return invalid("blocks must be a positive integer");
  if (d->layers_per_block < 1) return invalid("layers_per_block must be a positive integer");
  if (d->filter_width < 2) return invalid("filter_width must be at least 2");
  if (d->dilation_base < 2) return invalid("dilation_base must be at least 2");
  if (d->hidden_channels < 1) return invalid("hidden_channels must be a positive integer");
  if (d->activation != 0 && d->activation != 1) return invalid("activation must be 0 or 1");
  if (!d->taps || !d->bias) return invalid("weight pointers must not be null");
  if (batch < 1) return invalid("batch must be a positive integer");
  int ndev = 0;
  FW_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return invalid("device index out of range");
  FW_CUDA(cudaSetDevice(device));
  auto* fh = new (std::nothrow) fw_handle();
  if (!fh) return invalid("out of host memory");
  Handle& h = fh->h;
  h.is_plain = 1;
  h.device = device;
  h.batch = batch;
  const int n = d->blocks * d->layers_per_block, w = d->filter_width, C = d->hidden_channels;
  std::vector<int> dil(n), cin(n), cout(n);
  std::vector<int64_t> woff(n), boff(n), qoff(n), roff(n), soff(n);
  int64_t wt = 0, bt = 0, qt = 0, rt = 0, stt = 0;
  for (int l = 0; l < n; ++l) {
    int64_t dd = 1;
    for (int i = 0; i < l % d->layers_per_block; ++i) dd *= d->dilation_base;
    if (dd > (1 << 30)) {
      delete fh;
      return invalid("dilation too large");
    }
    dil[l] = (int)dd;
    cin[l] = l == 0 ? 1 : C;
    cout[l] = l == n - 1 ? 1 : C;
    woff[l] = wt;
    boff[l] = bt;
    qoff[l] = qt;
    roff[l] = rt;
    soff[l] = stt;
    wt += (int64_t)w * cout[l] * cin[l];
    bt += cout[l];
    qt += (int64_t)(w - 1) * dil[l] * batch * cin[l];
    rt += (int64_t)(w - 1) * cin[l];
    stt += cin[l];
  }
  PlainDev& p = h.p;
  p.n_layers = n;
  p.w = w;
  p.act = d->activation;
  p.cmax = C;
  p.rec_rows = rt;
  p.state_rows = stt;
  h.pdil = dil;
  h.pcin = cin;
  int rc = FW_OK;
  auto fail = [&](int code) {
    free_plain(h);
    delete fh;
    return code;
  };
  if ((rc = upload(&p.dil, dil.data(), n))) return fail(rc);
  if ((rc = upload(&p.cin, cin.data(), n))) return fail(rc);
  if ((rc = upload(&p.cout, cout.data(), n))) return fail(rc);
  if ((rc = upload(&p.woff, woff.data(), n))) return fail(rc);
  if ((rc = upload(&p.boff, boff.data(), n))) return fail(rc);
  if ((rc = upload(&p.qoff, qoff.data(), n))) return fail(rc);
  if ((rc = upload(&p.roff, roff.data(), n))) return fail(rc);
  if ((rc = upload(&p.soff, soff.data(), n))) return fail(rc);
  if ((rc = upload(&p.taps, d->taps, wt))) return fail(rc);
  if ((rc = upload(&p.bias, d->bias, bt))) return fail(rc);
  cudaError_t e = cudaMalloc(&p.queue, sizeof(double) * (size_t)qt);
  if (e != cudaSuccess) return fail(cuda_fail(e, "queue allocation"));
  e = cudaMemset(p.queue, 0, sizeof(double) * (size_t)qt);
  if (e != cudaSuccess) return fail(cuda_fail(e, "queue zero-fill"));
  h.queue_bytes = qt * 8;
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(cuda_fail(e, "create synchronize"));
  *out = fh;
  return FW_OK;
}

int fw_plain_naive(fw_handle* fh, const double* d_history, int32_t n, double* d_out,
                   void* stream) {
  int rc = check_handle(fh, true);
  if (rc) return rc;
  if (n < 1) return invalid("the history must hold at least one sample");
  if (!d_history || !d_out) return invalid("null device buffer");
  Handle& h = fh->h;
  FW_CUDA(cudaSetDevice(h.device));
  if ((rc = build_naive_plan(h))) return rc;
  FW_CUDA(launch_plain_naive(h, d_history, n, d_out, static_cast<cudaStream_t>(stream)));
  return FW_OK;
}

int fw_plain_step(fw_handle* fh, const double* d_in, double* d_out, void* stream) {
  return fw_plain_generate(fh, d_in, 1, 1, d_out, stream);
}

int fw_plain_generate(fw_handle* fh, const double* d_inputs, int32_t n_inputs, int32_t n_steps,
                      double* d_out, void* stream) {
  int rc = check_handle(fh, true);
  if (rc) return rc;
  Handle& h = fh->h;
  if (h.popped) {
    set_error("step on a popped state (missed push?)");
    return FW_ERR_STATE;
  }
  if (n_steps < 0) return invalid("steps must be non-negative");
  if (n_steps == 0) return FW_OK;
  if (n_inputs < 1 || !d_inputs || !d_out) return invalid("null buffer or no inputs");
  FW_CUDA(cudaSetDevice(h.device));
  cudaError_t e = launch_plain_generate(h, d_inputs, n_inputs, n_steps, d_out,
                                        static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "plain kernel launch");
  h.last_launches = 1;
  h.t += n_steps;
  return FW_OK;
}

int fw_plain_pop(fw_handle* fh, double* d_rec, void* stream) {
  int rc = check_handle(fh, true);
  if (rc) return rc;
  Handle& h = fh->h;
  if (h.popped) {
    set_error("pop phase on a queue below capacity");
    return FW_ERR_STATE;
  }
  if (!d_rec) return invalid("d_rec must not be null");
  FW_CUDA(cudaSetDevice(h.device));
  cudaError_t e = launch_plain_pop(h, d_rec, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "plain pop launch");
  h.popped = 1;
  return FW_OK;
}

int fw_plain_compute(fw_handle* fh, const double* d_in, const double* d_rec, double* d_out,
                     double* d_states, void* stream) {
  int rc = check_handle(fh, true);
  if (rc) return rc;
  if (!d_in || !d_rec || !d_out || !d_states) return invalid("null buffer");
  Handle& h = fh->h;
  FW_CUDA(cudaSetDevice(h.device));
  cudaError_t e = launch_plain_compute(h, d_in, d_rec, d_out, d_states,
                                       static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "plain compute launch");
  return FW_OK;
}

int fw_plain_push(fw_handle* fh, const double* d_states, void* stream) {
  int rc = check_handle(fh, true);
  if (rc) return rc;
  Handle& h = fh->h;
  if (!h.popped) {
    set_error("push phase on a queue not one short of capacity");
    return FW_ERR_STATE;
  }
  if (!d_states) return invalid("d_states must not be null");
  FW_CUDA(cudaSetDevice(h.device));
  cudaError_t e = launch_plain_push(h, d_states, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "plain push launch");
  h.popped = 0;
  h.t += 1;
  return FW_OK;
}

int fw_reset(fw_handle* fh, void* stream) {
  if (!fh) return invalid("null handle");
  Handle& h = fh->h;
  FW_CUDA(cudaSetDevice(h.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (h.is_plain)
    FW_CUDA(cudaMemsetAsync(h.p.queue, 0, (size_t)h.queue_bytes, st));
  else
    FW_CUDA(cudaMemsetAsync(h.d_queue, 0, (size_t)h.queue_bytes, st));
  h.t = 0;
  h.popped = 0;
  return FW_OK;
}

int fw_debug_trace(fw_handle* fh, int64_t* d_trace) {
  int rc = check_handle(fh, false);
  if (rc) return rc;
  if (fh->h.kernel != FW_KERNEL_TCGEN05) {
    fh->h.lat_trace = reinterpret_cast<long long*>(d_trace);  // small-batch kernel
    return FW_OK;
  }
  tc_set_trace(fh->h, reinterpret_cast<long long*>(d_trace));
  return FW_OK;
}

int fw_debug_timing(fw_handle* fh, int32_t enable) {
  int rc = check_handle(fh, false);
  if (rc) return rc;
  fh->h.timing = enable ? 1 : 0;
  return FW_OK;
}

int fw_debug_timing_read(fw_handle* fh, double* chain_ms, double* step_ms, int64_t* steps) {
  int rc = check_handle(fh, false);
  if (rc) return rc;
  if (!chain_ms || !step_ms || !steps) return invalid("null argument");
  Handle& h = fh->h;
  *chain_ms = *step_ms = 0.0;
  *steps = h.timed_steps;
  if (h.tev_used == 0) return FW_OK;
  FW_CUDA(cudaSetDevice(h.device));
  FW_CUDA(cudaEventSynchronize(h.tev[3 * h.tev_used - 1]));
  for (int i = 0; i < h.tev_used; ++i) {
    float a = 0.f, b = 0.f;
    FW_CUDA(cudaEventElapsedTime(&a, h.tev[3 * i], h.tev[3 * i + 1]));
    FW_CUDA(cudaEventElapsedTime(&b, h.tev[3 * i], h.tev[3 * i + 2]));
    *chain_ms += a;
    *step_ms += b;
  }
  return FW_OK;
}

int fw_debug_copy(const fw_handle* fh, int32_t which, void* d_dst, int64_t bytes, void* stream) {
  if (!fh || !d_dst) return invalid("null argument");
  const Handle& h = fh->h;
  const void* src = nullptr;
  int64_t have = 0;
  if (which == 0) {
    src = h.is_plain ? (const void*)h.p.queue : (const void*)h.d_queue;
    have = h.queue_bytes;
  } else if (!h.is_plain && h.kernel == FW_KERNEL_TCGEN05) {
    have = tc_debug_buffer(const_cast<Handle&>(h), which, &src);
  }
  if (!src) return invalid("unknown buffer selector");
  if (bytes < 0 || bytes > have) return invalid("byte count exceeds the buffer size");
  FW_CUDA(cudaSetDevice(h.device));
  FW_CUDA(cudaMemcpyAsync(d_dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice,
                          static_cast<cudaStream_t>(stream)));
  return FW_OK;
}

int fw_step_index(const fw_handle* fh, int64_t* out) {
  if (!fh || !out) return invalid("null argument");
  *out = fh->h.t;
  return FW_OK;
}

int fw_queue_bytes(const fw_handle* fh, int64_t* out) {
  if (!fh || !out) return invalid("null argument");
  *out = fh->h.queue_bytes;
  return FW_OK;
}

int fw_kernel_kind(const fw_handle* fh, int32_t* out) {
  if (!fh || !out) return invalid("null argument");
  *out = fh->h.kernel;
  return FW_OK;
}

int fw_last_launch_count(const fw_handle* fh, int64_t* out) {
  if (!fh || !out) return invalid("null argument");
  *out = fh->h.last_launches;
  return FW_OK;
}

int fw_destroy(fw_handle* fh) {
  if (!fh) return FW_OK;
  Handle& h = fh->h;
  cudaSetDevice(h.device);
  cudaDeviceSynchronize();
  if (h.is_plain)
    free_plain(h);
  else
    free_cell(h);
  if (h.d_io) cudaFree(h.d_io);
  delete fh;
  return FW_OK;
}

}  // extern "C"
