/*
 * fastwavenet.h -- C ABI of the B200 queue-cached generation step
 * (arXiv 1611.09482, "Fast WaveNet"), libfastwavenet.so.
 *
 * The reference (`streamconv`, pure Python + numba) exposes this path as
 * plain Python functions; there is no plugin/FFI registry to bind against
 * (SURVEY.md section 8(b)). Each entry point below states the reference
 * interface it replaces (file:line under /root/reference/pkg/src/streamconv).
 * The Python host side (paper_1611_09482_b200/fast.py, generate.py) keeps the
 * reference names on top of these calls; INTEGRATION.md shows the ctypes
 * binding a maintainer of the reference would add.
 *
 * Conventions
 *  - Plain C types only: sizes are int32/int64, device buffers are raw
 *    pointers (cudaMalloc'd or torch tensor data_ptr()), `stream` is a
 *    cudaStream_t passed as void* (NULL = legacy default stream). All work
 *    is enqueued on `stream`; nothing synchronises the host except the
 *    *_host entry points, which return after their device->host copy.
 *  - Return 0 on success. Nonzero codes map in the Python shim to the
 *    reference's exception types: FW_ERR_INVALID -> ValueError (the
 *    reference raises ValueError for config/shape/arity errors, model.py:48-64,
 *    fast.py:168-191, 218-219, 237-238), FW_ERR_STATE -> QueueStateError
 *    (fast.py:25-26; phase misuse), FW_ERR_CUDA -> RuntimeError.
 *    fw_last_error() returns a thread-local message for the last failure.
 *  - A handle owns its repacked device weights and its HBM ring-buffer
 *    queues; it is not thread-safe (as GenerationState, fast.py:98-103);
 *    use one handle per GPU per process.
 */
#ifndef FASTWAVENET_H
#define FASTWAVENET_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FW_OK 0
#define FW_ERR_INVALID 1
#define FW_ERR_STATE 2
#define FW_ERR_CUDA 3
#define FW_ERR_UNSUPPORTED 4

#define FW_DTYPE_F32 0
#define FW_DTYPE_BF16 1

#define FW_SAMPLE_ARGMAX 0 /* first maximum on ties (numpy argmax) */
#define FW_SAMPLE_INVCDF 1 /* smallest i with cumsum(exp(l-max))_i > u*total */
#define FW_SAMPLE_GUMBEL 2 /* argmax(logits - log(-log u)) */

#define FW_KERNEL_AUTO 0
#define FW_KERNEL_SIMT 1    /* fp32 CUDA-core persistent step kernel */
#define FW_KERNEL_TCGEN05 2 /* bf16 tcgen05/TMEM step kernels (large batch) */

typedef struct fw_handle fw_handle;

/* ---- gated cell (the north-star path) ---------------- */

/* Host float32 weights in the reference's (out, in) layout, tap 0 = current
 * step, tap 1 = `dilation` steps back (streamconv LayerWeights, model.py:98-129).
 * L = n_layers, R = residual, D = dilation (pre-gate 2D), S = skip,
 * H = head hidden, A = classes. For weight_dtype == FW_DTYPE_BF16 the values
 * are rounded to bf16 (nearest even) on upload. */
typedef struct fw_cell_desc {
  int32_t n_layers;
  const int32_t* dilations; /* [L] */
  int32_t residual_channels;
  int32_t dilation_channels;
  int32_t skip_channels;
  int32_t head_channels;
  int32_t classes;
  int32_t weight_dtype; /* FW_DTYPE_* */
  const float* embed;   /* [A][R]        */
  const float* dil_w;   /* [L][2][2D][R] */
  const float* dil_b;   /* [L][2D]       */
  const float* res_w;   /* [L][R][D]     */
  const float* res_b;   /* [L][R]        */
  const float* skip_w;  /* [L][S][D]     */
  const float* skip_b;  /* [L][S]        */
  const float* head1_w; /* [H][S]        */
  const float* head1_b; /* [H]           */
  const float* head2_w; /* [A][H]        */
  const float* head2_b; /* [A]           */
} fw_cell_desc;

typedef struct fw_sampler {
  int32_t mode;          /* FW_SAMPLE_* */
  uint32_t seed;         /* noise hash seed */
  int64_t stream_offset; /* global id of this handle's stream 0 (sharding) */
} fw_sampler;

/* = init_state (fast.py:122-128) for `batch` independent streams: uploads and
 * repacks the weights, allocates the per-layer ring queues
 * in HBM and zero-fills them: sum_l d_l * batch * R values, fp32 on the SIMT path and
 * fp16 on the tcgen05 path (the slot holds the MMA operand the tensor cores consume; every
 * pop would round to it anyway, so results are identical). Class ids outside [0, A) are
 * rejected by the host entry points and the Python shim; on the device they are clamped
 * into range (never read out of bounds). */
int fw_cell_create(const fw_cell_desc* desc, int32_t batch, int32_t device, int32_t kernel,
                   fw_handle** out);

/* = fast_step (fast.py:216-224) over all streams: pop -> compute -> push.
 * d_in [B] int32 class ids; d_out [B] int32 selected class; d_logits [B][A]
 * fp32 or NULL. Advances the step counter by one. */
int fw_cell_step(fw_handle* h, const int32_t* d_in, int32_t* d_out, float* d_logits,
                 const fw_sampler* sampler, void* stream);

/* = fast_generate (fast.py:227-252), all steps on the device in one launch
 * per chunk. Step i consumes d_inputs[i][:] for i < n_inputs (teacher / primer),
 * otherwise the class selected at step i-1. d_out [n_steps][B] receives the
 * class selected at every step; d_logits [n_logit_steps][B][A] (nullable)
 * receives the logits of the first n_logit_steps steps. The reference's
 * fast_generate(primer, steps) is n_inputs = len(primer),
 * n_steps = len(primer) - 1 + steps, result = d_out[len(primer)-1:]. */
int fw_cell_generate(fw_handle* h, const int32_t* d_inputs, int32_t n_inputs, int32_t n_steps,
                     int32_t* d_out, float* d_logits, int32_t n_logit_steps,
                     const fw_sampler* sampler, void* stream);

/* fw_cell_generate with HOST buffers: copies h_inputs in, runs, copies the
 * selected classes back to h_out [n_steps][B]; returns after the copy. This is
 * the end-to-end entry point the reference-facing shim calls. */
int fw_cell_generate_host(fw_handle* h, const int32_t* h_inputs, int32_t n_inputs,
                          int32_t n_steps, int32_t* h_out, const fw_sampler* sampler,
                          void* stream);

/* Full-sequence (time-parallel) forward over T given inputs per stream, from the
 * handle's current state: leaves the queues and the step counter exactly where T
 * teacher-forced steps of fw_cell_generate (n_inputs = n_steps = T) would, and writes
 * the logits of all T steps to d_logits [T][B][A] fp32 (nullable: queues only, the
 * skip sum and heads are skipped). The analogue of the reference's forward_full /
 * causal_dilated_conv (streamconv oracle.py:84-123) for the cell, used to prefill the
 * queues from a long primer (the reference steps primers, fast.py:244-245): the layers
 * run as GEMMs over all (time, stream) rows of a chunk instead of T dependent steps --
 * except on tcgen05 handles of >= 2,048 streams, where teacher-forced steps of the fused
 * step kernel are faster and are used instead (same end state; FW_PREFILL_MODE=gemm|steps
 * forces either). */
int fw_cell_prefill(fw_handle* h, const int32_t* d_inputs, int32_t T, float* d_logits,
                    void* stream);

/* The selection rule alone (the step kernels' final stage) over rows of
 * logits: row i of d_logits [n_rows][A] is stream i % B (global id stream_offset + i % B)
 * at step `step + i / B`, with the same counter-hash noise as the step kernels; the chosen
 * class goes to d_out[i]. The cache-free generator (naive.py:113-131's feedback rule on
 * the recomputed logits) selects through this. */
int fw_cell_select(fw_handle* h, const float* d_logits, int64_t n_rows, int64_t step,
                   const fw_sampler* sampler, int32_t* d_out, void* stream);

/* ---- plain mode: the reference's own stack, float64 (model.py, fast.py) ---- */

typedef struct fw_plain_desc {
  int32_t blocks;
  int32_t layers_per_block;
  int32_t filter_width;
  int32_t dilation_base;
  int32_t hidden_channels;
  int32_t activation; /* 0 linear, 1 tanh (kernel.py:18-27) */
  const double* taps; /* per layer (w, out, in), layers concatenated bottom to top */
  const double* bias; /* per layer (out,), concatenated */
} fw_plain_desc;

/* = init_state for `batch` scalar streams (fast.py:122-128). */
int fw_plain_create(const fw_plain_desc* desc, int32_t batch, int32_t device, fw_handle** out);

/* = fast_step (fast.py:216-224): d_in [B] float64 -> d_out [B] float64. */
int fw_plain_step(fw_handle* h, const double* d_in, double* d_out, void* stream);

/* = naive_step (naive.py:27-110): the sample that extends d_history [n][B] by one,
 * recomputed cache-free through the demand plan of its receptive field (every demanded
 * node of a layer in parallel, each in the pinned order of the cached path, so the result
 * equals it bit for bit). d_out [B]. The queues and the step counter are not touched. */
int fw_plain_naive(fw_handle* h, const double* d_history, int32_t n, double* d_out, void* stream);

/* = fast_generate's step loop: d_inputs [n_inputs][B], feedback afterwards,
 * d_out [n_steps][B] every step's output. */
int fw_plain_generate(fw_handle* h, const double* d_inputs, int32_t n_inputs, int32_t n_steps,
                      double* d_out, void* stream);

/* Phase-level API (pop_phase / compute_step / push_phase, fast.py:131-213):
 * fw_plain_pop copies each layer's w-1 tap values for every stream into
 * d_rec [sum_l (w-1)*C_in_l][B] (layer-major, tap k ascending, channel
 * ascending) and marks the queues popped; a second pop before a push returns
 * FW_ERR_STATE. fw_plain_push writes d_states [sum_l C_in_l][B] (each layer's
 * fresh input) into the slot of step t and advances t; a push without a pop
 * returns FW_ERR_STATE. fw_plain_compute evaluates the stack from d_in and
 * d_rec without touching the queues, writing d_out [B] and d_states. */
int fw_plain_pop(fw_handle* h, double* d_rec, void* stream);
int fw_plain_compute(fw_handle* h, const double* d_in, const double* d_rec, double* d_out,
                     double* d_states, void* stream);
int fw_plain_push(fw_handle* h, const double* d_states, void* stream);

/* ---- common ---------------------------------------------------------------- */

/* Zero all queues and reset the step counter (a fresh init_state). */
int fw_reset(fw_handle* h, void* stream);
/* Current step index (GenerationState.step_index, fast.py:114). */
int fw_step_index(const fw_handle* h, int64_t* out);
/* Bytes of HBM held by the queues (GenerationState.cached_scalar_count() * 4 or 8). */
int fw_queue_bytes(const fw_handle* h, int64_t* out);
/* Which kernel family the handle dispatches to (FW_KERNEL_SIMT / FW_KERNEL_TCGEN05). */
int fw_kernel_kind(const fw_handle* h, int32_t* out);
/* Number of kernel launches the last generate/step call enqueued. */
int fw_last_launch_count(const fw_handle* h, int64_t* out);
int fw_destroy(fw_handle* h);
const char* fw_last_error(void);
/* Diagnostics: record per-layer clock64() phase timestamps of CTA 0 of the
 * tcgen05 chain kernel into d_trace [n_layers][16] (NULL disables); on a SIMT handle the
 * small-batch cluster kernel instead writes %globaltimer stamps of its phases in step 1
 * of a launch, d_trace [n_layers + 4][8]. Not part of the reference's interface; used by
 * tools/trace_chain.py and tools/trace_lat.py. */
int fw_debug_trace(fw_handle* h, int64_t* d_trace);
/* Diagnostics: copy the first `bytes` of an internal device buffer to d_dst on `stream`.
 * which = 0: the HBM ring queues (layout in DESIGN.md); tcgen05 handles only: 1 z stash,
 * 2 ReLU(skip) images, 3 head-hidden images (fp16 operand images). */
int fw_debug_copy(const fw_handle* h, int32_t which, void* d_dst, int64_t bytes, void* stream);
/* Diagnostics: when enabled, cell generate calls record CUDA events around each step's
 * dominant (chain) kernel and the whole step, on the caller's stream. _read synchronises
 * and returns the summed milliseconds and the number of steps covered (up to 1,024). */
int fw_debug_timing(fw_handle* h, int32_t enable);
int fw_debug_timing_read(fw_handle* h, double* chain_ms, double* step_ms, int64_t* steps);
/* Library ABI version (major*100 + minor). */
int32_t fw_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FASTWAVENET_H */
