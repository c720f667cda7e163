// Internal definitions shared by the C-ABI (capi.cu) and the kernel files.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/fastwavenet.h"

namespace fw {

// Last-error slot (thread-local), set by every failing entry point.
void set_error(const std::string& msg);

// ---- noise hash (bit-identical to oracle/noise.py) -------------------------
__host__ __device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
constexpr uint32_t kSeedSalt = 0x243F6A88u;
constexpr uint32_t kUniformClass = 0xFFFFFFFFu;

// Hash prefix of (seed, stream, step); the class is mixed in last.
__host__ __device__ __forceinline__ uint32_t noise_prefix(uint32_t seed, uint32_t stream,
                                                          uint32_t step) {
  uint32_t h = mix32(seed ^ kSeedSalt);
  h = mix32(h ^ stream);
  return mix32(h ^ step);
}
// u in (0,1): ((h >> 8) + 0.5) * 2^-24 -- exact in fp32.
__host__ __device__ __forceinline__ float noise_uniform(uint32_t prefix, uint32_t cls) {
  uint32_t h = mix32(prefix ^ cls);
  return (static_cast<float>(h >> 8) + 0.5f) * (1.0f / 16777216.0f);
}

// Class id -> embedding row, kept inside [0, A): ids outside it (a caller bug the host
// entry points and the Python shim reject) must not read past the embedding table.
__host__ __device__ __forceinline__ int clamp_class(int c, int A) {
  return (unsigned)c < (unsigned)A ? c : (c < 0 ? 0 : A - 1);
}

// ---- cell problem description ------------------------------------------------
struct CellDims {
  int L, R, D, S, H, A;
  int dtype;  // FW_DTYPE_*
};

// Arguments of one generate call (device pointers), shared by all cell kernels.
struct CellRun {
  const int32_t* inputs;  // [n_inputs][B]
  int32_t n_inputs;
  int32_t n_steps;
  int32_t* out;           // [n_steps][B]
  float* logits;          // [n_logit_steps][B][A] or null
  int32_t n_logit_steps;
  int64_t t0;             // absolute step index of the first step
  int32_t mode;           // FW_SAMPLE_*
  uint32_t seed;
  int64_t stream_offset;
};

// fp32 SIMT weights: every matrix transposed to [in][out] so a warp's
// consecutive output channels read consecutive addresses.
struct SimtWeights {
  float* embed;  // [A][R]
  float* dilT;   // [L][2R][2D]  rows 0..R-1 tap 0 (current), R..2R-1 tap 1 (d back)
  float* dil_b;  // [L][2D]
  float* resT;   // [L][D][R]
  float* res_b;  // [L][R]
  float* skipT;  // [L][D][S]
  float* catT;   // [L][D][S+R]: skipT | resT per row (the staged kernel's one z GEMV)
  float* skip_b; // [L][S]
  float* h1T;    // [S][H]
  float* h1_b;   // [H]
  float* h2T;    // [H][A]
  float* h2_b;   // [A]
};

// Host copy of the cell's weights in the reference layouts (fw_cell_desc), rounded to bf16
// for bf16 configs: the source of the per-kernel images built lazily after create.
struct HostCell {
  std::vector<float> dil_w, dil_b, res_w, res_b, skip_w, skip_b, h1_w, h1_b, h2_w, h2_b;
};

// tcgen05 path device state (see cell_tc.cu).
struct TcState;
// small-batch cluster kernel's packed weights (see cell_lat.cu).
struct LatPlan;
// full-sequence prefill state (see prefill.cu).
struct PrefillState;
// warp-MMA kernel's fragment images (see cell_hmma.cu).
struct HmmaPlan;

struct Handle;

// Launchers (return cudaError_t of the launch); defined in the kernel files.
cudaError_t launch_cell_simt(Handle& h, const CellRun& run, cudaStream_t st,
                             int64_t* launches);
cudaError_t launch_cell_lat(Handle& h, const CellRun& run, int C, cudaStream_t st);
bool lat_supported(const CellDims& d, int C);
void lat_destroy(Handle& h);
cudaError_t launch_cell_hmma(Handle& h, const CellRun& run, cudaStream_t st);
bool hmma_supported(const CellDims& d);
void hmma_destroy(Handle& h);
cudaError_t launch_cell_tc(Handle& h, const CellRun& run, cudaStream_t st, int64_t* launches);
bool tc_supported(const CellDims& d, int batch, std::string* why);
int tc_create(Handle& h, const fw_cell_desc* desc);
void tc_destroy(Handle& h);
void tc_set_trace(Handle& h, long long* trace);
int64_t tc_debug_buffer(Handle& h, int which, const void** src);
int cell_prefill(Handle& h, const int32_t* d_inputs, int T, float* d_logits, cudaStream_t st);
void prefill_destroy(Handle& h);
cudaError_t launch_cell_select(const Handle& h, const float* d_logits, int64_t n_rows, int64_t t0,
                               int mode, uint32_t seed, int64_t stream_offset, int32_t* d_out,
                               cudaStream_t st);

struct PlainDev {
  int n_layers, w, act;
  int* dil;         // [n]
  int* cin;         // [n]
  int* cout;        // [n]
  int64_t* woff;    // [n] offset into taps
  int64_t* boff;    // [n] offset into bias
  int64_t* qoff;    // [n] offset into queue (doubles)
  int64_t* roff;    // [n] offset of the layer's rows in the rec buffer
  int64_t* soff;    // [n] offset of the layer's rows in the states buffer
  double* taps;
  double* bias;
  double* queue;
  int cmax;
  int64_t rec_rows, state_rows;
};

cudaError_t launch_plain_generate(const Handle& h, const double* inputs, int n_inputs,
                                  int n_steps, double* out, cudaStream_t st);
cudaError_t launch_plain_pop(const Handle& h, double* rec, cudaStream_t st);
cudaError_t launch_plain_compute(const Handle& h, const double* in, const double* rec,
                                 double* out, double* states, cudaStream_t st);
cudaError_t launch_plain_push(const Handle& h, const double* states, cudaStream_t st);

// Cache-free (demand-driven) plain step: the reference's naive_step (naive.py:27-110).
struct NaivePlan {
  int built = 0;
  int* count = nullptr;       // [n] demanded nodes per layer
  int64_t* goff = nullptr;    // [n] offset of layer l's gather rows in `gather`
  int* gather = nullptr;      // [nodes][w]: layer 0 -- history offset back from T; l > 0 --
                              // index of the input node in layer l-1's demanded list
  int* gsrc = nullptr;        // [nodes][w]: the input's offset back from T (a negative time
                              // reads zero, as the cached path's zero-filled queues)
  int64_t* voff = nullptr;    // [n] offset of layer l's node values (per stream)
  int64_t vals_per_stream = 0;
  double* vals = nullptr;     // [B][vals_per_stream] scratch
};
cudaError_t launch_plain_naive(const Handle& h, const double* history, int n, double* out,
                               cudaStream_t st);

struct Handle {
  int is_plain = 0;
  int device = 0;
  int kernel = FW_KERNEL_SIMT;
  int32_t batch = 0;       // streams on the device (tcgen05: padded to a multiple of 128)
  int32_t user_batch = 0;  // streams in the caller's buffers
  int64_t t = 0;
  int64_t last_launches = 0;
  int popped = 0;

  // cell
  CellDims dims{};
  std::vector<int> dil;
  int* d_dil = nullptr;
  int64_t* d_qoff = nullptr;
  float* d_queue = nullptr;
  int64_t queue_bytes = 0;
  SimtWeights w{};
  TcState* tc = nullptr;
  PrefillState* prefill = nullptr;
  LatPlan* lat = nullptr;
  HmmaPlan* hmma = nullptr;
  long long* lat_trace = nullptr;  // fw_debug_trace on a SIMT handle: small-batch kernel stamps
  HostCell host;

  // plain
  PlainDev p{};
  std::vector<int> pdil, pcin;
  NaivePlan naive{};

  // scratch for the *_host entry points
  int32_t* d_io = nullptr;
  int64_t d_io_elems = 0;
  // staging between the caller's [n][user_batch] and the device's [n][batch] layouts
  int32_t* d_pad = nullptr;
  int64_t d_pad_elems = 0;
  float* d_pad_lg = nullptr;
  int64_t d_pad_lg_elems = 0;

  // optional per-step kernel timing (fw_debug_timing): events [3i] before the chain
  // kernel of step i, [3i+1] after it, [3i+2] after the step's last kernel
  int timing = 0;
  std::vector<cudaEvent_t> tev;
  int tev_used = 0;      // event triples recorded by the last call
  int64_t timed_steps = 0;  // generation steps those triples cover
};

// Ensures events for up to min(steps, 1024) timed steps; returns how many steps are timed.
inline int timing_reserve(Handle& h, int steps) {
  const int n = steps < 1024 ? steps : 1024;
  while ((int)h.tev.size() < 3 * n) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) break;
    h.tev.push_back(e);
  }
  const int have = (int)h.tev.size() / 3;
  return have < n ? have : n;
}

}  // namespace fw

struct fw_handle {
  fw::Handle h;
};
