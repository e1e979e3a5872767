// Extrapolator-corrector of the asynchronous two-way coupling (
// PAPER.md §2.4, Eq. 14-16; C-ABI in include/scaletrack.h).
//
// One elementwise kernel per Eulerian step over the n values of a source field:
// fold the k newly received truths into the correction (Eq. 14 and the multi-step
// rule), extrapolate from the last two known truths (Eq. 16), emit
//     est = corr + dt_ratio * ext                                          (Eq. 15)
// rounded to fp32, and keep, for the later correction, the estimate of this step's own
// source = emitted − corr (reading C-25), all state in fp64.  The fp64 operations are
// written without contraction (__dadd_rn/__dmul_rn) in the order of the definition so
// that the emitted fp32 values are reproducible.  HBM-bound: ≈ 56 + 12 k B per value.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <string>

#include "scaletrack.h"

struct st_ec {
  st_ec_config cfg{};
  cudaStream_t s = nullptr;
  bool own_stream = false;
  int64_t n = 0;
  int B = 0;                      // ring capacity (max_backlog)
  int head = 0, count = 0;        // pending estimates: ring slots head .. head+count-1
  int known = 0;                  // true sources received so far, capped at 2
  double* last = nullptr;         // S^{n-1}
  double* prev = nullptr;         // S^{n-2}
  double* pend = nullptr;         // [B][n] estimates of pending steps' own sources
  double* cum_true = nullptr;
  double* cum_est = nullptr;
  float* stage_in = nullptr;      // [B][n] host-input staging
  float* stage_out = nullptr;     // [n] host-output staging
  double* d_tot = nullptr;        // [3] ledger totals
  std::string err;
};

namespace {

thread_local std::string g_ec_init_error;

st_status ec_fail(st_ec* e, st_status s, const std::string& m) {
  if (e) e->err = m;
  else g_ec_init_error = m;
  return s;
}

#define EC_CUDA(e, call)                                                                        \
  do {                                                                                          \
    cudaError_t _r = (call);                                                                    \
    if (_r != cudaSuccess) return ec_fail(e, ST_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_r)); \
  } while (0)

bool on_device(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct StepArgsEC {
  int64_t n;
  int k;                  // truths received this step
  const float* recv;      // [k][n]
  int B, head;            // ring: the k oldest pending are slots head .. head+k-1
  int tail;               // slot of this step's estimate
  int known_after;        // truths known after this step's receipts (0, 1, 2+)
  int mode;
  double dt_ratio;
  double* last;
  double* prev;
  double* pend;
  double* cum_true;
  double* cum_est;
  float* est;
};

__global__ void k_ec_step(StepArgsEC a) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    double corr = 0.0, last = a.last[i], prev = a.prev[i], ct = a.cum_true[i];
    for (int q = 0; q < a.k; ++q) {
      const double s = (double)a.recv[(int64_t)q * a.n + i];
      const int slot = (a.head + q) % a.B;
      corr = __dadd_rn(corr, __dsub_rn(s, a.pend[(int64_t)slot * a.n + i]));   // Eq. 14 / P:228
      ct = __dadd_rn(ct, s);
      prev = last;
      last = s;
    }
    double ext = 0.0;                                                            // Eq. 16a
    if (a.mode != ST_EC_ZERO && a.known_after >= 1)
      ext = (a.mode == ST_EC_CONSTANT || a.known_after == 1) ? last                // Eq. 16b (C-26)
                                                             : __dsub_rn(__dmul_rn(2.0, last), prev);   // Eq. 16c
    const double est = __dadd_rn(corr, __dmul_rn(a.dt_ratio, ext));             // Eq. 15 (C-27)
    const float e32 = __double2float_rn(est);
    a.pend[(int64_t)a.tail * a.n + i] = __dsub_rn((double)e32, corr);           // C-25
    a.cum_est[i] = __dadd_rn(a.cum_est[i], (double)e32);
    a.cum_true[i] = ct;
    a.last[i] = last;
    a.prev[i] = prev;
    a.est[i] = e32;
  }
}

// totals[0..2] = Σ cum_true, Σ cum_est, Σ pending (fp64 atomics over block sums)
__global__ void k_ec_totals(int64_t n, const double* cum_true, const double* cum_est, const double* pend, int B,
                            int head, int count, double* tot) {
  __shared__ double red[3][8];
  double t[3] = {0.0, 0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    t[0] += cum_true[i];
    t[1] += cum_est[i];
    for (int q = 0; q < count; ++q) t[2] += pend[(int64_t)((head + q) % B) * n + i];
  }
  for (int c = 0; c < 3; ++c) {
    double v = t[c];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[c][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[threadIdx.x][w];
    atomicAdd(tot + threadIdx.x, v);
  }
}

__global__ void k_ec_pending_sum(int64_t n, const double* pend, int B, int head, int count, double* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double v = 0.0;
    for (int q = 0; q < count; ++q) v += pend[(int64_t)((head + q) % B) * n + i];
    out[i] = v;
  }
}

unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (unsigned)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace

extern "C" {

st_status st_ec_init(const st_ec_config* cfg, st_ec** out) {
  if (!cfg || !out) return ec_fail(nullptr, ST_ERR_INVALID_ARG, "cfg and out must not be NULL");
  *out = nullptr;
  if (cfg->abi_version != ST_ABI_VERSION) return ec_fail(nullptr, ST_ERR_INVALID_ARG, "ABI version mismatch");
  if (cfg->mode < ST_EC_ZERO || cfg->mode > ST_EC_LINEAR) return ec_fail(nullptr, ST_ERR_INVALID_ARG, "mode must be 0, 1 or 2");
  if (cfg->n < 1) return ec_fail(nullptr, ST_ERR_INVALID_ARG, "n must be >= 1");
  if (cfg->max_backlog < 1 || cfg->max_backlog > 64) return ec_fail(nullptr, ST_ERR_INVALID_ARG, "max_backlog must be 1..64");
  st_ec* e = new st_ec();
  e->cfg = *cfg;
  e->n = cfg->n;
  e->B = cfg->max_backlog;
  auto bail = [&](st_status s) {
    g_ec_init_error = e->err;
    st_ec_destroy(e);
    return s;
  };
  st_status s;
#define EC_INIT(call)                                   \
  if ((s = [&]() -> st_status {                         \
         EC_CUDA(e, call);                              \
         return ST_OK;                                  \
       }()))                                            \
    return bail(s);
  EC_INIT(cudaSetDevice(cfg->device));
  if (cfg->stream) {
    e->s = (cudaStream_t)cfg->stream;
  } else {
    EC_INIT(cudaStreamCreateWithFlags(&e->s, cudaStreamNonBlocking));
    e->own_stream = true;
  }
  const size_t nd = (size_t)e->n * sizeof(double), nf = (size_t)e->n * sizeof(float);
  EC_INIT(cudaMalloc(&e->last, nd));
  EC_INIT(cudaMalloc(&e->prev, nd));
  EC_INIT(cudaMalloc(&e->cum_true, nd));
  EC_INIT(cudaMalloc(&e->cum_est, nd));
  EC_INIT(cudaMalloc(&e->pend, nd * e->B));
  EC_INIT(cudaMalloc(&e->stage_in, nf * e->B));
  EC_INIT(cudaMalloc(&e->stage_out, nf));
  EC_INIT(cudaMalloc(&e->d_tot, 3 * sizeof(double)));
  for (double* p : {e->last, e->prev, e->cum_true, e->cum_est}) EC_INIT(cudaMemsetAsync(p, 0, nd, e->s));
  EC_INIT(cudaStreamSynchronize(e->s));
#undef EC_INIT
  *out = e;
  return ST_OK;
}

st_status st_ec_destroy(st_ec* e) {
  if (!e) return ST_OK;
  if (e->s) cudaStreamSynchronize(e->s);
  for (void* p : {(void*)e->last, (void*)e->prev, (void*)e->pend, (void*)e->cum_true, (void*)e->cum_est,
                  (void*)e->stage_in, (void*)e->stage_out, (void*)e->d_tot})
    cudaFree(p);
  if (e->own_stream && e->s) cudaStreamDestroy(e->s);
  delete e;
  return ST_OK;
}

st_status st_ec_step(st_ec* e, int32_t k, const float* received, double dt_ratio, float* est) {
  if (!e) return ec_fail(nullptr, ST_ERR_INVALID_ARG, "NULL estimator");
  if (k < 0 || !(dt_ratio > 0.0) || !est || (k > 0 && !received))
    return ec_fail(e, ST_ERR_INVALID_ARG, "need k >= 0, dt_ratio > 0, est != NULL, received != NULL when k > 0");
  if (k > e->count)
    return ec_fail(e, ST_ERR_STATE, "protocol violation: a true source for a step that was never estimated");
  if (e->count - k + 1 > e->B) return ec_fail(e, ST_ERR_STATE, "backlog would exceed max_backlog");
  EC_CUDA(e, cudaSetDevice(e->cfg.device));
  const float* recv = received;
  if (k > 0 && !on_device(received)) {
    EC_CUDA(e, cudaMemcpyAsync(e->stage_in, received, (size_t)k * e->n * sizeof(float), cudaMemcpyHostToDevice, e->s));
    recv = e->stage_in;
  }
  const bool est_dev = on_device(est);
  StepArgsEC a;
  a.n = e->n;
  a.k = k;
  a.recv = recv;
  a.B = e->B;
  a.head = e->head;
  a.tail = (e->head + e->count) % e->B;   // the k oldest are consumed before this slot is reused
  a.known_after = e->known + k > 2 ? 2 : e->known + k;
  a.mode = e->cfg.mode;
  a.dt_ratio = dt_ratio;
  a.last = e->last;
  a.prev = e->prev;
  a.pend = e->pend;
  a.cum_true = e->cum_true;
  a.cum_est = e->cum_est;
  a.est = est_dev ? est : e->stage_out;
  // ring full (count == B): slot tail == head is read (q = 0) before the same thread
  // rewrites it, value by value
  k_ec_step<<<grid_for(e->n), 256, 0, e->s>>>(a);
  EC_CUDA(e, cudaGetLastError());
  if (!est_dev) EC_CUDA(e, cudaMemcpyAsync(est, e->stage_out, (size_t)e->n * sizeof(float), cudaMemcpyDeviceToHost, e->s));
  EC_CUDA(e, cudaStreamSynchronize(e->s));
  e->head = (e->head + k) % e->B;
  e->count = e->count - k + 1;
  e->known = a.known_after;
  e->err.clear();
  return ST_OK;
}

st_status st_ec_ledger(st_ec* e, double* cum_true, double* cum_est, double* pending, double* totals) {
  if (!e) return ec_fail(nullptr, ST_ERR_INVALID_ARG, "NULL estimator");
  EC_CUDA(e, cudaSetDevice(e->cfg.device));
  const size_t nd = (size_t)e->n * sizeof(double);
  if (cum_true) EC_CUDA(e, cudaMemcpyAsync(cum_true, e->cum_true, nd, cudaMemcpyDeviceToHost, e->s));
  if (cum_est) EC_CUDA(e, cudaMemcpyAsync(cum_est, e->cum_est, nd, cudaMemcpyDeviceToHost, e->s));
  if (pending) {
    // the free ring slot (if any) serves as scratch for the per-value pending sum
    double* tmp = nullptr;
    EC_CUDA(e, cudaMallocAsync(&tmp, nd, e->s));
    k_ec_pending_sum<<<grid_for(e->n), 256, 0, e->s>>>(e->n, e->pend, e->B, e->head, e->count, tmp);
    EC_CUDA(e, cudaGetLastError());
    EC_CUDA(e, cudaMemcpyAsync(pending, tmp, nd, cudaMemcpyDeviceToHost, e->s));
    EC_CUDA(e, cudaFreeAsync(tmp, e->s));
  }
  if (totals) {
    EC_CUDA(e, cudaMemsetAsync(e->d_tot, 0, 3 * sizeof(double), e->s));
    k_ec_totals<<<grid_for(e->n), 256, 0, e->s>>>(e->n, e->cum_true, e->cum_est, e->pend, e->B, e->head, e->count,
                                                  e->d_tot);
    EC_CUDA(e, cudaGetLastError());
    EC_CUDA(e, cudaMemcpyAsync(totals, e->d_tot, 3 * sizeof(double), cudaMemcpyDeviceToHost, e->s));
  }
  EC_CUDA(e, cudaStreamSynchronize(e->s));
  return ST_OK;
}

st_status st_ec_backlog(st_ec* e, int32_t* steps) {
  if (!e || !steps) return ec_fail(e, ST_ERR_INVALID_ARG, "NULL argument");
  *steps = e->count;
  return ST_OK;
}

const char* st_ec_last_error(const st_ec* e) { return e ? e->err.c_str() : g_ec_init_error.c_str(); }

}  // extern "C"
