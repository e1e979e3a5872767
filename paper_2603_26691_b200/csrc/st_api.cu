// C-ABI of the B200 SCALE-TRACK hot path (include/scaletrack.h).
// Owns the SoA particle store (ping-pong), the double-buffered fluid field and
// source accumulators (asynchronous coupling buffer), the
// compute and copy streams, and (nranks > 1) the NCCL communicator.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "st_comm.h"
#include "st_internal.h"
#include "st_step.h"

using namespace st;

struct st_ctx {
  st_config cfg{};
  std::string err;
  bool dead = false;

  // geometry
  Geom g{};
  Phys p{};
  int z0 = 0, z1 = 0, kz0 = 0, kz1 = 0, H = 0;
  int64_t local_cells = 0;   // nx*ny*(z1-z0)
  int32_t chunk_lo = 0, n_local_chunks = 0;
  int key_bits = 1;

  // streams
  cudaStream_t cs = nullptr;  // compute
  bool own_cs = false;
  cudaStream_t xs = nullptr;  // coupling buffer, field side (ingest)
  cudaStream_t xo = nullptr;  // coupling buffer, source side (readout): a readout waiting for
                              // the running step never delays the next field's copy
  cudaEvent_t ev_pinned_in{}; // last asynchronous copy from pinned host field memory
  bool pinned_in_flight = false;

  // store
  int64_t cap = 0, n = 0;
  Store S[2];
  int cur = 0;
  CUtensorMap tmap[4];        // [2 stores][float rows, ids] TMA descriptors (kernel parameters)
  CUtensorMap tmap_ip[2];     // [2 stores] float rows with the {68, 8} box of k_ip / k_fs
  CUtensorMap tmap_id66[2];   // [2 stores] ids with the {66, 1} box of k_fs
  CUtensorMap tmap_win[2][2]; // [field buffer][window shape] TMA descriptors of the fluid field
  long long* dtab = nullptr;  // [nbins][27] destination table of the fused scatter (k_dbase)
  int* far_cnt = nullptr;     // [nbins] far particles per destination bin (C-15b; k_count)
  unsigned long long* far_cur = nullptr;  // [nbins] far-tail cursors of the new layout (k_dbase)
  unsigned long long* d_far_n = nullptr;  // far particles placed by the last count (C-15b)
  int64_t general_rebins = 0;
  bool hist_ready = false;    // the last in-place step produced the next rebin's counts
  bool counts_from_ip = false; // the pending rebin's counts came from that step (not k_count)
  Comm* shard = nullptr;      // ST_DECOMP_SHARDED: communicator of the source all-reduce
  std::vector<int32_t> slab_copy;   // cfg.slab_planes, owned (the caller's array is read at init only)
  int shard_rank = 0, shard_nranks = 1;
  // ST_DECOMP_SHARDED: the Eulerian partition this rank owns (cell planes [eu_z0, eu_z1);
  // eu_zb = every rank's boundaries): the field comes in and the sources go out per owner
  int eu_z0 = 0, eu_z1 = 0;
  std::vector<int> eu_zb;
  int32_t* key[2] = {nullptr, nullptr};
  SortScratch sc;
  uint64_t next_id = 0;

  // binned layout (C-15): CSR per bin, warp items, slot histograms (k_step.cu)
  BinGeom bg{};
  bool binned = false;        // store sorted by bin key, off/items/hist valid
  bool rebin_due = false;     // contract rebin due (executed lazily, fused when possible)
  int lay = 0;                // index of the current layout in off/items
  int64_t* off[2] = {nullptr, nullptr};     // [nbins+1] current / next layout
  int* items[2] = {nullptr, nullptr};       // warp items (first bin of each)
  int* n_items[2] = {nullptr, nullptr};     // device counts
  int* hist = nullptr;                      // [27][nbins] slot counts of the current layout (k_count),
                                            // turned into run bases by k_rebin_prep
  uint32_t* new_cnt = nullptr;              // [nbins]
  uint32_t* item_flag = nullptr;            // [nbins]
  int64_t* item_pos = nullptr;              // [nbins+1]
  int* h_far = nullptr;                     // mapped pinned (1 rank): the rebin needs the general sort
  int* d_far = nullptr;
  unsigned long long* d_movers = nullptr;   // chunk movers counted by the last k_count
  cudaEvent_t ev_count = nullptr;           // k_count done (the far decision)
  // multi-GPU fused rebin (virtual neighbour planes)
  int64_t* voff[2] = {nullptr, nullptr};    // [nvb+1] offsets in the send buffers
  uint32_t* rcnt[2] = {nullptr, nullptr};   // [nvb] arrival counts (0: from below, 1: from above)
  int64_t* roff[2] = {nullptr, nullptr};    // [nvb+1]
  uint32_t* kept[2] = {nullptr, nullptr};   // [nvb]
  Store sbuf[2], rbuf[2];
  int64_t scap = 0;
  // far particles across ranks (C-15b): per neighbour-window cell counts (send / received),
  // d_fs = [counted per side 2 | scatter cursors 2 | received per side 2], keys of the far
  // region of each send buffer and of each receive buffer (+ a sort ping-pong)
  int* fv[2] = {nullptr, nullptr};
  int* rfv[2] = {nullptr, nullptr};
  int64_t nfv = 0;
  unsigned long long* d_fs = nullptr;
  int32_t* fs_key[2] = {nullptr, nullptr};    // sender's store index of each far mover
  int32_t* fs_cell[2] = {nullptr, nullptr};   // the cell it was counted for
  int32_t* fr_key[2] = {nullptr, nullptr};    // received
  int32_t* fr_cell[2] = {nullptr, nullptr};
  int64_t* h_fs = nullptr;   // pinned [4]: far sent lo / hi, far received dn / up
  int64_t* h_tot = nullptr;                 // pinned: send_lo, send_hi, recv_dn, recv_up
  int* h_farg = nullptr;                    // pinned: global far flag
  int* d_farg = nullptr;
  cudaEvent_t ev_tot{};
  cudaEvent_t ev_step_done{};

  // fields (double buffer)
  float4* field[2] = {nullptr, nullptr};
  int front = -1, pending = -1;
  cudaEvent_t ev_field_ready[2]{}, ev_field_reader[2]{};
  float* field_stage = nullptr;  // [3][ext planes][ny][nx] device staging
  int ext_z0 = 0, ext_nz = 0;    // planes held by field_stage (owned + halos)

  // sources (double buffer)
  float4* acc[2] = {nullptr, nullptr};
  int acc_cur = 0;
  double T_acc[2] = {0.0, 0.0};
  cudaEvent_t ev_acc_writer[2]{}, ev_acc_free[2]{};
  float* S_dev = nullptr;        // [3][local_cells]
  bool readout_pending = false;
  double readout_T = 0.0;
  cudaEvent_t ev_readout_done{};
  cudaEvent_t ev_in{};

  // errors and counters
  int* d_err = nullptr;
  int* item_ctr = nullptr;                  // dynamic item counter of the step kernels (reset per launch)
  int* far_long = nullptr;                  // [nbins] bins whose far tail is sorted by a CTA (k_far_order_b)
  int* far_long_n = nullptr;
  int* h_flags = nullptr;     // mapped pinned: consume_flags' atomic take of d_err
  int* d_flags = nullptr;
  int64_t calls = 0, rebins = 0, launches = 0, fused_rebins = 0, last_movers = 0;
  std::vector<int64_t> mig_row;
  int64_t last_sent = 0, last_recv = 0;

  // timing
  cudaEvent_t t_adv0{}, t_adv1{}, t_reb0{}, t_reb1{};
  // coupling-buffer trace (st_trace): a ring of [field copy begin/end (xs), step begin/end (cs),
  // readout begin/end (xo)] of the most recent calls, against a reference event
  static constexpr int kTrace = 64;
  cudaEvent_t tr_ref{}, tr[kTrace][6]{};
  int64_t tr_n[3] = {0, 0, 0};   // field copies, advances, readouts so far
  bool timed_adv = false, timed_reb = false;
  bool reb_t0 = false;        // t_reb0 already recorded for the rebin in progress (k_count)

  // multi-GPU
  Comm* comm = nullptr;
};

static thread_local std::string g_init_error;

#define ST_CUDA(ctx, call)                                                              \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      (ctx)->err = std::string(#call) + ": " + cudaGetErrorString(e_);                  \
      (ctx)->dead = true;                                                               \
      return e_ == cudaErrorMemoryAllocation ? ST_ERR_OOM : ST_ERR_CUDA;                \
    }                                                                                   \
  } while (0)

static st_status fail(st_ctx* c, st_status s, const std::string& msg) {
  c->err = msg;
  return s;
}

#define ST_ALIVE(ctx)                                                                   \
  do {                                                                                  \
    if (!(ctx)) return ST_ERR_INVALID_ARG;                                              \
    if ((ctx)->dead) return ST_ERR_CUDA;                                                \
  } while (0)

// page-locked host memory (cudaHostAlloc / cudaHostRegister): copies can be asynchronous
static bool is_pinned_host_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static st_status check_launch(st_ctx* c, int nl) {
  c->launches += nl;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    c->err = std::string("kernel launch: ") + cudaGetErrorString(e);
    c->dead = true;
    return ST_ERR_CUDA;
  }
  return ST_OK;
}

// Read and clear the device error flags, ordered on stream s (NULL: the compute stream):
// one atomic exchange into host-mapped memory, so nothing runs on the legacy default
// stream (a cudaMemcpy there would wait for the running step on the blocking compute
// stream and serialise the coupling buffer).  Flags raised by work still running on
// another stream are reported by a later call.
static st_status consume_flags(st_ctx* c, cudaStream_t s = nullptr) {
  if (!s) s = c->cs;
  *(volatile int*)c->h_flags = 0;
  st_status st = check_launch(c, launch_take_flags(c->d_err, c->d_flags, s));
  if (st) return st;
  ST_CUDA(c, cudaStreamSynchronize(s));
  const int h = *(volatile int*)c->h_flags;
  if (!h) return ST_OK;
  if (h & ERRF_CFL) return fail(c, ST_ERR_CFL, "displacement precondition violated (C-11/C-12: one wrap or bounce)");
  if (h & ERRF_WINDOW)
    return fail(c, ST_ERR_CFL, "a particle left this rank's field/source window between rebins (C-16)");
  if (h & ERRF_DOMAIN) return fail(c, ST_ERR_OUT_OF_DOMAIN, "position outside [lo, hi]");
  if (h & ERRF_SCATTER) return fail(c, ST_ERR_CFL, "rebin scatter found a particle outside its bin's neighbourhood");
  return ST_OK;
}

extern "C" {

static st_status flush_rebin(st_ctx* c);

int32_t st_abi_version(void) { return ST_ABI_VERSION; }

void st_config_default(st_config* c) {
  if (!c) return;
  memset(c, 0, sizeof(*c));
  c->abi_version = ST_ABI_VERSION;
  for (int a = 0; a < 3; ++a) {
    c->dims[a] = 16;
    c->origin[a] = 0.0;
    c->cell_size[a] = 1.0 / 16.0;
    c->bc[a] = ST_BC_PERIODIC;
    c->gravity[a] = 0.0;
  }
  c->chunk_cells = 8;
  c->rho_f = 1.2;
  c->nu_f = 1.5e-5;
  c->rho_p = 1000.0;
  c->drag_law = ST_DRAG_SCHILLER_NAUMANN;
  c->integrator = ST_INT_EXPONENTIAL;
  c->coupling = ST_TWO_WAY;
  c->rebin_interval = 1;
  c->capacity = 1000000;
  c->device = 0;
  c->stream = nullptr;
  c->rank = 0;
  c->nranks = 1;
  c->nccl_unique_id = nullptr;
  c->decomposition = ST_DECOMP_SLAB;
  c->slab_planes = nullptr;
}

// chunk planes [k0, k1) of rank r: equal split, or cfg->slab_planes
static void slab_range(const st_config* c, int ncz, int r, int* k0, int* k1) {
  if (c->slab_planes) {
    *k0 = c->slab_planes[r];
    *k1 = c->slab_planes[r + 1];
  } else {
    *k0 = (int)(((int64_t)r * ncz) / c->nranks);
    *k1 = (int)(((int64_t)(r + 1) * ncz) / c->nranks);
  }
}

// Cell-plane boundaries of the Eulerian partitions (rank r owns [zb[r], zb[r+1])): the
// slab rule of the slab decomposition (equal chunk planes, or cfg->slab_planes).
static void eulerian_slabs(const st_config* c, std::vector<int>& zb) {
  const int ncz = (c->dims[2] + c->chunk_cells - 1) / c->chunk_cells;
  zb.assign(c->nranks + 1, 0);
  for (int r = 0; r < c->nranks; ++r) {
    int k0, k1;
    slab_range(c, ncz, r, &k0, &k1);
    zb[r] = std::min(k0 * c->chunk_cells, c->dims[2]);
    zb[r + 1] = std::min(k1 * c->chunk_cells, c->dims[2]);
  }
}

// The geometry a rank sees: its own slab (ST_DECOMP_SLAB), or the whole domain as if
// alone (ST_DECOMP_SHARDED: the paper's Fig. 1c scheme, particles stay where injected).
static st_config geometry_view(const st_config* c) {
  st_config v = *c;
  if (c->decomposition == ST_DECOMP_SHARDED) {
    v.rank = 0;
    v.nranks = 1;
    v.decomposition = ST_DECOMP_SLAB;   // one rank's slab = the whole domain
    v.slab_planes = nullptr;            // (they bound the Eulerian partitions: eulerian_slabs)
  }
  return v;
}

const char* st_last_error(const st_ctx* c) { return c ? c->err.c_str() : g_init_error.c_str(); }

static st_status validate(const st_config* c, std::string& why) {
  if (c->abi_version != ST_ABI_VERSION) { why = "abi_version mismatch"; return ST_ERR_INVALID_ARG; }
  if (c->decomposition != ST_DECOMP_SLAB && c->decomposition != ST_DECOMP_SHARDED) {
    why = "decomposition must be ST_DECOMP_SLAB or ST_DECOMP_SHARDED";
    return ST_ERR_INVALID_ARG;
  }
  if (c->decomposition == ST_DECOMP_SHARDED) {
    if (c->nranks < 1 || c->rank < 0 || c->rank >= c->nranks) { why = "bad rank/nranks"; return ST_ERR_INVALID_ARG; }
    if (c->nranks > 1 && !c->nccl_unique_id) { why = "nccl_unique_id required when nranks > 1"; return ST_ERR_INVALID_ARG; }
    if (c->chunk_cells >= 1 && c->dims[2] >= 1 && c->nranks > (c->dims[2] + c->chunk_cells - 1) / c->chunk_cells) {
      why = "need at least one chunk plane per rank (Eulerian partitions)";
      return ST_ERR_INVALID_ARG;
    }
    if (c->slab_planes && c->chunk_cells >= 1) {
      const int ncz = (c->dims[2] + c->chunk_cells - 1) / c->chunk_cells;
      if (c->slab_planes[0] != 0 || c->slab_planes[c->nranks] != ncz) { why = "slab_planes must span [0, ncz]"; return ST_ERR_INVALID_ARG; }
      for (int r = 0; r < c->nranks; ++r)
        if (c->slab_planes[r + 1] <= c->slab_planes[r]) { why = "slab_planes must be strictly ascending"; return ST_ERR_INVALID_ARG; }
    }
    const st_config v = geometry_view(c);
    return validate(&v, why);
  }
  for (int a = 0; a < 3; ++a) {
    if (c->dims[a] < 1) { why = "dims must be >= 1"; return ST_ERR_INVALID_ARG; }
    if (!(c->cell_size[a] > 0.0)) { why = "cell_size must be > 0"; return ST_ERR_INVALID_ARG; }
    if (c->bc[a] != ST_BC_PERIODIC && c->bc[a] != ST_BC_REFLECT) { why = "bad bc"; return ST_ERR_INVALID_ARG; }
  }
  if (c->chunk_cells >= 1) {
    // chunk-padded bins x 27 slots must fit the 32-bit keys of the step kernel
    const int64_t cc = c->chunk_cells;
    const int64_t pad = ((c->dims[0] + cc - 1) / cc) * ((c->dims[1] + cc - 1) / cc) * ((c->dims[2] + cc - 1) / cc) * cc * cc * cc;
    if (pad * 27 > (int64_t)INT32_MAX) { why = "too many cells (padded bins x 27 must be < 2^31)"; return ST_ERR_INVALID_ARG; }
  }
  if (c->chunk_cells < 1) { why = "chunk_cells must be >= 1"; return ST_ERR_INVALID_ARG; }
  if (!(c->rho_f > 0 && c->nu_f > 0 && c->rho_p > 0)) { why = "densities and viscosity must be > 0"; return ST_ERR_INVALID_ARG; }
  if (c->drag_law < 0 || c->drag_law > 1 || c->integrator < 0 || c->integrator > 1 || c->coupling < 0 ||
      c->coupling > 1) { why = "bad enum"; return ST_ERR_INVALID_ARG; }
  if (c->rebin_interval < 1) { why = "rebin_interval must be >= 1"; return ST_ERR_INVALID_ARG; }
  if (c->capacity < 0) { why = "capacity must be >= 0"; return ST_ERR_INVALID_ARG; }
  // TMA box coordinates, store slots and far-tail indices are 32-bit in the step kernels
  if (c->capacity > (int64_t)INT32_MAX - 64) { why = "capacity must be <= 2^31 - 65 (32-bit store indices)"; return ST_ERR_INVALID_ARG; }
  if (c->nranks < 1 || c->rank < 0 || c->rank >= c->nranks) { why = "bad rank/nranks"; return ST_ERR_INVALID_ARG; }
  const int ncz = (c->dims[2] + c->chunk_cells - 1) / c->chunk_cells;
  if (c->nranks > ncz) { why = "need at least one chunk plane per rank"; return ST_ERR_INVALID_ARG; }
  if (c->nranks > 1 && !c->nccl_unique_id) { why = "nccl_unique_id required when nranks > 1"; return ST_ERR_INVALID_ARG; }
  if (c->slab_planes) {
    if (c->slab_planes[0] != 0 || c->slab_planes[c->nranks] != ncz) { why = "slab_planes must span [0, ncz]"; return ST_ERR_INVALID_ARG; }
    for (int r = 0; r < c->nranks; ++r)
      if (c->slab_planes[r + 1] <= c->slab_planes[r]) { why = "slab_planes must be strictly ascending"; return ST_ERR_INVALID_ARG; }
  }
  if (c->nranks > 1) {
    // every slab must hold the (chunk_cells + 1)-plane field halo its neighbour needs
    for (int r = 0; r < c->nranks; ++r) {
      int k0, k1;
      slab_range(c, ncz, r, &k0, &k1);
      const int zz1 = k1 * c->chunk_cells < c->dims[2] ? k1 * c->chunk_cells : c->dims[2];
      if (zz1 - k0 * c->chunk_cells < c->chunk_cells + 1) { why = "each rank needs >= chunk_cells+1 z planes"; return ST_ERR_INVALID_ARG; }
    }
  }
  return ST_OK;
}

static void build_geometry(st_ctx* c) {
  const st_config& f = c->cfg;
  Geom& g = c->g;
  memset(&g, 0, sizeof(g));
  for (int a = 0; a < 3; ++a) {
    g.n[a] = f.dims[a];
    g.lo[a] = (float)f.origin[a];
    g.ih[a] = (float)(1.0 / f.cell_size[a]);
    g.hi[a] = (float)(f.origin[a] + (double)f.dims[a] * f.cell_size[a]);
    g.L[a] = (float)((double)f.dims[a] * f.cell_size[a]);
    g.bc[a] = f.bc[a];
    g.NC[a] = (f.dims[a] + f.chunk_cells - 1) / f.chunk_cells;
  }
  g.cc = f.chunk_cells;
  const int G = f.nranks, r = f.rank;
  slab_range(&f, g.NC[2], r, &c->kz0, &c->kz1);
  c->z0 = c->kz0 * g.cc;
  c->z1 = c->kz1 * g.cc < g.n[2] ? c->kz1 * g.cc : g.n[2];
  c->H = G > 1 ? g.cc : 0;
  g.gx = g.n[0] + 2;
  g.gy = g.n[1] + 2;
  g.wz0 = c->z0 - c->H - 1;
  g.wnz = (c->z1 - c->z0) + 2 * c->H + 2;
  g.az0 = c->z0 - c->H;
  g.anz = (c->z1 - c->z0) + 2 * c->H;
  g.wrapz = (G > 1 && f.bc[2] == ST_BC_PERIODIC) ? 1 : 0;
  g.chunk_base = c->kz0 * g.NC[0] * g.NC[1];
  g.oz0 = c->z0;
  g.oz1 = c->z1;
  c->chunk_lo = g.chunk_base;
  c->n_local_chunks = (c->kz1 - c->kz0) * g.NC[0] * g.NC[1];
  c->local_cells = (int64_t)g.n[0] * g.n[1] * (c->z1 - c->z0);
  c->bg.cc3 = g.cc * g.cc * g.cc;
  c->bg.nbins = c->n_local_chunks * c->bg.cc3;
  c->bg.nkz = c->kz1 - c->kz0;
  c->bg.kz0 = c->kz0;
  c->bg.sh = -1;
  for (int s = 0; s < 16; ++s)
    if ((1 << s) == g.cc) c->bg.sh = s;
  c->bg.nvb = G > 1 ? g.NC[0] * g.NC[1] * g.cc * g.cc : 0;
  const bool pz = f.bc[2] == ST_BC_PERIODIC;
  c->bg.vz[0] = G > 1 ? (c->z0 > 0 ? c->z0 - 1 : (pz ? g.n[2] - 1 : -1)) : -1;
  c->bg.vz[1] = G > 1 ? (c->z1 < g.n[2] ? c->z1 : (pz ? 0 : -1)) : -1;
  // radix key = local bin (< nbins); multi-GPU pre-migration key = global chunk
  const int64_t kmax = std::max<int64_t>(c->bg.nbins, (int64_t)g.NC[0] * g.NC[1] * g.NC[2]);
  int bits = 1;
  while (((int64_t)1 << bits) < kmax) ++bits;
  c->key_bits = bits;
  // extended planes delivered to the ingest kernel (owned + one halo window each side)
  c->ext_z0 = c->z0 - c->H - 1;
  c->ext_nz = g.wnz;

  Phys& p = c->p;
  p.inv_nu = (float)(1.0 / f.nu_f);
  p.tau_c = (float)(f.rho_p / (18.0 * f.rho_f * f.nu_f));
  p.mass_c = (float)(M_PI / 6.0 * f.rho_p);
  for (int a = 0; a < 3; ++a) p.g[a] = (float)f.gravity[a];
  p.drag_law = f.drag_law;
  p.integrator = f.integrator;
  p.two_way = f.coupling == ST_TWO_WAY;
}

static st_status alloc_store(st_ctx* c, Store& s, int64_t cap_in) {
  const int64_t cap = cap_in > 0 ? cap_in : 1;
  const size_t bytes = (size_t)cap * (6 * sizeof(float) + 2 * sizeof(float) + sizeof(uint64_t)) + 1024;
  void* b = nullptr;
  ST_CUDA(c, cudaMalloc(&b, bytes));
  s.base = b;
  char* q = (char*)b;
  s.id = (uint64_t*)q;            // 8-byte aligned first
  q += (size_t)cap * sizeof(uint64_t);
  s.x = (float*)q;
  q += (size_t)cap * 3 * sizeof(float);
  s.u = (float*)q;
  q += (size_t)cap * 3 * sizeof(float);
  s.d = (float*)q;
  q += (size_t)cap * sizeof(float);
  s.w = (float*)q;
  return ST_OK;
}

// TMA descriptors of the particle stores (k_pstep input): the 8 float rows of a
// store are contiguous with stride cap (alloc_store), so one 2-D box {36, 8} stages
// a 32-particle batch from the 16-B aligned index below it; ids are a 2-D box {34, 1}
// of a {cap, 1} tensor.  Encoded through the driver entry
// point (no libcuda link dependency); passed as __grid_constant__ kernel parameters.
static st_status make_tensor_maps(st_ctx* c) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
      q != cudaDriverEntryPointSuccess)
    return fail(c, ST_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap* h = c->tmap;
  memset(h, 0, sizeof(c->tmap));
  for (int i = 0; i < 2; ++i) {
    const cuuint64_t dimf[2] = {(cuuint64_t)c->cap, 8};
    const cuuint64_t stridef[1] = {(cuuint64_t)c->cap * sizeof(float)};
    const cuuint32_t boxf[2] = {36, 8}, es[2] = {1, 1};   // k_pstep.cuh kBoxF
    CUresult r = encode(&h[2 * i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, c->S[i].x, dimf, stridef, boxf, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(c, ST_ERR_CUDA, "tensor map (float rows) encode failed: " + std::to_string((int)r));
    const cuuint32_t boxf64[2] = {68, 8};                // k_ip.cuh kIpBoxF
    r = encode(&c->tmap_ip[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, c->S[i].x, dimf, stridef, boxf64, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(c, ST_ERR_CUDA, "tensor map (float rows, 64) encode failed: " + std::to_string((int)r));
    const cuuint64_t dimi[2] = {(cuuint64_t)c->cap, 1};
    const cuuint64_t stridei[1] = {(cuuint64_t)c->cap * sizeof(uint64_t)};
    const cuuint32_t boxi[2] = {34, 1};                    // k_pstep.cuh kBoxI
    r = encode(&h[2 * i + 1], CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, c->S[i].id, dimi, stridei, boxi, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(c, ST_ERR_CUDA, "tensor map (ids) encode failed: " + std::to_string((int)r));
    const cuuint32_t boxi66[2] = {66, 1};                  // k_fs.cuh kFsBoxI
    r = encode(&c->tmap_id66[i], CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, c->S[i].id, dimi, stridei, boxi66, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(c, ST_ERR_CUDA, "tensor map (ids, 64) encode failed: " + std::to_string((int)r));
  }
  // fluid field float4 [wnz][gy][gx] seen as fp32 {4 gx, gy, wnz}: k_pstep's window boxes
  // of (10 + 2R) x (3 + 2R) x (3 + 2R) cells, R = 0 (in place) / 1 (fused scatter);
  // out-of-range planes/cells are zero-filled (never read by a lane inside the window)
  const Geom& g = c->g;
  for (int i = 0; i < 2; ++i)
    for (int w = 0; w < 2; ++w) {
      const cuuint64_t dimw[3] = {(cuuint64_t)g.gx * 4, (cuuint64_t)g.gy, (cuuint64_t)g.wnz};
      const cuuint64_t stridew[2] = {(cuuint64_t)g.gx * 16, (cuuint64_t)g.gx * g.gy * 16};
      const cuuint32_t boxw[3] = {(cuuint32_t)(4 * (10 + 2 * w)), (cuuint32_t)(3 + 2 * w), (cuuint32_t)(3 + 2 * w)};
      const cuuint32_t es3[3] = {1, 1, 1};
      CUresult r = encode(&c->tmap_win[i][w], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, c->field[i], dimw, stridew, boxw, es3,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(c, ST_ERR_CUDA, "tensor map (field window) encode failed: " + std::to_string((int)r));
    }
  return ST_OK;
}

static st_status init_impl(st_ctx* c) {
  ST_CUDA(c, cudaSetDevice(c->cfg.device));
  build_geometry(c);
  const Geom& g = c->g;
  if (g.wrapz && g.wnz > g.n[2]) return fail(c, ST_ERR_UNSUPPORTED, "periodic z needs (slab + 2 halos + 2) <= nz per rank");
  // SoA stride rounded to 32 particles: every component segment is 16-byte
  // aligned for the bulk (TMA) copies of k_step
  c->cap = (c->cfg.capacity + 31) / 32 * 32;
  if (c->cfg.stream) {
    c->cs = (cudaStream_t)c->cfg.stream;
  } else {
    // no stream given: a BLOCKING stream, so device inputs produced on the legacy
    // default stream (torch's default) are ordered before the library reads them
    ST_CUDA(c, cudaStreamCreateWithFlags(&c->cs, cudaStreamDefault));
    c->own_cs = true;
  }
  ST_CUDA(c, cudaStreamCreateWithFlags(&c->xs, cudaStreamNonBlocking));
  ST_CUDA(c, cudaStreamCreateWithFlags(&c->xo, cudaStreamNonBlocking));
  ST_CUDA(c, cudaEventCreateWithFlags(&c->ev_pinned_in, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) {
    st_status s = alloc_store(c, c->S[i], c->cap);
    if (s) return s;
    ST_CUDA(c, cudaMalloc(&c->key[i], (size_t)(c->cap > 0 ? c->cap : 1) * sizeof(int32_t)));
    ST_CUDA(c, cudaMalloc(&c->field[i], (size_t)g.wnz * g.gy * g.gx * sizeof(float4)));
    ST_CUDA(c, cudaMemset(c->field[i], 0, (size_t)g.wnz * g.gy * g.gx * sizeof(float4)));
    ST_CUDA(c, cudaMalloc(&c->acc[i], (size_t)g.anz * g.n[1] * g.n[0] * sizeof(float4)));
    ST_CUDA(c, cudaMemset(c->acc[i], 0, (size_t)g.anz * g.n[1] * g.n[0] * sizeof(float4)));
    ST_CUDA(c, cudaEventCreateWithFlags(&c->ev_field_ready[i], cudaEventDisableTiming));
    ST_CUDA(c, cudaEventCreateWithFlags(&c->ev_field_reader[i], cudaEventDisableTiming));
    ST_CUDA(c, cudaEventCreateWithFlags(&c->ev_acc_writer[i], cudaEventDisableTiming));
    ST_CUDA(c, cudaEventCreateWithFlags(&c->ev_acc_free[i], cudaEventDisableTiming));
  }
  ST_CUDA(c, cudaEventCreateWithFlags(&c->ev_readout_done, cudaEventDisableTiming));
  ST_CUDA(c, cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
  ST_CUDA(c, cudaEventCreate(&c->t_adv0));
  ST_CUDA(c, cudaEventCreate(&c->t_adv1));
  ST_CUDA(c, cudaEventCreate(&c->t_reb0));
  ST_CUDA(c, cudaEventCreate(&c->t_reb1));
  ST_CUDA(c, cudaEventCreate(&c->tr_ref));
  for (int i = 0; i < st_ctx::kTrace; ++i)
    for (int k = 0; k < 6; ++k) ST_CUDA(c, cudaEventCreate(&c->tr[i][k]));
  {
    st_status ts = make_tensor_maps(c);
    if (ts) return ts;
  }
  ST_CUDA(c, cudaMalloc(&c->field_stage, (size_t)3 * c->ext_nz * g.n[1] * g.n[0] * sizeof(float)));
  ST_CUDA(c, cudaMalloc(&c->S_dev, (size_t)3 * (c->local_cells > 0 ? c->local_cells : 1) * sizeof(float)));
  ST_CUDA(c, cudaMalloc(&c->d_err, sizeof(int)));
  ST_CUDA(c, cudaMemset(c->d_err, 0, sizeof(int)));
  ST_CUDA(c, cudaMalloc(&c->item_ctr, sizeof(int)));
  ST_CUDA(c, cudaHostAlloc(&c->h_flags, sizeof(int), cudaHostAllocMapped));
  ST_CUDA(c, cudaHostGetDevicePointer(&c->d_flags, c->h_flags, 0));
  const size_t nb = (size_t)c->bg.nbins;
  for (int i = 0; i < 2; ++i) {
    ST_CUDA(c, cudaMalloc(&c->off[i], (nb + 1) * sizeof(int64_t)));
    ST_CUDA(c, cudaMalloc(&c->items[i], (nb + 1) * sizeof(int)));
    ST_CUDA(c, cudaMalloc(&c->n_items[i], sizeof(int)));
  }
  ST_CUDA(c, cudaMalloc(&c->hist, nb * 27 * sizeof(int)));
  if (c->g.cc == 8) {
    ST_CUDA(c, cudaMalloc(&c->dtab, nb * 27 * sizeof(long long)));
    ST_CUDA(c, cudaMalloc(&c->far_cnt, nb * sizeof(int)));
    ST_CUDA(c, cudaMalloc(&c->far_cur, nb * sizeof(unsigned long long)));
    ST_CUDA(c, cudaMalloc(&c->far_long, nb * sizeof(int)));
    ST_CUDA(c, cudaMalloc(&c->far_long_n, sizeof(int)));
  }
  ST_CUDA(c, cudaMalloc(&c->new_cnt, (nb + 2 * (size_t)c->bg.nvb + 1) * sizeof(uint32_t)));
  if (c->bg.nvb > 0) {
    const size_t nv = (size_t)c->bg.nvb;
    c->scap = std::max<int64_t>(1 << 20, c->cap / 16);
    for (int i = 0; i < 2; ++i) {
      ST_CUDA(c, cudaMalloc(&c->voff[i], (nv + 1) * sizeof(int64_t)));
      ST_CUDA(c, cudaMalloc(&c->rcnt[i], nv * sizeof(uint32_t)));
      ST_CUDA(c, cudaMemset(c->rcnt[i], 0, nv * sizeof(uint32_t)));
      ST_CUDA(c, cudaMalloc(&c->roff[i], (nv + 1) * sizeof(int64_t)));
      ST_CUDA(c, cudaMalloc(&c->kept[i], nv * sizeof(uint32_t)));
      st_status s2 = alloc_store(c, c->sbuf[i], c->scap);
      if (s2) return s2;
      s2 = alloc_store(c, c->rbuf[i], c->scap);
      if (s2) return s2;
    }
    ST_CUDA(c, cudaHostAlloc(&c->h_tot, 4 * sizeof(int64_t), cudaHostAllocDefault));
    if (c->dtab) {   // 8^3 chunks: far particles across ranks stay on the fused path
      c->nfv = (int64_t)g.n[0] * g.n[1] * g.cc;
      for (int i = 0; i < 2; ++i) {
        ST_CUDA(c, cudaMalloc(&c->fv[i], c->nfv * sizeof(int)));
        ST_CUDA(c, cudaMemset(c->fv[i], 0, c->nfv * sizeof(int)));
        ST_CUDA(c, cudaMalloc(&c->rfv[i], c->nfv * sizeof(int)));
        ST_CUDA(c, cudaMemset(c->rfv[i], 0, c->nfv * sizeof(int)));   // stays 0 where no neighbour
        ST_CUDA(c, cudaMalloc(&c->fs_key[i], c->scap * sizeof(int32_t)));
        ST_CUDA(c, cudaMalloc(&c->fs_cell[i], c->scap * sizeof(int32_t)));
        ST_CUDA(c, cudaMalloc(&c->fr_key[i], c->scap * sizeof(int32_t)));
        ST_CUDA(c, cudaMalloc(&c->fr_cell[i], c->scap * sizeof(int32_t)));
      }
      ST_CUDA(c, cudaMalloc(&c->d_fs, 6 * sizeof(unsigned long long)));
      ST_CUDA(c, cudaMemset(c->d_fs, 0, 6 * sizeof(unsigned long long)));
      ST_CUDA(c, cudaHostAlloc(&c->h_fs, 4 * sizeof(int64_t), cudaHostAllocDefault));
    }
    ST_CUDA(c, cudaEventCreateWithFlags(&c->ev_tot, cudaEventDisableTiming));
  }
  ST_CUDA(c, cudaMalloc(&c->item_flag, (nb + 1) * sizeof(uint32_t)));
  ST_CUDA(c, cudaMalloc(&c->item_pos, (nb + 2) * sizeof(int64_t)));
  ST_CUDA(c, cudaHostAlloc(&c->h_far, sizeof(int), cudaHostAllocMapped));
  *c->h_far = 0;
  ST_CUDA(c, cudaHostGetDevicePointer(&c->d_far, c->h_far, 0));
  ST_CUDA(c, cudaEventCreateWithFlags(&c->ev_step_done, cudaEventDisableTiming));
  ST_CUDA(c, cudaEventCreateWithFlags(&c->ev_count, cudaEventDisableTiming));
  ST_CUDA(c, cudaHostAlloc(&c->h_farg, sizeof(int), cudaHostAllocDefault));
  ST_CUDA(c, cudaMalloc(&c->d_farg, sizeof(int)));
  ST_CUDA(c, cudaMalloc(&c->d_movers, sizeof(unsigned long long)));
  ST_CUDA(c, cudaMalloc(&c->d_far_n, sizeof(unsigned long long)));
  ST_CUDA(c, cudaMemset(c->d_far_n, 0, sizeof(unsigned long long)));
  ST_CUDA(c, cudaMemset(c->d_movers, 0, sizeof(unsigned long long)));
  // radix-sort scratch (also serves the scans over bins)
  c->sc.max_blocks = (c->cap + 4095) / 4096 + 1;
  const int64_t m = std::max<int64_t>(256 * c->sc.max_blocks, (int64_t)nb + 1);
  c->sc.partial_cap = (m + 4095) / 4096 + 1;
  ST_CUDA(c, cudaMalloc(&c->sc.hist, (size_t)m * sizeof(uint32_t)));
  ST_CUDA(c, cudaMalloc(&c->sc.offs, (size_t)(m + 1) * sizeof(int64_t)));
  ST_CUDA(c, cudaMalloc(&c->sc.partial, (size_t)c->sc.partial_cap * sizeof(int64_t)));
  c->mig_row.assign(c->cfg.nranks, 0);
  c->next_id = (uint64_t)c->cfg.rank << 40;
  if (c->cfg.nranks > 1) {
    std::string why;
    c->comm = comm_create(c->cfg.nccl_unique_id, c->cfg.rank, c->cfg.nranks, c->cfg.slab_planes, c->cs, why);
    if (!c->comm) return fail(c, ST_ERR_NCCL, why);
  }
  if (c->shard_nranks > 1) {   // particle-sharded: one communicator for the source sum
    std::string why;
    c->next_id = (uint64_t)c->shard_rank << 40;
    c->shard = comm_create(c->cfg.nccl_unique_id, c->shard_rank, c->shard_nranks, nullptr, c->cs, why);
    if (!c->shard) return fail(c, ST_ERR_NCCL, why);
  }
  ST_CUDA(c, cudaEventRecord(c->tr_ref, c->cs));
  ST_CUDA(c, cudaStreamSynchronize(c->cs));
  return ST_OK;
}

st_status st_destroy(st_ctx* c) {
  if (!c) return ST_OK;
  if (c->cs) cudaStreamSynchronize(c->cs);
  if (c->xs) cudaStreamSynchronize(c->xs);
  if (c->xo) cudaStreamSynchronize(c->xo);
  if (c->comm) comm_destroy(c->comm);
  if (c->shard) comm_destroy(c->shard);
  for (int i = 0; i < 2; ++i) {
    cudaFree(c->S[i].base);
    cudaFree(c->key[i]);
    cudaFree(c->field[i]);
    cudaFree(c->acc[i]);
    if (c->ev_field_ready[i]) cudaEventDestroy(c->ev_field_ready[i]);
    if (c->ev_field_reader[i]) cudaEventDestroy(c->ev_field_reader[i]);
    if (c->ev_acc_writer[i]) cudaEventDestroy(c->ev_acc_writer[i]);
    if (c->ev_acc_free[i]) cudaEventDestroy(c->ev_acc_free[i]);
  }
  cudaFree(c->field_stage);
  cudaFree(c->S_dev);
  cudaFree(c->d_err);
  if (c->h_flags) cudaFreeHost(c->h_flags);
  for (int i = 0; i < 2; ++i) {
    cudaFree(c->off[i]);
    cudaFree(c->items[i]);
    cudaFree(c->n_items[i]);
  }
  cudaFree(c->item_ctr);
  cudaFree(c->far_long);
  cudaFree(c->far_long_n);
  cudaFree(c->new_cnt);
  cudaFree(c->item_flag);
  cudaFree(c->item_pos);
  if (c->h_far) cudaFreeHost(c->h_far);
  cudaFree(c->d_movers);
  for (int i = 0; i < 2; ++i) {
    cudaFree(c->voff[i]);
    cudaFree(c->rcnt[i]);
    cudaFree(c->roff[i]);
    cudaFree(c->kept[i]);
    cudaFree(c->sbuf[i].base);
    cudaFree(c->rbuf[i].base);
  }
  if (c->h_tot) cudaFreeHost(c->h_tot);
  for (int i = 0; i < 2; ++i) {
    cudaFree(c->fv[i]);
    cudaFree(c->rfv[i]);
    cudaFree(c->fs_key[i]);
    cudaFree(c->fs_cell[i]);
    cudaFree(c->fr_key[i]);
    cudaFree(c->fr_cell[i]);
  }
  cudaFree(c->d_fs);
  if (c->h_fs) cudaFreeHost(c->h_fs);
  if (c->h_farg) cudaFreeHost(c->h_farg);
  cudaFree(c->d_farg);
  if (c->ev_tot) cudaEventDestroy(c->ev_tot);
  if (c->ev_step_done) cudaEventDestroy(c->ev_step_done);
  if (c->ev_count) cudaEventDestroy(c->ev_count);
  cudaFree(c->hist);
  cudaFree(c->dtab);
  cudaFree(c->far_cnt);
  cudaFree(c->far_cur);
  cudaFree(c->d_far_n);
  cudaFree(c->sc.hist);
  cudaFree(c->sc.offs);
  cudaFree(c->sc.partial);
  for (cudaEvent_t e : {c->ev_readout_done, c->ev_in, c->t_adv0, c->t_adv1, c->t_reb0, c->t_reb1, c->tr_ref})
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < st_ctx::kTrace; ++i)
    for (int k = 0; k < 6; ++k)
      if (c->tr[i][k]) cudaEventDestroy(c->tr[i][k]);
  if (c->own_cs && c->cs) cudaStreamDestroy(c->cs);
  if (c->xs) cudaStreamDestroy(c->xs);
  if (c->xo) cudaStreamDestroy(c->xo);
  if (c->ev_pinned_in) cudaEventDestroy(c->ev_pinned_in);
  cudaGetLastError();
  delete c;
  return ST_OK;
}

st_status st_init(const st_config* cfg, st_ctx** out) {
  if (!out) return ST_ERR_INVALID_ARG;
  *out = nullptr;
  if (!cfg) {
    g_init_error = "cfg is NULL";
    return ST_ERR_INVALID_ARG;
  }
  std::string why;
  st_status s = validate(cfg, why);
  if (s) {
    g_init_error = why;
    return s;
  }
  st_ctx* c = new st_ctx();
  c->cfg = geometry_view(cfg);
  if (c->cfg.slab_planes) {
    c->slab_copy.assign(c->cfg.slab_planes, c->cfg.slab_planes + c->cfg.nranks + 1);
    c->cfg.slab_planes = c->slab_copy.data();
  }
  if (cfg->decomposition == ST_DECOMP_SHARDED) {
    c->shard_rank = cfg->rank;
    c->shard_nranks = cfg->nranks;
    eulerian_slabs(cfg, c->eu_zb);
    c->eu_z0 = c->eu_zb[cfg->rank];
    c->eu_z1 = c->eu_zb[cfg->rank + 1];
  }
  s = init_impl(c);
  if (s) {
    g_init_error = c->err;
    st_destroy(c);
    return s;
  }
  *out = c;
  return ST_OK;
}

// ---------------------------------------------------------------- field in
st_status st_set_fluid_field(st_ctx* c, const float* u) {
  ST_ALIVE(c);
  if (!u) return fail(c, ST_ERR_INVALID_ARG, "u is NULL");
  const int back = c->pending >= 0 ? c->pending : (c->front < 0 ? 0 : 1 - c->front);
  // the back buffer may still be read by an advance enqueued earlier
  ST_CUDA(c, cudaStreamWaitEvent(c->xs, c->ev_field_reader[back], 0));
  const Geom& g = c->g;
  ST_CUDA(c, cudaEventRecord(c->tr[c->tr_n[0] % st_ctx::kTrace][0], c->xs));
  // cells the caller provides: this rank's slab (ST_DECOMP_SLAB) or its Eulerian
  // partition (ST_DECOMP_SHARDED; the other partitions arrive from their owners)
  const int in_z0 = c->shard ? c->eu_z0 : c->z0, in_z1 = c->shard ? c->eu_z1 : c->z1;
  const int64_t own_cells = (int64_t)g.n[0] * g.n[1] * (in_z1 - in_z0);
  const bool dev = is_device_ptr(u);
  const bool pinned = !dev && is_pinned_host_ptr(u);
  // the previous pinned copy is complete before this call returns (header contract: a
  // pinned buffer may be rewritten once the next st_set_fluid_field has returned)
  if (c->pinned_in_flight) {
    ST_CUDA(c, cudaEventSynchronize(c->ev_pinned_in));
    c->pinned_in_flight = false;
  }
  float* stage = c->field_stage;
  // staging layout: [3][ext_nz][ny][nx]; owned planes start at plane (z0 - ext_z0)
  const int64_t plane = (int64_t)g.n[0] * g.n[1];
  const int64_t comp = (int64_t)c->ext_nz * plane;
  const int own_off = c->z0 - c->ext_z0;
  if (dev) {
    ST_CUDA(c, cudaEventRecord(c->ev_in, c->cs));
    ST_CUDA(c, cudaStreamWaitEvent(c->xs, c->ev_in, 0));
  }
  const int in_off = in_z0 - c->ext_z0;
  for (int k = 0; k < 3; ++k)
    ST_CUDA(c, cudaMemcpyAsync(stage + k * comp + in_off * plane, u + k * own_cells, own_cells * sizeof(float),
                               dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->xs));
  if (pinned) {
    // pinned host input: stream-ordered like device input, overlapping the running step
    ST_CUDA(c, cudaEventRecord(c->ev_pinned_in, c->xs));
    c->pinned_in_flight = true;
  } else if (!dev) {
    // pageable host inputs are consumed before the call returns (header contract)
    ST_CUDA(c, cudaEventRecord(c->ev_in, c->xs));
    ST_CUDA(c, cudaEventSynchronize(c->ev_in));
  }
  int src_z0 = c->z0, src_nz = c->z1 - c->z0;
  if (c->shard) {   // Fig. 1c: every rank gets every owner's planes
    std::string why;
    if (comm_shard_field(c->shard, stage, comp, plane, -c->ext_z0, c->eu_zb, c->xs, why))
      return fail(c, ST_ERR_NCCL, why);
  }
  if (c->comm) {
    std::string why;
    if (comm_field_halo(c->comm, stage, comp, plane, c->ext_z0, c->ext_nz, c->z0, c->z1, g.n[2], g.bc[2], c->xs, why))
      return fail(c, ST_ERR_NCCL, why);
    src_z0 = c->ext_z0;
    src_nz = c->ext_nz;
  }
  const float* src = stage + (c->comm ? 0 : own_off * plane);
  st_status s = check_launch(c, launch_field_ingest(g, src, comp, src_z0, src_nz, c->field[back], c->xs));
  if (s) return s;
  ST_CUDA(c, cudaEventRecord(c->ev_field_ready[back], c->xs));
  ST_CUDA(c, cudaEventRecord(c->tr[c->tr_n[0] % st_ctx::kTrace][1], c->xs));
  c->tr_n[0] += 1;
  c->pending = back;
  return ST_OK;
}

// ---------------------------------------------------------------- inject
static st_status inject_local(st_ctx* c, int64_t n, const float* x, const float* u, const float* d, const float* w,
                    const uint64_t* id) {
  ST_ALIVE(c);
  if (n < 0) return fail(c, ST_ERR_INVALID_ARG, "n < 0");
  {
    st_status fr = flush_rebin(c);   // the contract sorted the store before this append
    if (fr) return fr;
  }
  if (n == 0) {
    if (c->comm) c->binned = c->hist_ready = false;   // collective: every rank leaves the binned state together
    return ST_OK;
  }
  if (!x || !u || !d) return fail(c, ST_ERR_INVALID_ARG, "x, u and d are required");
  if (c->n + n > c->cfg.capacity) return fail(c, ST_ERR_CAPACITY, "store capacity exceeded");
  Store s = c->S[c->cur];
  const int64_t o = c->n, cap = c->cap;
  auto kind = [](const void* p) { return is_device_ptr(p) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice; };
  for (int a = 0; a < 3; ++a) {
    ST_CUDA(c, cudaMemcpyAsync(s.x + a * cap + o, x + a * n, n * sizeof(float), kind(x), c->cs));
    ST_CUDA(c, cudaMemcpyAsync(s.u + a * cap + o, u + a * n, n * sizeof(float), kind(u), c->cs));
  }
  ST_CUDA(c, cudaMemcpyAsync(s.d + o, d, n * sizeof(float), kind(d), c->cs));
  int nl = 0;
  if (w) {
    ST_CUDA(c, cudaMemcpyAsync(s.w + o, w, n * sizeof(float), kind(w), c->cs));
  } else {
    nl += launch_fill_f32(s.w + o, n, 1.0f, c->cs);
  }
  if (id) {
    ST_CUDA(c, cudaMemcpyAsync(s.id + o, id, n * sizeof(uint64_t), kind(id), c->cs));
  } else {
    nl += launch_fill_u64_seq(s.id + o, n, c->next_id, c->cs);
  }
  nl += launch_check_domain(c->g, s.x + o, cap, n, c->d_err, c->cs);
  st_status st = check_launch(c, nl);
  if (st) return st;
  ST_CUDA(c, cudaStreamSynchronize(c->cs));
  st = consume_flags(c);
  if (st) return st;   // nothing appended: c->n unchanged
  if (!id) c->next_id += (uint64_t)n;
  c->n += n;
  c->binned = false;
  c->hist_ready = false;
  return ST_OK;
}

st_status st_inject(st_ctx* c, int64_t n, const float* x, const float* u, const float* d, const float* w,
                    const uint64_t* id) {
  ST_ALIVE(c);
  const int64_t n0 = c->n;
  const uint64_t id0 = c->next_id;
  st_status st = inject_local(c, n, x, u, d, w, id);
  if (!c->comm) return st;
  // collective: every rank learns whether any rank failed (else the others would run
  // into the next NCCL exchange alone and hang); ranks that appended roll back
  int flag = st != ST_OK ? 1 : 0;
  std::string why;
  ST_CUDA(c, cudaMemcpyAsync(c->d_farg, &flag, sizeof(int), cudaMemcpyHostToDevice, c->cs));
  if (comm_allreduce_max_i32(c->comm, c->d_farg, 1, c->cs, why)) return fail(c, ST_ERR_NCCL, why);
  ST_CUDA(c, cudaMemcpyAsync(&flag, c->d_farg, sizeof(int), cudaMemcpyDeviceToHost, c->cs));
  ST_CUDA(c, cudaStreamSynchronize(c->cs));
  if (flag) {   // every rank: nothing appended, leave the binned state together
    c->n = n0;
    c->next_id = id0;
    c->binned = c->hist_ready = false;
  }
  if (st != ST_OK) return st;
  if (flag) return fail(c, ST_ERR_STATE, "st_inject failed on another rank (nothing appended on any rank)");
  return ST_OK;
}

// ---------------------------------------------------------------- rebin
// C-15 / C-16.  Two implementations of the same contract:
//  * general: radix sort by the bin key (after injection, when a particle moved
//    more than one cell since its bin, and for the multi-GPU migration);
//  * neighbour scatter (k_step.cu): fused into the next advance (or standalone
//    when the store is observed first).
static StepArgs step_args(st_ctx* c, float dt, int nsteps) {
  StepArgs a;
  memset(&a, 0, sizeof(a));
  a.g = c->g;
  a.p = c->p;
  a.bg = c->bg;
  a.A = c->S[c->cur];
  a.B = c->S[1 - c->cur];
  a.tm_f = c->tmap[2 * c->cur];
  a.tm_id = c->tmap[2 * c->cur + 1];
  a.tm_f64 = c->tmap_ip[c->cur];
  a.tm_id66 = c->tmap_id66[c->cur];
  a.tm_win[0] = c->tmap_win[c->front < 0 ? 0 : c->front][0];
  a.tm_win[1] = c->tmap_win[c->front < 0 ? 0 : c->front][1];
  a.dtab = c->dtab;
  a.far_cur = c->far_cur;
  a.far_src = c->key[0];      // the radix keys are free outside the general sort: the far
  a.far_src_hi = c->key[1];   // tails' (hi, lo) sort keys
  a.cap = c->cap;
  a.n = c->n;
  a.off = c->off[c->lay];
  a.off_new = c->off[1 - c->lay];
  a.slot_base = c->hist;
  a.item_bin0 = c->items[c->lay];
  a.n_items = c->n_items[c->lay];
  a.item_ctr = c->item_ctr;
  a.nbins = c->bg.nbins;
  a.field = c->front >= 0 ? c->field[c->front] : nullptr;
  a.acc = c->acc[c->acc_cur];
  a.dt = dt;
  a.nsteps = nsteps;
  a.err = c->d_err;
  for (int k = 0; k < 2; ++k) {
    a.voff[k] = c->voff[k];
    a.sbuf[k] = c->sbuf[k];
  }
  a.scap = c->scap;
  return a;
}

static st_status general_rebin(st_ctx* c) {
  const Geom& g = c->g;
  if (!c->reb_t0) ST_CUDA(c, cudaEventRecord(c->t_reb0, c->cs));
  c->reb_t0 = false;
  int in_b = 0, nl = 0;
  st_status s;
  if (c->comm) {
    // owner segments: stable sort by global chunk, then kept ++ arrivals (C-16)
    nl = launch_keys(g, c->S[c->cur].x, c->cap, c->n, c->key[c->cur], c->cs);
    int ns = launch_stable_sort(c->S[c->cur], c->S[1 - c->cur], c->cap, c->n, c->key[c->cur], c->key[1 - c->cur],
                                c->key_bits, c->sc, &in_b, c->cs);
    if (ns < 0) return fail(c, ST_ERR_CAPACITY, "sort scratch too small");
    if ((s = check_launch(c, nl + ns))) return s;
    if (in_b) c->cur = 1 - c->cur;
    std::string why;
    int64_t n_new = 0;
    int ml = 0;
    int rc = comm_migrate(c->comm, g, c->S, &c->cur, c->key, c->cap, c->n, c->chunk_lo, c->n_local_chunks,
                          c->key_bits, c->sc, c->mig_row.data(), &n_new, &ml, c->cs, why);
    c->launches += ml;
    if (rc == 3) return fail(c, ST_ERR_CAPACITY, why);
    if (rc) return fail(c, ST_ERR_NCCL, why);
    c->last_sent = 0;
    for (int r = 0; r < c->cfg.nranks; ++r)
      if (r != c->cfg.rank) c->last_sent += c->mig_row[r];
    c->last_recv = n_new - c->mig_row[c->cfg.rank];
    c->n = n_new;
  } else {
    c->mig_row[0] = c->n;
  }
  nl = launch_bin_keys(g, c->bg, c->S[c->cur].x, c->cap, c->n, c->key[c->cur], c->d_err, c->cs);
  int ns = launch_stable_sort(c->S[c->cur], c->S[1 - c->cur], c->cap, c->n, c->key[c->cur], c->key[1 - c->cur],
                              c->key_bits, c->sc, &in_b, c->cs);
  if (ns < 0) return fail(c, ST_ERR_CAPACITY, "sort scratch too small");
  if ((s = check_launch(c, nl + ns))) return s;
  if (in_b) c->cur = 1 - c->cur;
  nl = launch_bin_offsets(c->key[c->cur], c->n, c->bg.nbins, c->off[c->lay], c->cs);
  nl += launch_items(c->off[c->lay], c->bg.nbins, g.cc, c->item_flag, c->item_pos, c->sc.partial, c->items[c->lay],
                     c->n_items[c->lay], c->cs);
  if ((s = check_launch(c, nl))) return s;
  ST_CUDA(c, cudaEventRecord(c->t_reb1, c->cs));
  c->timed_reb = true;
  c->binned = true;
  c->rebin_due = false;
  c->rebins += 1;
  c->general_rebins += 1;
  c->hist_ready = false;
  return ST_OK;
}

// Slot histogram of the current layout (k_count) before a neighbour-slot rebin.
// *far: some particle is more than one cell from its bin, so the rebin must take
// the general sort (1 rank: decided here, after the kernel; several ranks: the flag
// stays on the device and is reduced over all ranks inside scatter_rebin).
static st_status count_slots(st_ctx* c, bool* far) {
  *far = true;
  if (!c->binned) return ST_OK;
  c->counts_from_ip = c->hist_ready;
  if (c->hist_ready) {   // counted by the in-place step that made this rebin due
    c->hist_ready = false;
    ST_CUDA(c, cudaEventRecord(c->t_reb0, c->cs));
    c->reb_t0 = true;
    if (c->comm || c->far_cnt) {   // several ranks: decided on the device; 8^3 chunks on
      *far = false;                 // one rank: every far particle has a tail (no host sync)
      return ST_OK;
    }
    ST_CUDA(c, cudaEventSynchronize(c->ev_step_done));
    *far = *(volatile int*)c->h_far != 0;
    return ST_OK;
  }
  CountArgs ca;
  memset(&ca, 0, sizeof(ca));
  ca.g = c->g;
  ca.bg = c->bg;
  ca.x = c->S[c->cur].x;
  ca.cap = c->cap;
  ca.off = c->off[c->lay];
  ca.item_bin0 = c->items[c->lay];
  ca.n_items = c->n_items[c->lay];
  ca.nbins = c->bg.nbins;
  ca.hist = c->hist;
  ca.movers = c->d_movers;
  ca.far_n = c->d_far_n;
  ST_CUDA(c, cudaMemsetAsync(c->d_far_n, 0, sizeof(unsigned long long), c->cs));
  ca.far_cnt = c->far_cnt;   // NULL unless 8^3 chunks (k_pstep): then far particles stay on the fused path
  if (c->far_cnt) ST_CUDA(c, cudaMemsetAsync(c->far_cnt, 0, (size_t)c->bg.nbins * sizeof(int), c->cs));
  ST_CUDA(c, cudaEventRecord(c->t_reb0, c->cs));   // the rebin's timing starts with the count
  c->reb_t0 = true;
  ST_CUDA(c, cudaMemsetAsync(c->d_movers, 0, sizeof(unsigned long long), c->cs));
  if (c->comm) {
    ST_CUDA(c, cudaMemsetAsync(c->d_farg, 0, sizeof(int), c->cs));
    ca.far = c->d_farg;
    if (c->fv[0]) {   // k_count does not place far particles across ranks (they force the general path)
      for (int i = 0; i < 2; ++i) ST_CUDA(c, cudaMemsetAsync(c->fv[i], 0, c->nfv * sizeof(int), c->cs));
      ST_CUDA(c, cudaMemsetAsync(c->d_fs, 0, 2 * sizeof(unsigned long long), c->cs));
    }
  } else if (c->far_cnt) {
    ca.far = c->d_farg;             // never set on one rank with far tails: not read back
  } else {
    ST_CUDA(c, cudaEventSynchronize(c->ev_count));   // the previous count has read nothing since
    *c->h_far = 0;
    ca.far = c->d_far;
  }
  st_status s = check_launch(c, launch_count(ca, c->cs));
  if (s) return s;
  if (c->comm || c->far_cnt) {
    *far = false;
    return ST_OK;
  }
  ST_CUDA(c, cudaEventRecord(c->ev_count, c->cs));
  ST_CUDA(c, cudaEventSynchronize(c->ev_count));
  *far = *(volatile int*)c->h_far != 0;
  return ST_OK;
}

// Bitwise-OR-agree an error flag over all ranks (NCCL max of each bit pattern's
// disjoint flags is their OR for the small flags used here); host-blocking.
static st_status agree_flags(st_ctx* c, int* flags) {
  if (!c->comm) return ST_OK;
  std::string why;
  ST_CUDA(c, cudaMemcpyAsync(c->d_farg, flags, sizeof(int), cudaMemcpyHostToDevice, c->cs));
  if (comm_allreduce_max_i32(c->comm, c->d_farg, 1, c->cs, why)) return fail(c, ST_ERR_NCCL, why);
  ST_CUDA(c, cudaMemcpyAsync(flags, c->d_farg, sizeof(int), cudaMemcpyDeviceToHost, c->cs));
  ST_CUDA(c, cudaStreamSynchronize(c->cs));
  return ST_OK;
}

// Neighbour-slot scatter from the current layout into the other buffer; fused
// with the advance when `advance` (the field/accumulator must be set up).
// nranks > 1: the movers into the neighbour planes are scattered into send
// buffers, the counts are exchanged before the layout scan and the arrivals are
// inserted after the kernel (C-16); the "far" flag is reduced over all ranks and
// any rank's far particle makes every rank take the general path (*fell_back).
static st_status scatter_rebin(st_ctx* c, bool advance, float dt, int nsteps, bool* fell_back) {
  *fell_back = false;
  const Geom& g = c->g;
  const int nlay = 1 - c->lay;
  const int nb = c->bg.nbins, nv = c->bg.nvb;
  if (!c->reb_t0) ST_CUDA(c, cudaEventRecord(c->t_reb0, c->cs));
  c->reb_t0 = false;
  // chunk movers of the statistics: counted here when the in-place step produced the
  // counts (k_count counts them itself)
  int nl = launch_rebin_prep(g, c->bg, c->hist, c->new_cnt, c->far_cnt, c->counts_from_ip ? c->d_movers : nullptr,
                             c->cs);
  st_status s;
  if (c->comm) {
    if ((s = check_launch(c, nl))) return s;
    nl = 0;
    std::string why;
    if (comm_rebin_counts(c->comm, c->new_cnt + nb, c->new_cnt + nb + nv, c->rcnt[0], c->rcnt[1], nv, c->d_farg,
                          g.bc[2] == ST_BC_PERIODIC, c->cs, why, c->fv[0], c->fv[1], c->rfv[0], c->rfv[1], c->nfv))
      return fail(c, ST_ERR_NCCL, why);
    if (c->fv[0]) {   // far arrivals from the neighbours join the far tails of their bins
      ST_CUDA(c, cudaMemsetAsync(c->d_fs + 4, 0, 2 * sizeof(unsigned long long), c->cs));
      nl += launch_far_accept(g, c->bg, c->rfv[0], c->rfv[1], c->z0, c->z1, c->new_cnt, c->far_cnt, c->d_fs + 4,
                              c->d_err, c->cs);
    }
    nl += launch_vcombine(g, c->bg, c->new_cnt, c->rcnt[0], c->rcnt[1], c->kept[0], c->kept[1], c->z0, c->z1,
                          c->far_cnt, c->cs);
    nl += launch_exclusive_scan_u32(c->new_cnt + nb, nv, c->voff[0], c->sc.partial, c->cs);
    nl += launch_exclusive_scan_u32(c->new_cnt + nb + nv, nv, c->voff[1], c->sc.partial, c->cs);
    nl += launch_exclusive_scan_u32(c->rcnt[0], nv, c->roff[0], c->sc.partial, c->cs);
    nl += launch_exclusive_scan_u32(c->rcnt[1], nv, c->roff[1], c->sc.partial, c->cs);
    ST_CUDA(c, cudaMemcpyAsync(c->h_tot + 0, c->voff[0] + nv, sizeof(int64_t), cudaMemcpyDeviceToHost, c->cs));
    ST_CUDA(c, cudaMemcpyAsync(c->h_tot + 1, c->voff[1] + nv, sizeof(int64_t), cudaMemcpyDeviceToHost, c->cs));
    ST_CUDA(c, cudaMemcpyAsync(c->h_tot + 2, c->roff[0] + nv, sizeof(int64_t), cudaMemcpyDeviceToHost, c->cs));
    ST_CUDA(c, cudaMemcpyAsync(c->h_tot + 3, c->roff[1] + nv, sizeof(int64_t), cudaMemcpyDeviceToHost, c->cs));
    ST_CUDA(c, cudaMemcpyAsync(c->h_farg, c->d_farg, sizeof(int), cudaMemcpyDeviceToHost, c->cs));
    if (c->fv[0]) {
      // far send cursors start after the near movers of each send buffer
      for (int i = 0; i < 2; ++i)
        ST_CUDA(c, cudaMemcpyAsync(c->d_fs + 2 + i, c->voff[i] + nv, sizeof(int64_t), cudaMemcpyDeviceToDevice, c->cs));
      ST_CUDA(c, cudaMemcpyAsync(c->h_fs, c->d_fs, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, c->cs));
      ST_CUDA(c, cudaMemcpyAsync(c->h_fs + 2, c->d_fs + 4, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, c->cs));
    }
    ST_CUDA(c, cudaEventRecord(c->ev_tot, c->cs));
  }
  nl += launch_exclusive_scan_u32(c->new_cnt, nb, c->off[nlay], c->sc.partial, c->cs);
  if (c->dtab)
    nl += launch_dbase(g, c->bg, c->hist, c->off[nlay], nv > 0 ? c->voff[0] : nullptr, nv > 0 ? c->voff[1] : nullptr,
                       c->dtab, c->far_cnt, c->far_cur, c->cs);
  nl += launch_items(c->off[nlay], nb, g.cc, c->item_flag, c->item_pos, c->sc.partial, c->items[nlay], c->n_items[nlay],
                     c->cs);
  ST_CUDA(c, cudaEventRecord(c->t_reb1, c->cs));
  c->timed_reb = true;
  if ((s = check_launch(c, nl))) return s;
  int64_t n_new = c->n;
  if (c->comm) {
    ST_CUDA(c, cudaEventSynchronize(c->ev_tot));
    if (*c->h_farg) {
      *fell_back = true;
      return general_rebin(c);
    }
    const int64_t fs0 = c->fv[0] ? c->h_fs[0] : 0, fs1 = c->fv[0] ? c->h_fs[1] : 0;
    const int64_t fr0 = c->fv[0] ? c->h_fs[2] : 0, fr1 = c->fv[0] ? c->h_fs[3] : 0;
    int bad = 0;
    if (c->h_tot[0] + fs0 > c->scap || c->h_tot[1] + fs1 > c->scap || c->h_tot[2] + fr0 > c->scap ||
        c->h_tot[3] + fr1 > c->scap)
      bad |= 1;
    n_new = c->n - c->h_tot[0] - c->h_tot[1] - fs0 - fs1 + c->h_tot[2] + c->h_tot[3] + fr0 + fr1;
    if (n_new > c->cfg.capacity) bad |= 2;
    // every rank must take the same branch before the payload exchange (else the ranks
    // that did not fail would wait in ncclSend/Recv for ones that returned)
    if ((s = agree_flags(c, &bad))) return s;
    if (bad & 1) return fail(c, ST_ERR_CAPACITY, "migration buffer too small (more movers than cap/16) on some rank");
    if (bad & 2) return fail(c, ST_ERR_CAPACITY, "migration would exceed the store capacity on some rank");
  }
  StepArgs a = step_args(c, dt, nsteps);
  a.n = n_new;
  if (c->comm && c->fv[0]) {
    a.fs_cur = c->d_fs + 2;
    for (int i = 0; i < 2; ++i) {
      a.fs_key[i] = c->fs_key[i];
      a.fs_cell[i] = c->fs_cell[i];
    }
  }
  if (advance) ST_CUDA(c, cudaEventRecord(c->t_adv0, c->cs));
  if ((s = check_launch(c, launch_step(a, true, advance, c->cs)))) return s;
  if (c->comm) {
    std::string why;
    const int64_t fs0 = c->fv[0] ? c->h_fs[0] : 0, fs1 = c->fv[0] ? c->h_fs[1] : 0;
    const int64_t fr0 = c->fv[0] ? c->h_fs[2] : 0, fr1 = c->fv[0] ? c->h_fs[3] : 0;
    // near movers then far movers of each side in one payload (the far region follows)
    if (comm_rebin_payload(c->comm, c->sbuf, c->scap, c->h_tot[0] + fs0, c->h_tot[1] + fs1, c->rbuf, c->scap,
                           c->h_tot[2] + fr0, c->h_tot[3] + fr1, g.bc[2] == ST_BC_PERIODIC, c->cs, why))
      return fail(c, ST_ERR_NCCL, why);
    if (c->fv[0] && (fs0 + fs1 + fr0 + fr1) > 0 &&
        (comm_far_keys(c->comm, c->fs_key[0] + c->h_tot[0], fs0, c->fs_key[1] + c->h_tot[1], fs1, c->fr_key[0], fr0,
                       c->fr_key[1], fr1, g.bc[2] == ST_BC_PERIODIC, c->cs, why) ||
         comm_far_keys(c->comm, c->fs_cell[0] + c->h_tot[0], fs0, c->fs_cell[1] + c->h_tot[1], fs1, c->fr_cell[0], fr0,
                       c->fr_cell[1], fr1, g.bc[2] == ST_BC_PERIODIC, c->cs, why)))
      return fail(c, ST_ERR_NCCL, why);
    nl = 0;
    for (int side = 0; side < 2; ++side) {
      InsertArgs ia;
      memset(&ia, 0, sizeof(ia));
      ia.g = g;
      ia.bg = c->bg;
      ia.rbuf = c->rbuf[side];
      ia.rcap = c->scap;
      ia.count = c->h_tot[2 + side];
      ia.roff = c->roff[side];
      ia.kept = c->kept[side];
      ia.plane = side == 0 ? c->z0 : c->z1 - 1;
      ia.B = c->S[1 - c->cur];
      ia.cap = c->cap;
      ia.off_new = c->off[nlay];
      ia.nbins = nb;
      ia.err = c->d_err;
      nl += launch_insert(ia, c->cs);
    }
    if ((s = check_launch(c, nl))) return s;
    const int G = c->cfg.nranks, r = c->cfg.rank;
    const bool pz = g.bc[2] == ST_BC_PERIODIC;
    const int up = (r + 1 < G) ? r + 1 : (pz ? 0 : -1), dn = (r > 0) ? r - 1 : (pz ? G - 1 : -1);
    if (fr0 + fr1 > 0) {
      // far arrivals into the far tails: bin of the cell they were counted for, key
      // (1 + order of the source rank, sender's store index) — k_far_order_w sorts them after
      // the kept far particles, by source rank, in sender order (C-16, C-15b)
      const int64_t fr[2] = {fr0, fr1};
      const int src[2] = {dn, up};
      nl = 0;
      for (int side = 0; side < 2; ++side) {
        if (!fr[side]) continue;
        FarInsertArgs fa;
        memset(&fa, 0, sizeof(fa));
        fa.g = g;
        fa.bg = c->bg;
        Store rb = c->rbuf[side];
        const int64_t o = c->h_tot[2 + side];   // the far block follows the near arrivals
        rb.x += o; rb.u += o; rb.d += o; rb.w += o; rb.id += o;
        fa.r = rb;
        fa.rcap = c->scap;
        fa.count = fr[side];
        fa.key = c->fr_key[side];
        fa.cell = c->fr_cell[side];
        const int other = src[1 - side];
        fa.hi = 1 + ((other >= 0 && other < src[side]) ? 1 : 0);   // one source rank: both sides 1
        fa.far_cur = c->far_cur;
        fa.far_src = c->key[0];
        fa.far_src_hi = c->key[1];
        fa.B = c->S[1 - c->cur];
        fa.cap = c->cap;
        fa.err = c->d_err;
        nl += launch_far_insert(fa, c->cs);
      }
      if ((s = check_launch(c, nl))) return s;
    }
    c->mig_row.assign(c->cfg.nranks, 0);
    if (up >= 0) c->mig_row[up] += c->h_tot[1] + fs1;
    if (dn >= 0) c->mig_row[dn] += c->h_tot[0] + fs0;
    c->mig_row[r] = c->n - c->h_tot[0] - c->h_tot[1] - fs0 - fs1;
    c->last_sent = c->h_tot[0] + c->h_tot[1] + fs0 + fs1;
    c->last_recv = c->h_tot[2] + c->h_tot[3] + fr0 + fr1;
    c->n = n_new;
  } else {
    c->mig_row[0] = c->n;
  }
  // C-15b: far tails into prior store order (after the arrivals: they precede the tail)
  if ((s = check_launch(c, launch_far_order(c->bg, c->far_cnt, c->off[nlay], c->key[0], c->key[1], c->S[1 - c->cur],
                                            c->S[c->cur], c->cap, c->far_long, c->far_long_n, c->cs))))
    return s;
  if (advance) {
    ST_CUDA(c, cudaEventRecord(c->t_adv1, c->cs));
    c->timed_adv = true;
  }
  ST_CUDA(c, cudaEventRecord(c->ev_step_done, c->cs));
  c->cur = 1 - c->cur;
  c->lay = nlay;
  c->rebin_due = false;
  c->rebins += 1;
  if (advance) c->fused_rebins += 1;
  return ST_OK;
}

// Execute a due rebin before the store is observed or appended to (collective
// when nranks > 1).
static st_status flush_rebin(st_ctx* c) {
  if (!c->rebin_due) return ST_OK;
  bool far = true;
  st_status s = count_slots(c, &far);
  if (s) return s;
  if (far) return general_rebin(c);
  bool fell_back = false;
  return scatter_rebin(c, false, 0.0f, 0, &fell_back);
}

// ---------------------------------------------------------------- advance
st_status st_advance(st_ctx* c, double dt, int32_t nsteps) {
  ST_ALIVE(c);
  if (!(dt > 0.0) || nsteps < 1) return fail(c, ST_ERR_INVALID_ARG, "dt must be > 0 and nsteps >= 1");
  if (c->pending >= 0) {
    ST_CUDA(c, cudaStreamWaitEvent(c->cs, c->ev_field_ready[c->pending], 0));
    c->front = c->pending;
    c->pending = -1;
  }
  if (c->front < 0) return fail(c, ST_ERR_STATE, "st_advance before st_set_fluid_field (P:202: first step is synchronous)");
  // the accumulator must be free (its previous readout finished zeroing it)
  ST_CUDA(c, cudaStreamWaitEvent(c->cs, c->ev_acc_free[c->acc_cur], 0));
  ST_CUDA(c, cudaEventRecord(c->tr[c->tr_n[1] % st_ctx::kTrace][2], c->cs));
  st_status st = ST_OK;
  bool done = false;
  c->timed_reb = false;
  if (c->rebin_due) {
    // the rebin of the previous call (C-15), fused into this call when every
    // particle is still within one cell of its bin
    bool far = true;
    if ((st = count_slots(c, &far))) return st;
    if (!far) {
      bool fell_back = false;
      st = scatter_rebin(c, true, (float)dt, nsteps, &fell_back);
      if (st) return st;
      done = !fell_back;
    } else {
      st = general_rebin(c);
      if (st) return st;
    }
  }
  if (!done) {
    ST_CUDA(c, cudaEventRecord(c->t_adv0, c->cs));
    if (c->binned) {
      StepArgs a = step_args(c, (float)dt, nsteps);
      // this call makes a rebin due: let the in-place kernel count its bins' slots
      // (8^3 chunks: k_pstep) so the rebin needs no k_count pass
      if (c->dtab && (c->calls + 1) % c->cfg.rebin_interval == 0) {
        ST_CUDA(c, cudaMemsetAsync(c->d_movers, 0, sizeof(unsigned long long), c->cs));
        ST_CUDA(c, cudaMemsetAsync(c->d_far_n, 0, sizeof(unsigned long long), c->cs));
        ST_CUDA(c, cudaMemsetAsync(c->far_cnt, 0, (size_t)c->bg.nbins * sizeof(int), c->cs));
        if (c->comm) {
          ST_CUDA(c, cudaMemsetAsync(c->d_farg, 0, sizeof(int), c->cs));
          if (c->fv[0]) {   // far particles into a neighbour's window: counted per cell
            for (int i = 0; i < 2; ++i) {
              ST_CUDA(c, cudaMemsetAsync(c->fv[i], 0, c->nfv * sizeof(int), c->cs));
              a.cnt_fv[i] = c->fv[i];
            }
            ST_CUDA(c, cudaMemsetAsync(c->d_fs, 0, 2 * sizeof(unsigned long long), c->cs));
            a.cnt_fs_n = c->d_fs;
          }
        }
        a.cnt_far = c->d_farg;      // one rank: never set (8^3 chunks place every far particle)
        a.cnt_hist = c->hist;
        a.cnt_far_cnt = c->far_cnt;
        a.cnt_movers = c->d_movers;
        a.cnt_far_n = c->d_far_n;
        c->hist_ready = true;
      }
      st = check_launch(c, launch_step(a, false, true, c->cs));
      if (st) return st;
    } else {
      st = check_launch(c, launch_advance(c->g, c->p, c->field[c->front], c->acc[c->acc_cur], c->S[c->cur], c->cap,
                                          c->n, nullptr, 0, (float)dt, nsteps, nullptr, c->d_err, c->cs));
      if (st) return st;
    }
    ST_CUDA(c, cudaEventRecord(c->t_adv1, c->cs));
    ST_CUDA(c, cudaEventRecord(c->ev_step_done, c->cs));
    c->timed_adv = true;
  }
  ST_CUDA(c, cudaEventRecord(c->ev_field_reader[c->front], c->cs));
  ST_CUDA(c, cudaEventRecord(c->ev_acc_writer[c->acc_cur], c->cs));
  ST_CUDA(c, cudaEventRecord(c->tr[c->tr_n[1] % st_ctx::kTrace][3], c->cs));
  c->tr_n[1] += 1;
  c->T_acc[c->acc_cur] += (double)nsteps * dt;
  c->calls += 1;
  if (c->calls % c->cfg.rebin_interval == 0) {
    if (c->binned) {
      c->rebin_due = true;            // executed at the next advance / observation
    } else {
      st = general_rebin(c);          // first sort after injection: do it now
      if (st) return st;
    }
  }
  return ST_OK;
}

// ---------------------------------------------------------------- sources out
st_status st_request_sources(st_ctx* c) {
  ST_ALIVE(c);
  if (c->readout_pending) return fail(c, ST_ERR_STATE, "previous readout not yet waited for");
  const int old = c->acc_cur;
  c->acc_cur = 1 - old;
  c->readout_T = c->T_acc[old];
  c->T_acc[old] = 0.0;
  const Geom& g = c->g;
  ST_CUDA(c, cudaStreamWaitEvent(c->xo, c->ev_acc_writer[old], 0));
  ST_CUDA(c, cudaEventRecord(c->tr[c->tr_n[2] % st_ctx::kTrace][4], c->xo));
  if (c->comm) {
    std::string why;
    if (comm_source_halo(c->comm, c->acc[old], g, c->z0, c->z1, c->H, c->xo, why)) return fail(c, ST_ERR_NCCL, why);
  }
  if (c->shard) {   // particle-sharded: every rank deposited into the whole domain; each
    std::string why;  // owner receives the sum over ranks of its planes (reduce-scatter)
    if (comm_shard_sources(c->shard, c->acc[old], (int64_t)g.n[0] * g.n[1], c->eu_zb, c->xo, why))
      return fail(c, ST_ERR_NCCL, why);
  }
  const double V = c->cfg.cell_size[0] * c->cfg.cell_size[1] * c->cfg.cell_size[2];
  const float scale = c->readout_T > 0.0 ? (float)(1.0 / (V * c->readout_T)) : 0.0f;
  const int out_z0 = c->shard ? c->eu_z0 : c->z0, out_z1 = c->shard ? c->eu_z1 : c->z1;
  st_status s = check_launch(c, launch_source_readout(g, c->acc[old], out_z0, out_z1, scale, c->S_dev, c->xo));
  if (s) return s;
  ST_CUDA(c, cudaMemsetAsync(c->acc[old], 0, (size_t)g.anz * g.n[1] * g.n[0] * sizeof(float4), c->xo));
  ST_CUDA(c, cudaEventRecord(c->ev_acc_free[old], c->xo));
  ST_CUDA(c, cudaEventRecord(c->ev_readout_done, c->xo));
  c->readout_pending = true;
  return ST_OK;
}

st_status st_wait_sources(st_ctx* c, float* S, double* interval_s) {
  ST_ALIVE(c);
  if (!c->readout_pending) return fail(c, ST_ERR_STATE, "no readout requested");
  c->readout_pending = false;
  if (S) {
    const bool dev = is_device_ptr(S);
    const int64_t out_cells = c->shard ? (int64_t)c->g.n[0] * c->g.n[1] * (c->eu_z1 - c->eu_z0) : c->local_cells;
    ST_CUDA(c, cudaMemcpyAsync(S, c->S_dev, 3 * out_cells * sizeof(float),
                               dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->xo));
  }
  ST_CUDA(c, cudaEventRecord(c->tr[c->tr_n[2] % st_ctx::kTrace][5], c->xo));
  c->tr_n[2] += 1;
  if (interval_s) *interval_s = c->readout_T;
  return consume_flags(c, c->xo);   // syncs the readout stream only, not the running step
}

st_status st_get_sources(st_ctx* c, float* S, double* interval_s) {
  st_status s = st_request_sources(c);
  if (s) return s;
  return st_wait_sources(c, S, interval_s);
}

// ---------------------------------------------------------------- queries
st_status st_sync(st_ctx* c) {
  ST_ALIVE(c);
  ST_CUDA(c, cudaStreamSynchronize(c->cs));
  ST_CUDA(c, cudaStreamSynchronize(c->xs));
  ST_CUDA(c, cudaStreamSynchronize(c->xo));
  c->pinned_in_flight = false;
  return consume_flags(c);
}

st_status st_get_count(st_ctx* c, int64_t* n) {
  ST_ALIVE(c);
  if (!n) return ST_ERR_INVALID_ARG;
  if (c->comm) {
    st_status fr = flush_rebin(c);   // migration changes the local count
    if (fr) return fr;
  }
  *n = c->n;
  return ST_OK;
}

st_status st_get_particles(st_ctx* c, int64_t cap, int64_t* n_out, float* x, float* u, float* d, float* w,
                           uint64_t* id, int32_t* cell, int32_t* chunk) {
  ST_ALIVE(c);
  st_status fr = flush_rebin(c);
  if (fr) return fr;
  ST_CUDA(c, cudaStreamSynchronize(c->cs));
  st_status st = consume_flags(c);
  if (st) return st;
  if (n_out) *n_out = c->n;
  if (cap < c->n) return fail(c, ST_ERR_CAPACITY, "output capacity smaller than the store");
  const int64_t n = c->n;
  if (n == 0) return ST_OK;
  Store s = c->S[c->cur];
  auto kind = [](const void* p) { return is_device_ptr(p) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost; };
  for (int a = 0; a < 3; ++a) {
    if (x) ST_CUDA(c, cudaMemcpyAsync(x + a * cap, s.x + a * c->cap, n * sizeof(float), kind(x), c->cs));
    if (u) ST_CUDA(c, cudaMemcpyAsync(u + a * cap, s.u + a * c->cap, n * sizeof(float), kind(u), c->cs));
  }
  if (d) ST_CUDA(c, cudaMemcpyAsync(d, s.d, n * sizeof(float), kind(d), c->cs));
  if (w) ST_CUDA(c, cudaMemcpyAsync(w, s.w, n * sizeof(float), kind(w), c->cs));
  if (id) ST_CUDA(c, cudaMemcpyAsync(id, s.id, n * sizeof(uint64_t), kind(id), c->cs));
  if (cell || chunk) {
    int32_t* tmp = nullptr;
    ST_CUDA(c, cudaMallocAsync(&tmp, 2 * n * sizeof(int32_t), c->cs));
    st = check_launch(c, launch_locate(c->g, s.x, c->cap, n, tmp, tmp + n, c->cs));
    if (st) return st;
    if (cell) ST_CUDA(c, cudaMemcpyAsync(cell, tmp, n * sizeof(int32_t), kind(cell), c->cs));
    if (chunk) ST_CUDA(c, cudaMemcpyAsync(chunk, tmp + n, n * sizeof(int32_t), kind(chunk), c->cs));
    ST_CUDA(c, cudaFreeAsync(tmp, c->cs));
  }
  ST_CUDA(c, cudaStreamSynchronize(c->cs));
  return ST_OK;
}

st_status st_locate(st_ctx* c, int64_t n, const float* x, int32_t* cell, int32_t* chunk) {
  ST_ALIVE(c);
  if (n < 0 || (n > 0 && !x)) return fail(c, ST_ERR_INVALID_ARG, "bad arguments");
  if (n == 0) return ST_OK;
  float* dx = nullptr;
  int32_t* tmp = nullptr;
  const bool xdev = is_device_ptr(x);
  ST_CUDA(c, cudaMallocAsync(&tmp, 2 * n * sizeof(int32_t), c->cs));
  if (!xdev) {
    ST_CUDA(c, cudaMallocAsync(&dx, 3 * n * sizeof(float), c->cs));
    ST_CUDA(c, cudaMemcpyAsync(dx, x, 3 * n * sizeof(float), cudaMemcpyHostToDevice, c->cs));
  }
  st_status st = check_launch(c, launch_locate(c->g, xdev ? x : dx, n, n, tmp, tmp + n, c->cs));
  if (st) return st;
  auto kind = [](const void* p) { return is_device_ptr(p) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost; };
  if (cell) ST_CUDA(c, cudaMemcpyAsync(cell, tmp, n * sizeof(int32_t), kind(cell), c->cs));
  if (chunk) ST_CUDA(c, cudaMemcpyAsync(chunk, tmp + n, n * sizeof(int32_t), kind(chunk), c->cs));
  ST_CUDA(c, cudaFreeAsync(tmp, c->cs));
  if (dx) ST_CUDA(c, cudaFreeAsync(dx, c->cs));
  ST_CUDA(c, cudaStreamSynchronize(c->cs));
  return ST_OK;
}

st_status st_get_migration_counts(st_ctx* c, int64_t* row) {
  ST_ALIVE(c);
  if (!row) return ST_ERR_INVALID_ARG;
  st_status fr = flush_rebin(c);   // the contract's last rebin may still be pending
  if (fr) return fr;
  for (int r = 0; r < c->cfg.nranks; ++r) row[r] = c->mig_row[r];
  return ST_OK;
}

st_status st_get_layout(st_ctx* c, st_layout* o) {
  ST_ALIVE(c);
  if (!o) return ST_ERR_INVALID_ARG;
  o->z0 = c->z0;
  o->z1 = c->z1;
  o->kz0 = c->kz0;
  o->kz1 = c->kz1;
  o->n_chunks_global = c->g.NC[0] * c->g.NC[1] * c->g.NC[2];
  for (int a = 0; a < 3; ++a) o->nchunk[a] = c->g.NC[a];
  o->local_cells = c->local_cells;
  o->halo_cells = c->H;
  if (c->shard) {   // the Eulerian partition this rank feeds and reads (field in, sources out)
    o->z0 = c->eu_z0;
    o->z1 = c->eu_z1;
    o->kz0 = c->eu_z0 / c->g.cc;
    o->kz1 = (c->eu_z1 + c->g.cc - 1) / c->g.cc;
    o->local_cells = (int64_t)c->g.n[0] * c->g.n[1] * (c->eu_z1 - c->eu_z0);
  }
  return ST_OK;
}

st_status st_plan_partition(const st_config* cfg, const int64_t* counts, int32_t* out) {
  if (!cfg || !counts || !out) return ST_ERR_INVALID_ARG;
  st_config v = *cfg;
  v.slab_planes = nullptr;
  v.nccl_unique_id = (const void*)1;   // planning only
  std::string why;
  st_status s = validate(&v, why);
  if (s) {
    g_init_error = why;
    return s;
  }
  const int G = v.nranks, cc = v.chunk_cells, nz = v.dims[2];
  const int ncz = (nz + cc - 1) / cc;
  auto ok_slab = [&](int k0, int k1) {   // >= cc+1 cell planes (ragged top plane counted exactly)
    const int z1 = k1 * cc < nz ? k1 * cc : nz;
    return G == 1 || z1 - k0 * cc >= cc + 1;
  };
  std::vector<int64_t> pre(ncz + 1, 0);
  for (int k = 0; k < ncz; ++k) pre[k + 1] = pre[k] + (counts[k] > 0 ? counts[k] : 0);
  const int64_t INF = INT64_MAX;
  // best[g][k]: minimal largest slab count splitting planes [0, k) into g slabs
  std::vector<std::vector<int64_t>> best(G + 1, std::vector<int64_t>(ncz + 1, INF));
  std::vector<std::vector<int>> cut(G + 1, std::vector<int>(ncz + 1, -1));
  best[0][0] = 0;
  for (int gi = 1; gi <= G; ++gi)
    for (int k = 1; k <= ncz; ++k)
      for (int j = 0; j < k; ++j) {   // last slab [j, k); smallest j wins ties
        if (best[gi - 1][j] == INF || !ok_slab(j, k)) continue;
        const int64_t m = std::max(best[gi - 1][j], pre[k] - pre[j]);
        if (m < best[gi][k]) {
          best[gi][k] = m;
          cut[gi][k] = j;
        }
      }
  if (best[G][ncz] == INF) {
    g_init_error = "no split with >= chunk_cells+1 planes per rank";
    return ST_ERR_INVALID_ARG;
  }
  out[G] = ncz;
  for (int gi = G, k = ncz; gi > 0; --gi) {
    k = cut[gi][k];
    out[gi - 1] = k;
  }
  return ST_OK;
}

st_status st_plan_layout(const st_config* cfg, st_layout* o) {
  if (!cfg || !o) return ST_ERR_INVALID_ARG;
  std::string why;
  st_status s = validate(cfg, why);
  if (s) {
    g_init_error = why;
    return s;
  }
  st_ctx tmp;
  tmp.cfg = geometry_view(cfg);
  build_geometry(&tmp);
  o->z0 = tmp.z0;
  o->z1 = tmp.z1;
  o->kz0 = tmp.kz0;
  o->kz1 = tmp.kz1;
  o->n_chunks_global = tmp.g.NC[0] * tmp.g.NC[1] * tmp.g.NC[2];
  for (int a = 0; a < 3; ++a) o->nchunk[a] = tmp.g.NC[a];
  o->local_cells = tmp.local_cells;
  o->halo_cells = tmp.H;
  if (cfg->decomposition == ST_DECOMP_SHARDED) {
    std::vector<int> zb;
    eulerian_slabs(cfg, zb);
    o->z0 = zb[cfg->rank];
    o->z1 = zb[cfg->rank + 1];
    o->kz0 = o->z0 / cfg->chunk_cells;
    o->kz1 = (o->z1 + cfg->chunk_cells - 1) / cfg->chunk_cells;
    o->local_cells = (int64_t)cfg->dims[0] * cfg->dims[1] * (o->z1 - o->z0);
  }
  return ST_OK;
}

st_status st_get_stats(st_ctx* c, st_stats* o) {
  ST_ALIVE(c);
  if (!o) return ST_ERR_INVALID_ARG;
  unsigned long long mv = 0;
  ST_CUDA(c, cudaStreamSynchronize(c->cs));
  ST_CUDA(c, cudaMemcpy(&mv, c->d_movers, sizeof(mv), cudaMemcpyDeviceToHost));
  c->last_movers = (int64_t)mv;
  o->n_particles = c->n;
  o->calls = c->calls;
  o->rebins = c->rebins;
  o->last_movers = c->last_movers;
  o->last_sent_total = c->last_sent;
  o->last_recv_total = c->last_recv;
  o->fused_rebins = c->fused_rebins;
  o->kernel_launches = c->launches;
  unsigned long long fn = 0;
  ST_CUDA(c, cudaMemcpy(&fn, c->d_far_n, sizeof(fn), cudaMemcpyDeviceToHost));
  o->general_rebins = c->general_rebins;
  o->last_far = (int64_t)fn;
  return ST_OK;
}

// ---------------------------------------------------------------- rebalancing (f4)
// ST_DECOMP_SHARDED: equalise the particle counts of the ranks when the largest exceeds
// the mean by more than `tolerance` ("the partitioning would be regularly checked
// and ... particles can be exchanged between chunks").  Targets: total/G, the first
// total%G ranks one more.  Donors (above target) give their surplus from the END of
// their store — the last bins of their bin order, a spatially compact set — to the
// receivers (below target) in rank order (two-pointer water-filling, deterministic);
// receivers append in ascending donor rank.  Collective; the store is then unbinned.
st_status st_rebalance(st_ctx* c, double tolerance, int64_t* sent, int64_t* received) {
  ST_ALIVE(c);
  if (sent) *sent = 0;
  if (received) *received = 0;
  if (!(tolerance >= 0.0)) return fail(c, ST_ERR_INVALID_ARG, "tolerance must be >= 0");
  if (!c->shard) return ST_OK;   // one rank, or the slab decomposition (ownership is spatial)
  {
    st_status fr = flush_rebin(c);
    if (fr) return fr;
  }
  const int G = c->shard_nranks, r = c->shard_rank;
  std::string why;
  int64_t* d_cnt = reinterpret_cast<int64_t*>(c->sc.offs);   // scratch (>= G+1 int64)
  ST_CUDA(c, cudaMemcpyAsync(d_cnt + r, &c->n, sizeof(int64_t), cudaMemcpyHostToDevice, c->cs));
  if (comm_allgather_i64(c->shard, d_cnt, c->cs, why)) return fail(c, ST_ERR_NCCL, why);
  std::vector<int64_t> n(G);
  ST_CUDA(c, cudaMemcpyAsync(n.data(), d_cnt, G * sizeof(int64_t), cudaMemcpyDeviceToHost, c->cs));
  ST_CUDA(c, cudaStreamSynchronize(c->cs));
  int64_t tot = 0, mx = 0;
  for (int q = 0; q < G; ++q) {
    tot += n[q];
    mx = std::max(mx, n[q]);
  }
  if (tot == 0 || (double)mx <= (1.0 + tolerance) * ((double)tot / G)) return ST_OK;
  std::vector<int64_t> target(G), surplus(G);
  for (int q = 0; q < G; ++q) {
    target[q] = tot / G + (q < tot % G ? 1 : 0);
    surplus[q] = n[q] - target[q];
  }
  // water-filling plan T[src][dst]
  std::vector<std::vector<int64_t>> T(G, std::vector<int64_t>(G, 0));
  {
    int d = 0, q = 0;
    std::vector<int64_t> give(surplus);
    while (true) {
      while (d < G && give[d] <= 0) ++d;
      while (q < G && give[q] >= 0) ++q;
      if (d >= G || q >= G) break;
      const int64_t m = std::min(give[d], -give[q]);
      T[d][q] += m;
      give[d] -= m;
      give[q] += m;
    }
  }
  std::vector<int64_t> snd(G, 0), soff(G, 0), rcv(G, 0), roff(G, 0);
  int64_t out = 0, in = 0;
  for (int q = 0; q < G; ++q) out += T[r][q];
  for (int q = 0; q < G; ++q) in += T[q][r];
  if (c->n - out + in > c->cfg.capacity) why = "rebalance would exceed the store capacity";
  int bad = why.empty() ? 0 : 1;
  // every rank checks every rank's capacity the same way: agree before moving anything
  ST_CUDA(c, cudaMemcpyAsync(c->d_farg, &bad, sizeof(int), cudaMemcpyHostToDevice, c->cs));
  if (comm_allreduce_max_i32(c->shard, c->d_farg, 1, c->cs, why)) return fail(c, ST_ERR_NCCL, why);
  ST_CUDA(c, cudaMemcpyAsync(&bad, c->d_farg, sizeof(int), cudaMemcpyDeviceToHost, c->cs));
  ST_CUDA(c, cudaStreamSynchronize(c->cs));
  if (bad) return fail(c, ST_ERR_CAPACITY, why.empty() ? "rebalance would exceed the capacity of some rank" : why);
  int64_t o = c->n - out;   // the donor's tail, to destinations in ascending rank
  for (int q = 0; q < G; ++q) {
    snd[q] = T[r][q];
    soff[q] = o;
    o += T[r][q];
  }
  int64_t a = c->n - out;   // receivers append after what they keep, by ascending donor rank
  for (int q = 0; q < G; ++q) {
    rcv[q] = T[q][r];
    roff[q] = a;
    a += T[q][r];
  }
  // a rank is never both donor and receiver, so the sent tail and the appended block of
  // one rank never overlap
  if (comm_exchange_store(c->shard, c->S[c->cur], c->cap, snd, soff, rcv, roff, c->cs, why))
    return fail(c, ST_ERR_NCCL, why);
  ST_CUDA(c, cudaStreamSynchronize(c->cs));
  c->n = c->n - out + in;
  c->binned = false;
  c->hist_ready = false;
  c->rebin_due = false;
  if (sent) *sent = out;
  if (received) *received = in;
  return ST_OK;
}

st_status st_trace(st_ctx* c, int64_t k, double* t) {
  ST_ALIVE(c);
  if (!t) return fail(c, ST_ERR_INVALID_ARG, "t is NULL");
  for (int j = 0; j < 3; ++j) {   // j: 0 field copy, 1 advance, 2 readout
    t[2 * j] = t[2 * j + 1] = -1.0;
    const int64_t done = c->tr_n[j];
    if (k < 0 || k >= done || k < done - st_ctx::kTrace) continue;
    for (int e = 0; e < 2; ++e) {
      cudaEvent_t ev = c->tr[k % st_ctx::kTrace][2 * j + e];
      float ms = 0.0f;
      ST_CUDA(c, cudaEventSynchronize(ev));
      ST_CUDA(c, cudaEventElapsedTime(&ms, c->tr_ref, ev));
      t[2 * j + e] = ms;
    }
  }
  return ST_OK;
}

st_status st_last_timings(st_ctx* c, float* advance_ms, float* rebin_ms) {
  ST_ALIVE(c);
  if (advance_ms) {
    *advance_ms = 0.0f;
    if (c->timed_adv) {
      ST_CUDA(c, cudaEventSynchronize(c->t_adv1));
      ST_CUDA(c, cudaEventElapsedTime(advance_ms, c->t_adv0, c->t_adv1));
    }
  }
  if (rebin_ms) {
    *rebin_ms = 0.0f;
    if (c->timed_reb) {
      ST_CUDA(c, cudaEventSynchronize(c->t_reb1));
      ST_CUDA(c, cudaEventElapsedTime(rebin_ms, c->t_reb0, c->t_reb1));
    }
  }
  return ST_OK;
}

}  // extern "C"
