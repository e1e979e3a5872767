/*
 * scaletrack.h — C ABI of the B200-native SCALE-TRACK hot path
 * (arXiv 2603.26691, "SCALE-TRACK: Asynchronous Euler-Lagrange particle
 * tracking on heterogeneous computing architecture").
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * C-n = reading n in DESIGN.md §3 (where the paper is silent or ambiguous).
 *
 * What the library computes (one "particle step"):
 *   for every particle p and every sub-step of length dt:
 *     1. locate the cell of x_p                              (C-6)
 *     2. interpolate the fluid velocity u_f at x_p           (C-5)
 *     3. integrate Newton's law with drag (+ gravity)        (Eq. 9-10, C-1..C-4)
 *     4. deposit the drag reaction into the start cell       (Eq. 11, C-8..C-10)
 *     5. apply wall reflection / periodic wrap               (C-11, C-12)
 *     6. relocate to cell and chunk; rebin the SoA store     (C-14..C-16)
 *
 * Conventions shared by every entry point
 *   - Every call returns st_status; ST_OK == 0.  No C++ exception crosses the ABI.
 *     On error a message is kept per context (st_last_error).  CUDA errors are
 *     sticky: after ST_ERR_CUDA the context only accepts st_destroy.
 *   - Units are SI.  State is IEEE binary32 (C-19).
 *   - Array arguments are caller-owned.  Pointers may be host (pageable or
 *     pinned) or device memory of the context's GPU; the kind is detected with
 *     cudaPointerGetAttributes.  Device inputs are consumed in order on
 *     cfg.stream; host inputs are copied before the call returns, except the
 *     pinned-host field of st_set_fluid_field (see there).
 *   - Vectors are structure-of-arrays: x[3][n] means x[0..n) = x-components,
 *     x[n..2n) = y, x[2n..3n) = z.  Fields are [3][nz][ny][nx], x fastest.
 *   - Cell linear index: (cz*ny + cy)*nx + cx (global indices).
 *     Chunk id: (kz*NCy + ky)*NCx + kx with k_d = c_d / chunk_cells,
 *     NC_d = ceil(n_d / chunk_cells)                          (C-14)
 *   - Threading: one context per (process, GPU); calls on one context must
 *     not be concurrent.
 *   - Multi-GPU (nranks > 1): one process per GPU; rank r owns the z-slab of
 *     chunk planes [floor(r*NCz/G), floor((r+1)*NCz/G)) (C-16).  Calls marked
 *     "collective" must be made by every rank in the same order.
 */
#ifndef SCALETRACK_H
#define SCALETRACK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ST_ABI_VERSION 3   /* 3: st_micro_config.arithmetic */

typedef struct st_ctx st_ctx;   /* opaque; owns the particle store, fields, sources */
typedef int32_t st_status;

enum {
  ST_OK = 0,
  ST_ERR_INVALID_ARG = 1,   /* bad pointer / size / config value ("contract violation") */
  ST_ERR_STATE = 2,         /* call out of order (e.g. st_advance before any field) */
  ST_ERR_CAPACITY = 3,      /* store capacity exceeded */
  ST_ERR_OUT_OF_DOMAIN = 4, /* injected particle outside [lo, hi] (S:60 outside-marker) */
  ST_ERR_CFL = 5,           /* displacement precondition violated ("never silent") */
  ST_ERR_CUDA = 6,          /* CUDA runtime error (sticky) */
  ST_ERR_NCCL = 7,          /* NCCL error */
  ST_ERR_OOM = 8,           /* device allocation failed */
  ST_ERR_UNSUPPORTED = 9    /* feature not built / not available on this device */
};

enum { ST_BC_PERIODIC = 0, ST_BC_REFLECT = 1 };                 /* C-11, C-12 */
enum { ST_DRAG_STOKES = 0, ST_DRAG_SCHILLER_NAUMANN = 1 };      /* C-2 */
enum { ST_INT_EXPONENTIAL = 0, ST_INT_SEMI_IMPLICIT = 1 };      /* C-4 */
enum { ST_ONE_WAY = 0, ST_TWO_WAY = 1 };

/*
 * Configuration.  Fill with st_config_default() and override.
 *   dims, origin, cell_size : uniform Cartesian cell-centred mesh.
 *   chunk_cells             : edge of a cubic chunk in cells (8 -> 8^3-cell chunks, C-14).
 *   bc[3]                   : ST_BC_* per axis (both faces of an axis share the rule).
 *   rho_f, nu_f, rho_p      : fluid density, kinematic viscosity, particle density.
 *   gravity[3]              : body acceleration on particles (C-1; (0,0,0) = paper's
 *                             "only the drag force").
 *   drag_law, integrator, coupling : ST_DRAG_*, ST_INT_*, ST_ONE_WAY/ST_TWO_WAY.
 *   rebin_interval (K >= 1) : the store is stable-sorted by chunk after the last
 *                             sub-step of every K-th st_advance call (C-15).
 *   capacity                : maximum particles resident on this rank (<= 2^31 - 65: the step
 *                             kernels index the store with 32-bit TMA coordinates).
 *   device                  : CUDA ordinal; stream: cudaStream_t (NULL = the library creates a
 *                             BLOCKING stream of its own, ordered with the legacy default stream).
 *   rank, nranks            : position in the one-box job (nranks == 1: single GPU).
 *   nccl_unique_id          : 128-byte ncclUniqueId broadcast by the caller (nranks > 1).
 *   decomposition           : ST_DECOMP_SLAB (default): z-slabs of chunk planes, particles
 *                             migrate to the rank owning their chunk (north star).
 *                             ST_DECOMP_SHARDED: the paper's own scheme (Fig. 1c, P:181-185;
 *                             SURVEY §8(f2)): every rank holds the whole domain and the whole
 *                             fluid field, particles stay on the rank that injected them (no
 *                             migration), st_get_sources returns the sources of the whole
 *                             domain summed over all ranks (one NCCL all-reduce, collective).
 *   slab_planes             : ST_DECOMP_SLAB only: NULL = equal split of the chunk planes;
 *                             else nranks+1 ascending chunk-plane boundaries (slab of rank r =
 *                             planes [slab_planes[r], slab_planes[r+1]), [0] = 0, [nranks] =
 *                             ceil(dims[2]/chunk_cells)), e.g. from st_plan_partition: the
 *                             count-balanced owner ranges of SURVEY §8(f4)
 *                             along z.  Read during st_init only.
 */
typedef struct {
  int32_t abi_version;
  int32_t dims[3];
  double origin[3];
  double cell_size[3];
  int32_t chunk_cells;
  int32_t bc[3];
  double rho_f, nu_f, rho_p;
  double gravity[3];
  int32_t drag_law, integrator, coupling;
  int32_t rebin_interval;
  int64_t capacity;
  int32_t device;
  void* stream;
  int32_t rank, nranks;
  const void* nccl_unique_id;
  int32_t decomposition;
  const int32_t* slab_planes;
} st_config;

enum { ST_DECOMP_SLAB = 0, ST_DECOMP_SHARDED = 1 };

/* Geometry of this rank's share of the mesh (filled by st_get_layout). */
typedef struct {
  int32_t z0, z1;            /* owned cell planes [z0, z1) (global z index)          */
  int32_t kz0, kz1;          /* owned chunk planes [kz0, kz1)                         */
  int32_t n_chunks_global;   /* NCx*NCy*NCz                                           */
  int32_t nchunk[3];         /* NCx, NCy, NCz                                         */
  int64_t local_cells;       /* nx*ny*(z1-z0): size of one component of st_get_sources */
  int32_t halo_cells;        /* z-halo planes kept on each side (0 when nranks == 1)   */
} st_layout;

/* Counters of the last rebin and running totals (filled by st_get_stats). */
typedef struct {
  int64_t n_particles;       /* resident on this rank                                 */
  int64_t calls;             /* st_advance calls so far                               */
  int64_t rebins;            /* rebins performed                                      */
  int64_t last_movers;       /* particles that changed chunk in the last rebin        */
  int64_t last_sent_total;   /* particles sent to other ranks in the last rebin       */
  int64_t last_recv_total;   /* particles received in the last rebin                  */
  int64_t fused_rebins;      /* rebins fused into the advance kernel                  */
  int64_t kernel_launches;   /* kernels launched by the library so far                */
  int64_t general_rebins;    /* rebins that took the general radix sort               */
  int64_t last_far;          /* particles > 1 cell from their bin placed in bin tails
                                by the last neighbour-slot rebin (C-15b)              */
} st_stats;

/* Fill *cfg with defaults: 1 GPU, 16^3 unit box, periodic, chunk 8, air/water
 * properties (rho_f 1.2, nu_f 1.5e-5, rho_p 1000), no gravity, Schiller-Naumann,
 * exponential integrator, two-way, K = 1, capacity 1e6, device 0, NULL stream. */
void st_config_default(st_config* cfg);

/* Validate cfg, allocate the store (2 x capacity x 40 B), fields and source
 * buffers, create streams/events; nranks > 1: ncclCommInitRank (collective).
 * *out receives the context; on failure *out is NULL and the status says why. */
st_status st_init(const st_config* cfg, st_ctx** out);

/* Free everything.  NULL is accepted. */
st_status st_destroy(st_ctx* ctx);

/* Fluid state in ("receive the required states").  u = [3][z1-z0][ny][nx]
 * fp32 cell-centre velocities of the cells this rank owns.  Asynchronous: the
 * copy goes into the back buffer on the copy stream (it waits for the last
 * st_advance still reading that buffer); the next st_advance uses it.  The copy
 * stream is not shared with the source readout (st_request_sources), so a field
 * copy never waits behind a readout that waits for the running step (P:198-202,
 * field in and sources out overlap the Lagrangian step).  Pageable host u
 * is consumed before the call returns; PINNED host u (cudaHostAlloc) is copied
 * asynchronously and must stay unchanged until the next st_set_fluid_field or
 * st_sync returns (that call waits for the copy).  With nranks > 1 the halo planes
 * are exchanged with the neighbour ranks (collective). */
st_status st_set_fluid_field(st_ctx* ctx, const float* u);

/* Append n particles in the given order ("particles are created directly
 * on the GPUs").  x,u: [3][n]; d: [n] diameters (> 0); w: [n] parcel
 * multiplicity or NULL = 1; id: [n] or NULL = auto ((rank<<40)+counter).
 * Positions must satisfy lo <= x <= hi per axis, else ST_ERR_OUT_OF_DOMAIN and
 * nothing is appended.  With nranks > 1 the call is collective (every rank calls
 * it, n may be 0) and a rank injects only particles whose cell lies in its own
 * z-slab (st_get_layout z0..z1), else ST_ERR_OUT_OF_DOMAIN; the outcome is agreed
 * over ranks: if any rank fails, nothing is appended on any rank and the others
 * return ST_ERR_STATE (no rank is left alone in the next exchange).  st_get_particles
 * and st_get_count are collective too when nranks > 1 (they may execute a due
 * rebin, which exchanges movers). */
st_status st_inject(st_ctx* ctx, int64_t n, const float* x, const float* u,
                    const float* d, const float* w, const uint64_t* id);

/* Advance every particle by nsteps sub-steps of length dt (a fixed number
 * of sub-steps, interpolated values refreshed once per sub-step), depositing
 * two-way momentum sources.  Asynchronous (enqueued on the compute stream).
 * Rebin/migration per C-15/C-16 (collective when nranks > 1). */
st_status st_advance(st_ctx* ctx, double dt, int32_t nsteps);

/* Momentum source out ("send ... the calculated sources"; Eq. 11).
 * Closes the current accumulation interval (every st_advance enqueued so far)
 * and writes S = acc / (V_cell * T_acc), the time-averaged fluid-side rate in
 * N/m^3 (C-8, C-13), for the cells this rank owns ([3][z1-z0][ny][nx]), after
 * adding halo deposits received from the neighbour ranks (collective).
 * *interval_s (may be NULL) receives T_acc.  Blocks until S is written.
 * st_get_sources == st_request_sources + st_wait_sources. */
st_status st_get_sources(st_ctx* ctx, float* S, double* interval_s);

/* Split form (asynchronous coupling buffer): request closes
 * the interval and swaps the accumulation buffer, so st_advance calls made
 * after it deposit into the other buffer while the readout runs on the copy
 * stream; wait blocks until the readout is done and copies it into S. */
st_status st_request_sources(st_ctx* ctx);
st_status st_wait_sources(st_ctx* ctx, float* S, double* interval_s);

/* Number of particles resident on this rank (after any pending rebin). */
st_status st_get_count(st_ctx* ctx, int64_t* n);

/* Copy out the store in store order (blocking).  Any output pointer may be
 * NULL.  x,u: [3][cap] (component stride = cap); cell: global linear cell of
 * x (C-6); chunk: chunk id.  *n_out receives the count; ST_ERR_CAPACITY if
 * cap is too small (nothing copied). */
st_status st_get_particles(st_ctx* ctx, int64_t cap, int64_t* n_out,
                           float* x, float* u, float* d, float* w, uint64_t* id,
                           int32_t* cell, int32_t* chunk);

/* Locate n positions x[3][n] (host or device) with the kernel the store uses:
 * cell and chunk per C-6 / C-14.  Used to check the integer contract. */
st_status st_locate(st_ctx* ctx, int64_t n, const float* x, int32_t* cell, int32_t* chunk);

/* Migration counts of the last rebin: row[dst] = particles this rank sent to dst
 * (row[rank] = particles kept).  row has nranks entries.  Executes a due rebin
 * first (collective when nranks > 1). */
st_status st_get_migration_counts(st_ctx* ctx, int64_t* row);

st_status st_get_layout(st_ctx* ctx, st_layout* out);

/* Host-only: validate cfg and compute the layout of cfg->rank without touching
 * a GPU (the same slab rule st_init uses, C-16).  ST_ERR_INVALID_ARG on a bad cfg. */
st_status st_plan_layout(const st_config* cfg, st_layout* out);
st_status st_get_stats(st_ctx* ctx, st_stats* out);

/* Block until all work enqueued by this context has finished. */
st_status st_sync(st_ctx* ctx);

/* Time the most recent st_advance's kernels, in milliseconds, measured with
 * CUDA events on the stream they were launched on (blocks on those events).
 * advance_ms: the advance (+ fused rebin) kernel; rebin_ms: standalone rebin. */
st_status st_last_timings(st_ctx* ctx, float* advance_ms, float* rebin_ms);

/* Timeline of the asynchronous coupling buffer (SURVEY §8(d6) asks
 * for copy/compute overlap evidence).  The library records CUDA events on its streams
 * for every call; t[6] receives, in ms since the context was created, the begin and end
 * of the k-th field copy (st_set_fluid_field, copy-in stream), of the k-th st_advance
 * (compute stream) and of the k-th source readout (st_request_sources .. its copy out
 * in st_wait_sources, readout stream), counted from 0 since st_init; -1 where that
 * call has not happened or is older than the last 64.  Blocks on those events only,
 * so it can be read after a run without disturbing it. */
st_status st_trace(st_ctx* ctx, int64_t k, double* t);

/* Rebalance the particle counts of the ranks (ST_DECOMP_SHARDED; P:356
 * "the partitioning would be regularly checked and ... particles can be exchanged
 * between chunks").  Collective.  If the largest count exceeds the mean by more than
 * tolerance (relative), every rank ends with total/G particles (the first total%G ranks
 * one more): ranks above target send their surplus — the END of their store, i.e. the
 * last bins of their bin order, a compact set — to ranks below target in rank order
 * (water-filling), receivers append in ascending sender rank.  Afterwards the store
 * is unbinned (the next rebin is the plain stable sort, C-15b).  *sent / *received:
 * particles this rank gave / took.  No-op (ST_OK) for one rank or the slab
 * decomposition, whose ownership is spatial (use st_plan_partition there).
 * ST_ERR_CAPACITY on every rank, nothing moved, if any rank would overflow. */
st_status st_rebalance(st_ctx* ctx, double tolerance, int64_t* sent, int64_t* received);

/* Message of the last error on ctx ("" if none).  NULL ctx: last init error. */
const char* st_last_error(const st_ctx* ctx);

/* Count-balanced slab boundaries (the paper balances owner ranges by
 * particle count): given plane_counts[k] = particles in chunk plane k
 * (k < ceil(dims[2]/chunk_cells)), write the cfg->nranks+1 boundaries minimising the
 * largest slab count, every slab holding >= chunk_cells+1 cell planes (the halo the
 * neighbour needs); ties -> the lexicographically smallest boundaries.  Host-only.
 * ST_ERR_INVALID_ARG if cfg is invalid or no feasible split exists. */
st_status st_plan_partition(const st_config* cfg, const int64_t* plane_counts, int32_t* slab_planes);

/* 3-D Hilbert index of n cells ("initialization procedure using a
 * Hilbert space-filling curve"): xyz = [n][3] integer coordinates in
 * [0, 2^order), order 1..21; out[n] in [0, 8^order), a bijection along which
 * consecutive indices are face-adjacent cells (Skilling's transpose algorithm).
 * ST_ERR_INVALID_ARG for a coordinate out of range.  Host-only. */
st_status st_hilbert_index(int32_t order, int64_t n, const int32_t* xyz, uint64_t* out);

/* Count-balanced Hilbert partition of the chunks (SPEC
 * S:252-258 initialize_chunks): chunks ordered along the 3-D Hilbert curve of their
 * chunk coordinates are split into cfg->nranks contiguous, non-empty ranges minimising
 * the largest sum of chunk_counts (counts per global chunk id, chunk ids as in the
 * header conventions); owner[chunk] receives the rank.  With ST_DECOMP_SHARDED a rank
 * that injects the particles of the chunks it owns holds a compact, balanced share
 * (the bounding box of its particles covers few Eulerian partitions).  Host-only. */
st_status st_plan_hilbert(const st_config* cfg, const int64_t* chunk_counts, int32_t* owner);

/* ABI version the library was built with (== ST_ABI_VERSION). */
int32_t st_abi_version(void);

/* Write a fresh 128-byte ncclUniqueId into out (rank 0 calls it and broadcasts
 * the bytes to the other ranks before st_init).  ST_ERR_NCCL on failure. */
st_status st_nccl_unique_id(void* out);

/* ---------------------------------------------------------------------------------
 * Extrapolator-corrector for the asynchronously coupled Eulerian solve (SURVEY
 * §8(f1); §2.4 "Extrapolator-corrector method", Eq. 14-16).
 *
 * When the Eulerian step n starts before the true Lagrangian sources of the previous
 * step(s) are available, it uses the estimate
 *     S^n_est = ΔS^n_corr + dt_ratio · S^n_ext                         (Eq. 15)
 *     ΔS^n_corr = Σ_{newly received steps m} (S^m − S^m_est)          (Eq. 14 + P:228)
 *     S^n_ext = 0 | S^{n-1} | 2 S^{n-1} − S^{n-2}   (zero / constant / linear, Eq. 16)
 * with S^{n-1}, S^{n-2} the last two true sources received.  S^m_est is the estimate of
 * step m's own source: what step m emitted beyond its correction (C-25), so
 * the sequence is conservative: Σ emitted − Σ received = Σ estimates still pending.
 * Cell-wise over a whole field of n values (e.g. the 3 × cells of st_get_sources);
 * fp64 state on the device, fp32 emitted values.  Test oracle: oracle/extrapolator.py.
 * ------------------------------------------------------------------------------- */
typedef struct st_ec st_ec;
enum { ST_EC_ZERO = 0, ST_EC_CONSTANT = 1, ST_EC_LINEAR = 2 };

typedef struct {
  int32_t abi_version;   /* ST_ABI_VERSION */
  int32_t mode;          /* ST_EC_ZERO | ST_EC_CONSTANT | ST_EC_LINEAR */
  int64_t n;             /* values per source field, >= 1 */
  int32_t max_backlog;   /* steps whose truth may be outstanding, 1..64 */
  int32_t device;        /* CUDA device ordinal */
  void* stream;          /* cudaStream_t to run on, or NULL for a private stream */
} st_ec_config;

/* Create / destroy.  ST_ERR_INVALID_ARG on a bad config, ST_ERR_CUDA / ST_ERR_OOM on
 * device failures (message via st_ec_last_error(NULL)). */
st_status st_ec_init(const st_ec_config* cfg, st_ec** out);
st_status st_ec_destroy(st_ec* ec);

/* One Eulerian step.  received: k true source fields, oldest first, k*n floats
 * (host or device memory, caller-owned, read before return for host pointers; may be
 * NULL iff k == 0); they are the truths of the k oldest steps still pending.
 * dt_ratio > 0 scales the extrapolated term (C-27; 1 for rates or constant steps).
 * est: n floats (host or device) receive S^n_est.  Blocking: on return est is final.
 * Errors: ST_ERR_INVALID_ARG (k < 0, dt_ratio <= 0, NULL pointers),
 * ST_ERR_STATE (k > pending steps: a truth for a step never estimated — the protocol
 * violation; or the backlog would exceed max_backlog), ST_ERR_CUDA. */
st_status st_ec_step(st_ec* ec, int32_t k, const float* received, double dt_ratio, float* est);

/* Conservation ledger, fp64: per value (each array n doubles, host, NULL to skip)
 * Σ received truths, Σ emitted estimates, Σ estimates still pending; totals[3] (host,
 * NULL to skip) = the same three summed over the n values. */
st_status st_ec_ledger(st_ec* ec, double* cum_true, double* cum_est, double* pending, double* totals);

/* Number of emitted steps whose truth has not been received. */
st_status st_ec_backlog(st_ec* ec, int32_t* steps);

/* Message of the last error on ec ("" if none); NULL ec: last init error. */
const char* st_ec_last_error(const st_ec* ec);


/* ---------------------------------------------------------------------------------
 * Droplet microphysics step (§2.3 Eq. 7, 8, 9-11, 12, 13,
 * P:138-167; closures SPEC S:143-200; readings C-28..C-33 in DESIGN.md §3).
 *
 * For every droplet and each of nsteps sub-steps of length dt, field frozen (C-7):
 *   interpolate (u_f, T_f, rho_v) trilinearly at x (C-5); semi-implicit Euler drag
 *   (Schiller-Naumann or Stokes, + gravity); dm/dt = 2 pi D_v d rho_sat(T_f)
 *   (rho_v/rho_sat - S_v,p) (Eq. 7, Magnus rho_sat C-30); m' = max(m + dt dm/dt, 0.01 m)
 *   (C-32); T' = T + dt [pi Nu kappa d (T_f - T) - L dm/dt] / (m C_p) (Eq. 12, literal
 *   sign C-31); d' = (6 m'/(pi rho_p))^(1/3); into the cell of the start position add
 *   acc_u -= w (m'u' - m u - m g dt), acc_rv -= w (m' - m), acc_e -= w C_p (m'T' - m T)
 *   (Eq. 8, 11, 13; C-8, C-33); reflect / wrap at the walls (C-11, C-12).
 * State fp32, accumulators fp64; arithmetic fp64 by default (C-28) or fp32 when
 * cfg->arithmetic == ST_ARITH_FP32 (reading C-36: the same operations in the same order,
 * each rounded to binary32; each droplet's deposit is still added in fp64).  Test
 * oracle: oracle/microphysics.py (micro_advance(..., arith=np.float64 | np.float32)).
 * ------------------------------------------------------------------------------- */
typedef struct {
  int32_t abi_version;   /* ST_ABI_VERSION */
  int32_t dims[3];       /* cells (nx, ny, nz), each >= 1 */
  double origin[3];      /* m */
  double cell_size[3];   /* m, > 0 */
  int32_t bc[3];         /* ST_BC_PERIODIC | ST_BC_REFLECT per axis */
  double rho_f, nu_f, rho_p;
  double gravity[3];     /* m/s^2 */
  int32_t drag_law;      /* ST_DRAG_STOKES | ST_DRAG_SCHILLER_NAUMANN */
  double D_v;            /* vapour diffusivity, m^2/s */
  double kappa_f;        /* fluid conductivity, W/(m K) */
  double cp_p;           /* droplet specific heat, J/(kg K) */
  double latent;         /* latent heat, J/kg */
  double nusselt;        /* Nu_p */
  double s_vp;           /* surface saturation S_v,p */
  int32_t device;        /* CUDA device ordinal */
  void* stream;          /* cudaStream_t, NULL = the legacy default stream */
  int32_t arithmetic;    /* ST_ARITH_FP64 (default, C-28) | ST_ARITH_FP32 (C-36) */
} st_micro_config;

enum { ST_ARITH_FP64 = 0, ST_ARITH_FP32 = 1 };

/* Fill *cfg with the DESIGN.md C-30 constants (air / water, 1 m cells, reflecting). */
void st_micro_config_default(st_micro_config* cfg);

/* nsteps sub-steps of dt for n droplets.  Arrays are caller-owned, all DEVICE pointers
 * or all HOST pointers (host arrays are staged through device memory and the updated
 * ones copied back before the call returns):
 *   x, u: [3][n] fp32 (updated in place); d, T: [n] fp32 (updated); w: [n] fp32 weights;
 *   F: [5][nz][ny][nx] fp32 cell-centred (u_x, u_y, u_z, T_f, rho_v);
 *   acc: [5][nz][ny][nx] fp64 fluid-side accumulators (kg m/s x3, kg, J), ADDED to.
 * n_clamped (host, NULL to skip) receives the number of mass-floor clamps (C-32).
 * Runs on cfg->stream and blocks until done.  n == 0 is a no-op.
 * Errors: ST_ERR_INVALID_ARG (bad cfg, n < 0, nsteps < 0, dt <= 0, NULL arrays with
 * n > 0, a mix of host and device pointers), ST_ERR_CFL (a droplet still outside after one reflection /
 * wrap: the state is updated, the result is not trustworthy), ST_ERR_CUDA. */
st_status st_micro_advance(const st_micro_config* cfg, int64_t n, float* x, float* u, float* d, float* T,
                           const float* w, const float* F, double dt, int32_t nsteps, double* acc,
                           int64_t* n_clamped);

#ifdef __cplusplus
}
#endif
#endif /* SCALETRACK_H */
