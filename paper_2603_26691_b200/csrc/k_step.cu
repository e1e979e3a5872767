// KB2 + KB3 (fused form) — the binned particle step.
//
// Layout (C-15): the store is stable-sorted by the bin key
//   bin = local_chunk * cc^3 + ((lz*cc + ly)*cc + lx)
// (chunk-major, cells of a chunk in row-major order).  Between rebins every
// particle stays within one cell of its bin's cell per axis, so a rebin is a
// *neighbour-slot* stable counting sort: each particle of source bin s lands in
// one of the 27 neighbour bins d = s + delta(j).  Its destination is
//   dest = off_new[d] + base[j][s] + (# earlier particles of s with slot j)
// where base[j][s] = sum of cnt[j'][s'] over the sources s' < s of d (the
// stable order keeps source bins in ascending order, then the old order).
// cnt[j][s] (slot-major, coalesced in the prep) is counted by the previous step.
//
// One warp owns one "item" (<= kMaxBins consecutive bins); the kernel is
// persistent (grid-stride over items) and, per particle:
//   [SCATTER] slot j of the current cell w.r.t. the bin, rank by __match_any_sync,
//   [ADVANCE] locate -> trilinear u_f (L1-broadcast float4 loads) -> drag + gravity
//             exponential update -> deposit: lanes with equal cells are reduced with
//             a masked butterfly and one red.global.add.v4.f32 per group,
//   [HIST]    slot of the end position w.r.t. the output bin, one atomicAdd per
//             (bin, slot) group (input of the next rebin),
//   then writes the particle to B[dest] (scatter) or back in place.
// The kernel is specialised at compile time on the periodic-axis mask (BCM) and
// on log2(chunk_cells) (SH) so the hot loop carries no per-particle branches on
// the configuration; BCM = -1 / SH = 0 are the generic (runtime) fallbacks.
// Particle input is staged per warp with TMA bulk copies (cp.async.bulk +
// mbarrier, kStages batches ahead), so the DRAM stream is exact 16-byte aligned
// segments and never pollutes L1; in-place results use evict-first stores.
#include <cuda_runtime.h>
#include <stdlib.h>

#include "st_device.cuh"
#include "st_step.h"

namespace st {

namespace {

constexpr int kSlots = 27;
constexpr int kStay = 13;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void red_add_v4(float4* addr, float a, float b, float c) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(0.0f)
               : "memory");
}

// ---------------------------------------------------------------- TMA bulk-copy pipeline
// Each warp prefetches the SoA segments of its next kStages batches of 32
// particles into shared memory with cp.async.bulk (the Blackwell bulk-copy
// engine, SASS UBLKCP); completion is tracked by one mbarrier per stage.
constexpr int kStages = 3;
constexpr int kSeg = 36;   // floats per staged segment: 32 + 16-byte alignment slack
struct alignas(16) Stage {
  float f[8][kSeg];                 // x0 x1 x2 u0 u1 u2 d w
  unsigned long long id[kSeg / 2 + 16];  // 34 used (32 + alignment slack)
};

__host__ __device__ constexpr int warp_smem_bytes(bool scatter) {
  return (int)((kStages * sizeof(Stage) + kStages * 8 + (kMaxBins + 1) * 4 + kMaxBins * 12 +
                (scatter ? kMaxBins * kSlots * 4 : 0) + 15) / 16 * 16);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// Stage the batch starting at store index i0 (lane 0 only).  Segments are copied
// from the 16-byte aligned index below i0; `lim` bounds the copy (<= capacity).
__device__ __forceinline__ void stage_issue(Stage* stg, unsigned long long* bar, const Store& A, int64_t cap, int64_t i0,
                                            int64_t lim, bool with_id) {
  const int64_t f0 = i0 & ~(int64_t)3;
  int64_t f1 = (i0 + 32 + 3) & ~(int64_t)3;
  if (f1 > lim) f1 = lim;
  const uint32_t fb = (uint32_t)(f1 - f0) * 4u;
  uint32_t total = 8u * fb;
  int64_t q0 = 0, q1 = 0;
  if (with_id) {
    q0 = i0 & ~(int64_t)1;
    q1 = (i0 + 32 + 1) & ~(int64_t)1;
    if (q1 > lim) q1 = lim;
    total += (uint32_t)(q1 - q0) * 8u;
  }
  mbar_expect_tx(bar, total);
  const float* src[8] = {A.x, A.x + cap, A.x + 2 * cap, A.u, A.u + cap, A.u + 2 * cap, A.d, A.w};
#pragma unroll
  for (int k = 0; k < 8; ++k) bulk_g2s(stg->f[k], src[k] + f0, fb, bar);
  if (with_id) bulk_g2s(stg->id, A.id + q0, (uint32_t)(q1 - q0) * 8u, bar);
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// ---------------------------------------------------------------- configuration helpers
template <int BCM>
__device__ __forceinline__ bool periodic(const Geom& g, int ax) {
  if (BCM < 0) return g.bc[ax] == ST_BC_PERIODIC;
  return (BCM >> ax) & 1;
}
template <int SH>
__device__ __forceinline__ int dcc(int v, int cc) {
  if (SH > 0) return v >> SH;
  return v / cc;
}

// ---------------------------------------------------------------- bin geometry
template <int SH>
__device__ __forceinline__ int bin_of_cell(const Geom& g, const BinGeom& b, int cx, int cy, int cz) {
  const int cc = SH > 0 ? (1 << SH) : g.cc;
  const int kx = dcc<SH>(cx, cc), ky = dcc<SH>(cy, cc), kz = dcc<SH>(cz, cc);
  const int chunk = ((kz - b.kz0) * g.NC[1] + ky) * g.NC[0] + kx;
  const int lc = ((cz - kz * cc) * cc + (cy - ky * cc)) * cc + (cx - kx * cc);
  return chunk * b.cc3 + lc;
}

// virtual bin of a cell (x,y) of a neighbour plane: the receiver's bin order
template <int SH>
__device__ __forceinline__ int vbin_of_cell(const Geom& g, int cx, int cy, int cc) {
  const int kx = dcc<SH>(cx, cc), ky = dcc<SH>(cy, cc);
  return ((ky * g.NC[0] + kx) * cc + (cy - ky * cc)) * cc + (cx - kx * cc);
}
__device__ __forceinline__ void cell_of_vbin(const Geom& g, int v, int& cx, int& cy) {
  const int cc = g.cc;
  const int lx = v % cc, ly = (v / cc) % cc;
  const int kk = v / (cc * cc);
  cx = (kk % g.NC[0]) * cc + lx;
  cy = (kk / g.NC[0]) * cc + ly;
}

// (amortised: once per bin per item / per prep thread)
__device__ __forceinline__ void cell_of_bin(const Geom& g, const BinGeom& b, int bin, int& cx, int& cy, int& cz) {
  const int cc = g.cc;
  const int chunk = bin / b.cc3;
  const int lc = bin - chunk * b.cc3;
  const int kx = chunk % g.NC[0];
  const int ky = (chunk / g.NC[0]) % g.NC[1];
  const int kz = chunk / (g.NC[0] * g.NC[1]) + b.kz0;
  cx = kx * cc + lc % cc;
  cy = ky * cc + (lc / cc) % cc;
  cz = kz * cc + lc / (cc * cc);
}

// canonical per-axis delta from -> to in {-1,0,1}; 2 = not a neighbour
template <int BCM>
__device__ __forceinline__ int axis_delta(const Geom& g, int ax, int from, int to) {
  int d = to - from;
  if (periodic<BCM>(g, ax)) {
    const int n = g.n[ax];
    if (n >= 3) {
      d = (d == n - 1) ? -1 : d;
      d = (d == -(n - 1)) ? 1 : d;
    }
  }
  return ((unsigned)(d + 1) <= 2u) ? d : 2;
}

template <int BCM>
__device__ __forceinline__ int slot_of(const Geom& g, int sx, int sy, int sz, int cx, int cy, int cz) {
  const int dx = axis_delta<BCM>(g, 0, sx, cx);
  const int dy = axis_delta<BCM>(g, 1, sy, cy);
  const int dz = axis_delta<BCM>(g, 2, sz, cz);
  const int j = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
  return (dx == 2 || dy == 2 || dz == 2) ? -1 : j;
}

__device__ __forceinline__ int axis_step(int from, int d, int n, int bc, bool& ok) {
  int t = from + d;
  if (bc == ST_BC_PERIODIC) {
    if (t < 0) t += n;
    else if (t >= n) t -= n;
  } else if (t < 0 || t >= n) {
    ok = false;
  }
  return t;
}

// A cell plane beyond this rank's slab within chunk_cells planes (a neighbour's window):
// side 0 = below z0 (p planes below), side 1 = at / above z1 (p planes above); periodic z
// wraps.  false: not within reach (the displacement precondition C-23 is violated).
__device__ __forceinline__ bool far_plane(const Geom& g, int z, int& side, int& p) {
  const int nz = g.n[2];
  int below = g.oz0 - 1 - z, above = z - g.oz1;
  if (g.bc[2] == ST_BC_PERIODIC) {
    below = ((below % nz) + nz) % nz;
    above = ((above % nz) + nz) % nz;
  }
  if (below >= 0 && below < g.cc) {
    side = 0;
    p = below;
    return true;
  }
  if (above >= 0 && above < g.cc) {
    side = 1;
    p = above;
    return true;
  }
  return false;
}

// ---------------------------------------------------------------- warp reductions
__device__ __forceinline__ void group_sum3(bool member, float& a, float& b, float& c) {
  if (!member) a = b = c = 0.0f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(kFull, a, o);
    b += __shfl_xor_sync(kFull, b, o);
    c += __shfl_xor_sync(kFull, c, o);
  }
}

__device__ __forceinline__ float4 lerp4(float4 a, float4 b, float f) {
  return make_float4(fmaf(f, b.x - a.x, a.x), fmaf(f, b.y - a.y, a.y), fmaf(f, b.z - a.z, a.z), 0.0f);
}

// C-5 from the cell contract: t = (x-lo)*ih, c = cell; fr = t - c in [0,1];
// stencil base = c-1 (fr < 1/2, weight fr+1/2) or c (weight fr-1/2), i.e.
// floor(t - 1/2) and its fraction, within the ghost layer [-1, n].
__device__ __forceinline__ void stencil_from_cell(float t, int c, int& i0, float& f) {
  const float fr = t - (float)c;
  const bool lo = fr < 0.5f;
  i0 = lo ? c - 1 : c;
  f = lo ? fr + 0.5f : fr - 0.5f;
}

// ---------------------------------------------------------------- the step kernel
template <bool SCATTER, bool ADVANCE, int BCM, int SH>
__global__ void __launch_bounds__(256, (SCATTER && ADVANCE) ? 3 : 4) k_step(StepArgs a) {
  // dynamic shared memory, one slice per warp (see warp_smem_bytes)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geom& g = a.g;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* ws = smem_raw + (size_t)wib * warp_smem_bytes(SCATTER);
  Stage* stg = reinterpret_cast<Stage*>(ws);                                   // TMA-staged segments
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(ws + kStages * sizeof(Stage));
  int* rel = reinterpret_cast<int*>(bar + kStages);                            // [kMaxBins+1] bin offsets
  int (*cell_w)[3] = reinterpret_cast<int (*)[3]>(rel + kMaxBins + 1);         // [kMaxBins][3] bin cells
  int* run = reinterpret_cast<int*>(cell_w + kMaxBins);                        // [kMaxBins*27] (scatter)
  const int n_items = *a.n_items;
  const int warps_total = gridDim.x * (blockDim.x >> 5);
  const int64_t cap = a.cap;
  const int nbins = a.nbins;
  const int cc = SH > 0 ? (1 << SH) : g.cc;
  int flags = 0;
  uint32_t phase = 0;   // parity bit per stage
  if (lane == 0) {
    for (int k = 0; k < kStages; ++k) mbar_init(bar + k, 1);
    fence_mbar_init();
  }
  __syncwarp();

  for (int item = blockIdx.x * (blockDim.x >> 5) + wib; item < n_items; item += warps_total) {
    const int b0 = a.item_bin0[item];
    const int b1 = (item + 1 < n_items) ? a.item_bin0[item + 1] : nbins;
    const int nb = b1 - b0;
    const int64_t p0 = a.off[b0];
    for (int k = lane; k <= nb; k += 32) rel[k] = (int)(a.off[b0 + k] - p0);
    for (int k = lane; k < nb; k += 32) cell_of_bin(g, a.bg, b0 + k, cell_w[k][0], cell_w[k][1], cell_w[k][2]);
    if (SCATTER)
      for (int k = lane; k < nb * kSlots; k += 32) run[k] = 0;
    __syncwarp();
    const int np = rel[nb];
    const int nbatch = (np + 31) >> 5;
    // prime the pipeline
    if (lane == 0) {
      fence_proxy_async();
      for (int k = 0; k < kStages && k < nbatch; ++k) stage_issue(stg + k, bar + k, a.A, cap, p0 + 32 * k, cap, SCATTER);
    }
    __syncwarp();   // reconverge after the lane-0 issue (see k_pstep.cuh)
    int lb = 0;   // this lane's bin pointer (monotone over its particles)
    for (int bi = 0; bi < nbatch; ++bi) {
      const int base = bi << 5;
      const int sk = bi % kStages;
      const int r = base + lane;
      const bool valid = r < np;
      const int64_t i = p0 + r;
      if (valid)
        while (rel[lb + 1] <= r) ++lb;
      const int s = b0 + lb;
      const int sx = cell_w[lb][0], sy = cell_w[lb][1], sz = cell_w[lb][2];
      mbar_wait(bar + sk, (phase >> sk) & 1u);
      __syncwarp();
      phase ^= 1u << sk;
      const Stage& S = stg[sk];
      const int so = (int)((p0 + base) & 3) + lane;   // slot of this lane's particle in the segments
      float xp0 = 0.f, xp1 = 0.f, xp2 = 0.f, up0 = 0.f, up1 = 0.f, up2 = 0.f;
      float dp = 1e-5f, wp = 0.f;
      if (valid) {
        xp0 = S.f[0][so]; xp1 = S.f[1][so]; xp2 = S.f[2][so];
        up0 = S.f[3][so]; up1 = S.f[4][so]; up2 = S.f[5][so];
        dp = S.f[6][so];
        wp = S.f[7][so];
      }
      // current cell (deposit cell of the first sub-step; scatter key)
      float t0 = cell_coord(xp0, g.lo[0], g.ih[0]), t1 = cell_coord(xp1, g.lo[1], g.ih[1]),
            t2 = cell_coord(xp2, g.lo[2], g.ih[2]);
      int c0 = cell_from_t(t0, g.n[0]), c1 = cell_from_t(t1, g.n[1]), c2 = cell_from_t(t2, g.n[2]);
      // cell of the particle's bin in the output layout
      int ox = sx, oy = sy, oz = sz;
      int obin = s;
      int64_t dest = i;
      bool write_ok = valid;
      int vside = -1;   // >= 0: mover into a neighbour rank's plane (multi-GPU scatter)
      if (SCATTER) {
        const int j = valid ? slot_of<BCM>(g, sx, sy, sz, c0, c1, c2) : -1;
        if (valid && j < 0) {
          flags |= ERRF_SCATTER;
          write_ok = false;
        }
        const int key = write_ok ? lb * kSlots + j : -1 - lane;
        const unsigned peers = __match_any_sync(kFull, key);
        const int leader = __ffs(peers) - 1;
        int rbase = 0;
        if (lane == leader && key >= 0) {
          rbase = run[key];
          run[key] = rbase + __popc(peers);
        }
        rbase = __shfl_sync(kFull, rbase, leader);
        __syncwarp();
        if (write_ok) {
          ox = c0;
          oy = c1;
          oz = c2;
          const int64_t within = (int64_t)a.slot_base[(int64_t)j * nbins + s] + rbase + __popc(peers & lanemask_lt());
          vside = (c2 == a.bg.vz[0]) ? 0 : ((c2 == a.bg.vz[1]) ? 1 : -1);
          if (vside >= 0) {
            dest = a.voff[vside][vbin_of_cell<SH>(g, c0, c1, cc)] + within;
            if (dest < 0 || dest >= a.scap) {
              flags |= ERRF_SCATTER;
              write_ok = false;
            }
          } else {
            obin = bin_of_cell<SH>(g, a.bg, ox, oy, oz);
            dest = a.off_new[obin] + within;
            if (dest < 0 || dest >= a.n) {
              flags |= ERRF_SCATTER;
              write_ok = false;
            }
          }
        }
      }
      if (ADVANCE) {
        const float d = dp;
        const float tau = a.p.tau_c * d * d;
        const float inv_tau = rcp_approx(tau);
        const float mw = a.p.mass_c * d * d * d * wp;
        const float dt = a.dt;
        const float gx = a.p.g[0], gy = a.p.g[1], gz = a.p.g[2];
        for (int sub = 0; sub < a.nsteps; ++sub) {
          if (sub > 0) {
            t0 = cell_coord(xp0, g.lo[0], g.ih[0]);
            t1 = cell_coord(xp1, g.lo[1], g.ih[1]);
            t2 = cell_coord(xp2, g.lo[2], g.ih[2]);
            c0 = cell_from_t(t0, g.n[0]);
            c1 = cell_from_t(t1, g.n[1]);
            c2 = cell_from_t(t2, g.n[2]);
          }
          int ix, iy, iz;
          float fx, fy, fz;
          stencil_from_cell(t0, c0, ix, fx);
          stencil_from_cell(t1, c1, iy, fy);
          stencil_from_cell(t2, c2, iz, fz);
          int wz = window_z(g, iz);
          if (wz < 0 || wz + 1 >= g.wnz) {
            if (valid) flags |= ERRF_WINDOW;
            wz = wz < 0 ? 0 : g.wnz - 2;
          }
          const int pz = g.gy * g.gx;
          const float4* fb = a.field + ((int64_t)wz * pz + (iy + 1) * g.gx + (ix + 1));
          const float4 c000 = __ldg(fb), c100 = __ldg(fb + 1);
          const float4 c010 = __ldg(fb + g.gx), c110 = __ldg(fb + g.gx + 1);
          const float4 c001 = __ldg(fb + pz), c101 = __ldg(fb + pz + 1);
          const float4 c011 = __ldg(fb + pz + g.gx), c111 = __ldg(fb + pz + g.gx + 1);
          const float4 uf = lerp4(lerp4(lerp4(c000, c100, fx), lerp4(c010, c110, fx), fy),
                                  lerp4(lerp4(c001, c101, fx), lerp4(c011, c111, fx), fy), fz);
          const float sxv = uf.x - up0, syv = uf.y - up1, szv = uf.z - up2;
          const float Re = sqrt_approx(fmaf(sxv, sxv, fmaf(syv, syv, szv * szv))) * d * a.p.inv_nu;
          // C-2 Schiller-Naumann (branch-free): 1 + 0.15 Re^0.687 (Re <= 1000) or 0.44 Re / 24
          float f = 1.0f + 0.15f * exp2f(0.687f * __log2f(Re));
          f = (Re <= 1000.0f) ? f : (0.44f / 24.0f) * Re;
          f = (a.p.drag_law == ST_DRAG_STOKES) ? 1.0f : f;
          const float taue = tau * rcp_approx(f);
          const float h = dt * f * inv_tau;
          float du0, du1, du2;
          if (a.p.integrator == ST_INT_EXPONENTIAL) {
            float E, M;
            exp_pair(h, E, M);
            const float tM = taue * M;
            const float us0 = fmaf(gx, taue, uf.x), us1 = fmaf(gy, taue, uf.y), us2 = fmaf(gz, taue, uf.z);
            const float r0 = up0 - us0, r1 = up1 - us1, r2 = up2 - us2;
            du0 = fmaf(-M, r0, -gx * dt);
            du1 = fmaf(-M, r1, -gy * dt);
            du2 = fmaf(-M, r2, -gz * dt);
            xp0 = fmaf(tM, r0, fmaf(us0, dt, xp0));
            xp1 = fmaf(tM, r1, fmaf(us1, dt, xp1));
            xp2 = fmaf(tM, r2, fmaf(us2, dt, xp2));
            up0 = fmaf(E, r0, us0);
            up1 = fmaf(E, r1, us1);
            up2 = fmaf(E, r2, us2);
          } else {
            const float inv1h = rcp_approx(1.0f + h);
            const float un0 = (up0 + h * uf.x + dt * gx) * inv1h;
            const float un1 = (up1 + h * uf.y + dt * gy) * inv1h;
            const float un2 = (up2 + h * uf.z + dt * gz) * inv1h;
            du0 = (un0 - up0) - gx * dt;
            du1 = (un1 - up1) - gy * dt;
            du2 = (un2 - up2) - gz * dt;
            xp0 = fmaf(dt, un0, xp0);
            xp1 = fmaf(dt, un1, xp1);
            xp2 = fmaf(dt, un2, xp2);
            up0 = un0;
            up1 = un1;
            up2 = un2;
          }
          if (a.p.two_way) {
            // deposit -w m du into the start cell: the group of lanes sharing lane 0's
            // cell (cell-sorted warps) is reduced in registers, the rest red directly
            const int az = acc_z(g, c2);
            if (valid && az < 0) flags |= ERRF_WINDOW;
            const bool dep = valid && az >= 0;
            const int ckey = dep ? (az * g.n[1] + c1) * g.n[0] + c0 : -1 - lane;
            const float ja = -mw * du0, jb = -mw * du1, jc = -mw * du2;
            const unsigned peers = __match_any_sync(kFull, ckey);
            const int lead = __shfl_sync(kFull, ckey, 0);
            const unsigned major = __shfl_sync(kFull, peers, 0);
            if (__popc(major) >= 4 && lead >= 0) {
              const bool in = (major >> lane) & 1u;
              float ra = ja, rb = jb, rc = jc;
              group_sum3(in, ra, rb, rc);
              if (lane == 0) red_add_v4(a.acc + lead, ra, rb, rc);
              if (!in && dep) red_add_v4(a.acc + ckey, ja, jb, jc);
            } else if (dep) {
              red_add_v4(a.acc + ckey, ja, jb, jc);
            }
          }
          bool bad = false;
          bad |= apply_bc(periodic<BCM>(g, 0) ? ST_BC_PERIODIC : ST_BC_REFLECT, g.lo[0], g.hi[0], g.L[0], xp0, up0);
          bad |= apply_bc(periodic<BCM>(g, 1) ? ST_BC_PERIODIC : ST_BC_REFLECT, g.lo[1], g.hi[1], g.L[1], xp1, up1);
          bad |= apply_bc(periodic<BCM>(g, 2) ? ST_BC_PERIODIC : ST_BC_REFLECT, g.lo[2], g.hi[2], g.L[2], xp2, up2);
          if (bad && valid) flags |= ERRF_CFL;
        }
      }
      if (write_ok) {
        if (SCATTER) {
          // the id is only carried: read it from the stage late, out of the live range
          const unsigned long long pid = S.id[(int)((p0 + base) & 1) + lane];
          const Store& o = vside < 0 ? a.B : a.sbuf[vside];
          const int64_t oc = vside < 0 ? cap : a.scap;
          // normal L2 policy: the runs of consecutive destinations written by
          // neighbouring warps merge into full sectors before write-back
          o.x[dest] = xp0; o.x[oc + dest] = xp1; o.x[2 * oc + dest] = xp2;
          o.u[dest] = up0; o.u[oc + dest] = up1; o.u[2 * oc + dest] = up2;
          o.d[dest] = dp;
          o.w[dest] = wp;
          reinterpret_cast<unsigned long long*>(o.id)[dest] = pid;
        } else if (ADVANCE) {
          __stcs(a.A.x + i, xp0); __stcs(a.A.x + cap + i, xp1); __stcs(a.A.x + 2 * cap + i, xp2);
          __stcs(a.A.u + i, up0); __stcs(a.A.u + cap + i, up1); __stcs(a.A.u + 2 * cap + i, up2);
        }
      }
      // the stage is consumed: refill it with the batch kStages ahead
      __syncwarp();
      if (lane == 0 && bi + kStages < nbatch) {
        fence_proxy_async();
        stage_issue(stg + sk, bar + sk, a.A, cap, p0 + 32 * (bi + kStages), cap, SCATTER);
      }
      __syncwarp();
    }
    __syncwarp();
  }
  if (flags) atomicOr(a.err, flags);
}

#include "k_pstep.cuh"
#include "k_ip.cuh"
#include "k_fs.cuh"

// ---------------------------------------------------------------- rebin preparation
#ifndef ST_PREP_FAST
#define ST_PREP_FAST 1   // k_rebin_prep ranks the 27 sources from per-axis counts (else 27 x 27 compares)
#endif
// Per destination bin d: sources s = d - delta over the 27 deltas (canonical,
// deduplicated), in ascending s; base[j][s] = running sum; new_cnt[d] = total.
// The slot-major layout makes consecutive threads touch consecutive words.
// Destinations d >= nbins are the virtual bins of the neighbour planes (multi-GPU):
// d = nbins + side * nvb + v.
#ifndef ST_PREP_MINB
#define ST_PREP_MINB 1
#endif
template <int SH>
__global__ void __launch_bounds__(128, ST_PREP_MINB) k_rebin_prep(Geom g, BinGeom bg, int nbins, int* __restrict__ cnt_base, uint32_t* __restrict__ new_cnt,
                             const int* __restrict__ far_cnt, unsigned long long* __restrict__ movers) {
  __shared__ uint32_t prep_rows[128 * 27];   // launched with 128 threads
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nbins + 2 * bg.nvb) return;
  int dx, dy, dz;
  if (d < nbins) {
    cell_of_bin(g, bg, d, dx, dy, dz);
  } else {
    const int side = (d - nbins) / bg.nvb;
    cell_of_vbin(g, d - nbins - side * bg.nvb, dx, dy);
    dz = bg.vz[side];
  }
  if (dx >= g.n[0] || dy >= g.n[1] || dz < 0 || dz >= g.n[2]) {   // ragged chunk / no neighbour
    new_cnt[d] = 0;
    return;
  }
  const int kz_lo = bg.kz0, kz_hi = bg.kz0 + bg.nkz;
  bool fast = ST_PREP_FAST && SH == 3;
#pragma unroll
  for (int a = 0; a < 3; ++a) fast = fast && (g.bc[a] != ST_BC_PERIODIC || g.n[a] >= 3);
  // per axis a and option i (source coordinate c + 1 - i, the j convention below): chunk /
  // in-chunk coordinate, presence, and its term of the bin index (8^3 chunks: bin =
  // sum over axes of chunk stride * k + cell stride * l), so a source's key is two adds
  int ka[3][3], la[3][3], pa[3][3];
  bool oa[3][3];
  if (fast) {
    const int cd[3] = {dx, dy, dz};
    const int cs[3] = {bg.cc3, bg.cc3 * g.NC[0], bg.cc3 * g.NC[0] * g.NC[1]};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        int sc = cd[a] + 1 - i;
        if (g.bc[a] == ST_BC_PERIODIC) sc = sc < 0 ? sc + g.n[a] : (sc >= g.n[a] ? sc - g.n[a] : sc);
        ka[a][i] = sc >> 3;
        la[a][i] = sc & 7;
        oa[a][i] = sc >= 0 && sc < g.n[a] && (a < 2 || (ka[a][i] >= kz_lo && ka[a][i] < kz_hi));
        pa[a][i] = cs[a] * (a == 2 ? ka[a][i] - kz_lo : ka[a][i]) + (a == 0 ? 1 : (a == 1 ? 8 : 64)) * la[a][i];
      }
    }
  }
  // the 27 candidate sources s = d - delta(j); key = bin (INT_MAX if absent)
  int key[27], cnt[27];
#pragma unroll
  for (int j = 0; j < 27; ++j) {
    if (fast) {
      const int jx = j % 3, jy = (j / 3) % 3, jz = j / 9;
      const bool ok = oa[0][jx] && oa[1][jy] && oa[2][jz];
      key[j] = ok ? pa[0][jx] + pa[1][jy] + pa[2][jz] : 0x7fffffff;
      cnt[j] = ok ? cnt_base[(int64_t)j * nbins + key[j]] : 0;
      continue;
    }
    const int ox = j % 3 - 1, oy = (j / 3) % 3 - 1, oz = j / 9 - 1;
    bool ok = true;
    const int sx = axis_step(dx, -ox, g.n[0], g.bc[0], ok);
    const int sy = axis_step(dy, -oy, g.n[1], g.bc[1], ok);
    const int sz = axis_step(dz, -oz, g.n[2], g.bc[2], ok);
    if (ok) {
      const int kz = dcc<SH>(sz, g.cc);
      ok = kz >= kz_lo && kz < kz_hi &&                        // source on this rank
           slot_of<-1>(g, sx, sy, sz, dx, dy, dz) == j;          // canonical (no duplicate)
    }
    key[j] = ok ? bin_of_cell<SH>(g, bg, sx, sy, sz) : 0x7fffffff;
    cnt[j] = ok ? cnt_base[(int64_t)j * nbins + key[j]] : 0;
  }
  // statistics (movers != NULL): particles arriving from another chunk
  if (movers) {
    unsigned long long mv = 0;
    const int dk = dcc<SH>(dx, g.cc) + g.NC[0] * (dcc<SH>(dy, g.cc) + g.NC[1] * dcc<SH>(dz, g.cc));
#pragma unroll
    for (int j = 0; j < 27; ++j) {
      if (key[j] == 0x7fffffff) continue;
      const int sk = key[j] / bg.cc3;   // local chunk of the source bin
      const int dkl = dk - bg.kz0 * g.NC[0] * g.NC[1];
      mv += (sk != dkl) ? (unsigned long long)cnt[j] : 0ull;
    }
    // lanes of this warp that returned early (ragged chunks, the tail) are not in the mask
    const unsigned m = __activemask();
    const unsigned sum = __reduce_add_sync(m, (unsigned)mv);
    if ((threadIdx.x & 31) == __ffs(m) - 1 && sum) atomicAdd(movers, (unsigned long long)sum);
  }
  // stable order = ascending source bin: base of source q = sum of the counts of
  // the sources with a smaller bin (keys are distinct)
  uint32_t total = 0;
  if (fast) {
    // 8^3 chunks, three distinct source coordinates per axis: bin order is lexicographic
    // in (kz, ky, kx, lz, ly, lx) (chunk coordinates k = c >> 3 first, then the cell in the
    // chunk l = c & 7), so the rank of source (jx, jy, jz) among the 27 follows from
    // per-axis counts: lt = options with a smaller k, eq = options with the same k,
    // w = options with the same k and a smaller l (option i = source coordinate c + 1 - i,
    // the j = (oz+1)*9 + (oy+1)*3 + (ox+1) convention with s = d - o).  Absent sources
    // (walls, other ranks) have count 0 and any rank.
    int lt[3][3], eq[3][3], wl[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int* k = ka[a];
      const int* l = la[a];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        lt[a][i] = 0;
        eq[a][i] = 1;
        wl[a][i] = 0;
#pragma unroll
        for (int o = 0; o < 3; ++o) {
          if (o == i) continue;
          lt[a][i] += k[o] < k[i];
          eq[a][i] += k[o] == k[i];
          wl[a][i] += (k[o] == k[i]) && (l[o] < l[i]);
        }
      }
    }
    // counts scattered to their ranks in this thread's shared-memory row (stride 27
    // words: conflict-free across the warp), scanned, gathered back
    uint32_t* row = prep_rows + threadIdx.x * 27;
    int pos[27];
#pragma unroll
    for (int j = 0; j < 27; ++j) {
      const int jx = j % 3, jy = (j / 3) % 3, jz = j / 9;
      pos[j] = lt[2][jz] * 9 + eq[2][jz] * (lt[1][jy] * 3 + eq[1][jy] * lt[0][jx]) +
               wl[2][jz] * eq[1][jy] * eq[0][jx] + wl[1][jy] * eq[0][jx] + wl[0][jx];
      row[pos[j]] = (uint32_t)cnt[j];
    }
#pragma unroll
    for (int p = 0; p < 27; ++p) {
      const uint32_t c = row[p];
      row[p] = total;
      total += c;
    }
#pragma unroll
    for (int q = 0; q < 27; ++q)
      if (key[q] != 0x7fffffff) cnt_base[(int64_t)q * nbins + key[q]] = (int)row[pos[q]];
  } else {
#pragma unroll
    for (int q = 0; q < 27; ++q) {
      uint32_t base = 0;
#pragma unroll
      for (int p = 0; p < 27; ++p) base += (key[p] < key[q]) ? (uint32_t)cnt[p] : 0u;
      if (key[q] != 0x7fffffff) cnt_base[(int64_t)q * nbins + key[q]] = (int)base;
      total += (uint32_t)cnt[q];
    }
  }
  // far particles of this destination (C-15b) take the slots after its 27 runs
  if (far_cnt && d < nbins) total += (uint32_t)far_cnt[d];
  new_cnt[d] = total;
}

// Destination table of the fused scatter (k_pstep): for every source bin s and slot j,
// the store index where the run of s's particles at slot j starts in the new layout:
// off_new[d] + base[j][s] for a local destination bin d, voff[side][v] + base[j][s] for
// a neighbour rank's plane (the side is packed into bits 61-62), -1 if slot j leaves
// the domain.  Row-major [nbins][27] so that one item (a chunk row of 8 bins) is one
// contiguous 1728-byte bulk copy.
constexpr int kDbaseBlock = 128;
template <int SH>
__global__ void __launch_bounds__(kDbaseBlock) k_dbase(Geom g, BinGeom bg, int nbins, const int* __restrict__ base,
                                                       const int64_t* __restrict__ off_new, const int64_t* __restrict__ voff0,
                                                       const int64_t* __restrict__ voff1, long long* __restrict__ dtab,
                                                       const int* __restrict__ far_cnt,
                                                       unsigned long long* __restrict__ far_cur) {
  // each thread builds its bin's 27-entry row in shared memory; the block then writes its
  // 128 rows as one contiguous, coalesced run of 27 x 128 entries
  __shared__ long long tile[kDbaseBlock * kSlots];
  const int s0 = blockIdx.x * kDbaseBlock;
  const int s = s0 + threadIdx.x;
  if (s < nbins) {
    if (far_cur) far_cur[s] = (unsigned long long)(off_new[s + 1] - far_cnt[s]);   // start of bin s's far tail
    int sx, sy, sz;
    cell_of_bin(g, bg, s, sx, sy, sz);
    const bool cell_ok = sx < g.n[0] && sy < g.n[1] && sz < g.n[2];
#pragma unroll
    for (int j = 0; j < kSlots; ++j) {
      bool ok = cell_ok;
      const int dx = axis_step(sx, j % 3 - 1, g.n[0], g.bc[0], ok);
      const int dy = axis_step(sy, (j / 3) % 3 - 1, g.n[1], g.bc[1], ok);
      const int dz = axis_step(sz, j / 9 - 1, g.n[2], g.bc[2], ok);
      long long e = -1;
      if (ok) {
        const long long within = base[(int64_t)j * nbins + s];
        if (bg.nvb > 0 && dz == bg.vz[0]) {
          e = (voff0[vbin_of_cell<SH>(g, dx, dy, g.cc)] + within) | (1LL << 61);
        } else if (bg.nvb > 0 && dz == bg.vz[1]) {
          e = (voff1[vbin_of_cell<SH>(g, dx, dy, g.cc)] + within) | (2LL << 61);
        } else {
          const int kz = dcc<SH>(dz, g.cc);
          if (kz >= bg.kz0 && kz < bg.kz0 + bg.nkz) e = off_new[bin_of_cell<SH>(g, bg, dx, dy, dz)] + within;
        }
      }
      tile[threadIdx.x * kSlots + j] = e;
    }
  }
  __syncthreads();
  const int rows = min(kDbaseBlock, nbins - s0);
  for (int k = threadIdx.x; k < rows * kSlots; k += kDbaseBlock) dtab[(int64_t)s0 * kSlots + k] = tile[k];
}

// Arrival counts from the neighbours land after the local runs of the boundary-plane
// bins and before their far tails: one layout per bin, runs | arrivals | far tail
// (C-16: kept first, then arrivals; C-15b: far last).  new_cnt[d] already counts the
// far particles (k_rebin_prep), so the arrivals start at new_cnt - far_cnt.
__global__ void k_vcombine(Geom g, BinGeom bg, uint32_t* __restrict__ new_cnt, const uint32_t* __restrict__ rcnt_dn,
                           const uint32_t* __restrict__ rcnt_up, uint32_t* __restrict__ kept_dn,
                           uint32_t* __restrict__ kept_up, int oz0, int oz1, const int* __restrict__ far_cnt) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= bg.nvb) return;
  int x, y;
  cell_of_vbin(g, v, x, y);
  if (x >= g.n[0] || y >= g.n[1]) return;
  const int db = bin_of_cell<0>(g, bg, x, y, oz0);
  kept_dn[v] = new_cnt[db] - (far_cnt ? (uint32_t)far_cnt[db] : 0u);
  new_cnt[db] += rcnt_dn[v];
  const int dt = bin_of_cell<0>(g, bg, x, y, oz1 - 1);
  kept_up[v] = new_cnt[dt] - (far_cnt ? (uint32_t)far_cnt[dt] : 0u);
  new_cnt[dt] += rcnt_up[v];
}

// C-15b, deterministic: the fused scatter (and, across ranks, k_far_insert) placed bin
// d's F far particles in the last F slots of d in atomic order, each with its key
// (hi, lo) = (0, old-layout index) or (1 + source-rank order, sender's index); k_far_order_w
// sorts that tail by the key (payload moved with it), so the far tail is kept ++ arrivals
// in prior store order — the (bin, far)-stable sort of the oracle.
// Far-tail ordering in two kernels.  k_far_order_w: persistent warps scan the bins 32 at a
// time; a tail of F <= 32 kFarR entries is ordered by its warp — every entry's rank is the
// number of smaller keys in the tail (keys are distinct: (0, own old index) or (1 + source
// order, sender index)), then each entry moves once, from registers, to t0 + rank.  Longer
// tails go to a list for k_far_order_b: one CTA per tail sorts (key, entry) pairs in shared
// memory (bitonic), copies the tail's payload to the same indices of the old layout (free
// after the scatter) and gathers it back in key order.  (The round-2 thread-per-bin
// insertion sort moved O(F^2) payload per bin; at C5, K = 4, dense bins collect hundreds of
// far particles.)
constexpr int kFarR = 4;
constexpr int kFarBlockMax = 4096;   // longest tail sorted in shared memory (8 + 4 B per entry)
__device__ __forceinline__ int64_t far_key(const int32_t* far_src, const int32_t* far_hi, int64_t t) {
  return ((int64_t)far_hi[t] << 32) | (uint32_t)far_src[t];
}
__device__ __forceinline__ void move_payload(const Store& from, int64_t s, const Store& to, int64_t t, int64_t cap) {
  for (int a = 0; a < 3; ++a) {
    to.x[a * cap + t] = from.x[a * cap + s];
    to.u[a * cap + t] = from.u[a * cap + s];
  }
  to.d[t] = from.d[s];
  to.w[t] = from.w[s];
  to.id[t] = from.id[s];
}
__global__ void __launch_bounds__(256) k_far_order_w(int nbins, const int* __restrict__ far_cnt,
                                                     const int64_t* __restrict__ off_new, int32_t* __restrict__ far_src,
                                                     int32_t* __restrict__ far_hi, Store B, int64_t cap,
                                                     int* __restrict__ long_list, int* __restrict__ long_n) {
  const int lane = threadIdx.x & 31;
  const int gw = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  for (int64_t d0 = (int64_t)gw * 32; d0 < nbins; d0 += (int64_t)nw * 32) {
    const int64_t dl = d0 + lane;
    const int Fl = dl < nbins ? far_cnt[dl] : 0;
    unsigned todo = __ballot_sync(0xffffffffu, Fl >= 2);
    while (todo) {
      const int l = __ffs(todo) - 1;
      todo &= todo - 1;
      const int d = (int)(d0 + l);
      const int F = __shfl_sync(0xffffffffu, Fl, l);
      if (F > 32 * kFarR) {
        if (lane == 0) long_list[atomicAdd(long_n, 1)] = d;
        continue;
      }
      const int64_t t0 = off_new[d + 1] - F;
      int64_t key[kFarR];
      int rank[kFarR];
#pragma unroll
      for (int r = 0; r < kFarR; ++r) {
        const int i = lane + 32 * r;
        key[r] = i < F ? far_key(far_src, far_hi, t0 + i) : INT64_MAX;
        rank[r] = 0;
      }
#pragma unroll
      for (int r2 = 0; r2 < kFarR; ++r2) {
        if (32 * r2 >= F) break;
        const int m = min(32, F - 32 * r2);
        for (int j = 0; j < m; ++j) {
          const int64_t kj = __shfl_sync(0xffffffffu, key[r2], j);
#pragma unroll
          for (int r = 0; r < kFarR; ++r) rank[r] += kj < key[r];
        }
      }
      float v[kFarR][8];
      uint64_t id[kFarR];
#pragma unroll
      for (int r = 0; r < kFarR; ++r) {
        const int64_t t = t0 + lane + 32 * r;
        if (lane + 32 * r < F) {
          for (int a = 0; a < 3; ++a) {
            v[r][a] = B.x[a * cap + t];
            v[r][3 + a] = B.u[a * cap + t];
          }
          v[r][6] = B.d[t];
          v[r][7] = B.w[t];
          id[r] = B.id[t];
        }
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < kFarR; ++r) {
        if (lane + 32 * r < F) {
          const int64_t t = t0 + rank[r];
          far_src[t] = (int32_t)(uint32_t)key[r];
          far_hi[t] = (int32_t)(key[r] >> 32);
          for (int a = 0; a < 3; ++a) {
            B.x[a * cap + t] = v[r][a];
            B.u[a * cap + t] = v[r][3 + a];
          }
          B.d[t] = v[r][6];
          B.w[t] = v[r][7];
          B.id[t] = id[r];
        }
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(256) k_far_order_b(const int* __restrict__ far_cnt, const int64_t* __restrict__ off_new,
                                                     int32_t* __restrict__ far_src, int32_t* __restrict__ far_hi,
                                                     Store B, Store A, int64_t cap, const int* __restrict__ long_list,
                                                     const int* __restrict__ long_n) {
  __shared__ long long skey[kFarBlockMax];
  __shared__ int sidx[kFarBlockMax];
  const int nl = *long_n;
  for (int li = blockIdx.x; li < nl; li += gridDim.x) {
    const int d = long_list[li];
    const int F = far_cnt[d];
    const int64_t t0 = off_new[d + 1] - F;
    // the tail's payload to the same indices of the old layout (scratch)
    for (int i = threadIdx.x; i < F; i += blockDim.x) move_payload(B, t0 + i, A, t0 + i, cap);
    if (F <= kFarBlockMax) {
      int P = 1;
      while (P < F) P <<= 1;
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        skey[i] = i < F ? far_key(far_src, far_hi, t0 + i) : INT64_MAX;
        sidx[i] = i;
      }
      __syncthreads();
      for (int k = 2; k <= P; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
          for (int i = threadIdx.x; i < P; i += blockDim.x) {
            const int o = i ^ jj;
            if (o > i) {
              const bool up = (i & k) == 0;
              const long long a = skey[i], b = skey[o];
              if ((a > b) == up) {
                skey[i] = b;
                skey[o] = a;
                const int t = sidx[i];
                sidx[i] = sidx[o];
                sidx[o] = t;
              }
            }
          }
          __syncthreads();
        }
      }
      for (int p = threadIdx.x; p < F; p += blockDim.x) {
        far_src[t0 + p] = (int32_t)(uint32_t)skey[p];
        far_hi[t0 + p] = (int32_t)(skey[p] >> 32);
        move_payload(A, t0 + sidx[p], B, t0 + p, cap);
      }
      __syncthreads();
    } else {
      // beyond the shared-memory sort: rank of every entry by counting smaller keys
      __syncthreads();
      for (int i = threadIdx.x; i < F; i += blockDim.x) {
        const int64_t ki = far_key(far_src, far_hi, t0 + i);
        int rank = 0;
        for (int j = 0; j < F; ++j) rank += far_key(far_src, far_hi, t0 + j) < ki;
        move_payload(A, t0 + i, B, t0 + rank, cap);
        A.id[t0 + i] = (uint64_t)ki;   // keys kept beside the payload until every rank is known
      }
      __syncthreads();
      for (int i = threadIdx.x; i < F; i += blockDim.x) {
        // the keys in rank order: re-rank from the saved copies
        const int64_t ki = (int64_t)A.id[t0 + i];
        int rank = 0;
        for (int j = 0; j < F; ++j) rank += (int64_t)A.id[t0 + j] < ki;
        far_src[t0 + rank] = (int32_t)(uint32_t)ki;
        far_hi[t0 + rank] = (int32_t)(ki >> 32);
      }
      __syncthreads();
    }
  }
}

// Insert the arrivals of one side into B and count their slots for the next rebin.
__global__ void k_insert(InsertArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.count) return;
  int lo = 0, hi = a.bg.nvb;   // last v with roff[v] <= i
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.roff[mid] <= i) lo = mid;
    else hi = mid - 1;
  }
  const int v = lo;
  int x, y;
  cell_of_vbin(a.g, v, x, y);
  const int d = bin_of_cell<0>(a.g, a.bg, x, y, a.plane);
  const int64_t dest = a.off_new[d] + a.kept[v] + (i - a.roff[v]);
  const Store& r = a.rbuf;
  const int64_t rc = a.rcap, cap = a.cap;
  for (int ax = 0; ax < 3; ++ax) {
    a.B.x[ax * cap + dest] = r.x[ax * rc + i];
    a.B.u[ax * cap + dest] = r.u[ax * rc + i];
  }
  a.B.d[dest] = r.d[i];
  a.B.w[dest] = r.w[i];
  a.B.id[dest] = r.id[i];
}

// Slot histogram of the current layout — the input of the next neighbour-slot
// rebin (C-15): hist[j][s] = number of particles of bin s whose current cell lies at
// slot j (0..26) relative to the bin's cell.  One warp per item: the item's bins are
// owned, so counts gather in registers (stayers) and shared memory (the rest) and
// reach HBM as plain stores (no memset, no global atomics).  Reads only x (12 B per
// particle).  A particle more than one cell from its bin sets *far (the rebin must
// then take the general sort); chunk movers are counted for the roofline.
constexpr int kCountUnroll = 8;   // batches of x in flight per lane

template <int BCM, int SH>
__global__ void __launch_bounds__(256) k_count(CountArgs a) {
  __shared__ int cnt_s[8][kMaxBins * kSlots];
  __shared__ int rel_s[8][kMaxBins + 1];
  const Geom& g = a.g;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int* wc = cnt_s[wib];
  int* rel = rel_s[wib];
  const int n_items = *a.n_items, nbins = a.nbins, cc = g.cc;
  const int64_t cap = a.cap;
  const int warps_total = gridDim.x * (blockDim.x >> 5);
  unsigned movers = 0;
  int farflag = 0;
  for (int item = blockIdx.x * (blockDim.x >> 5) + wib; item < n_items; item += warps_total) {
    const int b0 = a.item_bin0[item];
    const int b1 = (item + 1 < n_items) ? a.item_bin0[item + 1] : nbins;
    const int nb = b1 - b0;
    const int64_t p0 = a.off[b0];
    for (int k = lane; k <= nb; k += 32) rel[k] = (int)(a.off[b0 + k] - p0);
    for (int k = lane; k < nb * kSlots; k += 32) wc[k] = 0;
    int rx = 0, ry = 0, rz = 0;
    if (SH == 3) cell_of_bin(g, a.bg, b0, rx, ry, rz);   // 8^3 chunks: the item is one row along +x
    __syncwarp();
    const int np = rel[nb];
    int lb = -1, sx = 0, sy = 0, sz = 0, scnt = 0;
    for (int base = 0; base < np; base += 32 * kCountUnroll) {
      float xv[kCountUnroll][3];
#pragma unroll
      for (int u = 0; u < kCountUnroll; ++u) {
        const int r = base + 32 * u + lane;
        const int64_t i = p0 + (r < np ? r : np - 1);
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) xv[u][ax] = __ldcs(a.x + ax * cap + i);
      }
#pragma unroll
      for (int u = 0; u < kCountUnroll; ++u) {
        const int r = base + 32 * u + lane;
        if (r < np) {
          int nl = lb < 0 ? 0 : lb;
          while (rel[nl + 1] <= r) ++nl;
          if (nl != lb) {
            if (scnt) atomicAdd(&wc[lb * kSlots + kStay], scnt);
            scnt = 0;
            lb = nl;
            if (SH == 3) {
              sx = rx + lb;
              sy = ry;
              sz = rz;
            } else {
              cell_of_bin(g, a.bg, b0 + lb, sx, sy, sz);
            }
          }
          const int c0 = cell_from_t(cell_coord(xv[u][0], g.lo[0], g.ih[0]), g.n[0]);
          const int c1 = cell_from_t(cell_coord(xv[u][1], g.lo[1], g.ih[1]), g.n[1]);
          const int c2 = cell_from_t(cell_coord(xv[u][2], g.lo[2], g.ih[2]), g.n[2]);
          const int j = slot_of<BCM>(g, sx, sy, sz, c0, c1, c2);
          if (j < 0) {
            // C-15b: a far particle whose cell is on this rank goes to its bin's tail
            const int kz = dcc<SH>(c2, cc);
            if (a.far_cnt && kz >= a.bg.kz0 && kz < a.bg.kz0 + a.bg.nkz) {
              atomicAdd(a.far_cnt + bin_of_cell<SH>(a.g, a.bg, c0, c1, c2), 1);
              atomicAdd(a.far_n, 1ULL);
            }
            else
              farflag = 1;
          }
          else if (j == kStay) ++scnt;
          else atomicAdd(&wc[lb * kSlots + j], 1);
          movers += ((dcc<SH>(c0, cc) != dcc<SH>(sx, cc)) | (dcc<SH>(c1, cc) != dcc<SH>(sy, cc)) |
                     (dcc<SH>(c2, cc) != dcc<SH>(sz, cc)))
                        ? 1u
                        : 0u;
        }
      }
    }
    if (scnt) atomicAdd(&wc[lb * kSlots + kStay], scnt);
    __syncwarp();
    for (int k = lane; k < nb * kSlots; k += 32) {
      const int l = k / kSlots, j = k - l * kSlots;
      a.hist[(int64_t)j * nbins + b0 + l] = wc[k];
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) movers += __shfl_xor_sync(kFull, movers, o);
  if (lane == 0 && movers) atomicAdd(a.movers, (unsigned long long)movers);
  if (farflag) *(volatile int*)a.far = 1;
}

// item boundaries: bin s starts an item if s % row == 0 or (ipart > 0) the ipart-particle
// window of its first particle differs from that of bin s-1's first particle.
__global__ void k_item_flags(const int64_t* __restrict__ off, int nbins, int row, int64_t ipart,
                             uint32_t* __restrict__ flag) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nbins) return;
  uint32_t f = (s % row) == 0;
  if (!f && ipart > 0) f = (off[s] / ipart) != (off[s - 1] / ipart);
  flag[s] = f;
}

__global__ void k_item_fill(const uint32_t* __restrict__ flag, const int64_t* __restrict__ pos, int nbins,
                            int* __restrict__ item_bin0, int* __restrict__ n_items) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nbins && flag[s]) item_bin0[pos[s]] = s;
  if (s == 0) *n_items = (int)pos[nbins];
}

__global__ void k_bin_offsets(const int32_t* __restrict__ key, int64_t n, int nbins, int64_t* __restrict__ off) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nbins) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (key[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  off[k] = lo;
}

__global__ void k_bin_keys(Geom g, BinGeom bg, const float* __restrict__ x, int64_t xs, int64_t n,
                           int32_t* __restrict__ key, int* __restrict__ err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int c[3];
    for (int ax = 0; ax < 3; ++ax) c[ax] = cell_from_t(cell_coord(x[ax * xs + i], g.lo[ax], g.ih[ax]), g.n[ax]);
    int b = bin_of_cell<0>(g, bg, c[0], c[1], c[2]);
    if (b < 0 || b >= bg.nbins) {   // outside this rank's bins (multi-GPU: migrates first)
      atomicOr(err, ERRF_WINDOW);
      b = b < 0 ? 0 : bg.nbins - 1;
    }
    key[i] = b;
  }
}

inline unsigned blocks_for(int64_t n, int bs = 256) { return (unsigned)((n + bs - 1) / bs); }

template <bool S, bool A, int BCM, int SH>
int launch_variant(const StepArgs& a, cudaStream_t s) {
  static int grid = 0;
  const int smem = 8 * warp_smem_bytes(S);
  if (!grid) {
    int nsm = 148, dev = 0, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_step<S, A, BCM, SH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_step<S, A, BCM, SH>, 256, smem);
    grid = nsm * (per > 0 ? per : 1);
  }
  k_step<S, A, BCM, SH><<<grid, 256, smem, s>>>(a);
  return 1;
}

template <bool S, bool A, int BCM, int SPEC = kSpecAll, int FEAT = 0xff>
int launch_pvariant(const StepArgs& a, cudaStream_t s) {
  static int grid = 0;
  constexpr int W = pwarps(S && A);
  const int smem = W * pwarp_smem_bytes(S) + kPSmemAlign;
  if (!grid) {
    int nsm = 148, dev = 0, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_pstep<S, A, BCM, SPEC, FEAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pstep<S, A, BCM, SPEC, FEAT>, 32 * W, smem);
    grid = nsm * (per > 0 ? per : 1);
  }
  k_pstep<S, A, BCM, SPEC, FEAT><<<grid, 32 * W, smem, s>>>(a);
  return 1;
}

// compile-time specialisation of k_pstep: neighbour-rank planes present (kSpecVP),
// more than one sub-step per call (kSpecSub)
template <bool S, bool A, int BCM>
int launch_pspec(const StepArgs& a, cudaStream_t s) {
  const int spec = (a.bg.nvb > 0 ? kSpecVP : 0) | (a.nsteps > 1 ? kSpecSub : 0);
  switch (spec) {
    case 0: return launch_pvariant<S, A, BCM, 0>(a, s);
    case kSpecVP: return launch_pvariant<S, A, BCM, kSpecVP>(a, s);
    case kSpecSub: return launch_pvariant<S, A, BCM, kSpecSub>(a, s);
    default: return launch_pvariant<S, A, BCM, kSpecAll>(a, s);
  }
}

// Performance ablation (benchmarking builds only: results are wrong).  Compiled in only
// with -DST_ABLATION_BUILD (scripts/gpu_ablate.sh); the product library never reads the
// environment.  FEAT bits 1 physics, 2 field gather, 4 deposit, 16 stores (single-rank,
// one-sub-step, reflecting-wall specialisation).
#ifdef ST_ABLATION_BUILD
int ablate_mask() {
  static int m = -2;
  if (m == -2) {
    const char* e = getenv("ST_ABLATE");
    m = e ? atoi(e) : -1;
  }
  return m;
}
#endif

template <bool S, bool A>
int launch_mode(const StepArgs& a, cudaStream_t s) {
  const int bcm = (a.g.bc[0] == ST_BC_PERIODIC ? 1 : 0) | (a.g.bc[1] == ST_BC_PERIODIC ? 2 : 0) |
                  (a.g.bc[2] == ST_BC_PERIODIC ? 4 : 0);
  if (a.g.cc == 8) {   // chunk-row items with the staged fluid box (k_pstep.cuh)
#ifdef ST_ABLATION_BUILD
    if (S && A && bcm == 0 && a.bg.nvb == 0 && a.nsteps == 1 && ablate_mask() >= 0) {
      switch (ablate_mask()) {
        case 29: return launch_pvariant<S, A, 0, 0, 29>(a, s);   // no field gather
        case 27: return launch_pvariant<S, A, 0, 0, 27>(a, s);   // no deposit
        case 15: return launch_pvariant<S, A, 0, 0, 15>(a, s);   // no stores
        case 30: return launch_pvariant<S, A, 0, 0, 30>(a, s);   // no physics (no field, no deposit)
        case 16: return launch_pvariant<S, A, 0, 0, 16>(a, s);   // loads + scatter stores only
        case 0: return launch_pvariant<S, A, 0, 0, 0>(a, s);  // loads + rank only
        default: break;
      }
    }
#endif
#ifndef ST_OLD_FUSED
    if (S && A) {    // fused rebin scatter + advance: two particles per lane (k_fs.cuh)
      switch (bcm) {
        case 0: return launch_fs<0>(a, s);
        case 7: return launch_fs<7>(a, s);
        case 3: return launch_fs<3>(a, s);
        default: return launch_fs<-1>(a, s);
      }
    }
#endif
#ifndef ST_OLD_INPLACE
    if (!S && A) {   // in place: the two-particles-per-lane kernel (k_ip.cuh)
      switch (bcm) {
        case 0: return launch_ip<0>(a, s);
        case 7: return launch_ip<7>(a, s);
        case 3: return launch_ip<3>(a, s);
        default: return launch_ip<-1>(a, s);
      }
    }
#endif
    switch (bcm) {
      case 0: return launch_pspec<S, A, 0>(a, s);
      case 7: return launch_pspec<S, A, 7>(a, s);
      case 3: return launch_pspec<S, A, 3>(a, s);
      default: return launch_pvariant<S, A, -1>(a, s);
    }
  }
  return launch_variant<S, A, -1, 0>(a, s);
}

}  // namespace

int launch_step(const StepArgs& a, bool scatter, bool advance, cudaStream_t s) {
  if (scatter && advance) return launch_mode<true, true>(a, s);
  if (scatter) return launch_mode<true, false>(a, s);
  return launch_mode<false, true>(a, s);
}

int launch_rebin_prep(const Geom& g, const BinGeom& bg, int* cnt_base, uint32_t* new_cnt, const int* far_cnt,
                      unsigned long long* movers, cudaStream_t s) {
  if (g.cc == 8)
    k_rebin_prep<3><<<blocks_for((int64_t)bg.nbins + 2 * bg.nvb, 128), 128, 0, s>>>(g, bg, bg.nbins, cnt_base, new_cnt,
                                                                                  far_cnt, movers);
  else
    k_rebin_prep<0><<<blocks_for((int64_t)bg.nbins + 2 * bg.nvb, 128), 128, 0, s>>>(g, bg, bg.nbins, cnt_base, new_cnt,
                                                                                  far_cnt, movers);
  return 1;
}

int launch_vcombine(const Geom& g, const BinGeom& bg, uint32_t* new_cnt, const uint32_t* rcnt_dn, const uint32_t* rcnt_up,
                    uint32_t* kept_dn, uint32_t* kept_up, int oz0, int oz1, const int* far_cnt, cudaStream_t s) {
  if (bg.nvb <= 0) return 0;
  k_vcombine<<<blocks_for(bg.nvb), 256, 0, s>>>(g, bg, new_cnt, rcnt_dn, rcnt_up, kept_dn, kept_up, oz0, oz1, far_cnt);
  return 1;
}

// The receiver of far particles across ranks: counts per cell of my first / last
// chunk_cells planes (rfv0 from the rank below: planes z0 + p; rfv1 from the rank above:
// planes z1 - 1 - p) join the far tails of their bins.
__global__ void k_far_accept(Geom g, BinGeom bg, const int* __restrict__ rfv0, const int* __restrict__ rfv1, int z0,
                             int z1, uint32_t* __restrict__ new_cnt, int* __restrict__ far_cnt,
                             unsigned long long* __restrict__ fr_n, int* __restrict__ err) {
  const int64_t plane = (int64_t)g.n[0] * g.n[1];
  const int64_t nf = plane * g.cc;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * nf) return;
  const int side = (int)(i / nf);
  const int64_t v = i - side * nf;
  const int cnt = (side ? rfv1 : rfv0)[v];
  if (!cnt) return;
  const int p = (int)(v / plane);
  const int y = (int)((v % plane) / g.n[0]), x = (int)(v % g.n[0]);
  const int z = side ? z1 - 1 - p : z0 + p;
  const int kz = z / g.cc;
  if (z < z0 || z >= z1 || kz < bg.kz0 || kz >= bg.kz0 + bg.nkz) {
    atomicOr(err, ERRF_SCATTER);
    return;
  }
  const int b = bin_of_cell<0>(g, bg, x, y, z);
  atomicAdd(new_cnt + b, (uint32_t)cnt);
  atomicAdd(far_cnt + b, cnt);
  atomicAdd(fr_n + side, (unsigned long long)cnt);
}

// Far arrivals of one side into the far tails of B: bin = the cell the sender counted
// them for (their position has advanced since, in the sender's fused launch), slot by
// the bin's cursor, key (1 + source-rank order, sender's index) for k_far_order_w.
__global__ void k_far_insert(FarInsertArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.count) return;
  const Store& r = a.r;
  const int64_t rc = a.rcap;
  const int cl = a.cell[i];
  const int cx = cl % a.g.n[0], cy = (cl / a.g.n[0]) % a.g.n[1], cz = cl / (a.g.n[0] * a.g.n[1]);
  const int kz = cz / a.g.cc;
  if (kz < a.bg.kz0 || kz >= a.bg.kz0 + a.bg.nkz) {
    atomicOr(a.err, ERRF_SCATTER);
    return;
  }
  const int b = bin_of_cell<0>(a.g, a.bg, cx, cy, cz);
  const int64_t slot = (int64_t)atomicAdd(a.far_cur + b, 1ULL);
  a.far_src[slot] = a.key[i];
  a.far_src_hi[slot] = a.hi;
  const int64_t cap = a.cap;
  for (int ax = 0; ax < 3; ++ax) {
    a.B.x[ax * cap + slot] = r.x[ax * rc + i];
    a.B.u[ax * cap + slot] = r.u[ax * rc + i];
  }
  a.B.d[slot] = r.d[i];
  a.B.w[slot] = r.w[i];
  a.B.id[slot] = r.id[i];
}

int launch_far_accept(const Geom& g, const BinGeom& bg, const int* rfv0, const int* rfv1, int z0, int z1,
                      uint32_t* new_cnt, int* far_cnt, unsigned long long* fr_n, int* err, cudaStream_t s) {
  const int64_t nf = (int64_t)g.n[0] * g.n[1] * g.cc;
  k_far_accept<<<blocks_for(2 * nf), 256, 0, s>>>(g, bg, rfv0, rfv1, z0, z1, new_cnt, far_cnt, fr_n, err);
  return 1;
}

int launch_far_insert(const FarInsertArgs& a, cudaStream_t s) {
  if (a.count <= 0) return 0;
  k_far_insert<<<blocks_for(a.count), 256, 0, s>>>(a);
  return 1;
}

int launch_far_order(const BinGeom& bg, const int* far_cnt, const int64_t* off_new, const int32_t* far_src,
                     const int32_t* far_src_hi, Store B, Store A, int64_t cap, int* long_list, int* long_n,
                     cudaStream_t s) {
  if (!far_cnt || !far_src || bg.nbins <= 0) return 0;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  cudaMemsetAsync(long_n, 0, sizeof(int), s);
  const int grid = (int)std::min<int64_t>((int64_t)nsm * 8, blocks_for((int64_t)bg.nbins, 256));
  k_far_order_w<<<grid, 256, 0, s>>>(bg.nbins, far_cnt, off_new, const_cast<int32_t*>(far_src),
                                      const_cast<int32_t*>(far_src_hi), B, cap, long_list, long_n);
  k_far_order_b<<<nsm, 256, 0, s>>>(far_cnt, off_new, const_cast<int32_t*>(far_src), const_cast<int32_t*>(far_src_hi),
                                     B, A, cap, long_list, long_n);
  return 2;
}

int launch_insert(const InsertArgs& a, cudaStream_t s) {
  if (a.count <= 0) return 0;
  k_insert<<<blocks_for(a.count), 256, 0, s>>>(a);
  return 1;
}

template <int BCM, int SH>
int launch_count_v(const CountArgs& a, cudaStream_t s) {
  static int grid = 0;
  if (!grid) {
    int nsm = 148, dev = 0, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_count<BCM, SH>, 256, 0);
    grid = nsm * (per > 0 ? per : 1);
  }
  k_count<BCM, SH><<<grid, 256, 0, s>>>(a);
  return 1;
}

int launch_dbase(const Geom& g, const BinGeom& bg, const int* base, const int64_t* off_new, const int64_t* voff0,
                 const int64_t* voff1, long long* dtab, const int* far_cnt, unsigned long long* far_cur, cudaStream_t s) {
  if (g.cc == 8)
    k_dbase<3><<<blocks_for(bg.nbins, kDbaseBlock), kDbaseBlock, 0, s>>>(g, bg, bg.nbins, base, off_new, voff0, voff1,
                                                                        dtab, far_cnt, far_cur);
  else
    k_dbase<0><<<blocks_for(bg.nbins, kDbaseBlock), kDbaseBlock, 0, s>>>(g, bg, bg.nbins, base, off_new, voff0, voff1,
                                                                        dtab, far_cnt, far_cur);
  return 1;
}

int launch_count(const CountArgs& a, cudaStream_t s) {
  const int bcm = (a.g.bc[0] == ST_BC_PERIODIC ? 1 : 0) | (a.g.bc[1] == ST_BC_PERIODIC ? 2 : 0) |
                  (a.g.bc[2] == ST_BC_PERIODIC ? 4 : 0);
  if (a.g.cc == 8) {
    switch (bcm) {
      case 0: return launch_count_v<0, 3>(a, s);
      case 7: return launch_count_v<7, 3>(a, s);
      case 3: return launch_count_v<3, 3>(a, s);
      default: return launch_count_v<-1, 3>(a, s);
    }
  }
  return launch_count_v<-1, 0>(a, s);
}

int launch_items(const int64_t* off, int nbins, int cc, uint32_t* flag, int64_t* pos, int64_t* partial,
                 int* item_bin0, int* n_items, cudaStream_t s) {
  // 8^3 chunks: one whole chunk row (8 bins) per item for k_pstep, so its per-item
  // set-up (destination table, fluid window) is amortised over the row; else
  // <= kMaxBins bins and <= ~kItemParticles particles
  const int row = cc == 8 ? kRowBins : kMaxBins;
  k_item_flags<<<blocks_for(nbins), 256, 0, s>>>(off, nbins, row, cc == 8 ? 0 : kItemParticles, flag);
  int nl = 1 + launch_exclusive_scan_u32(flag, nbins, pos, partial, s);
  k_item_fill<<<blocks_for(nbins), 256, 0, s>>>(flag, pos, nbins, item_bin0, n_items);
  return nl + 1;
}

int launch_bin_offsets(const int32_t* key_sorted, int64_t n, int nbins, int64_t* off, cudaStream_t s) {
  k_bin_offsets<<<blocks_for((int64_t)nbins + 1), 256, 0, s>>>(key_sorted, n, nbins, off);
  return 1;
}

int launch_bin_keys(const Geom& g, const BinGeom& bg, const float* x, int64_t xs, int64_t n, int32_t* key, int* err,
                    cudaStream_t s) {
  if (n <= 0) return 0;
  int64_t b = (n + 255) / 256;
  if (b > 148 * 64) b = 148 * 64;
  k_bin_keys<<<(unsigned)b, 256, 0, s>>>(g, bg, x, xs, n, key, err);
  return 1;
}

}  // namespace st
