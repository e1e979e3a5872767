// KB2 + KB3 (fused form) — the binned particle step.
//
// Layout (C-15): the store is stable-sorted by the bin key
//   bin = local_chunk * cc^3 + ((lz*cc + ly)*cc + lx)
// (chunk-major, cells of a chunk in row-major order).  Between rebins every
// particle stays within one cell of its bin's cell per axis, so a rebin is a
// *neighbour-slot* stable counting sort: each particle of source bin s lands in
// one of the 27 neighbour bins d = s + delta(j).  Its destination is
//   dest = off_new[d] + base[s][j] + (# earlier particles of s with slot j)
// where base[s][j] = sum of cnt[s'][j'] over the sources s' < s of d (the
// stable order keeps source bins in ascending order, then the old order).
// cnt[s][j] is the slot histogram counted by the previous advance.
//
// One warp owns one "item" (<= kMaxBins consecutive bins); the kernel is
// persistent (grid-stride over items) and, per particle:
//   [SCATTER] slot j of the current cell w.r.t. the bin, rank by __match_any_sync,
//   [ADVANCE] locate -> trilinear u_f (L1-broadcast float4 loads) -> drag + gravity
//             exponential update -> deposit by warp segmented reduction over
//             equal cells (one red.global.add.v4.f32 per segment) -> walls / wrap,
//   [HIST]    slot of the end position w.r.t. the output bin, counted by segmented
//             reduction + one atomicAdd per segment (input of the next rebin),
//   then writes the particle to B[dest] (scatter) or back in place.
#include <cuda_runtime.h>

#include "st_device.cuh"
#include "st_step.h"

namespace st {

namespace {

constexpr int kSlots = 27;
constexpr int kStay = 13;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void red_add_v4(float4* addr, float a, float b, float c) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(0.0f)
               : "memory");
}

// ---------------------------------------------------------------- bin geometry
__device__ __forceinline__ int bin_of_cell(const Geom& g, const BinGeom& b, int cx, int cy, int cz) {
  const int cc = g.cc;
  const int kx = cx / cc, ky = cy / cc, kz = cz / cc;
  const int chunk = (kz * g.NC[1] + ky) * g.NC[0] + kx - g.chunk_base;
  const int lc = ((cz - kz * cc) * cc + (cy - ky * cc)) * cc + (cx - kx * cc);
  return chunk * b.cc3 + lc;
}

__device__ __forceinline__ void cell_of_bin(const Geom& g, const BinGeom& b, int bin, int& cx, int& cy, int& cz) {
  const int cc = g.cc;
  const int chunk = bin / b.cc3 + g.chunk_base;
  const int lc = bin - (bin / b.cc3) * b.cc3;
  const int kx = chunk % g.NC[0];
  const int ky = (chunk / g.NC[0]) % g.NC[1];
  const int kz = chunk / (g.NC[0] * g.NC[1]);
  const int lx = lc % cc, ly = (lc / cc) % cc, lz = lc / (cc * cc);
  cx = kx * cc + lx;
  cy = ky * cc + ly;
  cz = kz * cc + lz;
}

// canonical per-axis delta from -> to in {-1,0,1}; 2 = not a neighbour
__device__ __forceinline__ int axis_delta(int from, int to, int n, int bc) {
  int d = to - from;
  if (bc == ST_BC_PERIODIC && n >= 3) {
    if (d == n - 1) d = -1;
    else if (d == -(n - 1)) d = 1;
  }
  return (d >= -1 && d <= 1) ? d : 2;
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

// slot of cell (cx,cy,cz) relative to the cell (sx,sy,sz); -1 if not a neighbour
__device__ __forceinline__ int slot_of(const Geom& g, int sx, int sy, int sz, int cx, int cy, int cz) {
  const int dx = axis_delta(sx, cx, g.n[0], g.bc[0]);
  const int dy = axis_delta(sy, cy, g.n[1], g.bc[1]);
  const int dz = axis_delta(sz, cz, g.n[2], g.bc[2]);
  if (dx == 2 || dy == 2 || dz == 2) return -1;
  return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
}

// ---------------------------------------------------------------- warp helpers
// Inclusive segmented sum over lanes with equal `key` in consecutive lanes; lanes
// whose key differs from the next lane's (segment tails) return true.
__device__ __forceinline__ bool seg_sum3(long long key, float& a, float& b, float& c) {
  const int lane = threadIdx.x & 31;
  const long long kprev = __shfl_up_sync(0xffffffffu, key, 1);
  const long long knext = __shfl_down_sync(0xffffffffu, key, 1);
  bool head = (lane == 0) || (kprev != key);
  for (int off = 1; off < 32; off <<= 1) {
    const float ua = __shfl_up_sync(0xffffffffu, a, off);
    const float ub = __shfl_up_sync(0xffffffffu, b, off);
    const float uc = __shfl_up_sync(0xffffffffu, c, off);
    const int uh = __shfl_up_sync(0xffffffffu, (int)head, off);
    if (lane >= off && !head) {
      a += ua;
      b += ub;
      c += uc;
      head = uh;
    }
  }
  return (lane == 31) || (knext != key);
}

__device__ __forceinline__ bool seg_count(long long key, int& cnt) {
  const int lane = threadIdx.x & 31;
  const long long kprev = __shfl_up_sync(0xffffffffu, key, 1);
  const long long knext = __shfl_down_sync(0xffffffffu, key, 1);
  bool head = (lane == 0) || (kprev != key);
  for (int off = 1; off < 32; off <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, cnt, off);
    const int uh = __shfl_up_sync(0xffffffffu, (int)head, off);
    if (lane >= off && !head) {
      cnt += u;
      head = uh;
    }
  }
  return (lane == 31) || (knext != key);
}

struct Stencil {
  int wx, wy, wz;
  float fx, fy, fz;
};

__device__ __forceinline__ void stencil_axis(float t, int n, int& i, float& f) {
  const float s = t - 0.5f;
  const float fl = floorf(s);
  i = (int)fl;
  f = s - fl;
  if (i < -1) { i = -1; f = 0.0f; }
  if (i > n - 1) { i = n - 1; f = 1.0f; }
}

__device__ __forceinline__ float4 lerp4(float4 a, float4 b, float f) {
  return make_float4(fmaf(f, b.x - a.x, a.x), fmaf(f, b.y - a.y, a.y), fmaf(f, b.z - a.z, a.z), 0.0f);
}

__device__ __forceinline__ float4 trilinear(const Geom& g, const float4* __restrict__ F, const Stencil& s) {
  const int64_t pz = (int64_t)g.gy * g.gx;
  const float4* b = F + (int64_t)s.wz * pz + (int64_t)s.wy * g.gx + s.wx;
  const float4 c000 = __ldg(b), c100 = __ldg(b + 1);
  const float4 c010 = __ldg(b + g.gx), c110 = __ldg(b + g.gx + 1);
  const float4 c001 = __ldg(b + pz), c101 = __ldg(b + pz + 1);
  const float4 c011 = __ldg(b + pz + g.gx), c111 = __ldg(b + pz + g.gx + 1);
  const float4 c00 = lerp4(c000, c100, s.fx), c10 = lerp4(c010, c110, s.fx);
  const float4 c01 = lerp4(c001, c101, s.fx), c11 = lerp4(c011, c111, s.fx);
  const float4 c0 = lerp4(c00, c10, s.fy), c1 = lerp4(c01, c11, s.fy);
  return lerp4(c0, c1, s.fz);
}

// ---------------------------------------------------------------- the step kernel
template <bool SCATTER, bool ADVANCE>
__global__ void __launch_bounds__(256) k_step(StepArgs a) {
  __shared__ int run_s[8][kMaxBins * kSlots];
  __shared__ long long off_s[8][kMaxBins + 1];
  const Geom& g = a.g;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int* run = run_s[wib];
  long long* offw = off_s[wib];
  const int n_items = *a.n_items;
  const int warps_total = gridDim.x * (blockDim.x >> 5);
  const int64_t cap = a.cap;
  int flags = 0, farflag = 0;

  for (int item = blockIdx.x * (blockDim.x >> 5) + wib; item < n_items; item += warps_total) {
    const int b0 = a.item_bin0[item];
    const int b1 = (item + 1 < n_items) ? a.item_bin0[item + 1] : a.nbins;
    const int nb = b1 - b0;
    for (int k = lane; k <= nb; k += 32) offw[k] = a.off[b0 + k];
    if (SCATTER)
      for (int k = lane; k < nb * kSlots; k += 32) run[k] = 0;
    __syncwarp();
    const int64_t p0 = offw[0], p1 = offw[nb];
    for (int64_t base = p0; base < p1; base += 32) {
      const int64_t i = base + lane;
      const bool valid = i < p1;
      // bin of particle i: last k with offw[k] <= i
      int lb = 0;
      if (valid) {
        int lo = 0, hi = nb - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (offw[mid] <= i) lo = mid;
          else hi = mid - 1;
        }
        lb = lo;
      }
      const int s = b0 + lb;
      float xp[3] = {0.f, 0.f, 0.f}, up[3] = {0.f, 0.f, 0.f};
      float dp = 1e-5f, wp = 0.f;
      unsigned long long pid = 0;
      if (valid) {
        xp[0] = a.A.x[i]; xp[1] = a.A.x[cap + i]; xp[2] = a.A.x[2 * cap + i];
        up[0] = a.A.u[i]; up[1] = a.A.u[cap + i]; up[2] = a.A.u[2 * cap + i];
        dp = a.A.d[i];
        wp = a.A.w[i];
        if (SCATTER) pid = a.A.id[i];
      }
      // current cell (deposit cell of the first sub-step; scatter key)
      float t[3];
      int c[3];
      for (int ax = 0; ax < 3; ++ax) {
        t[ax] = cell_coord(xp[ax], g.lo[ax], g.ih[ax]);
        c[ax] = cell_from_t(t[ax], g.n[ax]);
      }
      int sx, sy, sz;
      cell_of_bin(g, a.bg, s, sx, sy, sz);
      int obin = s;   // bin of the particle in the output layout
      int64_t dest = i;
      bool write_ok = valid;
      if (SCATTER) {
        int j = valid ? slot_of(g, sx, sy, sz, c[0], c[1], c[2]) : -1;
        if (valid && j < 0) {
          flags |= ERRF_SCATTER;
          write_ok = false;
        }
        const int key = (valid && j >= 0) ? lb * kSlots + j : -1 - lane;
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(peers) - 1;
        int rbase = 0;
        if (lane == leader && key >= 0) {
          rbase = run[key];
          run[key] = rbase + __popc(peers);
        }
        rbase = __shfl_sync(0xffffffffu, rbase, leader);
        __syncwarp();
        if (write_ok) {
          obin = bin_of_cell(g, a.bg, c[0], c[1], c[2]);
          dest = a.off_new[obin] + (int64_t)a.slot_base[(int64_t)s * kSlots + j] + rbase + __popc(peers & lanemask_lt());
          if (dest < 0 || dest >= a.n) {
            flags |= ERRF_SCATTER;
            write_ok = false;
          }
        }
      }
      if (ADVANCE) {
        const float d = dp;
        const float tau = a.p.tau_c * d * d;
        const float inv_tau = __frcp_rn(tau);
        const float mw = a.p.mass_c * d * d * d * wp;
        for (int sub = 0; sub < a.nsteps; ++sub) {
          if (sub > 0) {
            for (int ax = 0; ax < 3; ++ax) {
              t[ax] = cell_coord(xp[ax], g.lo[ax], g.ih[ax]);
              c[ax] = cell_from_t(t[ax], g.n[ax]);
            }
          }
          Stencil st;
          int ix, iy, iz;
          stencil_axis(t[0], g.n[0], ix, st.fx);
          stencil_axis(t[1], g.n[1], iy, st.fy);
          stencil_axis(t[2], g.n[2], iz, st.fz);
          st.wx = ix + 1;
          st.wy = iy + 1;
          st.wz = window_z(g, iz);
          if (st.wz < 0 || st.wz + 1 >= g.wnz) {
            if (valid) flags |= ERRF_WINDOW;
            st.wz = st.wz < 0 ? 0 : g.wnz - 2;
          }
          const float4 uf = trilinear(g, a.field, st);
          const float sxv = uf.x - up[0], syv = uf.y - up[1], szv = uf.z - up[2];
          const float Re = sqrtf(fmaf(sxv, sxv, fmaf(syv, syv, szv * szv))) * d * a.p.inv_nu;
          const float f = drag_factor(a.p.drag_law, Re);
          const float taue = tau * __frcp_rn(f);
          const float h = a.dt * f * inv_tau;
          const float ufa[3] = {uf.x, uf.y, uf.z};
          float du[3];
          if (a.p.integrator == ST_INT_EXPONENTIAL) {
            float E, M;
            exp_pair(h, E, M);
            const float tM = taue * M;
            for (int ax = 0; ax < 3; ++ax) {
              const float us = fmaf(a.p.g[ax], taue, ufa[ax]);
              const float rel = up[ax] - us;
              du[ax] = fmaf(-M, rel, -a.p.g[ax] * a.dt);
              xp[ax] = fmaf(tM, rel, fmaf(us, a.dt, xp[ax]));
              up[ax] = fmaf(E, rel, us);
            }
          } else {
            const float inv1h = __frcp_rn(1.0f + h);
            for (int ax = 0; ax < 3; ++ax) {
              const float un = (up[ax] + h * ufa[ax] + a.dt * a.p.g[ax]) * inv1h;
              du[ax] = (un - up[ax]) - a.p.g[ax] * a.dt;
              xp[ax] = fmaf(a.dt, un, xp[ax]);
              up[ax] = un;
            }
          }
          if (a.p.two_way) {
            // deposit -w m du into the start cell: warp segmented reduction over
            // equal cells (cell-sorted warps -> one reduction per segment)
            const int az = acc_z(g, c[2]);
            if (valid && az < 0) flags |= ERRF_WINDOW;
            const bool dep = valid && az >= 0;
            const long long ckey = dep ? ((long long)az * g.n[1] + c[1]) * g.n[0] + c[0] : -1 - lane;
            float ja = dep ? -mw * du[0] : 0.f, jb = dep ? -mw * du[1] : 0.f, jc = dep ? -mw * du[2] : 0.f;
            const bool tail = seg_sum3(ckey, ja, jb, jc);
            if (tail && ckey >= 0) red_add_v4(a.acc + ckey, ja, jb, jc);
          }
          for (int ax = 0; ax < 3; ++ax)
            if (apply_bc(g.bc[ax], g.lo[ax], g.hi[ax], g.L[ax], xp[ax], up[ax]) && valid) flags |= ERRF_CFL;
        }
      }
      // slot histogram of the end position w.r.t. the output bin (next rebin's input)
      {
        int e[3];
        for (int ax = 0; ax < 3; ++ax) e[ax] = cell_from_t(cell_coord(xp[ax], g.lo[ax], g.ih[ax]), g.n[ax]);
        int ox, oy, oz;
        cell_of_bin(g, a.bg, obin, ox, oy, oz);
        const int j2 = write_ok ? slot_of(g, ox, oy, oz, e[0], e[1], e[2]) : -1;
        if (write_ok && j2 < 0) farflag = 1;
        const long long hkey = (write_ok && j2 >= 0) ? (long long)obin * kSlots + j2 : -1 - lane;
        int cnt = (hkey >= 0) ? 1 : 0;
        const bool tail = seg_count(hkey, cnt);
        if (tail && hkey >= 0) atomicAdd(a.hist_next + hkey, cnt);
        // chunk movers w.r.t. the output bins (the algorithmic rebin traffic)
        const bool mover = write_ok && ((e[0] / g.cc) != (ox / g.cc) || (e[1] / g.cc) != (oy / g.cc) ||
                                        (e[2] / g.cc) != (oz / g.cc));
        const unsigned mb = __ballot_sync(0xffffffffu, mover);
        if (lane == 0 && mb) atomicAdd(a.movers, (unsigned long long)__popc(mb));
      }
      if (write_ok) {
        if (SCATTER) {
          a.B.x[dest] = xp[0]; a.B.x[cap + dest] = xp[1]; a.B.x[2 * cap + dest] = xp[2];
          a.B.u[dest] = up[0]; a.B.u[cap + dest] = up[1]; a.B.u[2 * cap + dest] = up[2];
          a.B.d[dest] = dp;
          a.B.w[dest] = wp;
          a.B.id[dest] = pid;
        } else if (ADVANCE) {
          a.A.x[i] = xp[0]; a.A.x[cap + i] = xp[1]; a.A.x[2 * cap + i] = xp[2];
          a.A.u[i] = up[0]; a.A.u[cap + i] = up[1]; a.A.u[2 * cap + i] = up[2];
        }
      }
    }
    __syncwarp();
  }
  if (flags) atomicOr(a.err, flags);
  if (farflag) *(volatile int*)a.far = 1;
}

// ---------------------------------------------------------------- rebin preparation
// Per destination bin d: sources s = d - delta over the 27 deltas (canonical,
// deduplicated), in ascending s; base[s][j] = running sum; new_cnt[d] = total.
__global__ void k_rebin_prep(Geom g, BinGeom bg, int nbins, int* __restrict__ cnt_base, uint32_t* __restrict__ new_cnt) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nbins) return;
  int dx, dy, dz;
  cell_of_bin(g, bg, d, dx, dy, dz);
  if (dx >= g.n[0] || dy >= g.n[1] || dz >= g.n[2]) {   // ragged chunk: no such cell
    new_cnt[d] = 0;
    return;
  }
  int src[27], slot[27], ns = 0;
  for (int oz = -1; oz <= 1; ++oz)
    for (int oy = -1; oy <= 1; ++oy)
      for (int ox = -1; ox <= 1; ++ox) {
        bool ok = true;
        const int sx = axis_step(dx, -ox, g.n[0], g.bc[0], ok);
        const int sy = axis_step(dy, -oy, g.n[1], g.bc[1], ok);
        const int sz = axis_step(dz, -oz, g.n[2], g.bc[2], ok);
        if (!ok) continue;
        const int kz = sz / g.cc;
        const int kz_lo = g.chunk_base / (g.NC[0] * g.NC[1]);
        if (kz < kz_lo || kz >= kz_lo + bg.nkz) continue;   // source outside this rank's bins
        const int j = slot_of(g, sx, sy, sz, dx, dy, dz);
        if (j != (oz + 1) * 9 + (oy + 1) * 3 + (ox + 1)) continue;   // non-canonical duplicate
        const int s = bin_of_cell(g, bg, sx, sy, sz);
        // insertion by ascending s
        int q = ns++;
        while (q > 0 && src[q - 1] > s) {
          src[q] = src[q - 1];
          slot[q] = slot[q - 1];
          --q;
        }
        src[q] = s;
        slot[q] = j;
      }
  uint32_t run = 0;
  for (int q = 0; q < ns; ++q) {
    int* e = cnt_base + (int64_t)src[q] * kSlots + slot[q];
    const int v = *e;
    *e = (int)run;
    run += (uint32_t)v;
  }
  new_cnt[d] = run;
}

__global__ void k_hist_all_stay(const int64_t* __restrict__ off, int nbins, int* __restrict__ hist) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (int64_t)nbins * kSlots) return;
  const int s = (int)(q / kSlots), j = (int)(q - (int64_t)s * kSlots);
  hist[q] = (j == kStay) ? (int)(off[s + 1] - off[s]) : 0;
}

// item boundaries: bin s starts an item if s % kMaxBins == 0 or the kItemParticles
// window of its first particle differs from that of bin s-1's first particle.
__global__ void k_item_flags(const int64_t* __restrict__ off, int nbins, uint32_t* __restrict__ flag) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nbins) return;
  uint32_t f = (s % kMaxBins) == 0;
  if (!f) f = (off[s] / kItemParticles) != (off[s - 1] / kItemParticles);
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
    int b = bin_of_cell(g, bg, c[0], c[1], c[2]);
    if (b < 0 || b >= bg.nbins) {   // outside this rank's bins (multi-GPU: migrates first)
      atomicOr(err, ERRF_WINDOW);
      b = b < 0 ? 0 : bg.nbins - 1;
    }
    key[i] = b;
  }
}

inline unsigned blocks_for(int64_t n, int bs = 256) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

int step_occupancy_grid(bool scatter, bool advance) {
  static int cache[4] = {0, 0, 0, 0};
  const int idx = (scatter ? 2 : 0) + (advance ? 1 : 0);
  if (cache[idx]) return cache[idx];
  int nsm = 148, dev = 0, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (scatter && advance) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_step<true, true>, 256, 0);
  else if (scatter) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_step<true, false>, 256, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_step<false, true>, 256, 0);
  cache[idx] = nsm * (per > 0 ? per : 1);
  return cache[idx];
}

int launch_step(const StepArgs& a, bool scatter, bool advance, cudaStream_t s) {
  const int grid = step_occupancy_grid(scatter, advance);
  if (scatter && advance) k_step<true, true><<<grid, 256, 0, s>>>(a);
  else if (scatter) k_step<true, false><<<grid, 256, 0, s>>>(a);
  else k_step<false, true><<<grid, 256, 0, s>>>(a);
  return 1;
}

int launch_rebin_prep(const Geom& g, const BinGeom& bg, int* cnt_base, uint32_t* new_cnt, cudaStream_t s) {
  k_rebin_prep<<<blocks_for(bg.nbins), 256, 0, s>>>(g, bg, bg.nbins, cnt_base, new_cnt);
  return 1;
}

int launch_hist_all_stay(const int64_t* off, int nbins, int* hist, cudaStream_t s) {
  k_hist_all_stay<<<blocks_for((int64_t)nbins * kSlots), 256, 0, s>>>(off, nbins, hist);
  return 1;
}

int launch_items(const int64_t* off, int nbins, uint32_t* flag, int64_t* pos, int64_t* partial, int* item_bin0,
                 int* n_items, cudaStream_t s) {
  k_item_flags<<<blocks_for(nbins), 256, 0, s>>>(off, nbins, flag);
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
