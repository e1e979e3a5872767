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
#include <cuda_runtime.h>

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

// ---------------------------------------------------------------- bin geometry
__device__ __forceinline__ int div_cc(const BinGeom& b, int v, int cc) { return b.sh >= 0 ? (v >> b.sh) : v / cc; }

__device__ __forceinline__ int bin_of_cell(const Geom& g, const BinGeom& b, int cx, int cy, int cz) {
  const int cc = g.cc;
  const int kx = div_cc(b, cx, cc), ky = div_cc(b, cy, cc), kz = div_cc(b, cz, cc);
  const int chunk = ((kz - b.kz0) * g.NC[1] + ky) * g.NC[0] + kx;
  const int lc = ((cz - kz * cc) * cc + (cy - ky * cc)) * cc + (cx - kx * cc);
  return chunk * b.cc3 + lc;
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

__device__ __forceinline__ int slot_of(const Geom& g, int sx, int sy, int sz, int cx, int cy, int cz) {
  const int dx = axis_delta(sx, cx, g.n[0], g.bc[0]);
  const int dy = axis_delta(sy, cy, g.n[1], g.bc[1]);
  const int dz = axis_delta(sz, cz, g.n[2], g.bc[2]);
  if (dx == 2 || dy == 2 || dz == 2) return -1;
  return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
}

// ---------------------------------------------------------------- warp reductions
// Sum (a,b,c) over the lanes of `grp` (a lane mask containing the caller when
// member) with a masked butterfly: every lane gets the group total.
__device__ __forceinline__ void group_sum3(bool member, float& a, float& b, float& c) {
  if (!member) a = b = c = 0.0f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(kFull, a, o);
    b += __shfl_xor_sync(kFull, b, o);
    c += __shfl_xor_sync(kFull, c, o);
  }
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
  const int pz = g.gy * g.gx;
  const float4* b = F + ((int64_t)s.wz * pz + s.wy * g.gx + s.wx);
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
__global__ void __launch_bounds__(256, 4) k_step(StepArgs a) {
  __shared__ int run_s[8][kMaxBins * kSlots];
  __shared__ int rel_s[8][kMaxBins + 1];     // particle offsets of the item's bins, relative to p0
  __shared__ int cell_s[8][kMaxBins][3];      // cell coordinates of the item's bins
  const Geom& g = a.g;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int* run = run_s[wib];
  int* rel = rel_s[wib];
  const int n_items = *a.n_items;
  const int warps_total = gridDim.x * (blockDim.x >> 5);
  const int64_t cap = a.cap;
  const int nbins = a.nbins;
  int flags = 0, farflag = 0;
  unsigned movers = 0;

  for (int item = blockIdx.x * (blockDim.x >> 5) + wib; item < n_items; item += warps_total) {
    const int b0 = a.item_bin0[item];
    const int b1 = (item + 1 < n_items) ? a.item_bin0[item + 1] : nbins;
    const int nb = b1 - b0;
    const int64_t p0 = a.off[b0];
    for (int k = lane; k <= nb; k += 32) rel[k] = (int)(a.off[b0 + k] - p0);
    for (int k = lane; k < nb; k += 32) cell_of_bin(g, a.bg, b0 + k, cell_s[wib][k][0], cell_s[wib][k][1], cell_s[wib][k][2]);
    if (SCATTER)
      for (int k = lane; k < nb * kSlots; k += 32) run[k] = 0;
    __syncwarp();
    const int np = rel[nb];
    int lb_base = 0;
    for (int base = 0; base < np; base += 32) {
      const int r = base + lane;
      const bool valid = r < np;
      const int64_t i = p0 + r;
      // bin of the particle: last k >= lb_base with rel[k] <= r
      int lb = lb_base;
      if (valid) {
        int hi = nb - 1;
        while (lb < hi) {
          const int mid = (lb + hi + 1) >> 1;
          if (rel[mid] <= r) lb = mid;
          else hi = mid - 1;
        }
      }
      lb_base = __shfl_sync(kFull, lb, 0);
      const int s = b0 + lb;
      const int sx = cell_s[wib][lb][0], sy = cell_s[wib][lb][1], sz = cell_s[wib][lb][2];
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
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        t[ax] = cell_coord(xp[ax], g.lo[ax], g.ih[ax]);
        c[ax] = cell_from_t(t[ax], g.n[ax]);
      }
      // cell of the particle's bin in the output layout
      int ox = sx, oy = sy, oz = sz;
      int obin = s;
      int64_t dest = i;
      bool write_ok = valid;
      if (SCATTER) {
        const int j = valid ? slot_of(g, sx, sy, sz, c[0], c[1], c[2]) : -1;
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
          ox = c[0];
          oy = c[1];
          oz = c[2];
          obin = bin_of_cell(g, a.bg, ox, oy, oz);
          dest = a.off_new[obin] + (int64_t)a.slot_base[(int64_t)j * nbins + s] + rbase + __popc(peers & lanemask_lt());
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
#pragma unroll
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
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
              const float us = fmaf(a.p.g[ax], taue, ufa[ax]);
              const float rl = up[ax] - us;
              du[ax] = fmaf(-M, rl, -a.p.g[ax] * a.dt);
              xp[ax] = fmaf(tM, rl, fmaf(us, a.dt, xp[ax]));
              up[ax] = fmaf(E, rl, us);
            }
          } else {
            const float inv1h = __frcp_rn(1.0f + h);
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
              const float un = (up[ax] + h * ufa[ax] + a.dt * a.p.g[ax]) * inv1h;
              du[ax] = (un - up[ax]) - a.p.g[ax] * a.dt;
              xp[ax] = fmaf(a.dt, un, xp[ax]);
              up[ax] = un;
            }
          }
          if (a.p.two_way) {
            // deposit -w m du into the start cell: the largest group of lanes with
            // equal cells (cell-sorted warps) is reduced in registers, the rest red
            // directly; one red.global.add.v4.f32 per group
            const int az = acc_z(g, c[2]);
            if (valid && az < 0) flags |= ERRF_WINDOW;
            const bool dep = valid && az >= 0;
            const int ckey = dep ? (az * g.n[1] + c[1]) * g.n[0] + c[0] : -1 - lane;
            float ja = -mw * du[0], jb = -mw * du[1], jc = -mw * du[2];
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
#pragma unroll
          for (int ax = 0; ax < 3; ++ax)
            if (apply_bc(g.bc[ax], g.lo[ax], g.hi[ax], g.L[ax], xp[ax], up[ax]) && valid) flags |= ERRF_CFL;
        }
      }
      // slot histogram of the end position w.r.t. the output bin (next rebin's input)
      {
        int e[3];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) e[ax] = cell_from_t(cell_coord(xp[ax], g.lo[ax], g.ih[ax]), g.n[ax]);
        const int j2 = write_ok ? slot_of(g, ox, oy, oz, e[0], e[1], e[2]) : -1;
        if (write_ok && j2 < 0) farflag = 1;
        const long long hkey = (write_ok && j2 >= 0) ? (long long)j2 * nbins + obin : -1 - lane;
        const unsigned peers = __match_any_sync(kFull, hkey);
        if (hkey >= 0 && (peers & lanemask_lt()) == 0) atomicAdd(a.hist_next + hkey, __popc(peers));
        // chunk movers w.r.t. the output bins (the algorithmic rebin traffic)
        const bool mover = write_ok && (div_cc(a.bg, e[0], g.cc) != div_cc(a.bg, ox, g.cc) ||
                                        div_cc(a.bg, e[1], g.cc) != div_cc(a.bg, oy, g.cc) ||
                                        div_cc(a.bg, e[2], g.cc) != div_cc(a.bg, oz, g.cc));
        movers += mover ? 1u : 0u;
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
  // warp totals -> one atomic per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) movers += __shfl_xor_sync(kFull, movers, o);
  if (lane == 0 && movers) atomicAdd(a.movers, (unsigned long long)movers);
  if (flags) atomicOr(a.err, flags);
  if (farflag) *(volatile int*)a.far = 1;
}

// ---------------------------------------------------------------- rebin preparation
// Per destination bin d: sources s = d - delta over the 27 deltas (canonical,
// deduplicated), in ascending s; base[j][s] = running sum; new_cnt[d] = total.
// The slot-major layout makes consecutive threads touch consecutive words.
__global__ void k_rebin_prep(Geom g, BinGeom bg, int nbins, int* __restrict__ cnt_base, uint32_t* __restrict__ new_cnt) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nbins) return;
  int dx, dy, dz;
  cell_of_bin(g, bg, d, dx, dy, dz);
  if (dx >= g.n[0] || dy >= g.n[1] || dz >= g.n[2]) {   // ragged chunk: no such cell
    new_cnt[d] = 0;
    return;
  }
  const int kz_lo = bg.kz0, kz_hi = bg.kz0 + bg.nkz;
  // the 27 candidate sources s = d - delta(j); key = bin (INT_MAX if absent)
  int key[27], cnt[27];
#pragma unroll
  for (int j = 0; j < 27; ++j) {
    const int ox = j % 3 - 1, oy = (j / 3) % 3 - 1, oz = j / 9 - 1;
    bool ok = true;
    const int sx = axis_step(dx, -ox, g.n[0], g.bc[0], ok);
    const int sy = axis_step(dy, -oy, g.n[1], g.bc[1], ok);
    const int sz = axis_step(dz, -oz, g.n[2], g.bc[2], ok);
    if (ok) {
      const int kz = div_cc(bg, sz, g.cc);
      ok = kz >= kz_lo && kz < kz_hi &&                    // source on this rank
           slot_of(g, sx, sy, sz, dx, dy, dz) == j;          // canonical (no duplicate)
    }
    key[j] = ok ? bin_of_cell(g, bg, sx, sy, sz) : 0x7fffffff;
    cnt[j] = ok ? cnt_base[(int64_t)j * nbins + key[j]] : 0;
  }
  // stable order = ascending source bin: base of source q = sum of the counts of
  // the sources with a smaller bin (keys are distinct), all in registers
  uint32_t total = 0;
#pragma unroll
  for (int q = 0; q < 27; ++q) {
    uint32_t base = 0;
#pragma unroll
    for (int p = 0; p < 27; ++p) base += (key[p] < key[q]) ? (uint32_t)cnt[p] : 0u;
    if (key[q] != 0x7fffffff) cnt_base[(int64_t)q * nbins + key[q]] = (int)base;
    total += (uint32_t)cnt[q];
  }
  new_cnt[d] = total;
}

__global__ void k_hist_stay(const int64_t* __restrict__ off, int nbins, int* __restrict__ hist_row13) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nbins) hist_row13[s] = (int)(off[s + 1] - off[s]);
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
  k_rebin_prep<<<blocks_for(bg.nbins, 128), 128, 0, s>>>(g, bg, bg.nbins, cnt_base, new_cnt);
  return 1;
}

int launch_hist_all_stay(const int64_t* off, int nbins, int* hist, cudaStream_t s) {
  cudaMemsetAsync(hist, 0, (size_t)nbins * kSlots * sizeof(int), s);
  k_hist_stay<<<blocks_for(nbins), 256, 0, s>>>(off, nbins, hist + (int64_t)kStay * nbins);
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
