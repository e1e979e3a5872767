// k_ip — the in-place particle step for 8^3-cell chunks, two particles per lane
// (included by k_step.cu after k_pstep.cuh: uses its bin geometry, slot, mbarrier, TMA
// and window helpers).  Rows a2-a7 of SURVEY §8(a) between rebins, plus the slot
// histogram of the next rebin when this call makes one due (COUNT).
//
// Why a separate kernel: at the bench's density (C5, ~377 particles per cell) the
// round-1 in-place launch issued ~520 warp-instructions per 32 particles and ran at
// the issue roofline (ncu r2a: 76 % issue-active).  Most of it was per-batch
// bookkeeping (bin walk, accumulator flush votes, mbarrier/TMA issue, reloaded kernel
// parameters) and MUFU denormal fix-ups.  Here:
//  * a batch is 64 particles (two per lane, lanes k and k+32 of one TMA box {68, 8}),
//    so every per-batch cost is paid once per 64 particles and the two particles give
//    the scheduler independent chains;
//  * the bin of a batch is warp-uniform in the common case (one compare against the
//    current bin's end); only batches that straddle a bin boundary walk per lane;
//  * the register accumulator of the deposit (and of the stayer count) belongs to the
//    warp's current bin cell, so it is flushed once per bin, not voted per batch;
//  * ex2/lg2/rcp/sqrt are the .ftz MUFU forms (no denormal range fix-ups).
// Semantics are the round-1 kernel's (same readings C-2..C-12, same deposit cell C-10,
// same slot / far rules C-15 / C-15b).
#pragma once

__device__ __forceinline__ float ex2_ftz(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2_ftz(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

#ifndef ST_DYN_ITEMS
#define ST_DYN_ITEMS 1   // step kernels take their items from a counter (k_ip, k_fs)
#endif


// Packed fp32 pairs (FADD2 / FMUL2 / FFMA2 of sm_100): the x and y components of a
// particle's vectors travel as one float2 and z alone, so each 3-vector operation is two
// instructions instead of three.  Every packed operation rounds each half exactly like
// the scalar one it replaces (same operands, same order, RN), so results are unchanged.
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 neg2(float2 v) { return make_float2(-v.x, -v.y); }
struct V3 {
  float2 xy;
  float z;
};
__device__ __forceinline__ V3 lerp3(const float4& a, const float4& b, float f) {
  V3 r;
  r.xy = __ffma2_rn(bc2(f), __fadd2_rn(f2(b.x, b.y), f2(-a.x, -a.y)), f2(a.x, a.y));
  r.z = fmaf(f, b.z - a.z, a.z);
  return r;
}
__device__ __forceinline__ V3 lerp3(const V3& a, const V3& b, float f) {
  V3 r;
  r.xy = __ffma2_rn(bc2(f), __fadd2_rn(b.xy, neg2(a.xy)), a.xy);
  r.z = fmaf(f, b.z - a.z, a.z);
  return r;
}
// C-5: the trilinear of trilerp() (same lerp tree, x then y then z)
__device__ __forceinline__ V3 trilerp3(const float4 (&q)[8], float fx, float fy, float fz) {
  return lerp3(lerp3(lerp3(q[0], q[1], fx), lerp3(q[2], q[3], fx), fy),
               lerp3(lerp3(q[4], q[5], fx), lerp3(q[6], q[7], fx), fy), fz);
}
// C-6 cell coordinates of (x, y): (x - lo) * ih per component, each rounded (cell_coord)
__device__ __forceinline__ float2 cell_coord2(float x, float y, float2 nlo, float2 ih) {
  return __fmul2_rn(__fadd2_rn(f2(x, y), nlo), ih);
}
// stencil_lo() of (tx, ty)
__device__ __forceinline__ void stencil_lo2(float2 t, int& i0, int& i1, float& f0, float& f1) {
  const float2 sh = __fadd2_rn(t, bc2(-0.5f));
  i0 = __float2int_rd(sh.x);
  i1 = __float2int_rd(sh.y);
  const float2 f = __fadd2_rn(sh, f2(-(float)i0, -(float)i1));
  f0 = f.x;
  f1 = f.y;
}

constexpr int kIpStages = 3;
constexpr int kIpBoxF = 68;                          // 64 particles + 4 floats of 16-B alignment slack
constexpr int kIpStageBytes = 8 * kIpBoxF * 4;       // 2176 = 17 x 128
constexpr int kIpWX = 12, kIpWYZ = 5;                // window of R = 1 (k_pstep.cuh, tm_win[1])
constexpr int kIpOffWin = kIpStages * kIpStageBytes;                 // 6528 (128-B aligned)
constexpr int kIpOffCnt = kIpOffWin + kIpWX * kIpWYZ * kIpWYZ * 16;  // + 4800
constexpr int kIpOffRel = kIpOffCnt + kTable * 4;                    // + 864
constexpr int kIpOffBar = kIpOffRel + 48;
constexpr int kIpWarpBytes = (kIpOffBar + 8 * (kIpStages + 1) + 127) / 128 * 128;   // 12288
constexpr int kIpWarps = 8;
constexpr uint32_t kIpTx = 8u * kIpBoxF * 4u;

template <int BCM, int SPEC, bool COUNT>
__global__ void __launch_bounds__(32 * kIpWarps, 2) k_ip(const __grid_constant__ StepArgs a) {
  constexpr int SH = 3;
  constexpr bool VP = (SPEC & kSpecVP) != 0;     // multi-rank window (z halos, wrap)
  constexpr bool SUB = (SPEC & kSpecSub) != 0;   // more than one sub-step per call
  extern __shared__ __align__(128) unsigned char ipsmem_raw[];
  const Geom& g = a.g;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* sbase = ipsmem_raw + ((kPSmemAlign - (smem_u32(ipsmem_raw) & (kPSmemAlign - 1))) & (kPSmemAlign - 1));
  unsigned char* ws = sbase + (size_t)wib * kIpWarpBytes;
  float4* win = reinterpret_cast<float4*>(ws + kIpOffWin);
  int* cnt_s = reinterpret_cast<int*>(ws + kIpOffCnt);
  int* rel = reinterpret_cast<int*>(ws + kIpOffRel);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(ws + kIpOffBar);
  unsigned long long* ibar = bar + kIpStages;
  const uint32_t stage0 = smem_u32(ws);
  const uint32_t win0 = smem_u32(win);
  const int n_items = *a.n_items;
  const int warps_total = gridDim.x * kIpWarps;
  const int64_t cap = a.cap;
  const int nbins = a.nbins;
  const bool two_way = a.p.two_way != 0;
  const float dt = a.dt;
  int cfar = 0, flags = 0;
  uint32_t phase = 0, iphase = 0;
  if (lane == 0) {
    for (int k = 0; k <= kIpStages; ++k) mbar_init(bar + k, 1);
    fence_mbar_init();
  }
  __syncwarp();

  // items: the first one per warp is static, the rest are handed out by a counter
  // (ST_DYN_ITEMS; clustered loads make item sizes uneven) and their headers are
  // fetched one item ahead, while the current item's batches run
  const bool dyn = ST_DYN_ITEMS && a.item_ctr != nullptr;
  int item = blockIdx.x * kIpWarps + wib;
  // the next item's header in two phases, so that no load is consumed right after it is
  // issued: its bins (after the first batch, once the counter's answer is in), then their
  // offsets (after the second batch); consumed at the next item's start
  int hb0 = 0, hb1 = 0;
  int64_t hp0 = 0, hoff = 0;
  auto header1 = [&](int it) {
    hb0 = a.item_bin0[it];
    hb1 = (it + 1 < n_items) ? a.item_bin0[it + 1] : nbins;
  };
  auto header2 = [&]() {
    hp0 = a.off[hb0];
    hoff = (lane <= hb1 - hb0) ? a.off[hb0 + lane] : hp0;
  };
  if (item < n_items) {
    header1(item);
    header2();
  }
  while (item < n_items) {
    const int b0 = hb0, b1 = hb1;
    const int nb = b1 - b0;                       // <= 8, one chunk row along +x
    const int64_t p0 = hp0;
    const int myrel = (int)(hoff - hp0);
    const int np = __shfl_sync(kFull, myrel, nb);
    const int nbatch = (np + 63) >> 6;
    int tk = 0;
    int next = item + warps_total;
    auto prefetch1 = [&]() {
      if (dyn) next = warps_total + __shfl_sync(kFull, tk, 0);
      if (next < n_items) header1(next);
    };
    auto prefetch2 = [&]() {
      if (next < n_items) header2();
    };
    int rx, ry, rz;
    cell_of_bin(g, a.bg, b0, rx, ry, rz);
    if (lane == 0) {
      fence_proxy_async();
      mbar_expect_tx(ibar, (uint32_t)(kIpWX * kIpWYZ * kIpWYZ * 16));
      tma_win(win, &a.tm_win[1], 4 * (rx - 1), ry - 1, window_z(g, rz) - 2, ibar);
      for (int k = 0; k < kIpStages && k < nbatch; ++k) {
        mbar_expect_tx(bar + k, kIpTx);
        tma_rows(ws + k * kIpStageBytes, &a.tm_f64, (int)((p0 + 64 * k) & ~3LL), bar + k);
      }
    }
    __syncwarp();
    // the next item from the counter, issued after this item's copies (the proxy fence
    // before them would otherwise wait for the atomic's round trip)
    if (dyn && lane == 0) tk = atomicAdd(a.item_ctr, 1);
    if (lane <= nb) rel[lane] = myrel;
    if (COUNT)
      for (int k = lane; k < kTable; k += 32) cnt_s[k] = 0;
    mbar_wait(ibar, iphase);
    iphase ^= 1u;
    __syncwarp();
    const int az_row = VP ? acc_z(g, rz) : rz - g.az0;
    // warp-uniform state: bin of the next batch's first particle (cb, ending at ce) and
    // the bin whose cell owns the register accumulators (acb)
    int cb = 0, ce = rel[1], acb = -1;
    float da0 = 0.f, da1 = 0.f, da2 = 0.f;
    int hc = 0;
    auto flush = [&]() {   // warp-uniform: acb's accumulators to HBM / the smem histogram
      if (acb < 0) return;
      if (two_way) {
        float ra = da0, rb = da1, rc = da2;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ra += __shfl_xor_sync(kFull, ra, o);
          rb += __shfl_xor_sync(kFull, rb, o);
          rc += __shfl_xor_sync(kFull, rc, o);
        }
        if (lane == 0) red_add_v4(a.acc + (uint32_t)((az_row * g.n[1] + ry) * g.n[0] + rx + acb), ra, rb, rc);
      }
      if (COUNT) {
        const int hs = (int)__reduce_add_sync(kFull, (unsigned)hc);
        if (lane == 0 && hs) cnt_s[acb * kSlots + kStay] += hs;
      }
      da0 = da1 = da2 = 0.f;
      hc = 0;
    };
    for (int bi = 0; bi < nbatch; ++bi) {
      const int base = bi << 6;
      while (ce <= base) ce = rel[++cb + 1];       // uniform: bin of the batch's first particle
      if (cb != acb) {
        __syncwarp();
        flush();
        acb = cb;
      }
      const int last = min(base + 63, np - 1);
      int lb[2] = {cb, cb};
      int r[2];
      bool valid[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int rr = base + 32 * q + lane;
        valid[q] = rr < np;
        r[q] = valid[q] ? rr : np - 1;             // idle lanes mirror a valid particle
      }
      if (last >= ce) {                            // the batch straddles a bin boundary
#pragma unroll
        for (int q = 0; q < 2; ++q)
          while (rel[lb[q] + 1] <= r[q]) ++lb[q];
      }
      // stage -> registers, then refill the stage kIpStages batches ahead
      const int sk = bi % kIpStages;
      mbar_wait(bar + sk, (phase >> sk) & 1u);
      __syncwarp();
      phase ^= 1u << sk;
      float x[2][3], u[2][3], dp[2], wp[2];
      {
        const uint32_t sa = stage0 + sk * kIpStageBytes + 4u * (uint32_t)(((p0 + base) & 3) + lane);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const uint32_t s = sa + 128u * q;
          // lanes past the end read the stage's zero-filled / stale tail: mirrored below
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x[q][0]) : "r"(s));
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x[q][1]) : "r"(s + 1u * kIpBoxF * 4));
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x[q][2]) : "r"(s + 2u * kIpBoxF * 4));
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(u[q][0]) : "r"(s + 3u * kIpBoxF * 4));
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(u[q][1]) : "r"(s + 4u * kIpBoxF * 4));
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(u[q][2]) : "r"(s + 5u * kIpBoxF * 4));
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(dp[q]) : "r"(s + 6u * kIpBoxF * 4));
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(wp[q]) : "r"(s + 7u * kIpBoxF * 4));
        }
      }
      if (base + 63 >= np) {   // tail batch (warp-uniform): idle lanes mirror lane 0's particle
        float m[8] = {x[0][0], x[0][1], x[0][2], u[0][0], u[0][1], u[0][2], dp[0], wp[0]};
#pragma unroll
        for (int k = 0; k < 8; ++k) m[k] = __shfl_sync(kFull, m[k], 0);
#pragma unroll
        for (int q = 0; q < 2; ++q)
          if (!valid[q]) {
            x[q][0] = m[0]; x[q][1] = m[1]; x[q][2] = m[2];
            u[q][0] = m[3]; u[q][1] = m[4]; u[q][2] = m[5];
            dp[q] = m[6]; wp[q] = m[7];
          }
      }
      __syncwarp();
      if (lane == 0 && bi + kIpStages < nbatch) {
        fence_proxy_async();
        mbar_expect_tx(bar + sk, kIpTx);
        tma_rows(ws + sk * kIpStageBytes, &a.tm_f64, (int)((p0 + base + 64 * kIpStages) & ~3LL), bar + sk);
      }
      __syncwarp();

      const float gx = a.p.g[0], gy = a.p.g[1], gz = a.p.g[2];
      const float2 gxy = f2(gx, gy), ngdt = f2(-gx * dt, -gy * dt);
      const float2 nlo = f2(-g.lo[0], -g.lo[1]), ihv = f2(g.ih[0], g.ih[1]);
      float tau[2], inv_tau[2], mw[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        tau[q] = a.p.tau_c * dp[q] * dp[q];
        inv_tau[q] = rcp_approx(tau[q]);
        mw[q] = a.p.mass_c * dp[q] * dp[q] * dp[q] * wp[q];
      }
      const int nsub = SUB ? a.nsteps : 1;
      for (int sub = 0; sub < nsub; ++sub) {
        int c[2][3];
        V3 ufq[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          int i0[3];
          float f[3];
          {
            const float2 txy = cell_coord2(x[q][0], x[q][1], nlo, ihv);
            const float tz = cell_coord(x[q][2], g.lo[2], g.ih[2]);
            c[q][0] = cell_from_t(txy.x, g.n[0]);
            c[q][1] = cell_from_t(txy.y, g.n[1]);
            c[q][2] = cell_from_t(tz, g.n[2]);
            stencil_lo2(txy, i0[0], i0[1], f[0], f[1]);
            stencil_lo(tz, i0[2], f[2]);
          }
          float4 q8[8];
          const bool inw = (unsigned)(i0[0] - rx + 2) <= 10u && (unsigned)(i0[1] - ry + 2) <= 3u &&
                           (unsigned)(i0[2] - rz + 2) <= 3u;
          if (__all_sync(kFull, inw)) {            // binned: the item's smem window
            const uint32_t w0 =
                win0 + 16u * (uint32_t)(((i0[2] - rz + 2) * kIpWYZ + (i0[1] - ry + 2)) * kIpWX + (i0[0] - rx + 2));
            constexpr uint32_t oy = kIpWX * 16, oz = kIpWYZ * kIpWX * 16;
            q8[0] = lds4(w0); q8[1] = lds4(w0 + 16); q8[2] = lds4(w0 + oy); q8[3] = lds4(w0 + oy + 16);
            q8[4] = lds4(w0 + oz); q8[5] = lds4(w0 + oz + 16); q8[6] = lds4(w0 + oz + oy);
            q8[7] = lds4(w0 + oz + oy + 16);
          } else {                                 // a lane left the window: generic loads
            int wz = VP ? window_z(g, i0[2]) : i0[2] - g.wz0;
            if (VP && (wz < 0 || wz + 1 >= g.wnz)) {
              if (valid[q]) flags |= ERRF_WINDOW;
              wz = wz < 0 ? 0 : g.wnz - 2;
            }
            const int pz = g.gy * g.gx;
            const float4* fb = inw ? win + ((i0[2] - rz + 2) * kIpWYZ + (i0[1] - ry + 2)) * kIpWX + (i0[0] - rx + 2)
                                   : a.field + ((int64_t)wz * pz + (i0[1] + 1) * g.gx + (i0[0] + 1));
            const int oy = inw ? kIpWX : g.gx, oz = inw ? kIpWYZ * kIpWX : pz;
            q8[0] = ld4(fb); q8[1] = ld4(fb + 1); q8[2] = ld4(fb + oy); q8[3] = ld4(fb + oy + 1);
            q8[4] = ld4(fb + oz); q8[5] = ld4(fb + oz + 1); q8[6] = ld4(fb + oz + oy);
            q8[7] = ld4(fb + oz + oy + 1);
          }
          ufq[q] = trilerp3(q8, f[0], f[1], f[2]);
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const V3 uf = ufq[q];
          const float2 sxy = __fadd2_rn(uf.xy, f2(-u[q][0], -u[q][1]));
          const float s0 = sxy.x, s1 = sxy.y, s2 = uf.z - u[q][2];
          const float Re = sqrt_approx(fmaf(s0, s0, fmaf(s1, s1, s2 * s2))) * dp[q] * a.p.inv_nu;
          float fd = fmaf(0.15f, ex2_ftz(0.687f * lg2_ftz(Re)), 1.0f);   // Re = 0: lg2 -> -inf, ex2 -> 0
          fd = (Re <= 1000.0f) ? fd : (0.44f / 24.0f) * Re;
          fd = (a.p.drag_law == ST_DRAG_STOKES) ? 1.0f : fd;
          const float taue = tau[q] * rcp_approx(fd);
          const float h = dt * fd * inv_tau[q];
          float2 duxy;
          float du2;
          if (a.p.integrator == ST_INT_EXPONENTIAL) {
            const float E = ex2_ftz(-1.44269504088896341f * h);
            const float Ms = h * (1.0f - h * (0.5f - h * (1.0f / 6.0f - h * (1.0f / 24.0f - h * (1.0f / 120.0f - h * (1.0f / 720.0f))))));
            const float M = h < 0.125f ? Ms : 1.0f - E;
            const float tM = taue * M;
            const float2 usxy = __ffma2_rn(gxy, bc2(taue), uf.xy);
            const float us2 = fmaf(gz, taue, uf.z);
            const float2 rxy = __fadd2_rn(f2(u[q][0], u[q][1]), neg2(usxy));
            const float r2 = u[q][2] - us2;
            duxy = __ffma2_rn(bc2(-M), rxy, ngdt);
            du2 = fmaf(-M, r2, -gz * dt);
            const float2 xn = __ffma2_rn(bc2(tM), rxy, __ffma2_rn(usxy, bc2(dt), f2(x[q][0], x[q][1])));
            x[q][0] = xn.x;
            x[q][1] = xn.y;
            x[q][2] = fmaf(tM, r2, fmaf(us2, dt, x[q][2]));
            const float2 un = __ffma2_rn(bc2(E), rxy, usxy);
            u[q][0] = un.x;
            u[q][1] = un.y;
            u[q][2] = fmaf(E, r2, us2);
          } else {
            const float inv1h = rcp_approx(1.0f + h);
            const float un0 = (u[q][0] + h * uf.xy.x + dt * gx) * inv1h;
            const float un1 = (u[q][1] + h * uf.xy.y + dt * gy) * inv1h;
            const float un2 = (u[q][2] + h * uf.z + dt * gz) * inv1h;
            duxy = f2((un0 - u[q][0]) - gx * dt, (un1 - u[q][1]) - gy * dt);
            du2 = (un2 - u[q][2]) - gz * dt;
            x[q][0] = fmaf(dt, un0, x[q][0]);
            x[q][1] = fmaf(dt, un1, x[q][1]);
            x[q][2] = fmaf(dt, un2, x[q][2]);
            u[q][0] = un0;
            u[q][1] = un1;
            u[q][2] = un2;
          }
          if (two_way) {
            // reaction into the sub-step start cell (Eq. 11, C-10): the warp's accumulator
            // cell in registers, any other cell by one red.global.add.v4
            const bool v = valid[q];
            const float2 jxy = __fmul2_rn(bc2(-mw[q]), duxy);
            const float ja = jxy.x, jb = jxy.y, jc = -mw[q] * du2;
            if (v && c[q][0] == rx + acb && c[q][1] == ry && c[q][2] == rz) {
              const float2 dn = __fadd2_rn(f2(da0, da1), jxy);
              da0 = dn.x;
              da1 = dn.y;
              da2 += jc;
            } else if (v) {
              const int az = VP ? acc_z(g, c[q][2]) : c[q][2] - g.az0;
              if (VP && az < 0) flags |= ERRF_WINDOW;
              else red_add_v4(a.acc + (uint32_t)((az * g.n[1] + c[q][1]) * g.n[0] + c[q][0]), ja, jb, jc);
            }
          }
        }
        // walls / wrap (C-11, C-12): one vote skips the axes when no lane left the box
        bool out = false;
#pragma unroll
        for (int q = 0; q < 2; ++q)
          out |= (x[q][0] < g.lo[0]) | (x[q][0] >= g.hi[0]) | (x[q][1] < g.lo[1]) | (x[q][1] >= g.hi[1]) |
                 (x[q][2] < g.lo[2]) | (x[q][2] >= g.hi[2]);
        if (__any_sync(kFull, out)) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            bool bad = false;
#pragma unroll
            for (int k = 0; k < 3; ++k)
              bad |= apply_bc(periodic<BCM>(g, k) ? ST_BC_PERIODIC : ST_BC_REFLECT, g.lo[k], g.hi[k], g.L[k], x[q][k],
                              u[q][k]);
            if (bad && valid[q]) flags |= ERRF_CFL;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (!valid[q]) continue;
        if (COUNT) {
          // slot of the end cell relative to the particle's bin (the next rebin's input)
          const int sx = rx + lb[q];
          const float2 exy = cell_coord2(x[q][0], x[q][1], nlo, ihv);
          const int e0 = cell_from_t(exy.x, g.n[0]);
          const int e1 = cell_from_t(exy.y, g.n[1]);
          const int e2 = cell_from_t(cell_coord(x[q][2], g.lo[2], g.ih[2]), g.n[2]);
          const int j = slot_of<BCM>(g, sx, ry, rz, e0, e1, e2);
          if (j == kStay && lb[q] == acb) {
            ++hc;
          } else if (j >= 0) {
            atomicAdd(&cnt_s[lb[q] * kSlots + j], 1);
          } else {   // far (C-15b): counted for the bin of its cell when that is on this rank
            const int kz = e2 >> SH;
            int side, pl;
            if (a.cnt_far_cnt && kz >= a.bg.kz0 && kz < a.bg.kz0 + a.bg.nkz) {
              atomicAdd(a.cnt_far_cnt + bin_of_cell<SH>(g, a.bg, e0, e1, e2), 1);
              atomicAdd(a.cnt_far_n, 1ULL);
            } else if (VP && a.cnt_fv[0] && far_plane(g, e2, side, pl)) {
              // a neighbour rank's cell: counted per cell of its window (k_far_accept there)
              atomicAdd(a.cnt_fv[side] + ((int64_t)pl * g.n[1] + e1) * g.n[0] + e0, 1);
              atomicAdd(a.cnt_fs_n + side, 1ULL);
              atomicAdd(a.cnt_far_n, 1ULL);
            } else {
              cfar = 1;
            }
          }
        }
        const int64_t i = p0 + r[q];
        __stcs(a.A.x + i, x[q][0]); __stcs(a.A.x + cap + i, x[q][1]); __stcs(a.A.x + 2 * cap + i, x[q][2]);
        __stcs(a.A.u + i, u[q][0]); __stcs(a.A.u + cap + i, u[q][1]); __stcs(a.A.u + 2 * cap + i, u[q][2]);
      }
      if (bi == 0) prefetch1();
      if (bi == 1) prefetch2();
    }
    if (nbatch == 0) prefetch1();
    if (nbatch <= 1) prefetch2();
    __syncwarp();
    flush();
    __syncwarp();
    if (COUNT) {   // the item's bins are this warp's: plain stores, every entry; lanes
      // 8s..8s+7 write one slot row's 8 consecutive bins (one 32-B sector of the slot-major
      // histogram) instead of 32 different rows
      for (int k = lane; k < kSlots * kRowBins; k += 32) {
        const int j = k >> 3, l = k & 7;
        if (l < nb) a.cnt_hist[(int64_t)j * nbins + b0 + l] = cnt_s[l * kSlots + j];
      }
      __syncwarp();
    }
    item = next;
  }
  // (the chunk movers of the statistics are summed from the histogram by k_rebin_prep)
  if (COUNT && cfar) *(volatile int*)a.cnt_far = 1;
  if (flags) atomicOr(a.err, flags);
}

template <int BCM, int SPEC, bool COUNT>
int launch_ip_variant(const StepArgs& a, cudaStream_t s) {
  static int grid = 0;
  const int smem = kIpWarps * kIpWarpBytes + kPSmemAlign;
  if (!grid) {
    int nsm = 148, dev = 0, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_ip<BCM, SPEC, COUNT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_ip<BCM, SPEC, COUNT>, 32 * kIpWarps, smem);
    grid = nsm * (per > 0 ? per : 1);
  }
  if (ST_DYN_ITEMS && a.item_ctr) cudaMemsetAsync(a.item_ctr, 0, sizeof(int), s);
  k_ip<BCM, SPEC, COUNT><<<grid, 32 * kIpWarps, smem, s>>>(a);
  return 1;
}

template <int BCM>
int launch_ip(const StepArgs& a, cudaStream_t s) {
  const int spec = (a.bg.nvb > 0 ? kSpecVP : 0) | (a.nsteps > 1 ? kSpecSub : 0);
  const bool count = a.cnt_hist != nullptr;
  switch (spec + 4 * count) {
    case 0: return launch_ip_variant<BCM, 0, false>(a, s);
    case kSpecVP: return launch_ip_variant<BCM, kSpecVP, false>(a, s);
    case kSpecSub: return launch_ip_variant<BCM, kSpecSub, false>(a, s);
    case kSpecAll: return launch_ip_variant<BCM, kSpecAll, false>(a, s);
    case 4: return launch_ip_variant<BCM, 0, true>(a, s);
    case 4 + kSpecVP: return launch_ip_variant<BCM, kSpecVP, true>(a, s);
    case 4 + kSpecSub: return launch_ip_variant<BCM, kSpecSub, true>(a, s);
    default: return launch_ip_variant<BCM, kSpecAll, true>(a, s);
  }
}
