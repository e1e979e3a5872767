// k_fs — the fused rebin scatter + advance for 8^3-cell chunks, two particles per lane
// (included by k_step.cu after k_ip.cuh).  Rows a2-a8 of SURVEY §8(a) in one pass: the
// neighbour-slot stable counting sort of C-15 (destination = run base of (bin, slot)
// from the item's destination table + rank within the run; far particles into their
// bin's tail, C-15b) fused with the step of the particle.
//
// Same structure as k_ip (64-particle batches staged by one TMA box {68, 8} of the float
// rows plus one box {66, 1} of the ids, a warp-uniform bin in the common case, the
// deposit accumulator owned by the warp's current bin cell) — the round-1 k_pstep<1,1>
// ran at 39 % issue-active, latency-bound on the per-batch bin walk and the rank chain;
// here the batch's two halves are ranked one after the other (lanes 0-31 are the first
// 32 particles in store order, lanes 0-31 of the second half the next 32), the stage is
// released only after the stores (the ids are read from it late), and the physics of
// the two particles of a lane interleave.
#pragma once

#ifndef ST_FS_STAGES
#define ST_FS_STAGES 3   // one CTA of 8 warps per SM (measured: 2 CTAs/SM with 2 stages or 6 warps are slower)
#endif
#ifndef ST_FS_WARPS
#define ST_FS_WARPS 10   // A/B at C5 K = 3 (r2y): 10 warps 1 % faster than 8; 12 and 2-stage 16 slower
#endif
constexpr int kFsStages = ST_FS_STAGES;
constexpr int kFsBoxI = 66;                                   // 64 ids + 2 of alignment slack
constexpr int kFsStageBytes = (8 * kIpBoxF * 4 + kFsBoxI * 8 + 127) / 128 * 128;   // 2176 + 528 -> 2816
constexpr int kFsOffId = 8 * kIpBoxF * 4;                     // ids after the float rows (128-B aligned)
constexpr int kFsOffWin = kFsStages * kFsStageBytes;          // 8448
constexpr int kFsOffTab = kFsOffWin + kIpWX * kIpWYZ * kIpWYZ * 16;   // + 4800: dtab i64[216]
constexpr int kFsOffRun = kFsOffTab + kTable * 8;             // run i32[216]
constexpr int kFsOffRel = kFsOffRun + kTable * 4;
constexpr int kFsOffBar = kFsOffRel + 48;
constexpr int kFsWarpBytes = (kFsOffBar + 8 * (kFsStages + 1) + 127) / 128 * 128;
constexpr int kFsWarps = ST_FS_WARPS;
constexpr uint32_t kFsTx = 8u * kIpBoxF * 4u + kFsBoxI * 8u;

template <int BCM, int SPEC>
__global__ void __launch_bounds__(32 * kFsWarps, kFsWarps > 8 ? 1 : 2) k_fs(const __grid_constant__ StepArgs a) {
  constexpr int SH = 3;
  constexpr bool VP = (SPEC & kSpecVP) != 0;
  constexpr bool SUB = (SPEC & kSpecSub) != 0;
  extern __shared__ __align__(128) unsigned char fssmem_raw[];
  const Geom& g = a.g;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* sbase = fssmem_raw + ((kPSmemAlign - (smem_u32(fssmem_raw) & (kPSmemAlign - 1))) & (kPSmemAlign - 1));
  unsigned char* ws = sbase + (size_t)wib * kFsWarpBytes;
  float4* win = reinterpret_cast<float4*>(ws + kFsOffWin);
  long long* dtab = reinterpret_cast<long long*>(ws + kFsOffTab);
  int* run = reinterpret_cast<int*>(ws + kFsOffRun);
  int* rel = reinterpret_cast<int*>(ws + kFsOffRel);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(ws + kFsOffBar);
  unsigned long long* ibar = bar + kFsStages;
  const uint32_t stage0 = smem_u32(ws);
  const uint32_t win0 = smem_u32(win);
  const int n_items = *a.n_items;
  const int warps_total = gridDim.x * kFsWarps;
  const int nbins = a.nbins;
  const bool two_way = a.p.two_way != 0;
  const float dt = a.dt;
  const float2 nlo = f2(-g.lo[0], -g.lo[1]), ihv = f2(g.ih[0], g.ih[1]);
  int flags = 0;
  uint32_t phase = 0, iphase = 0;
  const unsigned lt = lanemask_lt();
  if (lane == 0) {
    for (int k = 0; k <= kFsStages; ++k) mbar_init(bar + k, 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int k, int64_t first) {   // lane 0: stage k <- the 64-particle batch at `first`
    mbar_expect_tx(bar + k, kFsTx);
    unsigned char* st = ws + k * kFsStageBytes;
    tma_rows(st, &a.tm_f64, (int)(first & ~3LL), bar + k);
    tma_ids(st + kFsOffId, &a.tm_id66, (int)(first & ~1LL), bar + k);
  };

  const bool dyn = ST_DYN_ITEMS && a.item_ctr != nullptr;   // items as in k_ip
  int item = blockIdx.x * kFsWarps + wib;
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
      mbar_expect_tx(ibar, (uint32_t)(kIpWX * kIpWYZ * kIpWYZ * 16) + kTable * 8u);
      tma_win(win, &a.tm_win[1], 4 * (rx - 1), ry - 1, window_z(g, rz) - 2, ibar);
      bulk_g2s(dtab, a.dtab + (int64_t)b0 * kSlots, kTable * 8u, ibar);
      for (int k = 0; k < kFsStages && k < nbatch; ++k) issue(k, p0 + 64 * k);
    }
    __syncwarp();
    // the next item from the counter, issued after this item's copies (the proxy fence
    // before them would otherwise wait for the atomic's round trip)
    if (dyn && lane == 0) tk = atomicAdd(a.item_ctr, 1);
    if (lane <= nb) rel[lane] = myrel;
    for (int k = lane; k < kTable; k += 32) run[k] = 0;
    mbar_wait(ibar, iphase);
    iphase ^= 1u;
    __syncwarp();
    const int az_row = VP ? acc_z(g, rz) : rz - g.az0;
    int cb = 0, ce = rel[1], acb = -1;
    int carry_lb = -1, carry = 0;                 // stayers of bin carry_lb placed so far
    float da0 = 0.f, da1 = 0.f, da2 = 0.f;
    auto flush = [&]() {
      if (acb < 0 || !two_way) return;
      float ra = da0, rb = da1, rc = da2;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ra += __shfl_xor_sync(kFull, ra, o);
        rb += __shfl_xor_sync(kFull, rb, o);
        rc += __shfl_xor_sync(kFull, rc, o);
      }
      if (lane == 0) red_add_v4(a.acc + (uint32_t)((az_row * g.n[1] + ry) * g.n[0] + rx + acb), ra, rb, rc);
      da0 = da1 = da2 = 0.f;
    };
    for (int bi = 0; bi < nbatch; ++bi) {
      const int base = bi << 6;
      while (ce <= base) ce = rel[++cb + 1];
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
        r[q] = valid[q] ? rr : np - 1;
      }
      const bool straddle = last >= ce;             // warp-uniform
      if (straddle) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
          while (rel[lb[q] + 1] <= r[q]) ++lb[q];
      }
      const int sk = bi % kFsStages;
      mbar_wait(bar + sk, (phase >> sk) & 1u);
      __syncwarp();
      phase ^= 1u << sk;
      float x[2][3], u[2][3], dp[2], wp[2];
      const uint32_t sa = stage0 + sk * kFsStageBytes + 4u * (uint32_t)(((p0 + base) & 3) + lane);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t s = sa + 128u * q;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x[q][0]) : "r"(s));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x[q][1]) : "r"(s + 1u * kIpBoxF * 4));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x[q][2]) : "r"(s + 2u * kIpBoxF * 4));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(u[q][0]) : "r"(s + 3u * kIpBoxF * 4));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(u[q][1]) : "r"(s + 4u * kIpBoxF * 4));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(u[q][2]) : "r"(s + 5u * kIpBoxF * 4));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(dp[q]) : "r"(s + 6u * kIpBoxF * 4));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(wp[q]) : "r"(s + 7u * kIpBoxF * 4));
      }
      if (base + 63 >= np) {   // tail batch: idle lanes mirror lane 0's particle
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

      // ---- rebin scatter (a8): destination of each particle from its current cell ----
      int c[2][3];
      float t[2][3];
      int dest[2];
      int vside[2] = {-1, -1};
      bool wok[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        {
          const float2 txy = cell_coord2(x[q][0], x[q][1], nlo, ihv);
          t[q][0] = txy.x;
          t[q][1] = txy.y;
          t[q][2] = cell_coord(x[q][2], g.lo[2], g.ih[2]);
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) c[q][k] = cell_from_t(t[q][k], g.n[k]);
        const int sx = rx + lb[q];
        const int j = slot_of<BCM>(g, sx, ry, rz, c[q][0], c[q][1], c[q][2]);
        const int key = lb[q] * kSlots + (j < 0 ? kStay : j);
        const long long e = dtab[key];                 // -1: leaves the domain; bits 61-62: side + 1
        const long long db = e < 0 ? -1 : (e & ((1LL << 61) - 1));
        const bool farp = j < 0;
        bool ok = valid[q];
        if (ok && !farp && db < 0) {
          flags |= ERRF_SCATTER;
          ok = false;
        }
        int fdest = -1, fside = -1;
        if (ok && farp) {   // C-15b: the next slot of the destination bin's tail (k_far_order sorts it)
          const int kz = c[q][2] >> SH;
          int pl;
          if (a.far_cur && kz >= a.bg.kz0 && kz < a.bg.kz0 + a.bg.nkz) {
            fdest = (int)atomicAdd(a.far_cur + bin_of_cell<SH>(g, a.bg, c[q][0], c[q][1], c[q][2]), 1ULL);
            a.far_src[fdest] = (int32_t)(p0 + r[q]);
            a.far_src_hi[fdest] = 0;
          } else if (VP && a.fs_cur && far_plane(g, c[q][2], fside, pl)) {
            // a neighbour rank's cell: the far region of the send buffer, with its prior
            // index (the receiver's tail key) and the cell it was counted for
            fdest = (int)atomicAdd(a.fs_cur + fside, 1ULL);
            if ((int64_t)fdest < a.scap) {
              a.fs_key[fside][fdest] = (int32_t)(p0 + r[q]);
              a.fs_cell[fside][fdest] = (c[q][2] * g.n[1] + c[q][1]) * g.n[0] + c[q][0];
            }
          } else {
            flags |= ERRF_SCATTER;
            ok = false;
          }
        }
        const bool stay = ok && j == kStay;
        // stayers: rank inside the bin segment of this half (lanes of one bin are contiguous)
        const unsigned mstay = __ballot_sync(kFull, stay);
        int rank;
        if (!straddle) {   // the whole batch is one bin: a plain prefix of the stayer mask
          rank = (lb[q] == carry_lb ? carry : 0) + __popc(mstay & lt);
          carry = (lb[q] == carry_lb ? carry : 0) + __popc(mstay);
          carry_lb = lb[q];
        } else {
          const int lb_up = __shfl_up_sync(kFull, lb[q], 1);
          const unsigned starts = __ballot_sync(kFull, lane == 0 || lb[q] != lb_up);
          const int ss = 31 - __clz(starts & (lt | (1u << lane)));
          rank = (lb[q] == carry_lb ? carry : 0) + __popc(mstay & lt & ~((1u << ss) - 1u));
          const int lb31 = __shfl_sync(kFull, lb[q], 31);
          const int ss31 = 31 - __clz(starts);
          carry = (lb31 == carry_lb ? carry : 0) + __popc(mstay & ~((1u << ss31) - 1u));
          carry_lb = lb31;
        }
        // movers: groups of equal (bin, slot) keys take consecutive slots of the run
        const int mkey = (ok && !stay && !farp) ? key : -1;
        const unsigned movers = __ballot_sync(kFull, mkey >= 0);
        if (movers) {
          const unsigned peers = __match_any_sync(kFull, mkey);
          if (mkey >= 0) {
            const int leader = __ffs(peers) - 1;
            int rb0 = 0;
            if (lane == leader) {
              rb0 = run[mkey];
              run[mkey] = rb0 + __popc(peers);
            }
            rank = __shfl_sync(peers, rb0, leader) + __popc(peers & lt);
          }
          __syncwarp();
        }
        if (VP) vside[q] = farp ? fside : (e < 0 ? -1 : (int)(e >> 61) - 1);
        const long long dl = farp ? (long long)fdest : db + rank;
        if (ok && (uint64_t)dl >= (uint64_t)((VP && vside[q] >= 0) ? a.scap : a.n)) {
          flags |= ERRF_SCATTER;
          ok = false;
        }
        dest[q] = (int)dl;
        wok[q] = ok;
      }

      // ---- advance (a3-a7) ----
      const float gx = a.p.g[0], gy = a.p.g[1], gz = a.p.g[2];
      const float2 gxy = f2(gx, gy), ngdt = f2(-gx * dt, -gy * dt);
      float tau[2], inv_tau[2], mw[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        tau[q] = a.p.tau_c * dp[q] * dp[q];
        inv_tau[q] = rcp_approx(tau[q]);
        mw[q] = a.p.mass_c * dp[q] * dp[q] * dp[q] * wp[q];
      }
      const int nsub = SUB ? a.nsteps : 1;
      for (int sub = 0; sub < nsub; ++sub) {
        V3 ufq[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (sub > 0) {
            const float2 txy = cell_coord2(x[q][0], x[q][1], nlo, ihv);
            t[q][0] = txy.x;
            t[q][1] = txy.y;
            t[q][2] = cell_coord(x[q][2], g.lo[2], g.ih[2]);
#pragma unroll
            for (int k = 0; k < 3; ++k) c[q][k] = cell_from_t(t[q][k], g.n[k]);
          }
          int i0[3];
          float f[3];
          stencil_lo2(f2(t[q][0], t[q][1]), i0[0], i0[1], f[0], f[1]);
          stencil_lo(t[q][2], i0[2], f[2]);
          float4 q8[8];
          const bool inw = (unsigned)(i0[0] - rx + 2) <= 10u && (unsigned)(i0[1] - ry + 2) <= 3u &&
                           (unsigned)(i0[2] - rz + 2) <= 3u;
          if (__all_sync(kFull, inw)) {
            const uint32_t w0 =
                win0 + 16u * (uint32_t)(((i0[2] - rz + 2) * kIpWYZ + (i0[1] - ry + 2)) * kIpWX + (i0[0] - rx + 2));
            constexpr uint32_t oy = kIpWX * 16, oz = kIpWYZ * kIpWX * 16;
            q8[0] = lds4(w0); q8[1] = lds4(w0 + 16); q8[2] = lds4(w0 + oy); q8[3] = lds4(w0 + oy + 16);
            q8[4] = lds4(w0 + oz); q8[5] = lds4(w0 + oz + 16); q8[6] = lds4(w0 + oz + oy);
            q8[7] = lds4(w0 + oz + oy + 16);
          } else {
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
          float fd = fmaf(0.15f, ex2_ftz(0.687f * lg2_ftz(Re)), 1.0f);
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
            const float2 jxy = __fmul2_rn(bc2(-mw[q]), duxy);
            const float ja = jxy.x, jb = jxy.y, jc = -mw[q] * du2;
            if (valid[q] && c[q][0] == rx + acb && c[q][1] == ry && c[q][2] == rz) {
              const float2 dn = __fadd2_rn(f2(da0, da1), jxy);
              da0 = dn.x;
              da1 = dn.y;
              da2 += jc;
            } else if (valid[q]) {
              const int az = VP ? acc_z(g, c[q][2]) : c[q][2] - g.az0;
              if (VP && az < 0) flags |= ERRF_WINDOW;
              else red_add_v4(a.acc + (uint32_t)((az * g.n[1] + c[q][1]) * g.n[0] + c[q][0]), ja, jb, jc);
            }
          }
        }
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
      // ---- stores into the new layout (or a neighbour rank's send buffer) ----
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (!wok[q]) continue;
        unsigned long long pid;
        asm volatile("ld.shared.u64 %0, [%1];"
                     : "=l"(pid)
                     : "r"(stage0 + sk * kFsStageBytes + kFsOffId + 8u * (uint32_t)(((p0 + base) & 1) + 32 * q + lane)));
        const Store& o = (VP && vside[q] >= 0) ? a.sbuf[vside[q]] : a.B;
        const int64_t oc = (VP && vside[q] >= 0) ? a.scap : a.cap;
        const int64_t dd = dest[q];
        o.x[dd] = x[q][0]; o.x[oc + dd] = x[q][1]; o.x[2 * oc + dd] = x[q][2];
        o.u[dd] = u[q][0]; o.u[oc + dd] = u[q][1]; o.u[2 * oc + dd] = u[q][2];
        o.d[dd] = dp[q];
        o.w[dd] = wp[q];
        reinterpret_cast<unsigned long long*>(o.id)[dd] = pid;
      }
      // the stage is consumed (ids read last): refill it with the batch kFsStages ahead
      __syncwarp();
      if (lane == 0 && bi + kFsStages < nbatch) {
        fence_proxy_async();
        issue(sk, p0 + base + 64 * kFsStages);
      }
      __syncwarp();
      if (bi == 0) prefetch1();
      if (bi == 1) prefetch2();
    }
    if (nbatch == 0) prefetch1();
    if (nbatch <= 1) prefetch2();
    __syncwarp();
    flush();
    __syncwarp();
    item = next;
  }
  if (flags) atomicOr(a.err, flags);
}

template <int BCM, int SPEC>
int launch_fs_variant(const StepArgs& a, cudaStream_t s) {
  static int grid = 0;
  const int smem = kFsWarps * kFsWarpBytes + kPSmemAlign;
  if (!grid) {
    int nsm = 148, dev = 0, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_fs<BCM, SPEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_fs<BCM, SPEC>, 32 * kFsWarps, smem);
    grid = nsm * (per > 0 ? per : 1);
  }
  if (ST_DYN_ITEMS && a.item_ctr) cudaMemsetAsync(a.item_ctr, 0, sizeof(int), s);
  k_fs<BCM, SPEC><<<grid, 32 * kFsWarps, smem, s>>>(a);
  return 1;
}

template <int BCM>
int launch_fs(const StepArgs& a, cudaStream_t s) {
  const int spec = (a.bg.nvb > 0 ? kSpecVP : 0) | (a.nsteps > 1 ? kSpecSub : 0);
  switch (spec) {
    case 0: return launch_fs_variant<BCM, 0>(a, s);
    case kSpecVP: return launch_fs_variant<BCM, kSpecVP>(a, s);
    case kSpecSub: return launch_fs_variant<BCM, kSpecSub>(a, s);
    default: return launch_fs_variant<BCM, kSpecAll>(a, s);
  }
}
