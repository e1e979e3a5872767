// k_step v7 — latency-lean step kernel for 8^3-cell chunks (included by k_step.cu,
// which defines the helpers: Stage/TMA pipeline, bin geometry, slots, reductions).
//
// Measured on C5 (1e9 particles, scripts/gpu_ablate.sh): data movement alone runs
// at ~86 % of HBM peak, so the step is bound by the per-batch dependency chain of
// each warp.  This variant removes every global load from that chain:
//  * items are one chunk row (<= 8 consecutive bins);
//  * at item start the warp computes, for each (bin, slot) of the item, the base
//    of its destination run (off_new[d] + base[j][s], or the send-buffer offset of a
//    neighbour plane) into shared memory; a particle's destination is then
//    smem base + run counter + rank — no dependent L2 loads per batch;
//  * particle input arrives through a 2-stage TMA bulk pipeline (cp.async.bulk +
//    mbarrier); the fluid corners are L1-cached __ldg loads (cell-coherent warps);
//  * groups of equal keys use SHFL + VOTE (no MATCH.ANY); invalid lanes of a
//    partial batch mirror a valid particle with predicated side effects.
#pragma once

// Lanes holding the same key (what __match_any_sync returns), found by iterating
// over the distinct keys with one SHFL + one VOTE each; invalid lanes share one key.
__device__ __forceinline__ unsigned peers_of(int key) {
  unsigned todo = kFull, mine = 0;
  while (todo) {
    const int k = __shfl_sync(kFull, key, __ffs(todo) - 1);
    const unsigned m = __ballot_sync(kFull, key == k);
    mine = (key == k) ? m : mine;
    todo &= ~m;
  }
  return mine;
}

constexpr int kRowBins = 8;
constexpr int kPStages = 2;
constexpr int kBarBytes = 16;                               // kPStages mbarriers
// per-warp slice: stages | mbarriers | [scatter: dbase i64, run i32, side i8 — padded to 16] | rel[9]
constexpr int kScatterTable = (kRowBins * kSlots * 13 + 15) / 16 * 16;
__host__ __device__ constexpr int pwarp_smem_bytes(bool scatter) {
  return (int)((kPStages * sizeof(Stage) + kBarBytes + (scatter ? kScatterTable : 0) + (kRowBins + 1) * 4 + 15) /
               16 * 16);
}

template <bool SCATTER, bool ADVANCE, int BCM, int FEAT = 0xff>
__global__ void __launch_bounds__(256, (SCATTER && ADVANCE) ? 3 : 4) k_pstep(StepArgs a) {
  constexpr int SH = 3;   // chunk_cells == 8
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geom& g = a.g;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* ws = smem_raw + (size_t)wib * pwarp_smem_bytes(SCATTER);
  Stage* stg = reinterpret_cast<Stage*>(ws);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(ws + kPStages * sizeof(Stage));
  unsigned char* tail = ws + kPStages * sizeof(Stage) + kBarBytes;
  long long* dbase = reinterpret_cast<long long*>(tail);                      // [8*27] destination run bases
  int* run = reinterpret_cast<int*>(dbase + (SCATTER ? kRowBins * kSlots : 0));   // [8*27] run counters
  signed char* dside = reinterpret_cast<signed char*>(run + (SCATTER ? kRowBins * kSlots : 0));  // [8*27]
  int* rel = reinterpret_cast<int*>(tail + (SCATTER ? kScatterTable : 0));  // [kRowBins+1]
  const int n_items = *a.n_items;
  const int warps_total = gridDim.x * (blockDim.x >> 5);
  const int64_t cap = a.cap;
  const int nbins = a.nbins;
  const int pz = g.gy * g.gx;
  int flags = 0, farflag = 0;
  unsigned movers = 0;
  uint32_t phase = 0;
  if (lane == 0) {
    for (int k = 0; k < kPStages; ++k) mbar_init(bar + k, 1);
    fence_mbar_init();
  }
  __syncwarp();

  for (int item = blockIdx.x * (blockDim.x >> 5) + wib; item < n_items; item += warps_total) {
    const int b0 = a.item_bin0[item];
    const int b1 = (item + 1 < n_items) ? a.item_bin0[item + 1] : nbins;
    const int nb = b1 - b0;                       // <= kRowBins, one chunk row
    const int64_t p0 = a.off[b0];
    if (lane <= nb) rel[lane] = (int)(a.off[b0 + lane] - p0);
    int rx, ry, rz;                               // cell of the row's first bin (row along +x)
    cell_of_bin(g, a.bg, b0, rx, ry, rz);
    if (SCATTER) {
      // destination run bases of every (bin, slot) of the item
      for (int k = lane; k < nb * kSlots; k += 32) {
        const int lb = k / kSlots, j = k - lb * kSlots;
        bool ok = true;
        const int dx = axis_step(rx + lb, j % 3 - 1, g.n[0], g.bc[0], ok);
        const int dy = axis_step(ry, (j / 3) % 3 - 1, g.n[1], g.bc[1], ok);
        const int dz = axis_step(rz, j / 9 - 1, g.n[2], g.bc[2], ok);
        long long db = -1;
        signed char side = -1;
        if (ok) {
          const int within = a.slot_base[(int64_t)j * nbins + b0 + lb];
          side = (dz == a.bg.vz[0]) ? 0 : ((dz == a.bg.vz[1]) ? 1 : -1);
          if (side >= 0) db = a.voff[side][vbin_of_cell<SH>(g, dx, dy, 8)] + within;
          else if ((dz >> 3) >= a.bg.kz0 && (dz >> 3) < a.bg.kz0 + a.bg.nkz)
            db = a.off_new[bin_of_cell<SH>(g, a.bg, dx, dy, dz)] + within;
        }
        dbase[k] = db;
        dside[k] = side;
        run[k] = 0;
      }
    }
    __syncwarp();
    const int np = rel[nb];
    const int nbatch = (np + 31) >> 5;
    if (lane == 0) {
      fence_proxy_async();
      for (int k = 0; k < kPStages && k < nbatch; ++k) stage_issue(stg + k, bar + k, a.A, cap, p0 + 32 * k, cap, SCATTER);
    }
    int lb = 0;
    for (int bi = 0; bi < nbatch; ++bi) {
      const int base = bi << 5;
      const int sk = bi & (kPStages - 1);
      const bool valid = base + lane < np;
      const int r = valid ? base + lane : np - 1;          // invalid lanes mirror a valid particle
      while (rel[lb + 1] <= r) ++lb;
      const int s = b0 + lb;
      const int sx = rx + lb, sy = ry, sz = rz;             // bin cell (row along x)
      mbar_wait(bar + sk, (phase >> sk) & 1u);
      phase ^= 1u << sk;
      const Stage& S = stg[sk];
      const int so = (int)((p0 + base) & 3) + (r - base);
      float xp0 = S.f[0][so], xp1 = S.f[1][so], xp2 = S.f[2][so];
      float up0 = S.f[3][so], up1 = S.f[4][so], up2 = S.f[5][so];
      const float dp = S.f[6][so], wp = S.f[7][so];
      unsigned long long pid = 0;
      if (SCATTER) pid = S.id[(int)((p0 + base) & 1) + (r - base)];
      // the stage is consumed: refill it with the batch kPStages ahead
      __syncwarp();
      if (lane == 0 && bi + kPStages < nbatch) {
        fence_proxy_async();
        stage_issue(stg + sk, bar + sk, a.A, cap, p0 + 32 * (bi + kPStages), cap, SCATTER);
      }
      float t0 = cell_coord(xp0, g.lo[0], g.ih[0]), t1 = cell_coord(xp1, g.lo[1], g.ih[1]),
            t2 = cell_coord(xp2, g.lo[2], g.ih[2]);
      int c0 = cell_from_t(t0, g.n[0]), c1 = cell_from_t(t1, g.n[1]), c2 = cell_from_t(t2, g.n[2]);
      int ox = sx, oy = sy, oz = sz, obin = s, vside = -1;
      int64_t dest = p0 + r;
      bool write_ok = valid;
      if (SCATTER) {
        const int j = slot_of<BCM>(g, sx, sy, sz, c0, c1, c2);
        const int k = lb * kSlots + (j < 0 ? kStay : j);
        const long long db = dbase[k];
        if (valid && (j < 0 || db < 0)) {
          flags |= ERRF_SCATTER;
          write_ok = false;
        }
        const int key = write_ok ? k : -1;
        const unsigned peers = peers_of(key);
        const int leader = __ffs(peers) - 1;
        int rbase = 0;
        if (lane == leader && key >= 0) {
          rbase = run[key];
          run[key] = rbase + __popc(peers);
        }
        rbase = __shfl_sync(kFull, rbase, leader) + __popc(peers & lanemask_lt());
        __syncwarp();
        ox = c0;
        oy = c1;
        oz = c2;
        vside = dside[k];
        dest = db + rbase;
        if (vside < 0) obin = bin_of_cell<SH>(g, a.bg, ox, oy, oz);
        if (write_ok && (dest < 0 || dest >= (vside < 0 ? a.n : a.scap))) {
          flags |= ERRF_SCATTER;
          write_ok = false;
        }
      }
      if (ADVANCE && (FEAT & 1)) {
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
          float4 uf = make_float4(0.1f, 0.0f, 0.0f, 0.0f);   // (ablation value)
          if (FEAT & 2) {
            const float4* fb = a.field + ((int64_t)wz * pz + (iy + 1) * g.gx + (ix + 1));
            const float4 c000 = __ldg(fb), c100 = __ldg(fb + 1);
            const float4 c010 = __ldg(fb + g.gx), c110 = __ldg(fb + g.gx + 1);
            const float4 c001 = __ldg(fb + pz), c101 = __ldg(fb + pz + 1);
            const float4 c011 = __ldg(fb + pz + g.gx), c111 = __ldg(fb + pz + g.gx + 1);
            uf = lerp4(lerp4(lerp4(c000, c100, fx), lerp4(c010, c110, fx), fy),
                       lerp4(lerp4(c001, c101, fx), lerp4(c011, c111, fx), fy), fz);
          }
          const float sxv = uf.x - up0, syv = uf.y - up1, szv = uf.z - up2;
          const float Re = sqrt_approx(fmaf(sxv, sxv, fmaf(syv, syv, szv * szv))) * d * a.p.inv_nu;
          float f = 1.0f + 0.15f * exp2f(0.687f * __log2f(Re));
          f = (Re <= 1000.0f) ? f : (0.44f / 24.0f) * Re;
          f = (a.p.drag_law == ST_DRAG_STOKES) ? 1.0f : f;
          const float taue = tau * rcp_approx(f);
          const float h = dt * f * inv_tau;
          float du0, du1, du2;
          if (a.p.integrator == ST_INT_EXPONENTIAL) {
            // E = exp(-h); M = 1 - E (series below h = 1/8): both evaluated, selected
            const float E = __expf(-h);
            const float Ms = h * (1.0f - h * (0.5f - h * (1.0f / 6.0f - h * (1.0f / 24.0f - h * (1.0f / 120.0f - h * (1.0f / 720.0f))))));
            const float M = h < 0.125f ? Ms : 1.0f - E;
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
          if ((FEAT & 4) && a.p.two_way) {
            const int az = acc_z(g, c2);
            if (valid && az < 0) flags |= ERRF_WINDOW;
            const bool dep = valid && az >= 0;
            const int ckey = dep ? (az * g.n[1] + c1) * g.n[0] + c0 : -1;
            const float ja = -mw * du0, jb = -mw * du1, jc = -mw * du2;
            // anchors: the bin cells of lanes 0 and 31 (the first and last bin of the
            // batch) — their stayers, the bulk of a cell-sorted warp, are reduced in
            // registers with one red per anchor; the other lanes red individually
            const int bk = (acc_z(g, sz) * g.n[1] + sy) * g.n[0] + sx;
            const int kA = __shfl_sync(kFull, bk, 0), kB = __shfl_sync(kFull, bk, 31);
            const bool inA = dep && ckey == kA, inB = dep && kB != kA && ckey == kB;
            const unsigned mA = __ballot_sync(kFull, inA), mB = __ballot_sync(kFull, inB);
            if (mA) {
              float ra = ja, rb = jb, rc = jc;
              group_sum3(inA, ra, rb, rc);
              if (lane == 0) red_add_v4(a.acc + kA, ra, rb, rc);
            }
            if (mB) {
              float ra = ja, rb = jb, rc = jc;
              group_sum3(inB, ra, rb, rc);
              if (lane == 31) red_add_v4(a.acc + kB, ra, rb, rc);
            }
            if (dep && !inA && !inB) red_add_v4(a.acc + ckey, ja, jb, jc);
          }
          bool bad = false;
          bad |= apply_bc(periodic<BCM>(g, 0) ? ST_BC_PERIODIC : ST_BC_REFLECT, g.lo[0], g.hi[0], g.L[0], xp0, up0);
          bad |= apply_bc(periodic<BCM>(g, 1) ? ST_BC_PERIODIC : ST_BC_REFLECT, g.lo[1], g.hi[1], g.L[1], xp1, up1);
          bad |= apply_bc(periodic<BCM>(g, 2) ? ST_BC_PERIODIC : ST_BC_REFLECT, g.lo[2], g.hi[2], g.L[2], xp2, up2);
          if (bad && valid) flags |= ERRF_CFL;
        }
      }
      if (FEAT & 8) {   // slot histogram of the end position w.r.t. the output bin
        const int e0 = cell_from_t(cell_coord(xp0, g.lo[0], g.ih[0]), g.n[0]);
        const int e1 = cell_from_t(cell_coord(xp1, g.lo[1], g.ih[1]), g.n[1]);
        const int e2 = cell_from_t(cell_coord(xp2, g.lo[2], g.ih[2]), g.n[2]);
        const bool here = write_ok && vside < 0;
        const int j2 = slot_of<BCM>(g, ox, oy, oz, e0, e1, e2);
        if (here && j2 < 0) farflag = 1;
        const int hkey = (here && j2 >= 0) ? obin * kSlots + j2 : -1;
        // anchors: (bin, stay) of lanes 0 and 31 — one atomic per anchor group; the
        // remaining lanes (cell movers) add 1 each
        const int hb = s * kSlots + kStay;
        const int hA = __shfl_sync(kFull, hb, 0), hB = __shfl_sync(kFull, hb, 31);
        const bool inA = hkey == hA, inB = hkey == hB && hB != hA;
        const unsigned mA = __ballot_sync(kFull, inA), mB = __ballot_sync(kFull, inB);
        if (lane == 0 && mA) atomicAdd(a.hist_next + (int64_t)kStay * nbins + hA / kSlots, __popc(mA));
        if (lane == 31 && mB) atomicAdd(a.hist_next + (int64_t)kStay * nbins + hB / kSlots, __popc(mB));
        if (hkey >= 0 && !inA && !inB) atomicAdd(a.hist_next + (int64_t)j2 * nbins + obin, 1);
        const bool mover = write_ok && (((e0 >> SH) != (ox >> SH)) | ((e1 >> SH) != (oy >> SH)) | ((e2 >> SH) != (oz >> SH)));
        movers += mover ? 1u : 0u;
      }
      if ((FEAT & 16) && write_ok) {
        if (SCATTER) {
          const Store& o = vside < 0 ? a.B : a.sbuf[vside];
          const int64_t oc = vside < 0 ? cap : a.scap;
          o.x[dest] = xp0; o.x[oc + dest] = xp1; o.x[2 * oc + dest] = xp2;
          o.u[dest] = up0; o.u[oc + dest] = up1; o.u[2 * oc + dest] = up2;
          o.d[dest] = dp;
          o.w[dest] = wp;
          reinterpret_cast<unsigned long long*>(o.id)[dest] = pid;
        } else if (ADVANCE) {
          __stcs(a.A.x + dest, xp0); __stcs(a.A.x + cap + dest, xp1); __stcs(a.A.x + 2 * cap + dest, xp2);
          __stcs(a.A.u + dest, up0); __stcs(a.A.u + cap + dest, up1); __stcs(a.A.u + 2 * cap + dest, up2);
        }
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) movers += __shfl_xor_sync(kFull, movers, o);
  if (lane == 0 && movers) atomicAdd(a.movers, (unsigned long long)movers);
  if (flags) atomicOr(a.err, flags);
  if (farflag) *(volatile int*)a.far = 1;
}
