// k_step v8 — issue-lean step kernel for 8^3-cell chunks (included by k_step.cu,
// which defines the helpers: bin geometry, slots, reductions, mbarrier helpers).
//
// Measured on C5 (scripts/gpu_ablate.sh, profiles/README.md): data movement alone
// runs near the HBM roofline, so the step is bound by instruction issue per
// 32-particle batch.  v8 cuts the per-batch work of each warp:
//  * particle input: ONE 2-D TMA tensor copy of the 8 float rows (x0 x1 x2 u0 u1 u2
//    d w, contiguous rows of stride cap) + one copy of the ids per batch,
//    through a per-warp mbarrier pipeline (no per-array bulk copies);
//  * items are one chunk row (<= 8 bins); at item start the warp computes, for each
//    (bin, slot), the base of its destination run (off_new[d] + base[j][s], or the
//    send-buffer offset of a neighbour plane) into shared memory;
//  * stayers (end cell == bin cell, the bulk of a cell-sorted warp): rank from
//    segment ballots (lanes of one bin are contiguous), deposit and slot count
//    accumulated in registers per lane and flushed once per (lane, bin);
//  * movers: rank via MATCH.ANY over (bin, slot), individual red / atomic.
#pragma once

// one generic load of a cell (the window lives in smem, the rest of the field in
// global); ptxas narrows it to 8 + 4 bytes since the 4th lane is unused
__device__ __forceinline__ float4 ld4(const float4* p) {
  float4 v;
  asm("ld.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

__device__ __forceinline__ float4 trilerp(const float4 (&q)[8], float fx, float fy, float fz) {
  return lerp4(lerp4(lerp4(q[0], q[1], fx), lerp4(q[2], q[3], fx), fy),
               lerp4(lerp4(q[4], q[5], fx), lerp4(q[6], q[7], fx), fy), fz);
}

__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// trilinear stencil base and weight from the cell coordinate t = (x - lo)/h:
// i0 = floor(t - 1/2), f = t - 1/2 - i0 — exact in fp32 (t < 2^22), identical to
// deriving them from the cell (C-6) including the f = 1/2 tie and the clamped top cell
__device__ __forceinline__ void stencil_lo(float t, int& i0, float& f) {
  const float sh = t - 0.5f;
  i0 = __float2int_rd(sh);
  f = sh - (float)i0;
}

constexpr int kRowBins = 8;
constexpr int kPStages = 3;
// A tensor-copy box must start 16-byte aligned along the inner dimension (a
// misaligned start traps as an illegal instruction — measured, scripts/tma_probe.cu),
// so a batch at store index i0 is staged from i0 & ~3 (floats) / i0 & ~1 (ids) with
// 4 / 2 elements of slack.
constexpr int kBoxF = 36, kBoxI = 34;
struct alignas(128) TStage {
  float f[8][kBoxF];                // box {36, 8} of the float rows
  unsigned long long id[kBoxI];     // box {34, 1} of the ids (offset 1152: 128-B aligned)
};
constexpr int kTStageBytes = (int)sizeof(TStage);                   // 1536
constexpr uint32_t kTxF = 8 * kBoxF * 4, kTxI = kBoxI * 8;
// fluid window of an item, ghosted cells x in [rx-1-R, rx+8+R], y in [ry-1-R, ry+1+R],
// z in [rz-1-R, rz+1+R]: every trilinear stencil of a particle whose cell is within R of
// the row (R = 1 for the fused scatter: the whole neighbourhood a binned particle can
// be in; R = 0 in place).  Staged by one 3-D TMA tensor copy (tm_win[R]).
#ifndef ST_EARLY_GATHER
#define ST_EARLY_GATHER 1   // sub-step-0 corners issued before the rank (A/B: ~1 % faster)
#endif
#ifndef ST_PWIN_R
#define ST_PWIN_R 1   // window margin R of the fused scatter (A/B: R = 1 ~2.5 % faster than 0)
#endif
#ifndef ST_PWIN_R_IP
#define ST_PWIN_R_IP 1   // window margin of the in-place step (binned particles are within one cell)
#endif
__host__ __device__ constexpr int win_r(bool scatter) { return scatter ? ST_PWIN_R : ST_PWIN_R_IP; }
__host__ __device__ constexpr int win_x(bool scatter) { return kRowBins + 2 + 2 * win_r(scatter); }
__host__ __device__ constexpr int win_yz(bool scatter) { return 3 + 2 * win_r(scatter); }
__host__ __device__ constexpr int win_cells(bool scatter) { return win_x(scatter) * win_yz(scatter) * win_yz(scatter); }
constexpr int kTable = kRowBins * kSlots;           // destination table entries of an item (i64)
// per-warp slice: stages | fluid window | [scatter: table i64[216], run i32[216]] | rel[9] | mbarriers
// stage stride: the in-place step stages no ids (the float box only, 1152 B)
__host__ __device__ constexpr int stage_bytes(bool scatter) { return scatter ? kTStageBytes : 8 * kBoxF * 4; }
__host__ __device__ constexpr int off_win(bool scatter) { return kPStages * stage_bytes(scatter); }
__host__ __device__ constexpr int off_tab(bool scatter) { return off_win(scatter) + win_cells(scatter) * 16; }
__host__ __device__ constexpr int off_rel(bool scatter) { return off_tab(scatter) + (scatter ? kTable * 12 : kTable * 4); }
__host__ __device__ constexpr int off_bar(bool scatter) { return off_rel(scatter) + 48; }
__host__ __device__ constexpr int pwarp_smem_bytes(bool scatter) {
  return (off_bar(scatter) + 8 * (kPStages + 1) + 127) / 128 * 128;
}
constexpr int kPSmemAlign = 128;   // slack for aligning the dynamic smem base

__device__ __forceinline__ void tma_rows(void* dst, const void* tmap, int c0, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_ids(void* dst, const void* tmap, int c0, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_win(void* dst, const void* tmap, int c0, int c1, int c2, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tstage_issue(TStage* st, unsigned long long* bar, const void* tm_f, const void* tm_id,
                                             int i0, bool with_id) {
  mbar_expect_tx(bar, with_id ? kTxF + kTxI : kTxF);
  tma_rows(st->f, tm_f, i0 & ~3, bar);
  if (with_id) tma_ids(st->id, tm_id, i0 & ~1, bar);
}

#ifndef ST_PMINB
#define ST_PMINB 2      // CTAs per SM of the fused scatter
#endif
#ifndef ST_PMINB_IP
#define ST_PMINB_IP 3   // CTAs per SM of the in-place step (4: 64 registers, spills)
#endif
constexpr int kSpecVP = 1;    // neighbour-rank planes (send buffers) may be destinations
constexpr int kSpecSub = 2;   // more than one sub-step per call
constexpr int kSpecAll = 3;
#ifndef ST_PWARPS
#define ST_PWARPS 8     // warps per CTA of the fused scatter
#endif
__host__ __device__ constexpr int pwarps(bool scatter_advance) { return scatter_advance ? ST_PWARPS : 8; }
template <bool SCATTER, bool ADVANCE, int BCM, int SPEC = kSpecAll, int FEAT = 0xff>
__global__ void __launch_bounds__(32 * pwarps(SCATTER && ADVANCE), (SCATTER && ADVANCE) ? ST_PMINB : ST_PMINB_IP)
    k_pstep(const __grid_constant__ StepArgs a) {
  constexpr int SH = 3;   // chunk_cells == 8
  constexpr bool VP = (SPEC & kSpecVP) != 0;
  extern __shared__ __align__(128) unsigned char psmem_raw[];
  const Geom& g = a.g;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* sbase = psmem_raw + ((kPSmemAlign - (smem_u32(psmem_raw) & (kPSmemAlign - 1))) & (kPSmemAlign - 1));
  unsigned char* ws = sbase + (size_t)wib * pwarp_smem_bytes(SCATTER);
  auto stg = [&](int k) { return reinterpret_cast<TStage*>(ws + k * stage_bytes(SCATTER)); };
  float4* win = reinterpret_cast<float4*>(ws + off_win(SCATTER));
  long long* dtab = reinterpret_cast<long long*>(ws + off_tab(SCATTER));                 // [8*27]
  int* run = reinterpret_cast<int*>(ws + off_tab(SCATTER) + kTable * 8);                  // [8*27]
  int* cnt_s = reinterpret_cast<int*>(ws + off_tab(SCATTER));      // [8*27] slot counts (in place, counting)
  int* rel = reinterpret_cast<int*>(ws + off_rel(SCATTER));                               // [kRowBins+1]
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(ws + off_bar(SCATTER));  // stages | item
  unsigned long long* ibar = bar + kPStages;
  constexpr int WX = win_x(SCATTER), WYZ = win_yz(SCATTER), WR = win_r(SCATTER);
  const int n_items = *a.n_items;
  const int warps_total = gridDim.x * (blockDim.x >> 5);
  const int64_t cap = a.cap;
  const int nbins = a.nbins;
  const int pz = g.gy * g.gx;
  const bool two_way = (FEAT & 4) && a.p.two_way;
  // in place, when this call makes a rebin due: count the slot histogram of the item's
  // bins here (the warp owns them) instead of a later k_count pass over x
  const bool counting = !SCATTER && ADVANCE && a.cnt_hist != nullptr;
  unsigned cmov = 0;
  int cfar = 0;
  int flags = 0;
  uint32_t phase = 0, iphase = 0;
  if (lane == 0) {
    for (int k = 0; k <= kPStages; ++k) mbar_init(bar + k, 1);
    fence_mbar_init();
  }
  __syncwarp();

  for (int item = blockIdx.x * (blockDim.x >> 5) + wib; item < n_items; item += warps_total) {
    const int b0 = a.item_bin0[item];
    const int b1 = (item + 1 < n_items) ? a.item_bin0[item + 1] : nbins;
    const int nb = b1 - b0;                       // <= kRowBins, one chunk row
    const int64_t p0 = a.off[b0];
    const int64_t pe = a.off[b1];
    const int np = (int)(pe - p0);
    const int nbatch = (np + 31) >> 5;
    int rx, ry, rz;                               // cell of the row's first bin (row along +x)
    cell_of_bin(g, a.bg, b0, rx, ry, rz);
    // asynchronous item set-up: the destination table (one bulk copy of k_dbase's rows)
    // and the fluid window (one 3-D tensor copy), then the first particle batches
    if (lane == 0) {
      fence_proxy_async();
      const uint32_t tx = ((FEAT & 2) ? win_cells(SCATTER) * 16u : 0u) + (SCATTER ? kTable * 8u : 0u);
      if (tx) {
        mbar_expect_tx(ibar, tx);
        if (FEAT & 2) tma_win(win, &a.tm_win[WR], 4 * (rx - WR), ry - WR, window_z(g, rz) - 1 - WR, ibar);
        if (SCATTER) bulk_g2s(dtab, a.dtab + (int64_t)b0 * kSlots, kTable * 8u, ibar);
      }
      for (int k = 0; k < kPStages && k < nbatch; ++k)
        tstage_issue(stg(k), bar + k, &a.tm_f, &a.tm_id, (int)(p0 + 32 * k), SCATTER);
    }
    __syncwarp();
    if (lane <= nb) rel[lane] = (int)(a.off[b0 + lane] - p0);
    if (SCATTER)
      for (int k = lane; k < kTable; k += 32) run[k] = 0;
    if (counting)
      for (int k = lane; k < kTable; k += 32) cnt_s[k] = 0;
    if ((FEAT & 2) || SCATTER) {
      mbar_wait(ibar, iphase);
      iphase ^= 1u;
    }
    __syncwarp();
    const int az_row = acc_z(g, rz);
    int lb = 0;
    // per-lane stayer accumulators of bin st_lb: deposit (da*), slot count (hcnt)
    int st_lb = -1, hcnt = 0;
    float da0 = 0.f, da1 = 0.f, da2 = 0.f;
    int carry_lb = -1, carry = 0;                 // stayers of bin carry_lb placed by earlier batches
    for (int bi = 0; bi <= nbatch; ++bi) {
      const bool last = bi == nbatch;             // extra pass: flush only
      const int base = bi << 5;
      const bool valid = !last && base + lane < np;
      const int r = valid ? base + lane : np - 1;            // invalid lanes mirror a valid particle
      if (!last)
        while (rel[lb + 1] <= r) ++lb;
      // flush the stayer accumulators of lanes whose bin changed (one group per bin)
      if (two_way || counting) {
        const bool fl = st_lb >= 0 && (last || lb != st_lb);
        unsigned todo = __ballot_sync(kFull, fl);
        while (todo) {
          const int ld = __ffs(todo) - 1;
          const int kb = __shfl_sync(kFull, st_lb, ld);
          const bool in = fl && st_lb == kb;
          todo &= ~__ballot_sync(kFull, in);
          if (two_way) {
            float ra = da0, rb = da1, rc = da2;
            group_sum3(in, ra, rb, rc);
            if (lane == ld) red_add_v4(a.acc + (uint32_t)((az_row * g.n[1] + ry) * g.n[0] + rx + kb), ra, rb, rc);
          }
          if (counting) {
            const int hc = (int)__reduce_add_sync(kFull, in ? (unsigned)hcnt : 0u);
            if (lane == ld && hc) cnt_s[kb * kSlots + kStay] += hc;
          }
        }
        if (fl || st_lb < 0) {
          st_lb = lb;
          hcnt = 0;
          da0 = da1 = da2 = 0.f;
        }
      }
      if (last) break;
      const int sk = bi % kPStages;
      const int s = b0 + lb;
      const int sx = rx + lb, sy = ry, sz = rz;             // bin cell (row along x)
      mbar_wait(bar + sk, (phase >> sk) & 1u);
      __syncwarp();
      phase ^= 1u << sk;
      const TStage& S = *stg(sk);
      const int so = (int)((p0 + base) & 3) + (r - base);   // slot in the aligned-down box
      float xp0 = S.f[0][so], xp1 = S.f[1][so], xp2 = S.f[2][so];
      float up0 = S.f[3][so], up1 = S.f[4][so], up2 = S.f[5][so];
      const float dp = S.f[6][so], wp = S.f[7][so];
      unsigned long long pid = 0;
      if (SCATTER) pid = S.id[(int)((p0 + base) & 1) + (r - base)];
      // the stage is consumed: refill it with the batch kPStages ahead
      __syncwarp();
      if (lane == 0 && bi + kPStages < nbatch) {
        fence_proxy_async();
        tstage_issue(stg(sk), bar + sk, &a.tm_f, &a.tm_id, (int)(p0 + 32 * (bi + kPStages)), SCATTER);
      }
      __syncwarp();
      float t0 = cell_coord(xp0, g.lo[0], g.ih[0]), t1 = cell_coord(xp1, g.lo[1], g.ih[1]),
            t2 = cell_coord(xp2, g.lo[2], g.ih[2]);
      int c0 = cell_from_t(t0, g.n[0]), c1 = cell_from_t(t1, g.n[1]), c2 = cell_from_t(t2, g.n[2]);
      // fluid corners of a sub-step: from the smem window when the cell lies in the
      // item's row (the whole warp: shared loads), else from the global field
      float4 q[8];
      float fx, fy, fz;
      auto gather = [&](float s0, float s1, float s2, int k0, int k1, int k2) {
        int ix, iy, iz;
        stencil_lo(s0, ix, fx);
        stencil_lo(s1, iy, fy);
        stencil_lo(s2, iz, fz);
        int wz = window_z(g, iz);
        if (wz < 0 || wz + 1 >= g.wnz) {
          if (valid) flags |= ERRF_WINDOW;
          wz = wz < 0 ? 0 : g.wnz - 2;
        }
        if (FEAT & 2) {
          const bool inw = (unsigned)(k0 - rx + WR) < (unsigned)(kRowBins + 2 * WR) &&
                           (unsigned)(k1 - ry + WR) <= (unsigned)(2 * WR) && (unsigned)(k2 - rz + WR) <= (unsigned)(2 * WR);
          if (__all_sync(kFull, inw)) {   // the binned case: shared-memory loads only
            const uint32_t w0 = smem_u32(win + ((iz - rz + 1 + WR) * WYZ + (iy - ry + 1 + WR)) * WX + (ix - rx + 1 + WR));
            constexpr uint32_t oy = WX * 16, oz = WYZ * WX * 16;
            q[0] = lds4(w0); q[1] = lds4(w0 + 16); q[2] = lds4(w0 + oy); q[3] = lds4(w0 + oy + 16);
            q[4] = lds4(w0 + oz); q[5] = lds4(w0 + oz + 16); q[6] = lds4(w0 + oz + oy); q[7] = lds4(w0 + oz + oy + 16);
          } else {
            const float4* fb = inw ? win + ((iz - rz + 1 + WR) * WYZ + (iy - ry + 1 + WR)) * WX + (ix - rx + 1 + WR)
                                   : a.field + ((int64_t)wz * pz + (iy + 1) * g.gx + (ix + 1));
            const int oy = inw ? WX : g.gx, oz = inw ? WYZ * WX : pz;
            q[0] = ld4(fb); q[1] = ld4(fb + 1); q[2] = ld4(fb + oy); q[3] = ld4(fb + oy + 1);
            q[4] = ld4(fb + oz); q[5] = ld4(fb + oz + 1); q[6] = ld4(fb + oz + oy); q[7] = ld4(fb + oz + oy + 1);
          }
        }
      };
#if ST_EARLY_GATHER
      if (ADVANCE && (FEAT & 1)) gather(t0, t1, t2, c0, c1, c2);   // latency overlaps the rank
#endif
      int vside = -1;
      int64_t dest = p0 + r;
      bool write_ok = valid;
      if (SCATTER) {
        const int j = slot_of<BCM>(g, sx, sy, sz, c0, c1, c2);
        const int k = lb * kSlots + (j < 0 ? kStay : j);
        const long long e = dtab[k];                  // -1: leaves the domain; bits 61-62: side + 1
        const long long db = e < 0 ? -1 : (e & ((1LL << 61) - 1));
        const bool farp = j < 0;                      // more than one cell from its bin
        if (valid && !farp && db < 0) {
          flags |= ERRF_SCATTER;
          write_ok = false;
        }
        long long fdest = -1;
        int fside = -1;
        if (valid && farp) {
          // C-15b: a far particle takes the next slot of its destination bin's tail
          const int kz = c2 >> SH;
          int pl;
          if (a.far_cur && kz >= a.bg.kz0 && kz < a.bg.kz0 + a.bg.nkz) {
            fdest = (long long)atomicAdd(a.far_cur + bin_of_cell<SH>(g, a.bg, c0, c1, c2), 1ULL);
            a.far_src[fdest] = (int32_t)(p0 + r);   // prior index: k_far_order sorts the tail by it
            a.far_src_hi[fdest] = 0;
          } else if (VP && a.fs_cur && far_plane(g, c2, fside, pl)) {
            fdest = (long long)atomicAdd(a.fs_cur + fside, 1ULL);   // neighbour rank: far send region
            if (fdest < a.scap) {
              a.fs_key[fside][fdest] = (int32_t)(p0 + r);
              a.fs_cell[fside][fdest] = (c2 * g.n[1] + c1) * g.n[0] + c0;
            }
          } else {
            flags |= ERRF_SCATTER;
            write_ok = false;
          }
        }
        const bool stay = write_ok && j == kStay;
        // stayers: rank inside the lane's bin segment (lanes of one bin are contiguous)
        const unsigned mstay = __ballot_sync(kFull, stay);
        const int lb_up = __shfl_up_sync(kFull, lb, 1);
        const unsigned starts = __ballot_sync(kFull, lane == 0 || lb != lb_up);
        const unsigned lt = lanemask_lt();
        const int ss = 31 - __clz(starts & (lt | (1u << lane)));
        int rbase = (lb == carry_lb ? carry : 0) + __popc(mstay & lt & ~((1u << ss) - 1u));
        {
          const int lb31 = __shfl_sync(kFull, lb, 31);
          const int ss31 = 31 - __clz(starts);
          carry = (lb31 == carry_lb ? carry : 0) + __popc(mstay & ~((1u << ss31) - 1u));
          carry_lb = lb31;
        }
        // movers: groups of equal (bin, slot) keys
        const int key = (write_ok && !stay && !farp) ? k : -1;
        const unsigned peers = __match_any_sync(kFull, key);
        if (key >= 0) {
          const int leader = __ffs(peers) - 1;
          int rb0 = 0;
          if (lane == leader) {
            rb0 = run[key];
            run[key] = rb0 + __popc(peers);
          }
          rbase = __shfl_sync(peers, rb0, leader) + __popc(peers & lt);
        }
        __syncwarp();
        if (VP) vside = farp ? fside : (e < 0 ? -1 : (int)(e >> 61) - 1);
        dest = farp ? fdest : db + rbase;
        if (write_ok && (uint64_t)dest >= (uint64_t)((VP && vside >= 0) ? a.scap : a.n)) {
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
        const int nsub = (SPEC & kSpecSub) ? a.nsteps : 1;
        for (int sub = 0; sub < nsub; ++sub) {
          if (sub > 0) {
            t0 = cell_coord(xp0, g.lo[0], g.ih[0]);
            t1 = cell_coord(xp1, g.lo[1], g.ih[1]);
            t2 = cell_coord(xp2, g.lo[2], g.ih[2]);
            c0 = cell_from_t(t0, g.n[0]);
            c1 = cell_from_t(t1, g.n[1]);
            c2 = cell_from_t(t2, g.n[2]);
          }
#if ST_EARLY_GATHER
          if (sub > 0)
#endif
            gather(t0, t1, t2, c0, c1, c2);
          const float4 uf = (FEAT & 2) ? trilerp(q, fx, fy, fz) : make_float4(0.1f, 0.0f, 0.0f, 0.0f);
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
          if (two_way) {
            // reaction into the sub-step start cell (Eq. 11); the bin cell's share is
            // accumulated in registers, other cells take an individual red
            const int az = acc_z(g, c2);
            if (valid && az < 0) flags |= ERRF_WINDOW;
            const float ja = -mw * du0, jb = -mw * du1, jc = -mw * du2;
            if (valid && c0 == sx && c1 == sy && c2 == sz) {
              da0 += ja;
              da1 += jb;
              da2 += jc;
            } else if (valid && az >= 0) {
              red_add_v4(a.acc + (uint32_t)((az * g.n[1] + c1) * g.n[0] + c0), ja, jb, jc);
            }
          }
          // walls / wrap (C-11, C-12): one warp vote skips the three axes when no lane
          // left the box (the common case)
          const bool out = (xp0 < g.lo[0]) | (xp0 >= g.hi[0]) | (xp1 < g.lo[1]) | (xp1 >= g.hi[1]) |
                           (xp2 < g.lo[2]) | (xp2 >= g.hi[2]);
          if (__any_sync(kFull, out)) {
            bool bad = false;
            bad |= apply_bc(periodic<BCM>(g, 0) ? ST_BC_PERIODIC : ST_BC_REFLECT, g.lo[0], g.hi[0], g.L[0], xp0, up0);
            bad |= apply_bc(periodic<BCM>(g, 1) ? ST_BC_PERIODIC : ST_BC_REFLECT, g.lo[1], g.hi[1], g.L[1], xp1, up1);
            bad |= apply_bc(periodic<BCM>(g, 2) ? ST_BC_PERIODIC : ST_BC_REFLECT, g.lo[2], g.hi[2], g.L[2], xp2, up2);
            if (bad && valid) flags |= ERRF_CFL;
          }
        }
      }
      if (counting && valid) {
        // slot of the end cell relative to the bin (the next rebin's input)
        const int e0 = cell_from_t(cell_coord(xp0, g.lo[0], g.ih[0]), g.n[0]);
        const int e1 = cell_from_t(cell_coord(xp1, g.lo[1], g.ih[1]), g.n[1]);
        const int e2 = cell_from_t(cell_coord(xp2, g.lo[2], g.ih[2]), g.n[2]);
        const int j2 = slot_of<BCM>(g, sx, sy, sz, e0, e1, e2);
        if (j2 == kStay) {
          ++hcnt;
        } else if (j2 >= 0) {
          atomicAdd(&cnt_s[lb * kSlots + j2], 1);
        } else {   // far (C-15b): counted for the bin of its cell when that is on this rank
          const int kz = e2 >> SH;
          if (a.cnt_far_cnt && kz >= a.bg.kz0 && kz < a.bg.kz0 + a.bg.nkz) {
            atomicAdd(a.cnt_far_cnt + bin_of_cell<SH>(g, a.bg, e0, e1, e2), 1);
            atomicAdd(a.cnt_far_n, 1ULL);
          } else {
            cfar = 1;
          }
        }
        cmov += ((e0 >> SH) != (sx >> SH)) | ((e1 >> SH) != (sy >> SH)) | ((e2 >> SH) != (sz >> SH));
      }
      if ((FEAT & 16) && write_ok) {
        if (SCATTER) {
          const Store& o = (VP && vside >= 0) ? a.sbuf[vside] : a.B;
          const int64_t oc = (VP && vside >= 0) ? a.scap : cap;
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
    if (counting) {   // the item's bins are this warp's: plain stores, every entry
      for (int k = lane; k < nb * kSlots; k += 32) {
        const int l = k / kSlots, j = k - l * kSlots;
        a.cnt_hist[(int64_t)j * nbins + b0 + l] = cnt_s[k];
      }
      __syncwarp();
    }
  }
  if (counting) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cmov += __shfl_xor_sync(kFull, cmov, o);
    if (lane == 0 && cmov) atomicAdd(a.cnt_movers, (unsigned long long)cmov);
    if (cfar) *(volatile int*)a.cnt_far = 1;
  }
  if (flags) atomicOr(a.err, flags);
}
