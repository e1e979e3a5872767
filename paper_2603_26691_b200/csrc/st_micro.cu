// Droplet microphysics step (Eq. 7, 8, 9-11, 12, 13, P:138-167;
// C-ABI in include/scaletrack.h, readings C-28..C-33).
//
// One thread per droplet carries its state in registers through all nsteps sub-steps
// (the field is frozen within a call, C-7, so droplets are independent): the state is
// read and written once per call (24 B in + 24 B out + 4 B weight per droplet) and
// every sub-step adds 5 fp64 reductions into the start cell, one per run of lanes that
// share the cell (a binned store, C-15, makes those runs long).  Arithmetic is fp64 on
// fp32 storage (C-28); this file is compiled with -fmad=false so each operation rounds
// on its own, in the order the definition is written (the oracle's order); with the
// libm-vs-CUDA differences of exp/cbrt and the d^3, Re^0.687 forms (a few fp64 ulp) the
// fp32 state and the cell decisions match the oracle's except for rare last-bit flips.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "scaletrack.h"

namespace {

struct MicroArgs {
  int64_t n;
  int nx, ny, nz;
  double lo[3], hi[3], L[3], ih[3];
  int bc[3];
  double g[3];
  int drag_law;
  double dt;
  int nsteps;
  // host-folded constants (each folded the way the oracle writes it)
  double rho_p, nu_f, c18;    // c18 = 18 rho_f nu_f
  double c_m;                 // 2 pi D_v
  double c_q;                 // pi Nu kappa_f
  double c_d;                 // pi rho_p
  double c_m6;                // pi/6 rho_p
  double s_vp, latent, cp_p;
  float* x;
  float* u;
  float* d;
  float* T;
  const float* w;
  const float* F;
  double* acc;
  unsigned long long* counters;   // [0] clamps, [1] CFL violations
};

// Ghost mapping of i in [-1, n] (C-5): periodic wraps, reflecting replicates the edge.
__device__ __forceinline__ int ghost(int i, int n, int bc) {
  if (bc == ST_BC_PERIODIC) return i < 0 ? i + n : (i >= n ? i - n : i);
  return i < 0 ? 0 : (i > n - 1 ? n - 1 : i);
}

__device__ __forceinline__ int cell_axis(double x, double lo, double ih, int n) {
  double f = floor((x - lo) * ih);
  if (!(f >= 0.0)) return 0;
  if (f >= (double)n) return n - 1;
  return (int)f;
}

__global__ void __launch_bounds__(256, 4) k_micro(MicroArgs a) {
  const int64_t ncell = (int64_t)a.nx * a.ny * a.nz;
  const int dims[3] = {a.nx, a.ny, a.nz};
  unsigned long long clamps = 0, cfl = 0;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // whole warps iterate together (the deposit reduction below is warp-collective)
  const int64_t n_round = (a.n + 31) & ~(int64_t)31;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
    const bool valid = i < a.n;
    const int64_t j = valid ? i : a.n - 1;          // tail lanes shadow the last droplet
    float xs[3] = {a.x[j], a.x[a.n + j], a.x[2 * a.n + j]};
    float us[3] = {a.u[j], a.u[a.n + j], a.u[2 * a.n + j]};
    float ds = a.d[j], Ts = a.T[j];
    const double wn = valid ? -(double)a.w[j] : 0.0;
    for (int s = 0; s < a.nsteps; ++s) {
      double xp[3] = {xs[0], xs[1], xs[2]}, up[3] = {us[0], us[1], us[2]};
      const double dp = ds, Tp = Ts;
      // 1 deposit cell = cell of the start position (C-10)
      int c[3];
      for (int k = 0; k < 3; ++k) c[k] = cell_axis(xp[k], a.lo[k], a.ih[k], dims[k]);
      const int64_t cell = ((int64_t)c[2] * a.ny + c[1]) * a.nx + c[0];
      // 2 trilinear (u_f, T_f, rho_v) at x_p (C-5), loop order z, y, x as the oracle
      int i0[3];
      double fr[3];
      for (int k = 0; k < 3; ++k) {
        double t = (xp[k] - a.lo[k]) * a.ih[k];
        double sv = t - 0.5;
        double fl = floor(sv);
        int ii = (int)fl;
        double f = sv - fl;
        if (ii < -1) { ii = -1; f = 0.0; }
        if (ii > dims[k] - 1) { ii = dims[k] - 1; f = 1.0; }
        i0[k] = ii;
        fr[k] = f;
      }
      int gi[3][2];
      for (int k = 0; k < 3; ++k) {
        gi[k][0] = ghost(i0[k], dims[k], a.bc[k]);
        gi[k][1] = ghost(i0[k] + 1, dims[k], a.bc[k]);
      }
      double fv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int cz = 0; cz < 2; ++cz)
#pragma unroll
        for (int cy = 0; cy < 2; ++cy)
#pragma unroll
          for (int cx = 0; cx < 2; ++cx) {
            double wt = ((cx ? fr[0] : 1.0 - fr[0]) * (cy ? fr[1] : 1.0 - fr[1])) * (cz ? fr[2] : 1.0 - fr[2]);
            const int64_t cc = ((int64_t)gi[2][cz] * a.ny + gi[1][cy]) * a.nx + gi[0][cx];
#pragma unroll
            for (int k = 0; k < 5; ++k) fv[k] = fv[k] + wt * (double)__ldg(a.F + k * ncell + cc);
          }
      const double Tf = fv[3], rv = fv[4];
      // 3 drag, semi-implicit Euler (Eq. 9-10)
      double sl[3] = {fv[0] - up[0], fv[1] - up[1], fv[2] - up[2]};
      const double Re = sqrt((sl[0] * sl[0] + sl[1] * sl[1]) + sl[2] * sl[2]) * dp / a.nu_f;
      double fdr = 1.0;
      if (a.drag_law == ST_DRAG_SCHILLER_NAUMANN)
        fdr = Re <= 1000.0 ? 1.0 + 0.15 * exp2(0.687 * log2(Re)) : 0.44 * Re / 24.0;   // Re = 0 -> 1 (C-22)
      const double tau = a.rho_p * dp * dp / a.c18;
      const double h = a.dt / (tau / fdr);
      double un[3], xn[3];
      for (int k = 0; k < 3; ++k) {
        un[k] = ((up[k] + h * fv[k]) + a.dt * a.g[k]) / (1.0 + h);
        xn[k] = xp[k] + a.dt * un[k];
      }
      // 4 mass (Eq. 7, Magnus C-30) and temperature (Eq. 12), explicit Euler
      const double m = a.c_m6 * (dp * dp * dp);     // d^3 to <= 1.5 fp64 ulp of the oracle's pow
      const double tc = Tf - 273.15;
      const double es = 610.94 * exp(17.625 * tc / (tc + 243.04));
      const double rs = es / (461.5 * Tf);
      const double svf = rv / rs;
      const double mdot = a.c_m * dp * rs * (svf - a.s_vp);
      double mn = m + a.dt * mdot;
      const double mfloor = 0.01 * m;
      if (mn < mfloor) { mn = mfloor; clamps += valid; }
      const double q = a.c_q * dp * (Tf - Tp);
      const double Tn = Tp + a.dt * ((q - a.latent * mdot) / (m * a.cp_p));
      const double dn = cbrt(6.0 * mn / a.c_d);
      // 5 fluid-side sources into the start cell (Eq. 8, 11, 13; C-8, C-33)
      double dep[5];
      for (int k = 0; k < 3; ++k) dep[k] = wn * ((mn * un[k] - m * up[k]) - m * a.g[k] * a.dt);
      dep[3] = wn * (mn - m);
      dep[4] = wn * a.cp_p * (mn * Tn - m * Tp);
      // Runs of lanes with the same start cell (contiguous in a binned store) are summed
      // into the run's first lane by a segmented suffix scan; one fp64 reduction per run.
      const int key = valid ? (int)cell : -1 - lane;
      const int prev = __shfl_up_sync(0xffffffffu, key, 1);
      const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || prev != key);
      const unsigned above = lane == 31 ? 0u : heads & (0xffffffffu << (lane + 1));
      const int end = above ? __ffs(above) - 1 : 32;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const double o = __shfl_down_sync(0xffffffffu, dep[k], off);
          if (lane + off < end) dep[k] = dep[k] + o;
        }
      }
      if (valid && ((heads >> lane) & 1u))
        for (int k = 0; k < 5; ++k) atomicAdd(a.acc + k * ncell + cell, dep[k]);
      // 6 walls / periodic (C-11, C-12), round the state to fp32
      for (int k = 0; k < 3; ++k) {
        double v = xn[k];
        if (a.bc[k] == ST_BC_PERIODIC) {
          if (v < a.lo[k]) v = v + a.L[k];
          else if (v >= a.hi[k]) v = v - a.L[k];
          if (v < a.lo[k] || v >= a.hi[k]) cfl += valid;
        } else {
          if (v < a.lo[k]) { v = 2.0 * a.lo[k] - v; un[k] = -un[k]; if (v > a.hi[k]) cfl += valid; }
          else if (v > a.hi[k]) { v = 2.0 * a.hi[k] - v; un[k] = -un[k]; if (v < a.lo[k]) cfl += valid; }
        }
        xs[k] = (float)v;
        // C-12 fix-up in storage precision: a wrap that rounds onto hi is stored as lo
        if (a.bc[k] == ST_BC_PERIODIC && (xs[k] >= (float)a.hi[k] || xs[k] < (float)a.lo[k])) xs[k] = (float)a.lo[k];
        us[k] = (float)un[k];
      }
      ds = (float)dn;
      Ts = (float)Tn;
    }
    if (!valid) continue;
    for (int k = 0; k < 3; ++k) {
      a.x[k * a.n + i] = xs[k];
      a.u[k * a.n + i] = us[k];
    }
    a.d[i] = ds;
    a.T[i] = Ts;
  }
  if (clamps) atomicAdd(a.counters, clamps);
  if (cfl) atomicAdd(a.counters + 1, cfl);
}

bool is_device(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace

extern "C" void st_micro_config_default(st_micro_config* c) {
  if (!c) return;
  *c = st_micro_config{};
  c->abi_version = ST_ABI_VERSION;
  for (int k = 0; k < 3; ++k) {
    c->dims[k] = 1;
    c->origin[k] = 0.0;
    c->cell_size[k] = 1.0;
    c->bc[k] = ST_BC_REFLECT;
  }
  c->rho_f = 1.2;
  c->nu_f = 1.5e-5;
  c->rho_p = 1000.0;
  c->gravity[2] = -9.81;
  c->drag_law = ST_DRAG_SCHILLER_NAUMANN;
  c->D_v = 2.5e-5;
  c->kappa_f = 0.025;
  c->cp_p = 4186.0;
  c->latent = 2.45e6;
  c->nusselt = 2.0;
  c->s_vp = 1.0;
}

extern "C" st_status st_micro_advance(const st_micro_config* c, int64_t n, float* x, float* u, float* d,
                                      float* T, const float* w, const float* F, double dt, int32_t nsteps,
                                      double* acc, int64_t* n_clamped) {
  if (!c || c->abi_version != ST_ABI_VERSION || n < 0 || nsteps < 0 || !(dt > 0.0)) return ST_ERR_INVALID_ARG;
  for (int k = 0; k < 3; ++k)
    if (c->dims[k] < 1 || !(c->cell_size[k] > 0.0) || (c->bc[k] != ST_BC_PERIODIC && c->bc[k] != ST_BC_REFLECT))
      return ST_ERR_INVALID_ARG;
  if ((int64_t)c->dims[0] * c->dims[1] * c->dims[2] >= (1ll << 31)) return ST_ERR_INVALID_ARG;
  if (c->drag_law != ST_DRAG_STOKES && c->drag_law != ST_DRAG_SCHILLER_NAUMANN) return ST_ERR_INVALID_ARG;
  if (!(c->rho_p > 0.0) || !(c->rho_f > 0.0) || !(c->nu_f > 0.0) || !(c->cp_p > 0.0)) return ST_ERR_INVALID_ARG;
  if (n_clamped) *n_clamped = 0;
  if (n == 0 || nsteps == 0) return ST_OK;
  if (!x || !u || !d || !T || !w || !F || !acc) return ST_ERR_INVALID_ARG;
  if (cudaSetDevice(c->device) != cudaSuccess) return ST_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)c->stream;
  // host arrays (the other st_* calls accept host or device pointers too): stage every
  // array through device memory, run, copy the updated ones back (blocking)
  {
    const void* ptrs[7] = {x, u, d, T, w, F, acc};
    bool all_dev = true, any_dev = false;
    for (const void* p : ptrs) {
      const bool dv = is_device(p);
      all_dev &= dv;
      any_dev |= dv;
    }
    if (!all_dev) {
      if (any_dev) return ST_ERR_INVALID_ARG;   // mixed host / device arrays
      const int64_t nc = (int64_t)c->dims[0] * c->dims[1] * c->dims[2];
      const size_t bx = 3 * n * sizeof(float), b1 = n * sizeof(float), bF = 5 * nc * sizeof(float),
                   bA = 5 * nc * sizeof(double);
      char* buf = nullptr;
      if (cudaMallocAsync(&buf, 2 * bx + 3 * b1 + bF + bA, s) != cudaSuccess) return ST_ERR_CUDA;
      float* dx = (float*)buf;
      float* du = (float*)(buf + bx);
      float* dd = (float*)(buf + 2 * bx);
      float* dT = (float*)(buf + 2 * bx + b1);
      float* dw = (float*)(buf + 2 * bx + 2 * b1);
      float* dF = (float*)(buf + 2 * bx + 3 * b1);
      double* dA = (double*)(buf + 2 * bx + 3 * b1 + bF);
      cudaError_t e = cudaSuccess;
      const void* src[7] = {x, u, d, T, w, F, acc};
      void* dst[7] = {dx, du, dd, dT, dw, dF, dA};
      const size_t sz[7] = {bx, bx, b1, b1, b1, bF, bA};
      for (int k = 0; k < 7 && e == cudaSuccess; ++k) e = cudaMemcpyAsync(dst[k], src[k], sz[k], cudaMemcpyHostToDevice, s);
      st_status st = e == cudaSuccess ? st_micro_advance(c, n, dx, du, dd, dT, dw, dF, dt, nsteps, dA, n_clamped)
                                      : ST_ERR_CUDA;
      void* back[5] = {x, u, d, T, acc};
      const void* from[5] = {dx, du, dd, dT, dA};
      const size_t bsz[5] = {bx, bx, b1, b1, bA};
      for (int k = 0; k < 5 && (st == ST_OK || st == ST_ERR_CFL); ++k)
        if (cudaMemcpyAsync(back[k], from[k], bsz[k], cudaMemcpyDeviceToHost, s) != cudaSuccess) st = ST_ERR_CUDA;
      cudaFreeAsync(buf, s);
      if (cudaStreamSynchronize(s) != cudaSuccess) st = ST_ERR_CUDA;
      return st;
    }
  }

  MicroArgs a{};
  a.n = n;
  a.nx = c->dims[0];
  a.ny = c->dims[1];
  a.nz = c->dims[2];
  for (int k = 0; k < 3; ++k) {
    a.lo[k] = c->origin[k];
    a.hi[k] = c->origin[k] + (double)c->dims[k] * c->cell_size[k];
    a.L[k] = a.hi[k] - a.lo[k];
    a.ih[k] = 1.0 / c->cell_size[k];
    a.bc[k] = c->bc[k];
    a.g[k] = c->gravity[k];
  }
  a.drag_law = c->drag_law;
  a.dt = dt;
  a.nsteps = nsteps;
  const double pi = 3.141592653589793;
  a.rho_p = c->rho_p;
  a.nu_f = c->nu_f;
  a.c18 = 18.0 * c->rho_f * c->nu_f;
  a.c_m = 2.0 * pi * c->D_v;
  a.c_q = pi * c->nusselt * c->kappa_f;
  a.c_d = pi * c->rho_p;
  a.c_m6 = pi / 6.0 * c->rho_p;
  a.s_vp = c->s_vp;
  a.latent = c->latent;
  a.cp_p = c->cp_p;
  a.x = x;
  a.u = u;
  a.d = d;
  a.T = T;
  a.w = w;
  a.F = F;
  a.acc = acc;

  unsigned long long* cnt = nullptr;
  if (cudaMallocAsync(&cnt, 2 * sizeof(unsigned long long), s) != cudaSuccess) return ST_ERR_CUDA;
  cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), s);
  a.counters = cnt;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
  const int64_t need = (n + 255) / 256;   // block size 256 = 8 whole warps
  const int64_t cap = (int64_t)nsm * 8;            // 8 resident 256-thread CTAs per SM
  const int grid = (int)(need < cap ? need : cap);
  k_micro<<<grid, 256, 0, s>>>(a);
  unsigned long long h[2] = {0, 0};
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(cnt, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return ST_ERR_CUDA;
  if (n_clamped) *n_clamped = (int64_t)h[0];
  return h[1] ? ST_ERR_CFL : ST_OK;
}
