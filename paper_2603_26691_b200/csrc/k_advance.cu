// KB2 — the fused particle step:
//   locate -> trilinear u_f -> Re, f(Re), tau_e -> exponential (or semi-implicit)
//   update of u and x -> deposit -w m du_drag into the start cell -> walls/wrap
//   -> relocate (chunk key of the end position, consumed by the rebin).
// Paper: Eq. 9-11, sub-stepping, reflection.
#include <cuda_runtime.h>

#include "st_device.cuh"

namespace st {

namespace {

// red.global.add.v4.f32 (sm_90+): one 16-byte reduction per cell instead of three.
__device__ __forceinline__ void red_add_v4(float4* addr, float a, float b, float c) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
               "f"(c), "f"(0.0f)
               : "memory");
}

struct Stencil {
  int wx, wy, wz;       // window index of the lower corner
  float fx, fy, fz;     // fractional weights
};

// C-5: stencil base floor(t - 1/2), weights t - 1/2 - base, clamped to the
// ghost layer [-1, n-1] (positions are in [lo, hi], so clamping only absorbs
// rounding at the faces).
__device__ __forceinline__ void stencil_axis(float t, int n, int& i, float& f) {
  float s = t - 0.5f;
  float fl = floorf(s);
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
  float4 c000 = __ldg(b), c100 = __ldg(b + 1);
  float4 c010 = __ldg(b + g.gx), c110 = __ldg(b + g.gx + 1);
  float4 c001 = __ldg(b + pz), c101 = __ldg(b + pz + 1);
  float4 c011 = __ldg(b + pz + g.gx), c111 = __ldg(b + pz + g.gx + 1);
  float4 c00 = lerp4(c000, c100, s.fx), c10 = lerp4(c010, c110, s.fx);
  float4 c01 = lerp4(c001, c101, s.fx), c11 = lerp4(c011, c111, s.fx);
  float4 c0 = lerp4(c00, c10, s.fy), c1 = lerp4(c01, c11, s.fy);
  return lerp4(c0, c1, s.fz);
}

__global__ void __launch_bounds__(256) k_advance_v1(Geom g, Phys p, const float4* __restrict__ field,
                                                    float4* __restrict__ acc, float* __restrict__ x,
                                                    float* __restrict__ u, const float* __restrict__ dd,
                                                    const float* __restrict__ ww, int64_t cap, int64_t n,
                                                    float dt, int nsteps, int32_t* __restrict__ key_out,
                                                    int* __restrict__ err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float xp[3] = {x[i], x[cap + i], x[2 * cap + i]};
  float up[3] = {u[i], u[cap + i], u[2 * cap + i]};
  const float d = dd[i];
  const float w = ww[i];
  const float tau = p.tau_c * d * d;                 // C-3
  const float inv_tau = __frcp_rn(tau);
  const float mw = p.mass_c * d * d * d * w;         // w m_p (C-17, C-18)
  int flags = 0;
  for (int s = 0; s < nsteps; ++s) {
    // 1  deposit cell (C-6, C-10) and stencil (C-5) from the same t = (x-lo)*ih
    float t[3];
    int c[3];
    Stencil st;
    for (int a = 0; a < 3; ++a) {
      t[a] = cell_coord(xp[a], g.lo[a], g.ih[a]);
      c[a] = cell_from_t(t[a], g.n[a]);
    }
    int ix, iy, iz;
    stencil_axis(t[0], g.n[0], ix, st.fx);
    stencil_axis(t[1], g.n[1], iy, st.fy);
    stencil_axis(t[2], g.n[2], iz, st.fz);
    st.wx = ix + 1;
    st.wy = iy + 1;
    st.wz = window_z(g, iz);
    if (st.wz < 0 || st.wz + 1 >= g.wnz) {   // outside this rank's field window
      flags |= ERRF_WINDOW;
      st.wz = st.wz < 0 ? 0 : g.wnz - 2;
    }
    // 2  u_f at x_p, once per sub-step
    const float4 uf = trilinear(g, field, st);
    // 3  Re, f(Re), tau_e, h (C-2, C-3)
    const float sx = uf.x - up[0], sy = uf.y - up[1], sz = uf.z - up[2];
    const float Re = sqrtf(fmaf(sx, sx, fmaf(sy, sy, sz * sz))) * d * p.inv_nu;
    const float f = drag_factor(p.drag_law, Re);
    const float taue = tau * __frcp_rn(f);
    const float h = dt * f * inv_tau;
    const float ufa[3] = {uf.x, uf.y, uf.z};
    float du[3];
    // 4  integrate (C-4)
    if (p.integrator == ST_INT_EXPONENTIAL) {
      float E, M;
      exp_pair(h, E, M);
      const float tM = taue * M;
      for (int a = 0; a < 3; ++a) {
        const float us = fmaf(p.g[a], taue, ufa[a]);
        const float rel = up[a] - us;
        du[a] = fmaf(-M, rel, -p.g[a] * dt);
        xp[a] = fmaf(tM, rel, fmaf(us, dt, xp[a]));
        up[a] = fmaf(E, rel, us);
      }
    } else {
      const float inv1h = __frcp_rn(1.0f + h);
      for (int a = 0; a < 3; ++a) {
        const float un = (up[a] + h * ufa[a] + dt * p.g[a]) * inv1h;
        du[a] = (un - up[a]) - p.g[a] * dt;
        xp[a] = fmaf(dt, un, xp[a]);
        up[a] = un;
      }
    }
    // 5  two-way: fluid-side reaction into the start cell (Eq. 11, C-8, C-9)
    if (p.two_way) {
      const int az = acc_z(g, c[2]);
      if (az >= 0) {
        float4* cellp = acc + ((int64_t)az * g.n[1] + c[1]) * g.n[0] + c[0];
        red_add_v4(cellp, -mw * du[0], -mw * du[1], -mw * du[2]);
      } else {
        flags |= ERRF_WINDOW;
      }
    }
    // 6  walls / periodic (C-11, C-12)
    for (int a = 0; a < 3; ++a)
      if (apply_bc(g.bc[a], g.lo[a], g.hi[a], g.L[a], xp[a], up[a])) flags |= ERRF_CFL;
  }
  x[i] = xp[0]; x[cap + i] = xp[1]; x[2 * cap + i] = xp[2];
  u[i] = up[0]; u[cap + i] = up[1]; u[2 * cap + i] = up[2];
  if (key_out) {
    int c[3];
    for (int a = 0; a < 3; ++a) c[a] = cell_from_t(cell_coord(xp[a], g.lo[a], g.ih[a]), g.n[a]);
    key_out[i] = chunk_linear(g, c[0], c[1], c[2]);
  }
  if (flags) atomicOr(err, flags);
}

}  // namespace

int launch_advance(const Geom& g, const Phys& p, const float4* field, float4* acc, Store st, int64_t cap,
                   int64_t n, const Tile* tiles, int ntiles, float dt, int nsteps, int32_t* key_out, int* err,
                   cudaStream_t s) {
  (void)tiles;
  (void)ntiles;
  if (n <= 0) return 0;
  const int bs = 256;
  const int64_t nb = (n + bs - 1) / bs;
  k_advance_v1<<<(unsigned)nb, bs, 0, s>>>(g, p, field, acc, st.x, st.u, st.d, st.w, cap, n, dt, nsteps,
                                          key_out, err);
  return 1;
}

}  // namespace st
