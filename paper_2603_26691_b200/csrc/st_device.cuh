// Device-side building blocks of the particle step (sm_100a).
// Readings: C-2 drag, C-3 tau/Re, C-4 exponential integrator,
// C-5 trilinear, C-6 cell contract, C-10 deposit cell, C-11 reflect, C-12 wrap.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "st_internal.h"

namespace st {

// C-6: c = clamp(floor((x - lo) * ih), 0, n-1); subtraction and product each
// rounded to binary32 (explicit _rn intrinsics: never contracted into an FMA).
__device__ __forceinline__ float cell_coord(float x, float lo, float ih) {
  return __fmul_rn(__fsub_rn(x, lo), ih);
}
__device__ __forceinline__ int cell_from_t(float t, int n) {
  // cvt.rmi (floor; NaN -> 0, saturating) then clamp to [0, n-1]: identical to
  // "floor; <0 or NaN -> 0; >= n -> n-1" of the contract
  const int f = __float2int_rd(t);
  return min(max(f, 0), n - 1);
}

__device__ __forceinline__ int64_t cell_linear(const Geom& g, int cx, int cy, int cz) {
  return ((int64_t)cz * g.n[1] + cy) * g.n[0] + cx;
}
__device__ __forceinline__ int32_t chunk_linear(const Geom& g, int cx, int cy, int cz) {
  return (int32_t)(((cz / g.cc) * g.NC[1] + cy / g.cc) * g.NC[0] + cx / g.cc);
}

// Field window plane index of global plane gz (periodic z with a partial
// window wraps by the global size).  Returns -1 if outside the window.
__device__ __forceinline__ int window_z(const Geom& g, int gz) {
  int iz = gz - g.wz0;
  if (g.wrapz) {
    if (iz < 0) iz += g.n[2];
    else if (iz >= g.wnz) iz -= g.n[2];
  }
  return (iz >= 0 && iz < g.wnz) ? iz : -1;
}
__device__ __forceinline__ int acc_z(const Geom& g, int gz) {
  int ia = gz - g.az0;
  if (g.wrapz) {
    if (ia < 0) ia += g.n[2];
    else if (ia >= g.anz) ia -= g.n[2];
  }
  return (ia >= 0 && ia < g.anz) ? ia : -1;
}

// exp(-h) and M = -expm1(-h) = 1 - exp(-h), accurate to ~1e-7 relative for all
// h >= 0 (series below 1/8 avoids the cancellation of 1 - exp(-h)).
__device__ __forceinline__ void exp_pair(float h, float& E, float& M) {
  E = __expf(-h);
  if (h < 0.125f) {
    M = h * (1.0f - h * (0.5f - h * (1.0f / 6.0f - h * (1.0f / 24.0f - h * (1.0f / 120.0f - h * (1.0f / 720.0f))))));
  } else {
    M = 1.0f - E;
  }
}

// C-2: Schiller-Naumann factor f = C_D Re / 24.
__device__ __forceinline__ float drag_factor(int law, float Re) {
  if (law == ST_DRAG_STOKES) return 1.0f;
  if (Re <= 1000.0f) return 1.0f + 0.15f * exp2f(0.687f * __log2f(Re));
  return 0.44f / 24.0f * Re;
}

// C-11 / C-12 boundary rule for one axis; returns true if the displacement
// precondition is violated.
__device__ __forceinline__ bool apply_bc(int bc, float lo, float hi, float L, float& x, float& u) {
  float v = x;
  if (bc == ST_BC_PERIODIC) {
    bool bad = false;
    if (v < lo) {
      v = __fadd_rn(v, L);
      if (v >= hi) v = lo;
      else if (v < lo) bad = true;
    } else if (v >= hi) {
      v = __fsub_rn(v, L);
      if (v < lo) v = lo;
      else if (v >= hi) bad = true;
    }
    x = v;
    return bad;
  }
  if (v < lo) {
    v = __fsub_rn(__fmul_rn(2.0f, lo), v);
    u = -u;
    x = v;
    return v > hi;
  }
  if (v > hi) {
    v = __fsub_rn(__fmul_rn(2.0f, hi), v);
    u = -u;
    x = v;
    return v < lo;
  }
  return false;
}

}  // namespace st
