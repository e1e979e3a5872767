// KB1 field ingest, KB6 source readout, locate / key / domain-check kernels.
// Field ingest: cell-centred u_f [3][nz][ny][nx] -> float4 window with a ghost
// layer (periodic wrap or replicate, C-5).  Readout: S = acc/(V_cell T_acc) (C-13).
#include <cuda_runtime.h>

#include "st_device.cuh"

namespace st {

namespace {

__device__ __forceinline__ int ghost_map(int i, int n, int bc) {
  if (bc == ST_BC_PERIODIC) {
    if (i < 0) return i + n;
    if (i >= n) return i - n;
    return i;
  }
  return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

// One thread per window cell (x fastest): gathers 3 components and writes one
// 16-byte float4.
__global__ void k_field_ingest(Geom g, const float* __restrict__ src, int64_t comp_stride, int src_z0,
                               int src_nz, float4* __restrict__ field) {
  const int64_t total = (int64_t)g.wnz * g.gy * g.gx;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int ix = (int)(q % g.gx);
    const int iy = (int)((q / g.gx) % g.gy);
    const int iz = (int)(q / ((int64_t)g.gx * g.gy));
    const int x = ghost_map(ix - 1, g.n[0], g.bc[0]);
    const int y = ghost_map(iy - 1, g.n[1], g.bc[1]);
    int z = ghost_map(g.wz0 + iz, g.n[2], g.bc[2]);
    int sz = z - src_z0;
    if (g.bc[2] == ST_BC_PERIODIC) {
      if (sz < 0) sz += g.n[2];
      else if (sz >= src_nz) sz -= g.n[2];
    }
    sz = sz < 0 ? 0 : (sz >= src_nz ? src_nz - 1 : sz);
    const int64_t c = ((int64_t)sz * g.n[1] + y) * g.n[0] + x;
    field[q] = make_float4(src[c], src[comp_stride + c], src[2 * comp_stride + c], 0.0f);
  }
}

// out[k][z-z0][y][x] = acc[z][y][x].k * scale for owned planes [z0, z1); the
// accumulator window is then zeroed by the caller (cudaMemsetAsync).
__global__ void k_source_readout(Geom g, const float4* __restrict__ acc, int z0, int z1, float scale,
                                 float* __restrict__ out) {
  const int64_t plane = (int64_t)g.n[0] * g.n[1];
  const int64_t total = plane * (z1 - z0);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int z = z0 + (int)(q / plane);
    const int64_t r = q % plane;
    int ia = z - g.az0;
    if (g.wrapz) {
      if (ia < 0) ia += g.n[2];
      else if (ia >= g.anz) ia -= g.n[2];
    }
    const float4 v = acc[(int64_t)ia * plane + r];
    out[q] = v.x * scale;
    out[total + q] = v.y * scale;
    out[2 * total + q] = v.z * scale;
  }
}

__global__ void k_locate(Geom g, const float* __restrict__ x, int64_t xs, int64_t n, int32_t* __restrict__ cell,
                         int32_t* __restrict__ chunk) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int c[3];
    for (int a = 0; a < 3; ++a) c[a] = cell_from_t(cell_coord(x[a * xs + i], g.lo[a], g.ih[a]), g.n[a]);
    if (cell) cell[i] = (int32_t)cell_linear(g, c[0], c[1], c[2]);
    if (chunk) chunk[i] = chunk_linear(g, c[0], c[1], c[2]);
  }
}

__global__ void k_check_domain(Geom g, const float* __restrict__ x, int64_t xs, int64_t n, int* err) {
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int a = 0; a < 3; ++a) {
      const float v = x[a * xs + i];
      if (!(v >= g.lo[a] && v <= g.hi[a])) bad = 1;
    }
    // multi-GPU: the particle's cell must lie in this rank's slab
    const int cz = cell_from_t(cell_coord(x[2 * xs + i], g.lo[2], g.ih[2]), g.n[2]);
    if (cz < g.oz0 || cz >= g.oz1) bad = 1;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, ERRF_DOMAIN);
}

__global__ void k_fill_u64_seq(uint64_t* dst, int64_t n, uint64_t start) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = start + (uint64_t)i;
}

__global__ void k_fill_f32(float* dst, int64_t n, float v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = v;
}

inline unsigned grid_for(int64_t n, int bs = 256) {
  int64_t b = (n + bs - 1) / bs;
  if (b > 148 * 64) b = 148 * 64;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace

int launch_field_ingest(const Geom& g, const float* src, int64_t comp_stride, int src_z0, int src_nz,
                        float4* field, cudaStream_t s) {
  const int64_t total = (int64_t)g.wnz * g.gy * g.gx;
  k_field_ingest<<<grid_for(total), 256, 0, s>>>(g, src, comp_stride, src_z0, src_nz, field);
  return 1;
}

int launch_source_readout(const Geom& g, float4* acc, int z0, int z1, float scale, float* out, cudaStream_t s) {
  const int64_t total = (int64_t)g.n[0] * g.n[1] * (z1 - z0);
  if (total <= 0) return 0;
  k_source_readout<<<grid_for(total), 256, 0, s>>>(g, acc, z0, z1, scale, out);
  return 1;
}

int launch_locate(const Geom& g, const float* x, int64_t xs, int64_t n, int32_t* cell, int32_t* chunk,
                  cudaStream_t s) {
  if (n <= 0) return 0;
  k_locate<<<grid_for(n), 256, 0, s>>>(g, x, xs, n, cell, chunk);
  return 1;
}

int launch_keys(const Geom& g, const float* x, int64_t xs, int64_t n, int32_t* key, cudaStream_t s) {
  return launch_locate(g, x, xs, n, nullptr, key, s);
}

int launch_check_domain(const Geom& g, const float* x, int64_t xs, int64_t n, int* err, cudaStream_t s) {
  if (n <= 0) return 0;
  k_check_domain<<<grid_for(n), 256, 0, s>>>(g, x, xs, n, err);
  return 1;
}

int launch_fill_u64_seq(uint64_t* dst, int64_t n, uint64_t start, cudaStream_t s) {
  if (n <= 0) return 0;
  k_fill_u64_seq<<<grid_for(n), 256, 0, s>>>(dst, n, start);
  return 1;
}

// take the device error flags (read and clear in one atomic step) into host-mapped memory
__global__ void k_take_flags(int* err, int* out) { *out = atomicExch(err, 0); }

int launch_take_flags(int* err, int* out, cudaStream_t s) {
  k_take_flags<<<1, 1, 0, s>>>(err, out);
  return 1;
}

int launch_fill_f32(float* dst, int64_t n, float v, cudaStream_t s) {
  if (n <= 0) return 0;
  k_fill_f32<<<grid_for(n), 256, 0, s>>>(dst, n, v);
  return 1;
}

}  // namespace st
