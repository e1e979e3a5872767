// Internal declarations of the B200 SCALE-TRACK library (not part of the ABI).
// The ABI is include/scaletrack.h; the physics readings are DESIGN.md §3.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "scaletrack.h"

namespace st {

// ----------------------------------------------------------------------------
// Geometry and physics constants passed to kernels by value.
// ----------------------------------------------------------------------------
struct Geom {
  float lo[3], hi[3], L[3], ih[3];  // fp32 contract values (C-6, C-12)
  int n[3];                         // global cells per axis
  int bc[3];                        // ST_BC_*
  int cc;                           // chunk edge in cells
  int NC[3];                        // chunks per axis
  // field window: float4 [wnz][n1+2][n0+2]; window plane iz <-> global plane wz0+iz
  int gx, gy;                       // n0+2, n1+2
  int wz0, wnz;
  // source accumulator window: float4 [anz][n1][n0]; plane ia <-> global plane az0+ia
  int az0, anz;
  int wrapz;                        // 1: periodic z with a partial window (nranks > 1)
  int chunk_base;                   // first global chunk id owned by this rank
  int oz0, oz1;                     // owned cell planes [oz0, oz1)
};

struct Phys {
  float inv_nu;      // 1/nu_f
  float tau_c;       // rho_p / (18 rho_f nu_f):  tau_p = tau_c d^2   (C-3)
  float mass_c;      // (pi/6) rho_p:              m_p = mass_c d^3  (C-18)
  float g[3];        // body acceleration (C-1)
  int drag_law, integrator, two_way;
};

// Structure-of-arrays particle store (one of two ping-pong buffers).
struct Store {
  float* x = nullptr;   // [3][cap]
  float* u = nullptr;   // [3][cap]
  float* d = nullptr;   // [cap]
  float* w = nullptr;   // [cap]
  uint64_t* id = nullptr;
  void* base = nullptr;
};

// Device error flags (bit mask) written by kernels.
enum : int { ERRF_CFL = 1, ERRF_DOMAIN = 2, ERRF_WINDOW = 4, ERRF_SCATTER = 8 };

// Per-tile description for the advance kernel: particles [begin, end) all binned
// to local chunk `chunk` (or -1: unbinned, read the field from global memory).
struct Tile {
  int64_t begin, end;
  int32_t chunk;   // global chunk id or -1
  int32_t pad;
};

// ----------------------------------------------------------------------------
// Kernel launchers (k_*.cu).  All enqueue on the given stream and return the
// number of kernels launched.
// ----------------------------------------------------------------------------
int launch_field_ingest(const Geom& g, const float* src, int64_t plane_stride_src, int src_z0,
                        int src_nz, float4* field, cudaStream_t s);
int launch_advance(const Geom& g, const Phys& p, const float4* field, float4* acc, Store st,
                   int64_t cap, int64_t n, const Tile* tiles, int ntiles, float dt, int nsteps,
                   int32_t* key_out, int* err, cudaStream_t s);
int launch_locate(const Geom& g, const float* x, int64_t xstride, int64_t n, int32_t* cell,
                  int32_t* chunk, cudaStream_t s);
int launch_check_domain(const Geom& g, const float* x, int64_t xstride, int64_t n, int* err,
                        cudaStream_t s);
int launch_source_readout(const Geom& g, float4* acc, int z0, int z1, float scale, float* out,
                          cudaStream_t s);
int launch_fill_u64_seq(uint64_t* dst, int64_t n, uint64_t start, cudaStream_t s);
int launch_fill_f32(float* dst, int64_t n, float v, cudaStream_t s);
int launch_take_flags(int* err, int* out, cudaStream_t s);
int launch_keys(const Geom& g, const float* x, int64_t xstride, int64_t n, int32_t* key,
                cudaStream_t s);

// Stable counting sort of the store by key (LSD radix, 8-bit digits).  Moves the
// payload src -> dst (ping-pong) each pass; returns the buffer holding the result
// (0 = src, 1 = dst) through *result_in_dst.
struct SortScratch {
  uint32_t* hist = nullptr;   // [256 * max_blocks]
  int64_t* offs = nullptr;    // [256 * max_blocks + 1]
  int64_t* partial = nullptr; // scan partials
  int64_t max_blocks = 0;
  int64_t partial_cap = 0;
};
int launch_stable_sort(Store a, Store b, int64_t cap, int64_t n, int32_t* key_a, int32_t* key_b,
                       int key_bits, SortScratch& sc, int* result_in_b, cudaStream_t s);
int launch_exclusive_scan_u32(const uint32_t* in, int64_t m, int64_t* out, int64_t* partial,
                              cudaStream_t s);
int launch_chunk_offsets(const int32_t* key_sorted, int64_t n, int32_t key_lo, int32_t nkeys,
                         int64_t* offsets, cudaStream_t s);
int launch_build_tiles(const int64_t* offsets, int32_t key_lo, int32_t nkeys, int64_t tile_size,
                       Tile* tiles, int32_t* ntiles, int max_tiles, cudaStream_t s);

}  // namespace st
