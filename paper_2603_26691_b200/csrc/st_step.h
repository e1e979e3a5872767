// Binned particle step (k_step.cu): layout, arguments and launchers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "st_internal.h"

namespace st {

constexpr int kMaxBins = 32;          // bins per warp item
constexpr int kItemParticles = 1024;  // soft particle budget per warp item

struct BinGeom {
  int cc3;     // cells per chunk (bins per chunk)
  int nbins;   // local bins = local chunks * cc3
  int nkz;     // local chunk planes
  int kz0;     // first local chunk plane
  int sh;      // log2(chunk_cells) if a power of two, else -1
  // multi-GPU: the cell plane just below / above the slab belongs to the
  // neighbour rank; its cells are "virtual bins" v = ((ky*NCx+kx)*cc+ly)*cc+lx
  // (the receiver's bin order within one plane), nvb per side
  int nvb;
  int vz[2];   // global z of the lower / upper virtual plane, -1 if none (wall or 1 rank)
};

struct StepArgs {
  Geom g;
  Phys p;
  BinGeom bg;
  Store A, B;                 // input layout / output layout (scatter)
  CUtensorMap tm_f;           // TMA tensor map of A's float rows (2-D {cap, 8}; k_pstep)
  CUtensorMap tm_id;          // TMA tensor map of A's ids (2-D {cap, 1}; k_pstep)
  CUtensorMap tm_f64;         // TMA tensor map of A's float rows, box {68, 8} (k_ip / k_fs: 64-particle batches)
  CUtensorMap tm_id66;        // TMA tensor map of A's ids, box {66, 1} (k_fs)
  CUtensorMap tm_win[2];      // TMA maps of the front fluid field, window boxes of k_pstep:
                              // [0] 10x3x3 cells (in place), [1] 12x5x5 cells (fused scatter)
  int64_t cap, n;
  const int64_t* off;         // [nbins+1] CSR of A
  const int64_t* off_new;     // [nbins+1] CSR of B (scatter)
  const int* slot_base;       // [27][nbins] base[j][s] (scatter; rebin_prep output; k_step)
  const long long* dtab;      // [nbins][27] destination table (scatter; k_dbase output; k_pstep)
  unsigned long long* far_cur;// [nbins] next free slot of each bin's far tail (C-15b), or NULL
  int32_t* far_src;           // [cap] by new-layout slot: the tail sort key (hi, lo) of a far
  int32_t* far_src_hi;        // particle: (0, old-layout index) for this rank's own, (1 + order of
                              // the source rank, sender's index) for arrivals (k_far_order_w, C-15b)
  // multi-GPU far particles whose cell lies in a neighbour rank's slab (C-15b across ranks):
  // the scatter appends them to the far region of sbuf[side] (after the near movers),
  // fs_cur[side] = next free slot, fs_key[side][slot] = prior index (the receiver sorts by it)
  unsigned long long* fs_cur; // [2] or NULL: such a particle is an error (general path taken)
  int32_t* fs_key[2];
  int32_t* fs_cell[2];        // [scap] per side: the global cell it was counted for (its bin there)
  // ... and the in-place counting step counts them per cell of the neighbour's first
  // chunk_cells planes: cnt_fv[side][(p * ny + y) * nx + x], p = planes beyond the slab
  int* cnt_fv[2];             // or NULL: such a particle sets *cnt_far (general path)
  unsigned long long* cnt_fs_n;   // [2] totals per side
  // slot histogram produced by an in-place step whose call makes a rebin due (k_count's
  // outputs, same meaning; cnt_hist == NULL: not produced by this launch)
  int* cnt_hist;
  int* cnt_far;
  int* cnt_far_cnt;
  unsigned long long* cnt_movers;
  unsigned long long* cnt_far_n;
  const int* item_bin0;       // warp items of A
  const int* n_items;
  int* item_ctr;              // or NULL: items handed out dynamically (k_ip / k_fs; zeroed per launch)
  int nbins;
  const float4* field;
  float4* acc;
  float dt;
  int nsteps;
  int* err;                   // hard errors (ERRF_*)
  // multi-GPU scatter: movers into the neighbour planes go to send buffers
  const int64_t* voff[2];     // [nvb+1] offsets of the virtual bins in sbuf[side]
  Store sbuf[2];
  int64_t scap;               // capacity (particles) of each send buffer
};

// Multi-GPU rebin helpers (k_step.cu)
int launch_vcombine(const Geom& g, const BinGeom& bg, uint32_t* new_cnt, const uint32_t* rcnt_dn,
                    const uint32_t* rcnt_up, uint32_t* kept_dn, uint32_t* kept_up, int oz0, int oz1,
                    const int* far_cnt, cudaStream_t s);
// C-15b: sort every bin's far tail of the new layout B by the old-layout index (far_src)
int launch_far_order(const BinGeom& bg, const int* far_cnt, const int64_t* off_new, const int32_t* far_src,
                     const int32_t* far_src_hi, Store B, Store A, int64_t cap, int* long_list, int* long_n,
                     cudaStream_t s);
struct InsertArgs {
  Geom g;
  BinGeom bg;
  Store rbuf;                 // arrivals of one side (SoA, capacity rcap)
  int64_t rcap, count;
  const int64_t* roff;        // [nvb+1]
  const uint32_t* kept;       // [nvb] local count of the destination bin before arrivals
  int plane;                  // owned plane the arrivals land in (z0 or z1-1)
  Store B;
  int64_t cap;
  const int64_t* off_new;
  int nbins;
  int* err;
};
int launch_insert(const InsertArgs& a, cudaStream_t s);

int launch_step(const StepArgs& a, bool scatter, bool advance, cudaStream_t s);
// movers != NULL: add the particles arriving from another chunk (statistics; the counts
// came from the in-place step, which no longer counts them itself)
int launch_rebin_prep(const Geom& g, const BinGeom& bg, int* cnt_base, uint32_t* new_cnt, const int* far_cnt,
                      unsigned long long* movers, cudaStream_t s);
// Slot histogram of the current layout (k_count): input of the next neighbour-slot rebin
struct CountArgs {
  Geom g;
  BinGeom bg;
  const float* x;             // [3][cap] positions of the current layout
  int64_t cap;
  const int64_t* off;         // [nbins+1] CSR of the current layout
  const int* item_bin0;
  const int* n_items;
  int nbins;
  int* hist;                  // [27][nbins] out: hist[j][s] (every entry written)
  int* far;                   // set to 1 if a far particle cannot be placed by the fused rebin
  int* far_cnt;               // [nbins] far particles per destination bin (C-15b), or NULL:
                              // any particle more than one cell from its bin sets *far
  unsigned long long* movers; // += particles whose current chunk differs from their bin's chunk
  unsigned long long* far_n;  // += far particles placed in bin tails
};
// far particles across ranks (see StepArgs::fs_cur): the receiver adds the exchanged
// per-cell counts to its bins (new_cnt and far_cnt) and totals them per side
int launch_far_accept(const Geom& g, const BinGeom& bg, const int* rfv0, const int* rfv1, int z0, int z1,
                      uint32_t* new_cnt, int* far_cnt, unsigned long long* fr_n, int* err, cudaStream_t s);
// ... and puts the far arrivals of one side into the far tails of B
struct FarInsertArgs {
  Geom g;
  BinGeom bg;
  Store r;                    // far arrivals of this side (stride rcap), any order
  int64_t rcap, count;
  const int32_t* key;         // their sender store indices
  const int32_t* cell;        // the global cells they were counted for
  int32_t hi;                 // 1 + order of the source rank among this rank's sources (C-16)
  unsigned long long* far_cur;
  int32_t* far_src;
  int32_t* far_src_hi;
  Store B;
  int64_t cap;
  int* err;
};
int launch_far_insert(const FarInsertArgs& a, cudaStream_t s);
int launch_count(const CountArgs& a, cudaStream_t s);
// destination table [nbins][27] of k_pstep from the prep bases and the new offsets
int launch_dbase(const Geom& g, const BinGeom& bg, const int* base, const int64_t* off_new, const int64_t* voff0,
                 const int64_t* voff1, long long* dtab, const int* far_cnt, unsigned long long* far_cur,
                 cudaStream_t s);
int launch_items(const int64_t* off, int nbins, int cc, uint32_t* flag, int64_t* pos, int64_t* partial,
                 int* item_bin0, int* n_items, cudaStream_t s);
int launch_bin_offsets(const int32_t* key_sorted, int64_t n, int nbins, int64_t* off, cudaStream_t s);
int launch_bin_keys(const Geom& g, const BinGeom& bg, const float* x, int64_t xs, int64_t n, int32_t* key, int* err,
                    cudaStream_t s);

}  // namespace st
