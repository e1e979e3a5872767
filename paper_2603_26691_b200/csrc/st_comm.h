// Multi-GPU exchange over NCCL: z-slab ownership of
// chunk planes, field-halo exchange at ingest, halo-source exchange at readout,
// particle migration at rebin (counts by all-gather, payload by grouped send/recv).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "st_internal.h"

namespace st {

struct Comm;

// slab_planes: the nranks+1 chunk-plane boundaries of the slab decomposition (copied),
// NULL = equal split
Comm* comm_create(const void* unique_id, int rank, int nranks, const int32_t* slab_planes, cudaStream_t s,
                  std::string& why);
void comm_destroy(Comm* c);

// Fill the halo planes of the field staging buffer [3][ext_nz][ny][nx] (owned
// planes at ext index z0-ext_z0 ..) from the neighbour slabs.  Returns 0 on success.
int comm_field_halo(Comm* c, float* stage, int64_t comp_stride, int64_t plane, int ext_z0, int ext_nz, int z0,
                    int z1, int nz, int bc_z, cudaStream_t s, std::string& why);

// Send this rank's halo source planes to their owners and add the received ones
// into the owned planes of acc (float4 window [anz][ny][nx]).  Zeroing the
// whole window afterwards is the caller's job.
int comm_source_halo(Comm* c, float4* acc, const Geom& g, int z0, int z1, int H, cudaStream_t s, std::string& why);

// Particle-sharded decomposition (ST_DECOMP_SHARDED): sum the whole-domain source
// accumulator over all ranks in place (one all-reduce).  Returns 0 on success.
int comm_allreduce_sum(Comm* c, float* buf, size_t n, cudaStream_t s, std::string& why);
// Particle-sharded decomposition, the paper's Fig. 1c data flow: the
// Eulerian side stays partitioned (rank r owns cell planes [zb[r], zb[r+1])); every rank
// needs the whole field (its chunks may be anywhere) and every rank's deposits reach
// every owner.  Field: rank r's owned planes are broadcast from r into every rank's
// staging buffer (grouped ncclBroadcast, one per owner and component; stage plane index
// of global plane z is plane0 + z).  Sources: the whole-domain float4 accumulator is
// reduced onto each owner's planes (grouped ncclReduce, root = owner) — a reduce-scatter
// with per-rank sizes; non-owned planes are left as they were.  Returns 0 on success.
int comm_shard_field(Comm* c, float* stage, int64_t comp, int64_t plane, int plane0, const std::vector<int>& zb,
                     cudaStream_t s, std::string& why);
int comm_shard_sources(Comm* c, float4* acc, int64_t plane, const std::vector<int>& zb, cudaStream_t s,
                       std::string& why);
// All-gather one int64 per rank (device buffer of nranks; this rank's slot filled by the
// caller) — the counts of the sharded rebalance.
int comm_allgather_i64(Comm* c, int64_t* buf, cudaStream_t s, std::string& why);
// Sharded rebalance payload: this rank sends send[q] particles starting at store index
// send_off[q] to rank q and receives recv[q] from q at recv_off[q] (SoA x,u,d,w,id of
// capacity cap); one grouped send/recv.
int comm_exchange_store(Comm* c, const Store& A, int64_t cap, const std::vector<int64_t>& send,
                        const std::vector<int64_t>& send_off, const std::vector<int64_t>& recv,
                        const std::vector<int64_t>& recv_off, cudaStream_t s, std::string& why);
// max over ranks of n ints in place (collective agreement on a status)
int comm_allreduce_max_i32(Comm* c, int* buf, size_t n, cudaStream_t s, std::string& why);

// Migration after the local stable sort (store S[*cur] sorted by key[*cur]):
// send each owner segment to its rank, build kept ++ arrivals (ascending source
// rank) in the other buffer, and stable-sort it by chunk (C-16).  row[dst] gets
// this rank's send counts; *n_new the new local count; *launches the kernels.
// Returns 0 ok, 1 NCCL/CUDA error, 3 capacity.
int comm_migrate(Comm* c, const Geom& g, Store* S, int* cur, int32_t** key, int64_t cap, int64_t n,
                 int32_t chunk_lo, int32_t n_local_chunks, int key_bits, SortScratch& sc, int64_t* row,
                 int64_t* n_new, int* launches, cudaStream_t s, std::string& why);

// Fused neighbour-scatter rebin (C-16 without a global sort): all-reduce(max)
// of the "far" flag, then the virtual-plane counts: vcnt_hi (movers into the
// plane above) -> upper neighbour, vcnt_lo -> lower neighbour; rcnt_dn receives
// the lower neighbour's counts for my bottom plane, rcnt_up the upper's for my
// top plane.  Missing neighbours (walls) leave the receive arrays untouched.
// fv_lo / fv_hi (nf ints each, or NULL): far particles per cell of the lower / upper
// neighbour's window, exchanged the same way into rfv_dn / rfv_up.
int comm_rebin_counts(Comm* c, const uint32_t* vcnt_lo, const uint32_t* vcnt_hi, uint32_t* rcnt_dn, uint32_t* rcnt_up,
                      int nvb, int* d_far, bool periodic, cudaStream_t s, std::string& why, const int* fv_lo = nullptr,
                      const int* fv_hi = nullptr, int* rfv_dn = nullptr, int* rfv_up = nullptr, int64_t nf = 0);
// Keys of the far movers: send_lo keys from klo -> down, send_hi from khi -> up; recv_dn
// keys <- down into kdn, recv_up <- up into kup.
int comm_far_keys(Comm* c, const int32_t* klo, int64_t send_lo, const int32_t* khi, int64_t send_hi, int32_t* kdn,
                  int64_t recv_dn, int32_t* kup, int64_t recv_up, bool periodic, cudaStream_t s, std::string& why);
// Payload of the movers: sbuf[1] (send_hi particles) -> up, sbuf[0] (send_lo) ->
// down; rbuf[0] <- down (recv_dn), rbuf[1] <- up (recv_up).  SoA x,u,d,w,id.
int comm_rebin_payload(Comm* c, const Store* sbuf, int64_t scap, int64_t send_lo, int64_t send_hi, const Store* rbuf,
                       int64_t rcap, int64_t recv_dn, int64_t recv_up, bool periodic, cudaStream_t s, std::string& why);

}  // namespace st

extern "C" {
// Exported helper: write a fresh 128-byte ncclUniqueId into out (rank 0 calls it
// and broadcasts the bytes through torch.distributed).
st_status st_nccl_unique_id(void* out);
}
