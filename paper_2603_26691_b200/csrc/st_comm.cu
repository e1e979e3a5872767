// KB4/KB5 + NCCL plumbing for the one-box multi-GPU path.
// Rank r owns chunk planes [floor(r*NCz/G), floor((r+1)*NCz/G)) (C-16).  All
// NCCL calls run on one private stream in API-call order, so every rank issues
// them in the same order; the caller's stream is joined with events.
#include <cuda_runtime.h>
#include <nccl.h>
#include <string.h>

#include <string>
#include <vector>

#include "st_comm.h"

namespace st {

struct Comm {
  ncclComm_t nc = nullptr;
  int rank = 0, nranks = 1;
  std::vector<int32_t> planes;  // slab boundaries (chunk planes, nranks+1), empty = equal split
  cudaStream_t ns = nullptr;
  cudaEvent_t e_in = nullptr, e_out = nullptr;
  float4* halo_recv = nullptr;  // 2 * H * plane float4 (source halo receive)
  int64_t halo_cap = 0;
  int64_t* d_counts = nullptr;  // [nranks * nranks]
  int64_t* d_bounds = nullptr;  // [nranks + 1]
  int32_t* d_bases = nullptr;   // [nranks + 1]
  int* d_flag = nullptr;        // agreed error flag of comm_migrate
};

namespace {

__global__ void k_rank_bounds(const int32_t* __restrict__ key, int64_t n, const int32_t* __restrict__ bases, int nb,
                              int64_t* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nb) return;
  const int32_t target = bases[q];
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (key[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  out[q] = lo;
}

// KB5: acc[dst_plane + p] += recv[p] over `planes` planes.
__global__ void k_halo_add(float4* __restrict__ acc, const float4* __restrict__ recv, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = acc[i];
    const float4 b = recv[i];
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    acc[i] = a;
  }
}

// first chunk plane of rank r: the configured slab boundaries, else the equal split
inline int plane_owner_lo(const Comm* c, int r, int ncz) {
  if (!c->planes.empty()) return c->planes[r];
  return (int)(((int64_t)r * ncz) / c->nranks);
}

#define NCCK(call, why)                                                    \
  do {                                                                     \
    ncclResult_t r_ = (call);                                              \
    if (r_ != ncclSuccess) {                                               \
      why = std::string(#call) + ": " + ncclGetErrorString(r_);            \
      return 1;                                                            \
    }                                                                      \
  } while (0)
#define CUCK(call, why)                                                    \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess) {                                               \
      why = std::string(#call) + ": " + cudaGetErrorString(e_);            \
      return 1;                                                            \
    }                                                                      \
  } while (0)

int join_in(Comm* c, cudaStream_t s, std::string& why) {
  CUCK(cudaEventRecord(c->e_in, s), why);
  CUCK(cudaStreamWaitEvent(c->ns, c->e_in, 0), why);
  return 0;
}
int join_out(Comm* c, cudaStream_t s, std::string& why) {
  CUCK(cudaEventRecord(c->e_out, c->ns), why);
  CUCK(cudaStreamWaitEvent(s, c->e_out, 0), why);
  return 0;
}

}  // namespace

Comm* comm_create(const void* unique_id, int rank, int nranks, const int32_t* slab_planes, cudaStream_t s,
                  std::string& why) {
  (void)s;
  Comm* c = new Comm();
  c->rank = rank;
  c->nranks = nranks;
  if (slab_planes) c->planes.assign(slab_planes, slab_planes + nranks + 1);
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&c->nc, nranks, id, rank);
  if (r != ncclSuccess) {
    why = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
    delete c;
    return nullptr;
  }
  if (cudaStreamCreateWithFlags(&c->ns, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->e_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->e_out, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&c->d_counts, sizeof(int64_t) * nranks * nranks) != cudaSuccess ||
      cudaMalloc(&c->d_bounds, sizeof(int64_t) * (nranks + 1)) != cudaSuccess ||
      cudaMalloc(&c->d_bases, sizeof(int32_t) * (nranks + 1)) != cudaSuccess ||
      cudaMalloc(&c->d_flag, sizeof(int)) != cudaSuccess) {
    why = "comm_create: CUDA allocation failed";
    comm_destroy(c);
    return nullptr;
  }
  return c;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->ns) cudaStreamSynchronize(c->ns);
  if (c->nc) ncclCommDestroy(c->nc);
  if (c->ns) cudaStreamDestroy(c->ns);
  if (c->e_in) cudaEventDestroy(c->e_in);
  if (c->e_out) cudaEventDestroy(c->e_out);
  cudaFree(c->halo_recv);
  cudaFree(c->d_counts);
  cudaFree(c->d_bounds);
  cudaFree(c->d_bases);
  cudaFree(c->d_flag);
  delete c;
}

int comm_field_halo(Comm* c, float* stage, int64_t comp, int64_t plane, int ext_z0, int ext_nz, int z0, int z1,
                    int nz, int bc_z, cudaStream_t s, std::string& why) {
  const int G = c->nranks, r = c->rank;
  const bool periodic = bc_z == ST_BC_PERIODIC;
  const int up = (r + 1 < G) ? r + 1 : (periodic ? 0 : -1);
  const int dn = (r > 0) ? r - 1 : (periodic ? G - 1 : -1);
  const int own = z0 - ext_z0;              // = H + 1 planes of halo below
  const int nh = own;                       // planes exchanged per side
  const int slab = z1 - z0;
  (void)ext_nz;
  (void)nz;
  const size_t cnt = (size_t)nh * plane;
  if (join_in(c, s, why)) return 1;
  NCCK(ncclGroupStart(), why);
  for (int k = 0; k < 3; ++k)  // my top nh owned planes -> upper neighbour's lower halo
    if (up >= 0) NCCK(ncclSend(stage + k * comp + (int64_t)(own + slab - nh) * plane, cnt, ncclFloat, up, c->nc, c->ns), why);
  for (int k = 0; k < 3; ++k)  // my bottom nh owned planes -> lower neighbour's upper halo
    if (dn >= 0) NCCK(ncclSend(stage + k * comp + (int64_t)own * plane, cnt, ncclFloat, dn, c->nc, c->ns), why);
  for (int k = 0; k < 3; ++k)
    if (dn >= 0) NCCK(ncclRecv(stage + k * comp, cnt, ncclFloat, dn, c->nc, c->ns), why);
  for (int k = 0; k < 3; ++k)
    if (up >= 0) NCCK(ncclRecv(stage + k * comp + (int64_t)(own + slab) * plane, cnt, ncclFloat, up, c->nc, c->ns), why);
  NCCK(ncclGroupEnd(), why);
  return join_out(c, s, why);
}

int comm_source_halo(Comm* c, float4* acc, const Geom& g, int z0, int z1, int H, cudaStream_t s, std::string& why) {
  const int G = c->nranks, r = c->rank;
  const bool periodic = g.bc[2] == ST_BC_PERIODIC;
  const int up = (r + 1 < G) ? r + 1 : (periodic ? 0 : -1);
  const int dn = (r > 0) ? r - 1 : (periodic ? G - 1 : -1);
  const int64_t plane = (int64_t)g.n[0] * g.n[1];
  const int slab = z1 - z0;
  const int64_t cnt = (int64_t)H * plane;   // float4 per side
  if (c->halo_cap < 2 * cnt) {
    cudaFree(c->halo_recv);
    c->halo_recv = nullptr;
    CUCK(cudaMalloc(&c->halo_recv, sizeof(float4) * 2 * cnt), why);
    c->halo_cap = 2 * cnt;
  }
  float4* from_up = c->halo_recv;         // adds to my top H owned planes
  float4* from_dn = c->halo_recv + cnt;   // adds to my bottom H owned planes
  if (join_in(c, s, why)) return 1;
  NCCK(ncclGroupStart(), why);
  if (dn >= 0) NCCK(ncclSend(acc, (size_t)cnt * 4, ncclFloat, dn, c->nc, c->ns), why);                       // lower halo
  if (up >= 0) NCCK(ncclSend(acc + (int64_t)(H + slab) * plane, (size_t)cnt * 4, ncclFloat, up, c->nc, c->ns), why);  // upper halo
  if (up >= 0) NCCK(ncclRecv(from_up, (size_t)cnt * 4, ncclFloat, up, c->nc, c->ns), why);
  if (dn >= 0) NCCK(ncclRecv(from_dn, (size_t)cnt * 4, ncclFloat, dn, c->nc, c->ns), why);
  NCCK(ncclGroupEnd(), why);
  const unsigned grid = (unsigned)((cnt + 255) / 256 < 148 * 16 ? (cnt + 255) / 256 : 148 * 16);
  if (up >= 0) k_halo_add<<<grid, 256, 0, c->ns>>>(acc + (int64_t)slab * plane, from_up, cnt);
  if (dn >= 0) k_halo_add<<<grid, 256, 0, c->ns>>>(acc + (int64_t)H * plane, from_dn, cnt);
  CUCK(cudaGetLastError(), why);
  return join_out(c, s, why);
}

static bool equal_slabs(const std::vector<int>& zb) {
  for (size_t r = 1; r + 1 < zb.size(); ++r)
    if (zb[r + 1] - zb[r] != zb[1] - zb[0]) return false;
  return true;
}

int comm_shard_field(Comm* c, float* stage, int64_t comp, int64_t plane, int plane0, const std::vector<int>& zb,
                     cudaStream_t s, std::string& why) {
  if (join_in(c, s, why)) return 1;
  if (equal_slabs(zb)) {   // equal partitions: one all-gather per component (NVLS-capable)
    const size_t cnt = (size_t)(zb[1] - zb[0]) * plane;
    NCCK(ncclGroupStart(), why);
    for (int k = 0; k < 3; ++k) {
      float* base = stage + k * comp + (int64_t)plane0 * plane;
      NCCK(ncclAllGather(base + (int64_t)zb[c->rank] * plane, base, cnt, ncclFloat, c->nc, c->ns), why);
    }
    NCCK(ncclGroupEnd(), why);
    return join_out(c, s, why);
  }
  NCCK(ncclGroupStart(), why);
  for (int r = 0; r < c->nranks; ++r) {
    const size_t cnt = (size_t)(zb[r + 1] - zb[r]) * plane;
    if (!cnt) continue;
    for (int k = 0; k < 3; ++k) {
      float* p = stage + k * comp + (int64_t)(plane0 + zb[r]) * plane;
      NCCK(ncclBroadcast(p, p, cnt, ncclFloat, r, c->nc, c->ns), why);
    }
  }
  NCCK(ncclGroupEnd(), why);
  return join_out(c, s, why);
}

int comm_shard_sources(Comm* c, float4* acc, int64_t plane, const std::vector<int>& zb, cudaStream_t s,
                       std::string& why) {
  if (join_in(c, s, why)) return 1;
  if (equal_slabs(zb)) {   // equal partitions: one reduce-scatter, in place (NVLS-capable)
    const size_t cnt = (size_t)(zb[1] - zb[0]) * plane * 4;
    float* base = reinterpret_cast<float*>(acc);
    NCCK(ncclReduceScatter(base, base + (int64_t)zb[c->rank] * plane * 4, cnt, ncclFloat, ncclSum, c->nc, c->ns), why);
    return join_out(c, s, why);
  }
  NCCK(ncclGroupStart(), why);
  for (int r = 0; r < c->nranks; ++r) {
    const size_t cnt = (size_t)(zb[r + 1] - zb[r]) * plane * 4;
    if (!cnt) continue;
    float* p = reinterpret_cast<float*>(acc + (int64_t)zb[r] * plane);
    NCCK(ncclReduce(p, p, cnt, ncclFloat, ncclSum, r, c->nc, c->ns), why);
  }
  NCCK(ncclGroupEnd(), why);
  return join_out(c, s, why);
}

int comm_allgather_i64(Comm* c, int64_t* buf, cudaStream_t s, std::string& why) {
  if (join_in(c, s, why)) return 1;
  NCCK(ncclAllGather(buf + c->rank, buf, 1, ncclInt64, c->nc, c->ns), why);
  return join_out(c, s, why);
}

int comm_exchange_store(Comm* c, const Store& A, int64_t cap, const std::vector<int64_t>& send,
                        const std::vector<int64_t>& send_off, const std::vector<int64_t>& recv,
                        const std::vector<int64_t>& recv_off, cudaStream_t s, std::string& why) {
  if (join_in(c, s, why)) return 1;
  NCCK(ncclGroupStart(), why);
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) continue;
    if (send[q] > 0) {
      const int64_t o = send_off[q], m = send[q];
      for (int a = 0; a < 3; ++a) NCCK(ncclSend(A.x + a * cap + o, m, ncclFloat, q, c->nc, c->ns), why);
      for (int a = 0; a < 3; ++a) NCCK(ncclSend(A.u + a * cap + o, m, ncclFloat, q, c->nc, c->ns), why);
      NCCK(ncclSend(A.d + o, m, ncclFloat, q, c->nc, c->ns), why);
      NCCK(ncclSend(A.w + o, m, ncclFloat, q, c->nc, c->ns), why);
      NCCK(ncclSend(A.id + o, m, ncclUint64, q, c->nc, c->ns), why);
    }
    if (recv[q] > 0) {
      const int64_t o = recv_off[q], m = recv[q];
      for (int a = 0; a < 3; ++a) NCCK(ncclRecv(A.x + a * cap + o, m, ncclFloat, q, c->nc, c->ns), why);
      for (int a = 0; a < 3; ++a) NCCK(ncclRecv(A.u + a * cap + o, m, ncclFloat, q, c->nc, c->ns), why);
      NCCK(ncclRecv(A.d + o, m, ncclFloat, q, c->nc, c->ns), why);
      NCCK(ncclRecv(A.w + o, m, ncclFloat, q, c->nc, c->ns), why);
      NCCK(ncclRecv(A.id + o, m, ncclUint64, q, c->nc, c->ns), why);
    }
  }
  NCCK(ncclGroupEnd(), why);
  return join_out(c, s, why);
}

int comm_allreduce_max_i32(Comm* c, int* buf, size_t n, cudaStream_t s, std::string& why) {
  if (join_in(c, s, why)) return 1;
  NCCK(ncclAllReduce(buf, buf, n, ncclInt32, ncclMax, c->nc, c->ns), why);
  return join_out(c, s, why);
}

int comm_allreduce_sum(Comm* c, float* buf, size_t n, cudaStream_t s, std::string& why) {
  if (join_in(c, s, why)) return 1;
  NCCK(ncclAllReduce(buf, buf, n, ncclFloat, ncclSum, c->nc, c->ns), why);
  return join_out(c, s, why);
}

int comm_migrate(Comm* c, const Geom& g, Store* S, int* cur, int32_t** key, int64_t cap, int64_t n, int32_t chunk_lo,
                 int32_t n_local_chunks, int key_bits, SortScratch& sc, int64_t* row, int64_t* n_new, int* launches,
                 cudaStream_t s, std::string& why) {
  (void)chunk_lo;
  (void)n_local_chunks;
  const int G = c->nranks, r = c->rank;
  const int ncxy = g.NC[0] * g.NC[1];
  std::vector<int32_t> bases(G + 1);
  for (int q = 0; q <= G; ++q) bases[q] = plane_owner_lo(c, q, g.NC[2]) * ncxy;
  CUCK(cudaMemcpyAsync(c->d_bases, bases.data(), sizeof(int32_t) * (G + 1), cudaMemcpyHostToDevice, s), why);
  k_rank_bounds<<<1, 64, 0, s>>>(key[*cur], n, c->d_bases, G + 1, c->d_bounds);
  *launches += 1;
  std::vector<int64_t> b(G + 1), cnt(G), M((size_t)G * G);
  CUCK(cudaMemcpyAsync(b.data(), c->d_bounds, sizeof(int64_t) * (G + 1), cudaMemcpyDeviceToHost, s), why);
  CUCK(cudaStreamSynchronize(s), why);
  b[0] = 0;
  b[G] = n;
  for (int q = 0; q < G; ++q) cnt[q] = b[q + 1] - b[q];
  CUCK(cudaMemcpyAsync(c->d_counts + (size_t)r * G, cnt.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice, s), why);
  if (join_in(c, s, why)) return 1;
  NCCK(ncclAllGather(c->d_counts + (size_t)r * G, c->d_counts, G, ncclInt64, c->nc, c->ns), why);
  CUCK(cudaMemcpyAsync(M.data(), c->d_counts, sizeof(int64_t) * G * G, cudaMemcpyDeviceToHost, c->ns), why);
  CUCK(cudaStreamSynchronize(c->ns), why);
  for (int q = 0; q < G; ++q) row[q] = M[(size_t)r * G + q];
  int64_t total = M[(size_t)r * G + r];
  for (int src = 0; src < G; ++src)
    if (src != r) total += M[(size_t)src * G + r];
  {
    // agree on the capacity check before any payload moves (a rank that returned alone
    // would leave the others waiting in the grouped send/recv)
    int bad = total > cap ? 1 : 0;
    CUCK(cudaMemcpyAsync(c->d_flag, &bad, sizeof(int), cudaMemcpyHostToDevice, c->ns), why);
    NCCK(ncclAllReduce(c->d_flag, c->d_flag, 1, ncclInt32, ncclMax, c->nc, c->ns), why);
    CUCK(cudaMemcpyAsync(&bad, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->ns), why);
    CUCK(cudaStreamSynchronize(c->ns), why);
    if (bad) {
      join_out(c, s, why);
      why = total > cap ? "migration would exceed the store capacity" : "migration would exceed the store capacity on another rank";
      return 3;
    }
  }
  const int o = 1 - *cur;
  Store A = S[*cur], B = S[o];
  // kept segment first (in order)
  const int64_t kept = cnt[r], k0 = b[r];
  if (kept > 0) {
    for (int a = 0; a < 3; ++a) {
      CUCK(cudaMemcpyAsync(B.x + a * cap, A.x + a * cap + k0, kept * sizeof(float), cudaMemcpyDeviceToDevice, c->ns), why);
      CUCK(cudaMemcpyAsync(B.u + a * cap, A.u + a * cap + k0, kept * sizeof(float), cudaMemcpyDeviceToDevice, c->ns), why);
    }
    CUCK(cudaMemcpyAsync(B.d, A.d + k0, kept * sizeof(float), cudaMemcpyDeviceToDevice, c->ns), why);
    CUCK(cudaMemcpyAsync(B.w, A.w + k0, kept * sizeof(float), cudaMemcpyDeviceToDevice, c->ns), why);
    CUCK(cudaMemcpyAsync(B.id, A.id + k0, kept * sizeof(uint64_t), cudaMemcpyDeviceToDevice, c->ns), why);
  }
  NCCK(ncclGroupStart(), why);
  for (int q = 0; q < G; ++q) {
    if (q == r || cnt[q] == 0) continue;
    const int64_t o0 = b[q], m = cnt[q];
    for (int a = 0; a < 3; ++a) NCCK(ncclSend(A.x + a * cap + o0, m, ncclFloat, q, c->nc, c->ns), why);
    for (int a = 0; a < 3; ++a) NCCK(ncclSend(A.u + a * cap + o0, m, ncclFloat, q, c->nc, c->ns), why);
    NCCK(ncclSend(A.d + o0, m, ncclFloat, q, c->nc, c->ns), why);
    NCCK(ncclSend(A.w + o0, m, ncclFloat, q, c->nc, c->ns), why);
    NCCK(ncclSend(A.id + o0, m, ncclUint64, q, c->nc, c->ns), why);
  }
  int64_t pos = kept;
  for (int src = 0; src < G; ++src) {
    const int64_t m = M[(size_t)src * G + r];
    if (src == r || m == 0) continue;
    for (int a = 0; a < 3; ++a) NCCK(ncclRecv(B.x + a * cap + pos, m, ncclFloat, src, c->nc, c->ns), why);
    for (int a = 0; a < 3; ++a) NCCK(ncclRecv(B.u + a * cap + pos, m, ncclFloat, src, c->nc, c->ns), why);
    NCCK(ncclRecv(B.d + pos, m, ncclFloat, src, c->nc, c->ns), why);
    NCCK(ncclRecv(B.w + pos, m, ncclFloat, src, c->nc, c->ns), why);
    NCCK(ncclRecv(B.id + pos, m, ncclUint64, src, c->nc, c->ns), why);
    pos += m;
  }
  NCCK(ncclGroupEnd(), why);
  if (join_out(c, s, why)) return 1;
  // kept ++ arrivals now sit in the other buffer; the caller stable-sorts it by
  // bin key (C-16), which refines the chunk order each segment already has
  (void)key_bits;
  (void)sc;
  (void)key;
  *cur = o;
  *n_new = total;
  CUCK(cudaGetLastError(), why);
  return 0;
}

namespace {
void neighbours(const Comm* c, bool periodic, int& up, int& dn) {
  const int G = c->nranks, r = c->rank;
  up = (r + 1 < G) ? r + 1 : (periodic ? 0 : -1);
  dn = (r > 0) ? r - 1 : (periodic ? G - 1 : -1);
}

int send_store(Comm* c, const Store& b, int64_t cap, int64_t n, int peer, std::string& why) {
  for (int a = 0; a < 3; ++a) NCCK(ncclSend(b.x + a * cap, n, ncclFloat, peer, c->nc, c->ns), why);
  for (int a = 0; a < 3; ++a) NCCK(ncclSend(b.u + a * cap, n, ncclFloat, peer, c->nc, c->ns), why);
  NCCK(ncclSend(b.d, n, ncclFloat, peer, c->nc, c->ns), why);
  NCCK(ncclSend(b.w, n, ncclFloat, peer, c->nc, c->ns), why);
  NCCK(ncclSend(b.id, n, ncclUint64, peer, c->nc, c->ns), why);
  return 0;
}

int recv_store(Comm* c, const Store& b, int64_t cap, int64_t n, int peer, std::string& why) {
  for (int a = 0; a < 3; ++a) NCCK(ncclRecv(b.x + a * cap, n, ncclFloat, peer, c->nc, c->ns), why);
  for (int a = 0; a < 3; ++a) NCCK(ncclRecv(b.u + a * cap, n, ncclFloat, peer, c->nc, c->ns), why);
  NCCK(ncclRecv(b.d, n, ncclFloat, peer, c->nc, c->ns), why);
  NCCK(ncclRecv(b.w, n, ncclFloat, peer, c->nc, c->ns), why);
  NCCK(ncclRecv(b.id, n, ncclUint64, peer, c->nc, c->ns), why);
  return 0;
}
}  // namespace

int comm_rebin_counts(Comm* c, const uint32_t* vcnt_lo, const uint32_t* vcnt_hi, uint32_t* rcnt_dn, uint32_t* rcnt_up,
                      int nvb, int* d_far, bool periodic, cudaStream_t s, std::string& why, const int* fv_lo,
                      const int* fv_hi, int* rfv_dn, int* rfv_up, int64_t nf) {
  int up, dn;
  neighbours(c, periodic, up, dn);
  if (join_in(c, s, why)) return 1;
  NCCK(ncclAllReduce(d_far, d_far, 1, ncclInt32, ncclMax, c->nc, c->ns), why);
  NCCK(ncclGroupStart(), why);
  if (up >= 0) NCCK(ncclSend(vcnt_hi, nvb, ncclUint32, up, c->nc, c->ns), why);
  if (dn >= 0) NCCK(ncclSend(vcnt_lo, nvb, ncclUint32, dn, c->nc, c->ns), why);
  if (dn >= 0) NCCK(ncclRecv(rcnt_dn, nvb, ncclUint32, dn, c->nc, c->ns), why);
  if (up >= 0) NCCK(ncclRecv(rcnt_up, nvb, ncclUint32, up, c->nc, c->ns), why);
  if (nf > 0) {
    if (up >= 0) NCCK(ncclSend(fv_hi, nf, ncclInt32, up, c->nc, c->ns), why);
    if (dn >= 0) NCCK(ncclSend(fv_lo, nf, ncclInt32, dn, c->nc, c->ns), why);
    if (dn >= 0) NCCK(ncclRecv(rfv_dn, nf, ncclInt32, dn, c->nc, c->ns), why);
    if (up >= 0) NCCK(ncclRecv(rfv_up, nf, ncclInt32, up, c->nc, c->ns), why);
  }
  NCCK(ncclGroupEnd(), why);
  return join_out(c, s, why);
}

int comm_far_keys(Comm* c, const int32_t* klo, int64_t send_lo, const int32_t* khi, int64_t send_hi, int32_t* kdn,
                  int64_t recv_dn, int32_t* kup, int64_t recv_up, bool periodic, cudaStream_t s, std::string& why) {
  int up, dn;
  neighbours(c, periodic, up, dn);
  if (join_in(c, s, why)) return 1;
  NCCK(ncclGroupStart(), why);
  if (up >= 0 && send_hi > 0) NCCK(ncclSend(khi, send_hi, ncclInt32, up, c->nc, c->ns), why);
  if (dn >= 0 && send_lo > 0) NCCK(ncclSend(klo, send_lo, ncclInt32, dn, c->nc, c->ns), why);
  if (dn >= 0 && recv_dn > 0) NCCK(ncclRecv(kdn, recv_dn, ncclInt32, dn, c->nc, c->ns), why);
  if (up >= 0 && recv_up > 0) NCCK(ncclRecv(kup, recv_up, ncclInt32, up, c->nc, c->ns), why);
  NCCK(ncclGroupEnd(), why);
  return join_out(c, s, why);
}

int comm_rebin_payload(Comm* c, const Store* sbuf, int64_t scap, int64_t send_lo, int64_t send_hi, const Store* rbuf,
                       int64_t rcap, int64_t recv_dn, int64_t recv_up, bool periodic, cudaStream_t s, std::string& why) {
  int up, dn;
  neighbours(c, periodic, up, dn);
  if (join_in(c, s, why)) return 1;
  NCCK(ncclGroupStart(), why);
  if (up >= 0 && send_hi > 0 && send_store(c, sbuf[1], scap, send_hi, up, why)) return 1;
  if (dn >= 0 && send_lo > 0 && send_store(c, sbuf[0], scap, send_lo, dn, why)) return 1;
  if (dn >= 0 && recv_dn > 0 && recv_store(c, rbuf[0], rcap, recv_dn, dn, why)) return 1;
  if (up >= 0 && recv_up > 0 && recv_store(c, rbuf[1], rcap, recv_up, up, why)) return 1;
  NCCK(ncclGroupEnd(), why);
  return join_out(c, s, why);
}

}  // namespace st

extern "C" st_status st_nccl_unique_id(void* out) {
  if (!out) return ST_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return ST_ERR_NCCL;
  memcpy(out, &id, sizeof(id));
  return ST_OK;
}
