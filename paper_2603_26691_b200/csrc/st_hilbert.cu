// Hilbert space-filling curve and the count-balanced Hilbert partition of the chunks
// ("an initialization procedure using a Hilbert
// space-filling curve ... to place the particles into chunks compactly"
// balancing; SPEC S:245-262 hilbert_index / initialize_chunks).  Host code (the
// planning is O(chunks)); exported through include/scaletrack.h.
//
// hilbert3: Skilling's transpose algorithm ("Programming the Hilbert curve", AIP Conf.
// Proc. 707, 2004): Gray-decode the axes from the top bit down, undoing the excess work
// of each level's rotation/reflection, then interleave the bits (x is the most
// significant axis of each 3-bit digit).  Consecutive indices are face-adjacent cells
// (tests/test_hilbert.py checks bijectivity and adjacency against brute force).
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "scaletrack.h"

namespace {

uint64_t hilbert3(uint32_t x, uint32_t y, uint32_t z, int order) {
  uint32_t X[3] = {x, y, z};
  const uint32_t M = 1u << (order - 1);
  // inverse undo excess work
  for (uint32_t Q = M; Q > 1; Q >>= 1) {
    const uint32_t P = Q - 1;
    for (int i = 0; i < 3; ++i) {
      if (X[i] & Q) {
        X[0] ^= P;                       // invert
      } else {
        const uint32_t t = (X[0] ^ X[i]) & P;   // exchange
        X[0] ^= t;
        X[i] ^= t;
      }
    }
  }
  // Gray encode
  for (int i = 1; i < 3; ++i) X[i] ^= X[i - 1];
  uint32_t t = 0;
  for (uint32_t Q = M; Q > 1; Q >>= 1)
    if (X[2] & Q) t ^= Q - 1;
  for (int i = 0; i < 3; ++i) X[i] ^= t;
  // interleave the transposed bits: digit b = (X0_b, X1_b, X2_b)
  uint64_t h = 0;
  for (int b = order - 1; b >= 0; --b)
    for (int i = 0; i < 3; ++i) h = (h << 1) | ((X[i] >> b) & 1u);
  return h;
}

}  // namespace

extern "C" {

st_status st_hilbert_index(int32_t order, int64_t n, const int32_t* xyz, uint64_t* out) {
  if (order < 1 || order > 21 || n < 0 || (n > 0 && (!xyz || !out))) return ST_ERR_INVALID_ARG;
  const int64_t side = (int64_t)1 << order;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    if (x < 0 || y < 0 || z < 0 || x >= side || y >= side || z >= side) return ST_ERR_INVALID_ARG;
    out[i] = hilbert3((uint32_t)x, (uint32_t)y, (uint32_t)z, order);
  }
  return ST_OK;
}

st_status st_plan_hilbert(const st_config* cfg, const int64_t* chunk_counts, int32_t* owner) {
  if (!cfg || !chunk_counts || !owner || cfg->chunk_cells < 1 || cfg->nranks < 1) return ST_ERR_INVALID_ARG;
  int nc[3], ncmax = 1;
  for (int a = 0; a < 3; ++a) {
    if (cfg->dims[a] < 1) return ST_ERR_INVALID_ARG;
    nc[a] = (cfg->dims[a] + cfg->chunk_cells - 1) / cfg->chunk_cells;
    ncmax = std::max(ncmax, nc[a]);
  }
  int order = 1;                       // chunk coordinates on a 2^order cube
  while ((1 << order) < ncmax) ++order;
  const int64_t n = (int64_t)nc[0] * nc[1] * nc[2];
  const int G = cfg->nranks;
  if (G > n) return ST_ERR_INVALID_ARG;
  // chunks in Hilbert order of their chunk coordinates (ties impossible: bijective)
  std::vector<std::pair<uint64_t, int64_t>> key((size_t)n);
  for (int64_t c = 0; c < n; ++c) {
    const int kx = (int)(c % nc[0]), ky = (int)((c / nc[0]) % nc[1]), kz = (int)(c / ((int64_t)nc[0] * nc[1]));
    key[(size_t)c] = {hilbert3((uint32_t)kx, (uint32_t)ky, (uint32_t)kz, order), c};
  }
  std::sort(key.begin(), key.end());
  std::vector<int64_t> w((size_t)n);
  int64_t tot = 0, wmax = 0;
  for (int64_t i = 0; i < n; ++i) {
    w[(size_t)i] = std::max<int64_t>(0, chunk_counts[key[(size_t)i].second]);
    tot += w[(size_t)i];
    wmax = std::max(wmax, w[(size_t)i]);
  }
  // minimal largest segment count over contiguous splits into <= G non-empty segments:
  // binary search on the bound with the greedy feasibility test (linear partition)
  auto segments = [&](int64_t bound) {
    int s = 1;
    int64_t acc = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (acc + w[(size_t)i] > bound) {
        ++s;
        acc = 0;
      }
      acc += w[(size_t)i];
    }
    return s;
  };
  int64_t lo = wmax, hi = std::max<int64_t>(tot, 1);
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (segments(mid) <= G) hi = mid;
    else lo = mid + 1;
  }
  // greedy fill under the optimal bound; a rank advances early only when every later
  // rank would otherwise be left without a chunk (then the remaining chunks go one each)
  int r = 0;
  int64_t acc = 0;
  for (int64_t i = 0; i < n; ++i) {
    const bool must = (int64_t)(G - 1 - r) >= n - i;
    if (i > 0 && r < G - 1 && (acc + w[(size_t)i] > lo || must)) {
      ++r;
      acc = 0;
    }
    owner[key[(size_t)i].second] = r;
    acc += w[(size_t)i];
  }
  return ST_OK;
}

}  // extern "C"
