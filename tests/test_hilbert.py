"""the 3-D Hilbert index and the count-balanced Hilbert partition of the
chunks (st_hilbert_index / st_plan_hilbert, host functions of the library; no GPU).

Pins: a bijection onto [0, 8^order) whose consecutive
indices are face-adjacent cells (exhaustive at order <= 4 — a wrong rotation table or
bit interleave breaks adjacency); the planner's ranges are contiguous along that curve,
non-empty, and their largest count equals the brute-force optimum over every contiguous
split on small inputs; and the locality property the paper uses the curve for: chunks
of a Hilbert range touch fewer Eulerian slabs than a random assignment."""
import itertools

import numpy as np
import pytest

from paper_2603_26691_b200 import Config, hilbert_index, plan_hilbert


@pytest.mark.parametrize("order", [1, 2, 3, 4])
def test_hilbert_bijective_and_face_adjacent(order):
    n = 1 << order
    cells = np.array(list(itertools.product(range(n), repeat=3)), np.int32)
    h = hilbert_index(order, cells)
    assert sorted(h.tolist()) == list(range(n ** 3))
    path = cells[np.argsort(h)]
    steps = np.abs(np.diff(path.astype(np.int64), axis=0)).sum(axis=1)
    assert np.all(steps == 1)
    assert h[0] == 0                      # starts at the origin cell


def test_hilbert_rejects_out_of_range():
    from paper_2603_26691_b200 import StError
    with pytest.raises(StError):
        hilbert_index(2, [[4, 0, 0]])
    with pytest.raises(StError):
        hilbert_index(2, [[0, -1, 0]])


def _chunk_hilbert_order(cfg):
    nc = [(d + cfg.chunk_cells - 1) // cfg.chunk_cells for d in cfg.dims]
    order = 1
    while (1 << order) < max(nc):
        order += 1
    ids = np.arange(nc[0] * nc[1] * nc[2])
    xyz = np.stack([ids % nc[0], (ids // nc[0]) % nc[1], ids // (nc[0] * nc[1])], 1)
    return ids[np.argsort(hilbert_index(order, xyz))], nc


def _brute_best(w, G):
    """Smallest largest-segment sum over all splits of w into G contiguous non-empty parts."""
    n = len(w)
    best = None
    for cuts in itertools.combinations(range(1, n), G - 1):
        b = [0, *cuts, n]
        m = max(sum(w[b[i]:b[i + 1]]) for i in range(G))
        best = m if best is None else min(best, m)
    return best


@pytest.mark.parametrize("G,seed", [(2, 0), (3, 1), (4, 2), (5, 3)])
def test_plan_hilbert_contiguous_balanced_optimal(G, seed):
    cfg = Config(dims=(16, 16, 24), chunk_cells=8, nranks=G)      # 2 x 2 x 3 = 12 chunks
    order, nc = _chunk_hilbert_order(cfg)
    rng = np.random.default_rng(seed)
    counts = rng.integers(0, 1000, order.size) * (rng.random(order.size) < 0.8)
    owner = plan_hilbert(cfg, counts)
    seq = owner[order]
    assert np.all(np.diff(seq) >= 0) and seq[0] == 0 and seq[-1] == G - 1     # contiguous ranges
    assert set(seq.tolist()) == set(range(G))                                # none empty
    loads = [int(counts[owner == r].sum()) for r in range(G)]
    assert max(loads) == _brute_best([int(counts[c]) for c in order], G)


def test_plan_hilbert_locality_vs_random():
    """S:257 locality oracle: with 4 Eulerian z-slabs and 16 chunk ranges, a range from the
    Hilbert split needs fewer slabs (its chunks' planes) than a random equal-size set."""
    cfg = Config(dims=(64, 64, 64), chunk_cells=8, nranks=16)      # 512 chunks
    counts = np.ones(512, np.int64)
    owner = plan_hilbert(cfg, counts)
    kz = np.arange(512) // 64
    slab = kz // 2                                                    # 4 slabs of 2 chunk planes
    hil = np.mean([len(set(slab[owner == r].tolist())) for r in range(16)])
    rng = np.random.default_rng(0)
    rnd = np.mean([np.mean([len(set(slab[p].tolist())) for p in np.array_split(rng.permutation(512), 16)])
                   for _ in range(20)])
    assert hil < rnd, (hil, rnd)
    assert np.bincount(owner, minlength=16).tolist() == [32] * 16
