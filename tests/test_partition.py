"""Count-balanced slab partition (st_plan_partition): the planner's
largest slab count is the minimum over every feasible split (brute force), each slab
keeps the chunk_cells+1 halo planes, uniform counts give the equal split, and the
library's layout follows the chosen boundaries.  CPU only."""
import itertools

import numpy as np
import pytest

from paper_2603_26691_b200 import Config, StError, plan_layout, plan_partition


def _feasible(split, nz, cc):
    return all(min(b * cc, nz) - a * cc >= cc + 1 for a, b in zip(split[:-1], split[1:]))


@pytest.mark.parametrize("seed,G,ncz", [(0, 3, 10), (1, 4, 11), (2, 2, 9), (3, 3, 12)])
def test_minimax_against_brute_force(seed, G, ncz):
    rng = np.random.default_rng(seed)
    cc = 8
    nz = ncz * cc - int(rng.integers(0, 4))          # ragged top plane
    counts = rng.integers(0, 1000, ncz) * (rng.random(ncz) < 0.7)
    cfg = Config(dims=(16, 16, nz), cell_size=(1 / 16,) * 3, chunk_cells=cc, nranks=G)
    split = plan_partition(cfg, counts)
    assert split[0] == 0 and split[-1] == ncz and all(b > a for a, b in zip(split[:-1], split[1:]))
    assert _feasible(split, nz, cc)
    load = max(int(counts[a:b].sum()) for a, b in zip(split[:-1], split[1:]))
    best = None
    for cuts in itertools.combinations(range(1, ncz), G - 1):
        s = (0,) + cuts + (ncz,)
        if _feasible(s, nz, cc):
            m = max(int(counts[a:b].sum()) for a, b in zip(s[:-1], s[1:]))
            best = m if best is None else min(best, m)
    assert load == best


def test_uniform_counts_give_equal_split_and_layout_follows():
    cfg = Config(dims=(32, 32, 288), cell_size=(1 / 32,) * 3, nranks=4)
    assert plan_partition(cfg, np.ones(36)) == (0, 9, 18, 27, 36)
    counts = np.exp(-np.arange(36) / 6.0) * 1e6       # clustered at the bottom
    split = plan_partition(cfg, counts)
    loads = [counts[a:b].sum() for a, b in zip(split[:-1], split[1:])]
    assert max(loads) < 0.35 * counts.sum()           # equal planes would give 0.78
    for r in range(4):
        cfg.rank, cfg.slab_planes = r, split
        lay = plan_layout(cfg)
        assert (lay.kz0, lay.kz1) == (split[r], split[r + 1])


def test_bad_split_rejected():
    cfg = Config(dims=(32, 32, 64), cell_size=(1 / 32,) * 3, nranks=2, slab_planes=(0, 1, 8))
    with pytest.raises(StError):                      # slab 0 has 8 < 9 cell planes
        plan_layout(cfg)
    cfg.slab_planes = (0, 5, 7)                        # does not end at ncz = 8
    with pytest.raises(StError):
        plan_layout(cfg)
