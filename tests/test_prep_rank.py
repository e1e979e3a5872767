"""Host-side check of the rank rule k_rebin_prep uses for 8^3 chunks:
the bin order of a destination's 27 neighbour sources is lexicographic in
(kz, ky, kx, lz, ly, lx), so each source's rank among the 27 follows from per-axis
counts.  Brute force: the rule must order the valid sources exactly as sorting their
bin keys does, on random geometries (periodic / walls, ragged chunks)."""
import random


def _bin_key(c, NC):
    k = [ci >> 3 for ci in c]
    l = [ci & 7 for ci in c]
    return ((k[2] * NC[1] + k[1]) * NC[0] + k[0]) * 512 + (l[2] * 8 + l[1]) * 8 + l[0]


def _positions(d, n, periodic):
    lt = [[0] * 3 for _ in range(3)]
    eq = [[1] * 3 for _ in range(3)]
    wl = [[0] * 3 for _ in range(3)]
    coords = [[0] * 3 for _ in range(3)]
    for a in range(3):
        k, l = [0] * 3, [0] * 3
        for i in range(3):
            sc = d[a] + 1 - i                       # option i = source coordinate c + 1 - i
            if periodic[a]:
                sc = sc + n[a] if sc < 0 else (sc - n[a] if sc >= n[a] else sc)
            coords[a][i] = sc
            k[i], l[i] = sc >> 3, sc & 7
        for i in range(3):
            for o in range(3):
                if o != i:
                    lt[a][i] += k[o] < k[i]
                    eq[a][i] += k[o] == k[i]
                    wl[a][i] += k[o] == k[i] and l[o] < l[i]
    pos, src = {}, {}
    for j in range(27):
        jx, jy, jz = j % 3, (j // 3) % 3, j // 9
        pos[j] = (lt[2][jz] * 9 + eq[2][jz] * (lt[1][jy] * 3 + eq[1][jy] * lt[0][jx])
                  + wl[2][jz] * eq[1][jy] * eq[0][jx] + wl[1][jy] * eq[0][jx] + wl[0][jx])
        src[j] = (coords[0][jx], coords[1][jy], coords[2][jz])
    return pos, src


def test_prep_rank_rule_matches_key_sort():
    rng = random.Random(7)
    for _ in range(5000):
        n = [rng.choice([3, 4, 5, 8, 9, 16, 17, 24]) for _ in range(3)]
        periodic = [rng.random() < 0.5 for _ in range(3)]
        NC = [(v + 7) // 8 for v in n]
        d = [rng.randrange(v) for v in n]
        pos, src = _positions(d, n, periodic)
        assert sorted(pos.values()) == list(range(27))
        valid = [j for j in range(27) if all(0 <= src[j][a] < n[a] for a in range(3))]
        by_key = sorted(valid, key=lambda j: _bin_key(src[j], NC))
        by_pos = sorted(valid, key=lambda j: pos[j])
        assert by_key == by_pos, (n, periodic, d)
