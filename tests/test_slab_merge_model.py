"""CPU tier: the distributed CCL design of paper_2510_01592_b200.slabs /
csrc/k_slab.cu, restated in numpy, against whole-graph union-find.

Random steppable sets on a small window with a random symmetric edge
predicate restricted to the (2w+1)^3 window (what build_adjacency,
segmentation.cpp:112-130, can produce) are split into x-slabs (including
slabs thinner than w). Each slab labels its extended list locally, emits the
boundary triples, the replicated zone union-find merges them, and the owners
assemble their clusters from the exported members. The result must be the
canonical labelling (component-minimum ordinal, segmentation.cpp:147-194) and
the single-grid cluster member lists (ascending ordinal)."""
import numpy as np
import pytest

from paper_2510_01592_b200.slabs import SlabLayout, split_x


def uf_labels(n, edges):
    parent = list(range(n))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for a, b in edges:
        ra, rb = find(a), find(b)
        if ra != rb:
            lo, hi = min(ra, rb), max(ra, rb)
            parent[hi] = lo
    return np.array([find(i) for i in range(n)], np.int64)


def random_case(rng, ex, ey, ez, density, w, p_edge):
    occ = rng.random((ex, ey, ez)) < density
    idx = np.argwhere(occ)  # lexicographic = ordinal order
    n = len(idx)
    salt = int(rng.integers(1 << 30))

    def edge(i, j):  # symmetric pseudo-random predicate
        a, b = (i, j) if i < j else (j, i)
        h = (a * 1000003 + b * 7919 + salt) * 2654435761 % (1 << 32)
        return h / (1 << 32) < p_edge

    pos = {tuple(v): k for k, v in enumerate(idx)}
    edges = []
    for i, (x, y, z) in enumerate(idx):
        for X in range(x, min(ex, x + w + 1)):
            for Y in range(max(0, y - w), min(ey, y + w + 1)):
                for Z in range(max(0, z - w), min(ez, z + w + 1)):
                    j = pos.get((X, Y, Z))
                    if j is not None and j > i and edge(i, j):
                        edges.append((i, j))
    return idx, edges


def distributed_labels(idx, edges, ranges, w, ex):
    """Mirror of vp_slab_extend/label/merge/export/segment_owned."""
    counts = np.bincount(idx[:, 0], minlength=ex)
    lay = SlabLayout(ranges, counts, w)
    P = lay.P
    edge_set = set(edges)
    # zone (k_slab.cu: [B - w, B + w) around internal boundaries, merged)
    zone = []
    for a, _ in lay.ranges[1:]:
        lo, hi = max(0, a - w), min(ex, a + w)
        if zone and lo <= zone[-1][1]:
            zone[-1][1] = max(zone[-1][1], hi)
        else:
            zone.append([lo, hi])
    dbase, zsize = [], 0
    for lo, hi in zone:
        dbase.append(zsize)
        zsize += int(P[hi] - P[lo])

    def zidx(o):
        x = idx[o, 0]
        for (lo, hi), d in zip(zone, dbase):
            if lo <= x < hi:
                return d + int(o - P[lo])
        return -1

    triples, local = [], []
    for k in range(lay.n):
        lo, hi = lay.ext(k)
        base = int(P[lo])
        n_ext = lay.n_ext(k)
        ext_edges = [(a - base, b - base) for (a, b) in edge_set
                     if base <= a < base + n_ext and base <= b < base + n_ext]
        lab = uf_labels(n_ext, ext_edges)  # local index of the local min
        bmin = {}
        for i in range(n_ext):
            if zidx(base + i) >= 0:
                bmin[lab[i]] = min(bmin.get(lab[i], i), i)
        for i in range(n_ext):
            if zidx(base + i) >= 0:
                triples.append((zidx(base + i), zidx(base + bmin[lab[i]]), base + lab[i]))
        local.append((base, lab, bmin))
    # replicated merge
    zl = uf_labels(zsize, [(a, b) for a, b, _ in triples])
    minlab = {}
    for a, b, L in triples:
        r = zl[b]
        minlab[r] = min(minlab.get(r, L), L)
    labels = np.zeros(len(idx), np.int64)
    for k, (base, lab, bmin) in enumerate(local):
        a, b = lay.ranges[k]
        nl = lay.n_left(k)
        for j in range(lay.n_own(k)):
            r = lab[nl + j]
            if r in bmin:
                labels[int(P[a]) + j] = minlab[zl[zidx(base + bmin[r])]]
            else:
                labels[int(P[a]) + j] = base + r
    # cluster gather: owner = slab holding the label; members own ++ received (slab order)
    owner_of = lambda L: max(k for k in range(lay.n) if P[lay.ranges[k][0]] <= L)  # noqa: E731
    clusters = {}
    for k in range(lay.n):
        a, _ = lay.ranges[k]
        mine = [(int(P[a]) + j) for j in range(lay.n_own(k))]
        recv = [o for s in range(k + 1, lay.n) for o in range(int(P[lay.ranges[s][0]]),
                                                               int(P[lay.ranges[s][1]]))
                if owner_of(labels[o]) == k and labels[o] < P[lay.ranges[s][0]]]
        for o in mine + recv:
            if owner_of(labels[o]) == k:
                clusters.setdefault(int(labels[o]), []).append(o)
    return labels, clusters


CASES = [
    dict(ex=12, ey=5, ez=4, density=0.5, w=1, p_edge=0.6),
    dict(ex=20, ey=4, ez=4, density=0.45, w=2, p_edge=0.5),
    dict(ex=16, ey=3, ez=3, density=0.7, w=3, p_edge=0.3),
]


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("nslab", [1, 2, 3, 5])
def test_merge_equals_whole_graph(case, nslab):
    c = CASES[case]
    rng = np.random.default_rng(100 * case + nslab)
    for trial in range(3):
        idx, edges = random_case(rng, c["ex"], c["ey"], c["ez"], c["density"], c["w"], c["p_edge"])
        ref = uf_labels(len(idx), edges)
        if nslab == 5:  # ragged, some slabs thinner than w
            cuts = sorted(rng.choice(np.arange(1, c["ex"]), 4, replace=False).tolist())
            ranges = list(zip([0] + cuts, cuts + [c["ex"]]))
        else:
            ranges = split_x(c["ex"], nslab)
        labels, clusters = distributed_labels(idx, edges, ranges, c["w"], c["ex"])
        assert np.array_equal(labels, ref)
        ref_clusters = {}
        for o, L in enumerate(ref):
            ref_clusters.setdefault(int(L), []).append(o)
        assert clusters == ref_clusters


def test_layout_transfers_cover_extended_lists():
    rng = np.random.default_rng(7)
    ex = 30
    counts = rng.integers(0, 5, ex)
    for ranges in (split_x(ex, 4), [(0, 1), (1, 2), (2, 29), (29, 30)], [(0, 30)]):
        lay = SlabLayout(ranges, counts, 3)
        filled = [np.zeros(lay.n_ext(k), int) for k in range(lay.n)]
        for k in range(lay.n):
            nl, no = lay.n_left(k), lay.n_own(k)
            filled[k][nl:nl + no] += 1
        for s, d, s0, cnt, d0 in lay.transfers():
            assert 0 <= s0 and s0 + cnt <= lay.n_own(s)
            filled[d][d0:d0 + cnt] += 1
            # the same global ordinals on both sides
            assert lay.P[lay.ranges[s][0]] + s0 == lay.P[lay.ext(d)[0]] + d0
        assert all((f == 1).all() for f in filled)
