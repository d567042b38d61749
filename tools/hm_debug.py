"""Height-map regions vs a plain-Python restatement of hm_segment's BFS
(heightmap.cpp:44-79) on the baseline stream (tests/golden)."""
import collections
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from paper_2510_01592_b200 import native  # noqa: E402
from paper_2510_01592_b200.frames import read_frames  # noqa: E402
from workloads import GOLDEN  # noqa: E402


def py_bfs(h, v, dth):
    ex, ey = v.shape
    region = -np.ones((ex, ey), np.int64)
    order = []
    for x in range(ex):
        for y in range(ey):
            if not v[x, y] or region[x, y] >= 0:
                continue
            lab = x * ey + y
            q = collections.deque([(x, y)])
            region[x, y] = lab
            while q:
                cx, cy = q.popleft()
                order.append(cx * ey + cy)
                for sx, sy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                    nx, ny = cx + sx, cy + sy
                    if not (0 <= nx < ex and 0 <= ny < ey) or not v[nx, ny] or region[nx, ny] >= 0:
                        continue
                    if abs(h[nx, ny] - h[cx, cy]) >= dth:
                        continue
                    region[nx, ny] = lab
                    q.append((nx, ny))
    return order, region


frames = read_frames(f"{GOLDEN}/baseline_frames.bin")
hm = native.HeightMap(0.01, (140, 140), (0.0, 0.0))
p = native.default_params(seed=77, refine_exact=True)
for i, f in enumerate(frames):
    hm.integrate(f.points, f.rotation, f.translation)
    hm.segment(p)
    h, v = hm.cells()
    visit, root = hm.regions()
    order, region = py_bfs(h, v, p.seg.distance_th)
    ok_root = np.array_equal(np.where(v, root, -1), np.where(v, region, -1))
    # per region member order
    g_by = collections.defaultdict(list)
    for c in visit:
        g_by[int(root.reshape(-1)[c])].append(int(c))
    r_by = collections.defaultdict(list)
    for c in order:
        r_by[int(region.reshape(-1)[c])].append(int(c))
    bad = [k for k in r_by if r_by[k] != g_by.get(k)]
    print(f"frame {i}: valid {v.sum()} visited {len(visit)} py {len(order)} roots equal {ok_root} "
          f"regions {len(r_by)} mismatched {len(bad)}", flush=True)
    if bad:
        k = bad[0]
        a, b = r_by[k], g_by.get(k, [])
        j = next((t for t in range(min(len(a), len(b))) if a[t] != b[t]), None)
        print("  first region", k, "len", len(a), len(b), "first diff at", j, a[j - 2:j + 3] if j else None,
              b[j - 2:j + 3] if j else None)
        missing = sorted(set(a) - set(b))[:3]
        for c in missing:
            x, y = divmod(c, 140)
            print("   cell", c, (x, y), "gpu root", root[x, y], "h", h[x, y])
            for sx, sy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                nx, ny = x + sx, y + sy
                print("     nb", (nx, ny), "valid", v[nx, ny], "h", h[nx, ny], "dh", abs(h[nx, ny] - h[x, y]),
                      "gpu root", root[nx, ny], "py", region[nx, ny])

# every edge of the 4-neighbour graph must join two cells of the same region
h, v = hm.cells()
visit, root = hm.regions()
d = p.seg.distance_th
bad = 0
for x in range(139):
    for y in range(140):
        if v[x, y] and v[x + 1, y] and abs(h[x + 1, y] - h[x, y]) < d and root[x, y] != root[x + 1, y]:
            bad += 1
            if bad <= 3:
                print("x-edge", (x, y), root[x, y], root[x + 1, y])
print("violating x-edges", bad)
for rep in range(3):
    hm.segment(p)
    _, r2 = hm.regions()
    print("rep", rep, "roots identical to previous:", np.array_equal(r2, root))
    root = r2
