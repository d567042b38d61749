/* voxplane_oracle.c — CPU ORACLE, TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference hot path
 * (/root/reference/proj/core/src) used as the checker for the B200 library.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it. It is pinned against the compiled reference (oracle/_ref, built
 * from the unmodified sources by oracle/Makefile) stage by stage, and through
 * it against the golden files in proj/test_scratch (tests/test_oracle.py).
 *
 * Arithmetic contract (shared with the shim and the CUDA kernels): no FMA
 * contraction (-ffp-contract=off); 3-term dot products (a0b0 + a1b1) + a2b2;
 * 3x3 * vec3 rows 0,1 as (r0 v0 + r1 v1) + r2 v2 and row 2 as
 * r0 v0 + (r1 v1 + r2 v2) (Eigen 3.4 SSE2 coefficient-based product).
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "voxplane_b200.h"
#include "voxplane_trace.h"

/* ---------------------------------------------------------------- vectors */
typedef struct { double v[3]; } V3;
typedef struct { int32_t v[3]; } V3i;
typedef struct { double m[3][3]; } M3; /* m[row][col] */
typedef struct { double x, y; } V2;

static V3 v3(double a, double b, double c) { V3 r = {{a, b, c}}; return r; }
static V3 vadd(V3 a, V3 b) { return v3(a.v[0] + b.v[0], a.v[1] + b.v[1], a.v[2] + b.v[2]); }
static V3 vsub(V3 a, V3 b) { return v3(a.v[0] - b.v[0], a.v[1] - b.v[1], a.v[2] - b.v[2]); }
static V3 vscale(double s, V3 a) { return v3(s * a.v[0], s * a.v[1], s * a.v[2]); }
static V3 vdiv(V3 a, double s) { return v3(a.v[0] / s, a.v[1] / s, a.v[2] / s); }
static V3 vneg(V3 a) { return v3(-a.v[0], -a.v[1], -a.v[2]); }
static double dot3(V3 a, V3 b) { return (a.v[0] * b.v[0] + a.v[1] * b.v[1]) + a.v[2] * b.v[2]; }
static double sqnorm3(V3 a) { return dot3(a, a); }
static V3 normalized3(V3 a) { /* Eigen normalized(): guarded by > 0 */
  const double z = sqnorm3(a);
  return z > 0.0 ? vdiv(a, sqrt(z)) : a;
}
static V3 cross3(V3 a, V3 b) {
  return v3(a.v[1] * b.v[2] - a.v[2] * b.v[1], a.v[2] * b.v[0] - a.v[0] * b.v[2],
            a.v[0] * b.v[1] - a.v[1] * b.v[0]);
}
static V3 matvec(const M3* r, V3 p) {
  return v3((r->m[0][0] * p.v[0] + r->m[0][1] * p.v[1]) + r->m[0][2] * p.v[2],
            (r->m[1][0] * p.v[0] + r->m[1][1] * p.v[1]) + r->m[1][2] * p.v[2],
            r->m[2][0] * p.v[0] + (r->m[2][1] * p.v[1] + r->m[2][2] * p.v[2]));
}
static int finite3(V3 p) { return isfinite(p.v[0]) && isfinite(p.v[1]) && isfinite(p.v[2]); }

/* types.hpp:43-52 */
static V3 orient_up(V3 n, V3 up) {
  const double d = dot3(n, up);
  if (d < 0.0) return vneg(n);
  if (d > 0.0) return n;
  for (int k = 0; k < 3; ++k) {
    if (n.v[k] > 0.0) return n;
    if (n.v[k] < 0.0) return vneg(n);
  }
  return n;
}

/* voxel_grid.cpp:13-17 (r^T r via the same product order as the shim) */
static int is_valid_rotation(const M3* r) {
  const double tol = 1e-6;
  M3 t, p;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t.m[i][j] = r->m[j][i];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i)
      p.m[i][j] = i < 2 ? (t.m[i][0] * r->m[0][j] + t.m[i][1] * r->m[1][j]) + t.m[i][2] * r->m[2][j]
                        : t.m[i][0] * r->m[0][j] + (t.m[i][1] * r->m[1][j] + t.m[i][2] * r->m[2][j]);
  double mx = 0.0;
  int first = 1;
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) {
      double v = p.m[i][j] - (i == j ? 1.0 : 0.0);
      v = v < 0.0 ? -v : v;
      if (first || mx < v) mx = v;
      first = 0;
    }
  if (mx > tol) return 0;
  const double(*m)[3] = r->m;
#define H(a, b, c) (m[0][a] * (m[1][b] * m[2][c] - m[1][c] * m[2][b]))
  const double det = H(0, 1, 2) - H(1, 0, 2) + H(2, 0, 1);
#undef H
  return fabs(det - 1.0) <= tol;
}

/* ------------------------------------------------------------------- grid */
typedef struct {
  double sx, sy, sz;
  uint32_t count;
  uint8_t status;
} Cell; /* voxel_grid.hpp:19-23 */

typedef struct {
  double res;
  int32_t ext[3];
  double origin[3];
  Cell* cells;
  size_t ncells;
  size_t occupied;
  uint8_t* mask; /* clear_rays scratch (voxel_grid.hpp:90) */
} Grid;

static size_t gflat(const Grid* g, const int32_t* i) {
  return ((size_t)i[0] * (size_t)g->ext[1] + (size_t)i[1]) * (size_t)g->ext[2] + (size_t)i[2];
}
static int in_bounds(const Grid* g, const int32_t* i) {
  return i[0] >= 0 && i[1] >= 0 && i[2] >= 0 && i[0] < g->ext[0] && i[1] < g->ext[1] &&
         i[2] < g->ext[2];
}
/* voxel_grid.cpp:31-35 */
static V3i world_to_index(const Grid* g, V3 p) {
  V3i r;
  for (int k = 0; k < 3; ++k) r.v[k] = (int32_t)floor((p.v[k] - g->origin[k]) / g->res);
  return r;
}
/* voxel_grid.cpp:19-25 */
static int grid_init(Grid* g, double res, const int32_t* ext, const double* c) {
  if (!(res > 0.0) || ext[0] <= 0 || ext[1] <= 0 || ext[2] <= 0) return VP_EINVAL;
  g->res = res;
  for (int k = 0; k < 3; ++k) {
    g->ext[k] = ext[k];
    g->origin[k] = c[k] - (double)ext[k] * (0.5 * res);
  }
  g->ncells = (size_t)ext[0] * ext[1] * ext[2];
  g->cells = (Cell*)calloc(g->ncells, sizeof(Cell));
  g->mask = (uint8_t*)calloc(g->ncells, 1);
  g->occupied = 0;
  return g->cells && g->mask ? VP_OK : VP_ENOMEM;
}

static M3 pose_rot(const double* R) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = R[3 * i + j];
  return r;
}

/* SensorFrame point -> world: pose.apply(pf.cast<double>()) (types.hpp:31) */
static V3 to_world(const M3* r, const double* t, const float* pf) {
  V3 q = matvec(r, v3((double)pf[0], (double)pf[1], (double)pf[2]));
  return v3(q.v[0] + t[0], q.v[1] + t[1], q.v[2] + t[2]);
}

typedef struct {
  int64_t key;
  uint32_t idx;
} KeyIdx;
static int cmp_keyidx(const void* a, const void* b) {
  const KeyIdx* x = (const KeyIdx*)a;
  const KeyIdx* y = (const KeyIdx*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* voxel_grid.cpp:59-115 */
static int integrate_frame(Grid* g, const float* xyz, uint64_t n, const double* R, const double* t,
                           vp_update_stats* st) {
  M3 r = pose_rot(R);
  st->voxels_touched = st->points_discarded = 0;
  if (!is_valid_rotation(&r)) return VP_EINVAL;
  if (n == 0) return VP_OK;
  V3* world = (V3*)malloc(sizeof(V3) * n);
  KeyIdx* keys = (KeyIdx*)malloc(sizeof(KeyIdx) * n);
  for (uint64_t i = 0; i < n; ++i) {
    const V3 p = to_world(&r, t, xyz + 3 * i);
    world[i] = p;
    int64_t key = -1;
    if (finite3(p)) {
      V3i idx = world_to_index(g, p);
      if (in_bounds(g, idx.v)) key = (int64_t)gflat(g, idx.v);
    }
    keys[i].key = key;
    keys[i].idx = (uint32_t)i;
  }
  qsort(keys, n, sizeof(KeyIdx), cmp_keyidx);
  uint64_t first = 0;
  while (first < n && keys[first].key == -1) ++first;
  st->points_discarded = first;
  for (uint64_t i = first; i < n;) {
    uint64_t j = i + 1;
    while (j < n && keys[j].key == keys[i].key) ++j;
    Cell* c = &g->cells[keys[i].key];
    if (c->count == 0) g->occupied++;
    for (uint64_t k = i; k < j; ++k) {
      const V3 p = world[keys[k].idx];
      c->sx += p.v[0];
      c->sy += p.v[1];
      c->sz += p.v[2];
      c->count++;
    }
    c->status = 1; /* Occupied */
    st->voxels_touched++;
    i = j;
  }
  free(world);
  free(keys);
  return VP_OK;
}

/* voxel_grid.cpp:122-178 */
static void walk_segment(Grid* g, V3 a, V3 b) {
  const double res = g->res;
  const V3 d = vsub(b, a);
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = g->origin[k];
    hi[k] = lo[k] + (double)g->ext[k] * res;
  }
  double t0 = 0.0, t1 = 1.0;
  for (int k = 0; k < 3; ++k) {
    if (d.v[k] == 0.0) {
      if (a.v[k] < lo[k] || a.v[k] >= hi[k]) return;
      continue;
    }
    double ta = (lo[k] - a.v[k]) / d.v[k];
    double tb = (hi[k] - a.v[k]) / d.v[k];
    if (ta > tb) {
      const double s = ta;
      ta = tb;
      tb = s;
    }
    t0 = t0 > ta ? t0 : ta; /* std::max(t0, ta) */
    t1 = tb < t1 ? tb : t1; /* std::min(t1, tb) */
    if (t0 > t1) return;
  }
  const V3i oc = world_to_index(g, a);
  const V3i ec = world_to_index(g, b);
  const V3 entry = vadd(a, vscale(t0, d));
  V3i cell = world_to_index(g, entry);
  for (int k = 0; k < 3; ++k) {
    if (cell.v[k] < 0) cell.v[k] = 0;
    if (cell.v[k] > g->ext[k] - 1) cell.v[k] = g->ext[k] - 1;
  }
  int step[3] = {0, 0, 0};
  double tmax[3] = {INFINITY, INFINITY, INFINITY}, tdelta[3] = {INFINITY, INFINITY, INFINITY};
  for (int k = 0; k < 3; ++k) {
    if (d.v[k] > 0.0) {
      step[k] = 1;
      tmax[k] = t0 + (lo[k] + (double)(cell.v[k] + 1) * res - entry.v[k]) / d.v[k];
      tdelta[k] = res / d.v[k];
    } else if (d.v[k] < 0.0) {
      step[k] = -1;
      tmax[k] = t0 + (lo[k] + (double)cell.v[k] * res - entry.v[k]) / d.v[k];
      tdelta[k] = res / -d.v[k];
    }
  }
  const int max_steps = g->ext[0] + g->ext[1] + g->ext[2] + 4;
  for (int i = 0; i < max_steps; ++i) {
    const int is_o = cell.v[0] == oc.v[0] && cell.v[1] == oc.v[1] && cell.v[2] == oc.v[2];
    const int is_e = cell.v[0] == ec.v[0] && cell.v[1] == ec.v[1] && cell.v[2] == ec.v[2];
    if (!is_o && !is_e) g->mask[gflat(g, cell.v)] = 1;
    int m = 0;
    if (tmax[1] < tmax[m]) m = 1;
    if (tmax[2] < tmax[m]) m = 2;
    if (tmax[m] >= t1) break;
    cell.v[m] += step[m];
    if (cell.v[m] < 0 || cell.v[m] >= g->ext[m]) break;
    tmax[m] += tdelta[m];
  }
}

/* voxel_grid.cpp:182-215 */
static int clear_rays(Grid* g, const float* xyz, uint64_t n, const double* R, const double* t,
                      vp_clear_stats* st) {
  M3 r = pose_rot(R);
  st->voxels_cleared = st->voxels_freed = 0;
  if (!is_valid_rotation(&r)) return VP_EINVAL;
  if (n == 0) return VP_OK;
  memset(g->mask, 0, g->ncells);
  const V3 sensor = v3(t[0], t[1], t[2]);
  for (uint64_t i = 0; i < n; ++i) {
    const V3 p = to_world(&r, t, xyz + 3 * i);
    if (!finite3(p)) continue;
    walk_segment(g, sensor, p);
  }
  for (size_t f = 0; f < g->ncells; ++f) {
    if (!g->mask[f]) continue;
    st->voxels_cleared++;
    if (g->cells[f].count > 0) st->voxels_freed++;
    memset(&g->cells[f], 0, sizeof(Cell));
  }
  g->occupied -= st->voxels_freed;
  return VP_OK;
}

/* voxel_grid.cpp:217-252 */
static void recenter(Grid* g, const double* c, vp_shift_stats* st) {
  memset(st, 0, sizeof(*st));
  double wc[3];
  for (int k = 0; k < 3; ++k) wc[k] = g->origin[k] + (double)g->ext[k] * (0.5 * g->res);
  for (int k = 0; k < 3; ++k) st->shift[k] = (int32_t)llround((c[k] - wc[k]) / g->res);
  if (st->shift[0] == 0 && st->shift[1] == 0 && st->shift[2] == 0) return;
  for (int k = 0; k < 3; ++k) g->origin[k] += (double)st->shift[k] * g->res;
  const int32_t* e = g->ext;
  const int32_t* s = st->shift;
  int x0 = s[0] >= 0 ? 0 : e[0] - 1, xs = s[0] >= 0 ? 1 : -1;
  int y0 = s[1] >= 0 ? 0 : e[1] - 1, ys = s[1] >= 0 ? 1 : -1;
  int z0 = s[2] >= 0 ? 0 : e[2] - 1, zs = s[2] >= 0 ? 1 : -1;
  size_t after = 0;
  for (int xi = 0, x = x0; xi < e[0]; ++xi, x += xs)
    for (int yi = 0, y = y0; yi < e[1]; ++yi, y += ys)
      for (int zi = 0, z = z0; zi < e[2]; ++zi, z += zs) {
        const int32_t dst[3] = {x, y, z};
        const int32_t src[3] = {x + s[0], y + s[1], z + s[2]};
        Cell* out = &g->cells[gflat(g, dst)];
        if (in_bounds(g, src))
          *out = g->cells[gflat(g, src)];
        else
          memset(out, 0, sizeof(Cell));
        if (out->count > 0) ++after;
      }
  st->voxels_dropped = g->occupied - after;
  g->occupied = after;
}

/* ----------------------------------------------------------------- Jacobi */
/* jacobi.cpp:13-38 */
static void jrotate(double a[3][3], double v[3][3], int p, int q) {
  const double apq = a[p][q];
  if (apq == 0.0) return;
  const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
  const double t = copysign(1.0, theta) / (fabs(theta) + sqrt(theta * theta + 1.0));
  const double c = 1.0 / sqrt(t * t + 1.0);
  const double s = t * c;
  const double app = a[p][p], aqq = a[q][q];
  a[p][p] = app - t * apq;
  a[q][q] = aqq + t * apq;
  a[p][q] = 0.0;
  a[q][p] = 0.0;
  const int r = 3 - p - q;
  const double arp = a[r][p], arq = a[r][q];
  a[r][p] = a[p][r] = c * arp - s * arq;
  a[r][q] = a[q][r] = s * arp + c * arq;
  for (int i = 0; i < 3; ++i) {
    const double vip = v[i][p], viq = v[i][q];
    v[i][p] = c * vip - s * viq;
    v[i][q] = s * vip + c * viq;
  }
}
static double off_diag(double a[3][3]) {
  return sqrt(2.0 * (a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2]));
}
/* jacobi.cpp:46-81: eigenvalues ascending, vec[k] = eigenvector column k */
static void jacobi3(const double in[3][3], double val[3], V3 vec[3]) {
  double a[3][3] = {{in[0][0], 0.5 * (in[0][1] + in[1][0]), 0.5 * (in[0][2] + in[2][0])},
                    {0.0, in[1][1], 0.5 * (in[1][2] + in[2][1])},
                    {0.0, 0.0, in[2][2]}};
  a[1][0] = a[0][1];
  a[2][0] = a[0][2];
  a[2][1] = a[1][2];
  double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 30 && off_diag(a) >= 1e-10; ++sweep) {
    jrotate(a, v, 0, 1);
    jrotate(a, v, 0, 2);
    jrotate(a, v, 1, 2);
  }
  double ev[3] = {a[0][0], a[1][1], a[2][2]};
  int order[3] = {0, 1, 2};
  for (int i = 0; i < 2; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (ev[order[j]] < ev[order[i]]) {
        const int s = order[i];
        order[i] = order[j];
        order[j] = s;
      }
  for (int k = 0; k < 3; ++k) {
    val[k] = ev[order[k]];
    vec[k] = v3(v[0][order[k]], v[1][order[k]], v[2][order[k]]);
  }
  double m[3][3];
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) m[i][k] = vec[k].v[i];
#define H(a_, b_, c_) (m[0][a_] * (m[1][b_] * m[2][c_] - m[1][c_] * m[2][b_]))
  const double det = H(0, 1, 2) - H(1, 0, 2) + H(2, 0, 1);
#undef H
  if (det < 0.0) vec[2] = vneg(vec[2]);
}

/* ------------------------------------------------------------ segmentation */
typedef struct {
  int32_t idx[3];
  V3 mean;
  uint32_t count;
  uint8_t status;
} Occ;

/* voxel_grid.cpp:254-263 */
static Occ* occupied_voxels(const Grid* g, size_t* n_out) {
  Occ* out = (Occ*)malloc(sizeof(Occ) * (g->occupied ? g->occupied : 1));
  size_t n = 0;
  const size_t ey = (size_t)g->ext[1], ez = (size_t)g->ext[2];
  for (size_t f = 0; f < g->ncells; ++f) {
    const Cell* c = &g->cells[f];
    if (c->count == 0) continue;
    Occ* o = &out[n++];
    o->idx[0] = (int32_t)(f / (ez * ey));
    o->idx[1] = (int32_t)((f / ez) % ey);
    o->idx[2] = (int32_t)(f % ez);
    o->mean = vdiv(v3(c->sx, c->sy, c->sz), (double)c->count); /* cell_mean */
    o->count = c->count;
    o->status = c->status;
  }
  *n_out = n;
  return out;
}

typedef struct {
  V3 normal;
  int32_t ncount;
  uint8_t valid;
  double angle;
} Est;

/* segmentation.cpp:19-67 */
static Est* estimate_normals(const Grid* g, const Occ* occ, size_t n, const vp_seg_params* p) {
  Est* est = (Est*)calloc(n ? n : 1, sizeof(Est));
  const int r = p->neighbor_radius;
  const V3 up = v3(p->up[0], p->up[1], p->up[2]);
  for (size_t i = 0; i < n; ++i) {
    V3 sum = v3(0, 0, 0);
    double sq[3][3] = {{0}};
    int cnt = 0;
    int32_t idx[3];
    for (int dx = -r; dx <= r; ++dx) {
      idx[0] = occ[i].idx[0] + dx;
      for (int dy = -r; dy <= r; ++dy) {
        idx[1] = occ[i].idx[1] + dy;
        for (int dz = -r; dz <= r; ++dz) {
          idx[2] = occ[i].idx[2] + dz;
          if (!in_bounds(g, idx)) continue;
          const Cell* c = &g->cells[gflat(g, idx)];
          if (c->count == 0) continue;
          const V3 m = vdiv(v3(c->sx, c->sy, c->sz), (double)c->count);
          sum = vadd(sum, m);
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) sq[a][b] = sq[a][b] + m.v[b] * m.v[a];
          ++cnt;
        }
      }
    }
    est[i].ncount = cnt;
    if (cnt < 3) continue;
    const V3 mean = vdiv(sum, (double)cnt);
    double cov[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) cov[a][b] = sq[a][b] / (double)cnt - mean.v[b] * mean.v[a];
    double val[3];
    V3 vec[3];
    jacobi3(cov, val, vec);
    if (val[1] <= 1e-12 + 1e-9 * fabs(val[2])) continue;
    est[i].normal = orient_up(normalized3(vec[0]), up);
    double d = dot3(est[i].normal, up);
    d = d < 0.0 ? 0.0 : (d > 1.0 ? 1.0 : d);
    est[i].angle = acos(d) * 57.295779513082320876798;
    est[i].valid = 1;
  }
  return est;
}

typedef struct {
  int32_t idx[3];
  V3 mean, normal;
} Step;

/* segmentation.cpp:69-85 */
static Step* classify_steppable(Grid* g, const Occ* occ, const Est* est, size_t n,
                                const vp_seg_params* p, size_t* ns) {
  Step* out = (Step*)malloc(sizeof(Step) * (n ? n : 1));
  size_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    const int ok = est[i].valid && est[i].ncount >= p->min_neighbors &&
                   est[i].angle <= p->max_angle_deg;
    if (ok) {
      memcpy(out[k].idx, occ[i].idx, sizeof out[k].idx);
      out[k].mean = occ[i].mean;
      out[k].normal = est[i].normal;
      ++k;
    }
    g->cells[gflat(g, occ[i].idx)].status = ok ? 2 : 1;
  }
  *ns = k;
  return out;
}

/* segmentation.cpp:87-132 + 147-194: adjacency over the steppable bounding
 * box, then min-label propagation until a full pass is quiet. The single
 * thread visits chunks in order, so this is the reference's loop with one
 * worker; the fixed point (component minimum) is order independent. */
static int32_t* label_components(const Step* s, size_t n, const vp_seg_params* p, double res) {
  int32_t* labels = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
  for (size_t i = 0; i < n; ++i) labels[i] = (int32_t)i;
  if (n == 0) return labels;
  int w = (int)ceil(p->distance_th / res);
  if (w < 1) w = 1;
  const double d2 = p->distance_th * p->distance_th;
  const double cth = cos(p->adjacency_angle_deg * 0.017453292519943295769237);
  int32_t lo[3], hi[3];
  for (int k = 0; k < 3; ++k) lo[k] = hi[k] = s[0].idx[k];
  for (size_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      if (s[i].idx[k] < lo[k]) lo[k] = s[i].idx[k];
      if (s[i].idx[k] > hi[k]) hi[k] = s[i].idx[k];
    }
  const size_t dims[3] = {(size_t)(hi[0] - lo[0] + 1), (size_t)(hi[1] - lo[1] + 1),
                          (size_t)(hi[2] - lo[2] + 1)};
  const size_t vol = dims[0] * dims[1] * dims[2];
  int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * vol);
  for (size_t f = 0; f < vol; ++f) ord[f] = -1;
#define SLOT(x, y, z) ((((size_t)((x)-lo[0])) * dims[1] + (size_t)((y)-lo[1])) * dims[2] + (size_t)((z)-lo[2]))
  for (size_t i = 0; i < n; ++i) ord[SLOT(s[i].idx[0], s[i].idx[1], s[i].idx[2])] = (int32_t)i;
  /* adjacency as CSR, lists ascending (scan order) */
  size_t cap = 1024, ne = 0;
  int32_t* cols = (int32_t*)malloc(sizeof(int32_t) * cap);
  size_t* rows = (size_t*)malloc(sizeof(size_t) * (n + 1));
  for (size_t i = 0; i < n; ++i) {
    rows[i] = ne;
    int32_t wl[3], wh[3];
    for (int k = 0; k < 3; ++k) {
      wl[k] = s[i].idx[k] - w < lo[k] ? lo[k] : s[i].idx[k] - w;
      wh[k] = s[i].idx[k] + w > hi[k] ? hi[k] : s[i].idx[k] + w;
    }
    for (int x = wl[0]; x <= wh[0]; ++x)
      for (int y = wl[1]; y <= wh[1]; ++y)
        for (int z = wl[2]; z <= wh[2]; ++z) {
          const int32_t j = ord[SLOT(x, y, z)];
          if (j < 0 || j == (int32_t)i) continue;
          if (sqnorm3(vsub(s[i].mean, s[j].mean)) >= d2) continue;
          if (dot3(s[i].normal, s[j].normal) <= cth) continue;
          if (ne == cap) {
            cap *= 2;
            cols = (int32_t*)realloc(cols, sizeof(int32_t) * cap);
          }
          cols[ne++] = j;
        }
  }
  rows[n] = ne;
#undef SLOT
  free(ord);
  int changed = 1;
  while (changed) {
    changed = 0;
    for (size_t i = 0; i < n; ++i)
      for (size_t e = rows[i]; e < rows[i + 1]; ++e) {
        const int32_t j = cols[e];
        const int32_t li = labels[i], lj = labels[j];
        if (li > lj) {
          labels[i] = lj;
          changed = 1;
        } else if (lj > li) {
          labels[j] = li;
          changed = 1;
        }
      }
  }
  free(cols);
  free(rows);
  return labels;
}

/* ------------------------------------------------------------------ RANSAC */
/* rng.hpp:13-64 */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
typedef struct { uint64_t s; } Rng;
static Rng rng_make(uint64_t seed, uint64_t k1, uint64_t k2) {
  Rng r;
  r.s = mix64(seed + 0x9e3779b97f4a7c15ULL);
  r.s = mix64(r.s ^ mix64(k1 + 0xbf58476d1ce4e5b9ULL));
  r.s = mix64(r.s ^ mix64(k2 + 0x94d049bb133111ebULL));
  return r;
}
static uint64_t rng_next(Rng* r) {
  r->s += 0x9e3779b97f4a7c15ULL;
  return mix64(r->s);
}
static uint32_t rng_below(Rng* r, uint32_t n) {
  return (uint32_t)(((unsigned __int128)rng_next(r) * n) >> 64);
}

typedef struct {
  V3 normal;
  double offset;
  int inliers;
} Cand;

/* plane_fit.cpp:21-43 */
static Cand sample_candidate(const V3* pts, uint32_t n, int32_t label, int it,
                             const vp_ransac_params* p) {
  Rng rng = rng_make(p->seed, (uint64_t)(uint32_t)label, (uint64_t)it);
  const uint32_t a = rng_below(&rng, n);
  uint32_t b = rng_below(&rng, n);
  while (b == a) b = rng_below(&rng, n);
  uint32_t c = rng_below(&rng, n);
  while (c == a || c == b) c = rng_below(&rng, n);
  const V3 p0 = pts[a];
  const V3 cr = cross3(vsub(pts[b], p0), vsub(pts[c], p0));
  const double norm = sqrt(sqnorm3(cr));
  Cand cand;
  cand.normal = v3(0, 0, 0);
  cand.offset = 0.0;
  cand.inliers = -1;
  if (0.5 * norm <= 1e-10) return cand;
  cand.normal = orient_up(vdiv(cr, norm), v3(p->up[0], p->up[1], p->up[2]));
  cand.offset = dot3(cand.normal, p0);
  cand.inliers = 0;
  return cand;
}

typedef struct {
  vp_plane model;
  size_t n_in;
  V3* inliers;
} Fit;

/* plane_fit.cpp:55-131 (both execution modes compute the same values) */
static Fit* fit_planes(size_t nc, const int32_t* labels, const size_t* off, const V3* means,
                       const vp_ransac_params* p, size_t* nfit, uint64_t* skipped,
                       uint64_t* unfit) {
  Fit* out = (Fit*)calloc(nc ? nc : 1, sizeof(Fit));
  *nfit = 0;
  *skipped = *unfit = 0;
  const int ni = p->iterations;
  Cand* cands = (Cand*)malloc(sizeof(Cand) * (size_t)(ni > 0 ? ni : 1));
  for (size_t c = 0; c < nc; ++c) {
    const size_t m = off[c + 1] - off[c];
    if (m < 3) {
      ++*skipped;
      continue;
    }
    const V3* pts = means + off[c];
    for (int i = 0; i < ni; ++i) {
      cands[i] = sample_candidate(pts, (uint32_t)m, labels[c], i, p);
      if (cands[i].inliers >= 0) {
        int cnt = 0;
        for (size_t k = 0; k < m; ++k)
          if (fabs(dot3(cands[i].normal, pts[k]) - cands[i].offset) <= p->inlier_eps) ++cnt;
        cands[i].inliers = cnt;
      }
    }
    int best = -1, best_count = -1;
    for (int i = 0; i < ni; ++i)
      if (cands[i].inliers > best_count) {
        best_count = cands[i].inliers;
        best = i;
      }
    if (best_count < 0) {
      ++*unfit;
      continue;
    }
    Fit* f = &out[(*nfit)++];
    const Cand* w = &cands[best];
    memcpy(f->model.normal, w->normal.v, sizeof f->model.normal);
    f->model.offset = w->offset;
    f->model.inlier_count = w->inliers;
    f->model.cluster_label = labels[c];
    f->inliers = (V3*)malloc(sizeof(V3) * (size_t)(w->inliers > 0 ? w->inliers : 1));
    for (size_t k = 0; k < m; ++k)
      if (fabs(dot3(w->normal, pts[k]) - w->offset) <= p->inlier_eps) f->inliers[f->n_in++] = pts[k];
  }
  free(cands);
  return out;
}

/* plane_fit.cpp:133-154 */
static vp_plane refine_plane(const V3* in, size_t n, vp_plane init, V3 up) {
  if (n < 3) return init;
  V3 sum = v3(0, 0, 0);
  for (size_t i = 0; i < n; ++i) sum = vadd(sum, in[i]);
  const V3 cen = vdiv(sum, (double)n);
  double cov[3][3] = {{0}};
  for (size_t i = 0; i < n; ++i) {
    const V3 d = vsub(in[i], cen);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) cov[a][b] = cov[a][b] + d.v[b] * d.v[a];
  }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) cov[a][b] = cov[a][b] / (double)n;
  double val[3];
  V3 vec[3];
  jacobi3(cov, val, vec);
  if (val[1] <= 1e-12 + 1e-9 * fabs(val[2])) return init;
  vp_plane r = init;
  const V3 nrm = orient_up(normalized3(vec[0]), up);
  memcpy(r.normal, nrm.v, sizeof r.normal);
  r.offset = dot3(nrm, cen);
  return r;
}

/* -------------------------------------------------------------- polygonize */
static double cross2(V2 o, V2 a, V2 b) {
  return (a.x - o.x) * (b.y - o.y) - (a.y - o.y) * (b.x - o.x);
}
static int lex_less(V2 a, V2 b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }
static int cmp_lex(const void* a, const void* b) {
  const V2 x = *(const V2*)a, y = *(const V2*)b;
  return lex_less(x, y) ? -1 : (lex_less(y, x) ? 1 : 0);
}

typedef struct { V3 u, v, origin; } Basis;

/* polygonize.cpp:21-34 */
static Basis plane_basis(V3 n, double offset) {
  int least = 0;
  for (int k = 1; k < 3; ++k)
    if (fabs(n.v[k]) < fabs(n.v[least])) least = k;
  V3 axis = v3(0, 0, 0);
  axis.v[least] = 1.0;
  Basis b;
  b.u = normalized3(vsub(axis, vscale(dot3(n, axis), n)));
  b.v = cross3(n, b.u);
  b.origin = vscale(offset, n);
  return b;
}

/* polygonize.cpp:116-139; returns hull size, writes into out (cap >= 2n) */
static size_t monotone_chain(const V2* in, size_t n0, V2* out) {
  V2* pts = (V2*)malloc(sizeof(V2) * (n0 ? n0 : 1));
  memcpy(pts, in, sizeof(V2) * n0);
  qsort(pts, n0, sizeof(V2), cmp_lex);
  size_t n = 0;
  for (size_t i = 0; i < n0; ++i)
    if (n == 0 || !(pts[i].x == pts[n - 1].x && pts[i].y == pts[n - 1].y)) pts[n++] = pts[i];
  if (n < 3) {
    free(pts);
    return 0;
  }
  V2* h = (V2*)malloc(sizeof(V2) * 2 * n);
  size_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    while (k >= 2 && cross2(h[k - 2], h[k - 1], pts[i]) <= 0.0) --k;
    h[k++] = pts[i];
  }
  const size_t lower = k + 1;
  for (size_t i = n - 1; i-- > 0;) {
    while (k >= lower && cross2(h[k - 2], h[k - 1], pts[i]) <= 0.0) --k;
    h[k++] = pts[i];
  }
  size_t m = k - 1;
  if (m < 3) m = 0;
  memcpy(out, h, sizeof(V2) * m);
  free(h);
  free(pts);
  return m;
}

/* polygonize.cpp:50-114 (chunked partial maxima reduce to the same total-order
 * maximum: larger dot, ties to the lexicographically smaller point) */
static size_t hull_filter(const V2* pts, size_t n, int dirs_n, V2* out) {
  if (n <= 3 || dirs_n < 3) {
    memcpy(out, pts, sizeof(V2) * n);
    return n;
  }
  V2 ext[64];
  for (int j = 0; j < dirs_n; ++j) {
    const double a = 2.0 * M_PI * j / dirs_n;
    const V2 d = {cos(a), sin(a)};
    double best = -INFINITY;
    V2 bp = {0.0, 0.0};
    for (size_t i = 0; i < n; ++i) {
      const double dd = pts[i].x * d.x + pts[i].y * d.y;
      if (dd > best || (dd == best && lex_less(pts[i], bp))) {
        best = dd;
        bp = pts[i];
      }
    }
    ext[j] = bp;
  }
  V2 inner[128];
  const size_t ni = monotone_chain(ext, (size_t)dirs_n, inner);
  if (ni < 3) {
    memcpy(out, pts, sizeof(V2) * n);
    return n;
  }
  size_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    for (size_t e = 0; e < ni; ++e)
      if (cross2(inner[e], inner[(e + 1) % ni], pts[i]) <= 0.0) {
        out[k++] = pts[i];
        break;
      }
  }
  return k;
}

typedef struct {
  vp_plane plane;
  size_t nv;
  V2* v2;
  V3* v3;
  double area;
} Poly;

/* polygonize.cpp:166-182; returns 0 for nullopt */
static int make_polygon(vp_plane pl, const V3* in, size_t n, int dirs, Poly* out) {
  if (n < 3) return 0;
  const V3 nrm = v3(pl.normal[0], pl.normal[1], pl.normal[2]);
  const Basis b = plane_basis(nrm, pl.offset);
  V2* proj = (V2*)malloc(sizeof(V2) * n);
  for (size_t i = 0; i < n; ++i) {
    const V3 d = vsub(in[i], b.origin);
    proj[i].x = dot3(d, b.u);
    proj[i].y = dot3(d, b.v);
  }
  V2* surv = (V2*)malloc(sizeof(V2) * n);
  const size_t ns = hull_filter(proj, n, dirs, surv);
  V2* ring = (V2*)malloc(sizeof(V2) * 2 * (ns ? ns : 1));
  const size_t m = monotone_chain(surv, ns, ring);
  free(proj);
  free(surv);
  if (m < 3) {
    free(ring);
    return 0;
  }
  out->plane = pl;
  out->nv = m;
  out->v2 = ring;
  out->v3 = (V3*)malloc(sizeof(V3) * m);
  for (size_t i = 0; i < m; ++i) /* lift_from_plane (polygonize.cpp:46-48) */
    out->v3[i] = vadd(vadd(b.origin, vscale(ring[i].x, b.u)), vscale(ring[i].y, b.v));
  double twice = 0.0; /* polygon_area (polygonize.cpp:146-154) */
  for (size_t i = 0; i < m; ++i) {
    const V2 a = ring[i], c = ring[(i + 1) % m];
    twice += a.x * c.y - c.x * a.y;
  }
  out->area = 0.5 * twice;
  return 1;
}

/* ------------------------------------------------------------------ trace */
typedef struct {
  uint8_t* b;
  size_t n, cap;
} Buf;
static void bput(Buf* w, const void* p, size_t k) {
  if (w->n + k > w->cap) {
    while (w->n + k > w->cap) w->cap = w->cap ? 2 * w->cap : 4096;
    w->b = (uint8_t*)realloc(w->b, w->cap);
  }
  memcpy(w->b + w->n, p, k);
  w->n += k;
}
#define PUT(w, T, v)   \
  do {                 \
    T tmp_ = (T)(v);   \
    bput(w, &tmp_, sizeof(T)); \
  } while (0)
static void put3(Buf* w, V3 v) { bput(w, v.v, 24); }

/* ------------------------------------------------------------ session ABI */
typedef struct {
  Grid g;
  vp_pipeline_params p;
  int32_t last_cell[3];
  uint32_t frame;
  int fixed; /* 1: fixed window, never recentered */
} Session;

/* pipeline.cpp:37-41 */
static void global_cell(const double* t, double res, int32_t* c) {
  for (int k = 0; k < 3; ++k) c[k] = (int32_t)floor(t[k] / res);
}

void* oracle_session_create(double res, const int32_t ext[3], const double center[3],
                            const vp_pipeline_params* p) {
  Session* s = (Session*)calloc(1, sizeof(Session));
  if (grid_init(&s->g, res, ext, center) != VP_OK) {
    free(s->g.cells);
    free(s->g.mask);
    free(s);
    return NULL;
  }
  s->p = *p;
  global_cell(center, res, s->last_cell);
  return s;
}

/* Fixed-window mode: clear_rays + integrate_frame + voxel_frame_polygons per
 * frame with no recenter (the C5 map and the slab path). */
void oracle_session_set_fixed(void* sp, int fixed) { ((Session*)sp)->fixed = fixed; }

void oracle_session_destroy(void* sp) {
  Session* s = (Session*)sp;
  if (!s) return;
  free(s->g.cells);
  free(s->g.mask);
  free(s);
}

void oracle_free(void* p) { free(p); }

int oracle_session_cells(void* sp, double* sums, uint32_t* counts, uint8_t* status) {
  Session* s = (Session*)sp;
  for (size_t f = 0; f < s->g.ncells; ++f) {
    sums[3 * f] = s->g.cells[f].sx;
    sums[3 * f + 1] = s->g.cells[f].sy;
    sums[3 * f + 2] = s->g.cells[f].sz;
    counts[f] = s->g.cells[f].count;
    status[f] = s->g.cells[f].status;
  }
  return 0;
}

/* One run_frames iteration (pipeline.cpp:199-213) + voxel_frame_polygons
 * (pipeline.cpp:43-85), serialised per voxplane_trace.h. */
int oracle_session_frame(void* sp, const float* xyz, uint64_t n, const double R[9],
                         const double t[3], uint8_t** out, uint64_t* out_len) {
  Session* s = (Session*)sp;
  Grid* g = &s->g;
  const vp_pipeline_params* P = &s->p;
  Buf w = {0};
  bput(&w, "VPTR", 4);
  PUT(&w, uint32_t, VP_TRACE_VERSION);
  PUT(&w, uint32_t, s->frame++);

  vp_clear_stats cs;
  vp_update_stats us;
  int rc = clear_rays(g, xyz, n, R, t, &cs);
  if (rc == VP_OK) rc = integrate_frame(g, xyz, n, R, t, &us);
  if (rc != VP_OK) {
    free(w.b);
    return rc;
  }
  int32_t cell[3];
  global_cell(t, g->res, cell);
  vp_shift_stats ss;
  memset(&ss, 0, sizeof ss);
  uint8_t rec = 0;
  if (!s->fixed && (cell[0] != s->last_cell[0] || cell[1] != s->last_cell[1] || cell[2] != s->last_cell[2])) {
    recenter(g, t, &ss);
    memcpy(s->last_cell, cell, sizeof cell);
    rec = 1;
  }
  PUT(&w, uint64_t, cs.voxels_cleared);
  PUT(&w, uint64_t, cs.voxels_freed);
  PUT(&w, uint64_t, us.voxels_touched);
  PUT(&w, uint64_t, us.points_discarded);
  PUT(&w, uint8_t, rec);
  bput(&w, ss.shift, 12);
  PUT(&w, uint64_t, ss.voxels_dropped);
  bput(&w, g->origin, 24);
  PUT(&w, uint64_t, g->occupied);

  if (g->occupied == 0) {
    for (int k = 0; k < 7; ++k) PUT(&w, uint64_t, 0);
  } else {
    size_t V;
    Occ* occ = occupied_voxels(g, &V);
    PUT(&w, uint64_t, V);
    for (size_t i = 0; i < V; ++i) bput(&w, occ[i].idx, 12);
    for (size_t i = 0; i < V; ++i) put3(&w, occ[i].mean);
    for (size_t i = 0; i < V; ++i) PUT(&w, uint32_t, occ[i].count);
    for (size_t i = 0; i < V; ++i) PUT(&w, uint8_t, occ[i].status);
    Est* est = estimate_normals(g, occ, V, &P->seg);
    for (size_t i = 0; i < V; ++i) put3(&w, est[i].normal);
    for (size_t i = 0; i < V; ++i) PUT(&w, int32_t, est[i].ncount);
    for (size_t i = 0; i < V; ++i) PUT(&w, uint8_t, est[i].valid);
    size_t S;
    Step* st = classify_steppable(g, occ, est, V, &P->seg, &S);
    PUT(&w, uint64_t, S);
    for (size_t i = 0; i < S; ++i) bput(&w, st[i].idx, 12);
    for (size_t i = 0; i < S; ++i) put3(&w, st[i].mean);
    for (size_t i = 0; i < S; ++i) put3(&w, st[i].normal);
    int32_t* lab = label_components(st, S, &P->seg, g->res);
    bput(&w, lab, 4 * S);
    /* label_components grouping (segmentation.cpp:182-193) + filter_clusters
       (:196-201): ascending label, members ascending ordinal */
    size_t* cnt = (size_t*)calloc(S ? S : 1, sizeof(size_t));
    for (size_t i = 0; i < S; ++i) cnt[lab[i]]++;
    size_t K = 0;
    for (size_t i = 0; i < S; ++i)
      if (cnt[i] > 0 && cnt[i] >= (size_t)(P->seg.min_cluster_size > 0 ? P->seg.min_cluster_size : 0)) ++K;
    int32_t* klab = (int32_t*)malloc(sizeof(int32_t) * (K ? K : 1));
    size_t* koff = (size_t*)malloc(sizeof(size_t) * (K + 1));
    V3* kmem = (V3*)malloc(sizeof(V3) * (S ? S : 1));
    size_t* kpos = (size_t*)malloc(sizeof(size_t) * (S ? S : 1));
    PUT(&w, uint64_t, K);
    size_t k = 0, tot = 0;
    for (size_t i = 0; i < S; ++i)
      if (cnt[i] > 0 && (long)cnt[i] >= (long)P->seg.min_cluster_size) {
        klab[k] = (int32_t)i;
        koff[k] = tot;
        kpos[i] = tot;
        tot += cnt[i];
        PUT(&w, int32_t, (int32_t)i);
        PUT(&w, uint64_t, cnt[i]);
        ++k;
      }
    koff[K] = tot;
    for (size_t i = 0; i < S; ++i) {
      const size_t l = (size_t)lab[i];
      if (cnt[l] > 0 && (long)cnt[l] >= (long)P->seg.min_cluster_size) kmem[kpos[l]++] = st[i].mean;
    }
    size_t F;
    uint64_t skipped, unfit;
    Fit* fits = fit_planes(K, klab, koff, kmem, &P->ransac, &F, &skipped, &unfit);
    PUT(&w, uint64_t, skipped);
    PUT(&w, uint64_t, unfit);
    PUT(&w, uint64_t, F);
    for (size_t f = 0; f < F; ++f) {
      bput(&w, fits[f].model.normal, 24);
      PUT(&w, double, fits[f].model.offset);
      PUT(&w, int32_t, fits[f].model.inlier_count);
      PUT(&w, int32_t, fits[f].model.cluster_label);
      PUT(&w, uint64_t, fits[f].n_in);
      for (size_t i = 0; i < fits[f].n_in; ++i) put3(&w, fits[f].inliers[i]);
    }
    Poly* polys = (Poly*)calloc(F ? F : 1, sizeof(Poly));
    size_t np = 0;
    const V3 rup = v3(P->ransac.up[0], P->ransac.up[1], P->ransac.up[2]);
    for (size_t f = 0; f < F; ++f) {
      vp_plane model = fits[f].model;
      if (P->refine) { /* pipeline.cpp:74-78 */
        model = refine_plane(fits[f].inliers, fits[f].n_in, model, rup);
        model.inlier_count = fits[f].model.inlier_count;
        model.cluster_label = fits[f].model.cluster_label;
      }
      bput(&w, model.normal, 24);
      PUT(&w, double, model.offset);
      Poly poly;
      if (make_polygon(model, fits[f].inliers, fits[f].n_in, 16, &poly)) {
        if (poly.area >= P->min_polygon_area) {
          polys[np++] = poly;
        } else {
          free(poly.v2);
          free(poly.v3);
        }
      }
    }
    PUT(&w, uint64_t, np);
    for (size_t i = 0; i < np; ++i) {
      bput(&w, polys[i].plane.normal, 24);
      PUT(&w, double, polys[i].plane.offset);
      PUT(&w, int32_t, polys[i].plane.inlier_count);
      PUT(&w, int32_t, polys[i].plane.cluster_label);
      PUT(&w, uint64_t, polys[i].nv);
      for (size_t j = 0; j < polys[i].nv; ++j) {
        PUT(&w, double, polys[i].v2[j].x);
        PUT(&w, double, polys[i].v2[j].y);
      }
      for (size_t j = 0; j < polys[i].nv; ++j) put3(&w, polys[i].v3[j]);
      PUT(&w, double, polys[i].area);
      free(polys[i].v2);
      free(polys[i].v3);
    }
    free(polys);
    for (size_t f = 0; f < F; ++f) free(fits[f].inliers);
    free(fits);
    free(kpos);
    free(kmem);
    free(koff);
    free(klab);
    free(cnt);
    free(lab);
    free(st);
    free(est);
    free(occ);
  }
  *out = w.b;
  *out_len = w.n;
  return VP_OK;
}

/* ---- single-stage entry points for unit-level parity tests ------------- */

/* segmentation.cpp:87-194 on a given steppable list */
int oracle_label_components(size_t n, const int32_t* idx, const double* mean, const double* normal,
                            const vp_seg_params* p, double res, int32_t* labels) {
  Step* s = (Step*)malloc(sizeof(Step) * (n ? n : 1));
  for (size_t i = 0; i < n; ++i) {
    memcpy(s[i].idx, idx + 3 * i, 12);
    s[i].mean = v3(mean[3 * i], mean[3 * i + 1], mean[3 * i + 2]);
    s[i].normal = v3(normal[3 * i], normal[3 * i + 1], normal[3 * i + 2]);
  }
  int32_t* l = label_components(s, n, p, res);
  memcpy(labels, l, 4 * n);
  free(l);
  free(s);
  return 0;
}

/* plane_fit.cpp:55-131: writes models[nc], inlier counts n_in[nc] (0 when
 * unfit/skipped), fitted[nc] flags; inliers written at off[c] into inl. */
int oracle_fit_planes(size_t nc, const int32_t* labels, const uint64_t* off, const double* means,
                      const vp_ransac_params* p, vp_plane* models, uint8_t* fitted,
                      double* inl, uint64_t* n_in, uint64_t* skipped, uint64_t* unfit) {
  size_t* o = (size_t*)malloc(sizeof(size_t) * (nc + 1));
  for (size_t c = 0; c <= nc; ++c) o[c] = (size_t)off[c];
  const size_t tot = nc ? o[nc] : 0;
  V3* m = (V3*)malloc(sizeof(V3) * (tot ? tot : 1));
  for (size_t i = 0; i < tot; ++i) m[i] = v3(means[3 * i], means[3 * i + 1], means[3 * i + 2]);
  size_t F;
  Fit* fits = fit_planes(nc, labels, o, m, p, &F, skipped, unfit);
  size_t f = 0;
  for (size_t c = 0; c < nc; ++c) {
    fitted[c] = 0;
    n_in[c] = 0;
    if (f < F && fits[f].model.cluster_label == labels[c]) {
      models[c] = fits[f].model;
      fitted[c] = 1;
      n_in[c] = fits[f].n_in;
      memcpy(inl + 3 * o[c], fits[f].inliers, sizeof(V3) * fits[f].n_in);
      free(fits[f].inliers);
      ++f;
    }
  }
  free(fits);
  free(m);
  free(o);
  return 0;
}

int oracle_refine_plane(size_t n, const double* pts, const vp_plane* init, const double up[3],
                        vp_plane* out) {
  V3* p = (V3*)malloc(sizeof(V3) * (n ? n : 1));
  for (size_t i = 0; i < n; ++i) p[i] = v3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
  *out = refine_plane(p, n, *init, v3(up[0], up[1], up[2]));
  free(p);
  return 0;
}

/* make_polygon; returns vertex count (0 = nullopt); v2 cap 2n, v3 cap 3n */
int oracle_make_polygon(const vp_plane* pl, size_t n, const double* pts, int dirs, double* v2,
                        double* v3o, double* area) {
  V3* p = (V3*)malloc(sizeof(V3) * (n ? n : 1));
  for (size_t i = 0; i < n; ++i) p[i] = v3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
  Poly poly;
  int nv = 0;
  if (make_polygon(*pl, p, n, dirs, &poly)) {
    nv = (int)poly.nv;
    for (size_t i = 0; i < poly.nv; ++i) {
      v2[2 * i] = poly.v2[i].x;
      v2[2 * i + 1] = poly.v2[i].y;
      memcpy(v3o + 3 * i, poly.v3[i].v, 24);
    }
    *area = poly.area;
    free(poly.v2);
    free(poly.v3);
  }
  free(p);
  return nv;
}

/* CounterRng stream (rng.hpp:13-36) for known-answer tests */
void oracle_rng_stream(uint64_t seed, uint64_t k1, uint64_t k2, uint32_t below_n, size_t count,
                       uint64_t* raw, uint32_t* below) {
  Rng r = rng_make(seed, k1, k2);
  for (size_t i = 0; i < count; ++i) raw[i] = rng_next(&r);
  r = rng_make(seed, k1, k2);
  for (size_t i = 0; i < count; ++i) below[i] = rng_below(&r, below_n);
}

/* jacobi_eigen_sym3 (jacobi.cpp:46-81); a row-major 9, vecs column-major 9 */
void oracle_jacobi(const double a[9], double vals[3], double vecs[9]) {
  double in[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) in[i][j] = a[3 * i + j];
  V3 v[3];
  jacobi3(in, vals, v);
  for (int k = 0; k < 3; ++k) memcpy(vecs + 3 * k, v[k].v, 24);
}
