/* TEST INFRASTRUCTURE ONLY — see tc_oracle.h. Single-threaded C restatement
 * of the reference DBSCAN path; every function cites the reference lines it
 * follows (REF = /root/reference/proj/src). Built with -ffp-contract=off so the
 * fp64 distance chain is never fused (REF geometry.hpp:72-93). */
#include "tc_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  float lo[3], hi[3];
} Box;

enum { KIND_POINT = 0, KIND_DENSE = 1 };

typedef struct { /* REF bvh.hpp:12-17 */
  uint8_t kind;
  int32_t id;
  Box b;
} Prim;

typedef struct { /* REF bvh.hpp:89-94 */
  Box box;
  int32_t left, right, max_rank;
} Node;

typedef struct {
  int dim;
  int32_t m;
  Prim* leaves;
  uint64_t* codes;
  Node* nodes;
} Tree;

/* ---- geometry (REF geometry.hpp:72-156) ---- */

static double dist2(const float* a, const float* b, int dim) {
  double s = 0.0;
  for (int k = 0; k < dim; ++k) {
    double d = (double)a[k] - (double)b[k];
    s += d * d;
  }
  return s;
}

static double box_dist2(const float* p, const Box* b, int dim) {
  double s = 0.0;
  for (int k = 0; k < dim; ++k) {
    double d = 0.0;
    if (p[k] < b->lo[k])
      d = (double)b->lo[k] - (double)p[k];
    else if (p[k] > b->hi[k])
      d = (double)p[k] - (double)b->hi[k];
    s += d * d;
  }
  return s;
}

static uint64_t expand2(uint64_t x) {
  x &= 0xffffffffull;
  x = (x | (x << 16)) & 0x0000ffff0000ffffull;
  x = (x | (x << 8)) & 0x00ff00ff00ff00ffull;
  x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}

static uint64_t expand3(uint64_t x) {
  x &= 0x1fffffull;
  x = (x | (x << 32)) & 0x001f00000000ffffull;
  x = (x | (x << 16)) & 0x001f0000ff0000ffull;
  x = (x | (x << 8)) & 0x100f00f00f00f00full;
  x = (x | (x << 4)) & 0x10c30c30c30c30c3ull;
  x = (x | (x << 2)) & 0x1249249249249249ull;
  return x;
}

static uint32_t quantize(float v, float lo, float hi, int bits) { /* REF :132-141 */
  uint64_t cells = 1ull << bits;
  double w = (double)hi - (double)lo;
  if (w <= 0.0) return 0;
  double t = ((double)v - (double)lo) / w;
  if (t < 0.0) t = 0.0;
  uint64_t q = (uint64_t)(t * (double)cells);
  if (q >= cells) q = cells - 1;
  return (uint32_t)q;
}

static uint64_t morton(const float* p, const float* lo, const float* hi, int dim) {
  if (dim == 2) {
    uint64_t x = quantize(p[0], lo[0], hi[0], 31), y = quantize(p[1], lo[1], hi[1], 31);
    return expand2(x) | (expand2(y) << 1);
  }
  uint64_t x = quantize(p[0], lo[0], hi[0], 21), y = quantize(p[1], lo[1], hi[1], 21),
           z = quantize(p[2], lo[2], hi[2], 21);
  return expand3(x) | (expand3(y) << 1) | (expand3(z) << 2);
}

void oracle_morton_codes(const float* coords, int64_t n, int dim, const float* lo,
                         const float* hi, uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = morton(coords + i * dim, lo, hi, dim);
}

/* ---- LBVH (REF bvh.cpp:10-124) ---- */

typedef struct {
  uint64_t code;
  int32_t idx;
} KeyIdx;

static int cmp_key_idx(const void* a, const void* b) {
  const KeyIdx* x = (const KeyIdx*)a;
  const KeyIdx* y = (const KeyIdx*)b;
  if (x->code != y->code) return x->code < y->code ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static int clz64(uint64_t x) { return x ? __builtin_clzll(x) : 64; }
static int clz32(uint32_t x) { return x ? __builtin_clz(x) : 32; }

static int delta(const Tree* t, int64_t i, int64_t j) { /* REF bvh.cpp:49-56 */
  if (j < 0 || j >= t->m) return -1;
  uint64_t ci = t->codes[i], cj = t->codes[j];
  if (ci != cj) return clz64(ci ^ cj);
  return 64 + clz32((uint32_t)i ^ (uint32_t)j);
}

static void topology(Tree* t) { /* REF bvh.cpp:58-86 */
  for (int64_t i = 0; i < t->m - 1; ++i) {
    int d = delta(t, i, i + 1) > delta(t, i, i - 1) ? 1 : -1;
    int dmin = delta(t, i, i - d);
    int64_t lmax = 2;
    while (delta(t, i, i + lmax * d) > dmin) lmax *= 2;
    int64_t l = 0;
    for (int64_t s = lmax / 2; s >= 1; s /= 2)
      if (delta(t, i, i + (l + s) * d) > dmin) l += s;
    int64_t j = i + l * d;
    int dnode = delta(t, i, j);
    int64_t s = 0, w = l;
    do {
      w = (w + 1) / 2;
      if (delta(t, i, i + (s + w) * d) > dnode) s += w;
    } while (w > 1);
    int64_t gamma = i + s * d + (d < 0 ? d : 0);
    int64_t lo = i < j ? i : j, hi = i < j ? j : i;
    t->nodes[i].left = lo == gamma ? ~(int32_t)gamma : (int32_t)gamma;
    t->nodes[i].right = hi == gamma + 1 ? ~(int32_t)(gamma + 1) : (int32_t)(gamma + 1);
  }
}

static void box_grow(Box* a, const Box* b, int dim) {
  for (int k = 0; k < dim; ++k) {
    if (b->lo[k] < a->lo[k]) a->lo[k] = b->lo[k];
    if (b->hi[k] > a->hi[k]) a->hi[k] = b->hi[k];
  }
}

/* Refit by recursion from the root: same boxes / max ranks as the reference's
 * bottom-up arrival walk (REF bvh.cpp:88-124). */
static void refit(Tree* t, int32_t node) {
  Node* nd = &t->nodes[node];
  int32_t kids[2] = {nd->left, nd->right};
  for (int c = 0; c < 2; ++c) {
    const Box* b;
    int32_t mr;
    if (kids[c] < 0) {
      b = &t->leaves[~kids[c]].b;
      mr = ~kids[c];
    } else {
      refit(t, kids[c]);
      b = &t->nodes[kids[c]].box;
      mr = t->nodes[kids[c]].max_rank;
    }
    if (c == 0) {
      nd->box = *b;
      nd->max_rank = mr;
    } else {
      box_grow(&nd->box, b, t->dim);
      if (mr > nd->max_rank) nd->max_rank = mr;
    }
  }
}

static int tree_build(Tree* t, const Prim* prims, int32_t m, int dim) {
  t->dim = dim;
  t->m = m;
  t->leaves = (Prim*)malloc(sizeof(Prim) * (size_t)m);
  t->codes = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)m);
  t->nodes = (Node*)calloc((size_t)(m > 1 ? m - 1 : 1), sizeof(Node));
  KeyIdx* ki = (KeyIdx*)malloc(sizeof(KeyIdx) * (size_t)m);
  if (!t->leaves || !t->codes || !t->nodes || !ki) return 1;
  float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
  for (int32_t i = 0; i < m; ++i)
    for (int k = 0; k < dim; ++k) { /* centroid (REF geometry.hpp:67-69) */
      float c = 0.5f * (prims[i].b.lo[k] + prims[i].b.hi[k]);
      if (c < lo[k]) lo[k] = c;
      if (c > hi[k]) hi[k] = c;
    }
  for (int32_t i = 0; i < m; ++i) {
    float c[3];
    for (int k = 0; k < dim; ++k) c[k] = 0.5f * (prims[i].b.lo[k] + prims[i].b.hi[k]);
    ki[i].code = morton(c, lo, hi, dim);
    ki[i].idx = i;
  }
  qsort(ki, (size_t)m, sizeof(KeyIdx), cmp_key_idx);
  for (int32_t r = 0; r < m; ++r) {
    t->leaves[r] = prims[ki[r].idx];
    t->codes[r] = ki[r].code;
  }
  free(ki);
  if (m > 1) {
    topology(t);
    refit(t, 0);
  }
  return 0;
}

static void tree_free(Tree* t) {
  free(t->leaves);
  free(t->codes);
  free(t->nodes);
}

/* query_sphere_masked (REF bvh.hpp:45-72); visit returns 0 to stop. */
typedef int (*VisitFn)(void* ctx, int32_t rank, const Prim* prim);

static void tree_query(const Tree* t, const float* p, double radius, int32_t min_rank,
                       VisitFn visit, void* ctx) {
  double r2 = radius * radius;
  if (t->m == 1) {
    if (min_rank <= 0 && box_dist2(p, &t->leaves[0].b, t->dim) <= r2) visit(ctx, 0, &t->leaves[0]);
    return;
  }
  int32_t stack[128];
  int top = 0;
  stack[top++] = 0;
  while (top > 0) {
    const Node* nd = &t->nodes[stack[--top]];
    int32_t kids[2] = {nd->left, nd->right};
    for (int c = 0; c < 2; ++c) {
      int32_t child = kids[c];
      if (child < 0) {
        int32_t rank = ~child;
        if (rank < min_rank) continue;
        if (box_dist2(p, &t->leaves[rank].b, t->dim) <= r2)
          if (!visit(ctx, rank, &t->leaves[rank])) return;
      } else {
        const Node* cn = &t->nodes[child];
        if (cn->max_rank < min_rank) continue;
        if (box_dist2(p, &cn->box, t->dim) <= r2) stack[top++] = child;
      }
    }
  }
}

static Prim* point_prims(const float* coords, int64_t n, int dim) { /* REF dbscan.cpp:27-34 */
  Prim* prims = (Prim*)malloc(sizeof(Prim) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    prims[i].kind = KIND_POINT;
    prims[i].id = (int32_t)i;
    memset(&prims[i].b, 0, sizeof(Box));
    for (int k = 0; k < dim; ++k) prims[i].b.lo[k] = prims[i].b.hi[k] = coords[i * dim + k];
  }
  return prims;
}

int oracle_point_bvh(const float* coords, int64_t n, int dim, int32_t* leaf_ids, int32_t* left,
                     int32_t* right, int32_t* max_rank, float* boxes) {
  Prim* prims = point_prims(coords, n, dim);
  Tree t;
  if (tree_build(&t, prims, (int32_t)n, dim)) return 1;
  for (int32_t r = 0; r < t.m; ++r) leaf_ids[r] = t.leaves[r].id;
  for (int32_t i = 0; i + 1 < t.m; ++i) {
    left[i] = t.nodes[i].left;
    right[i] = t.nodes[i].right;
    max_rank[i] = t.nodes[i].max_rank;
    for (int k = 0; k < 3; ++k) {
      boxes[6 * i + k] = k < dim ? t.nodes[i].box.lo[k] : 0.f;
      boxes[6 * i + 3 + k] = k < dim ? t.nodes[i].box.hi[k] : 0.f;
    }
  }
  tree_free(&t);
  free(prims);
  return 0;
}

/* ---- dense grid (REF dense_grid.cpp:12-98) ---- */

typedef struct {
  uint64_t id;
  int32_t begin, end;
  int dense;
} Cell;

typedef struct {
  int32_t* perm;
  int32_t* cell_of_point;
  Cell* cells;
  int64_t num_cells;
} Grid;

static int64_t cell_coord(float v, float origin, double h, int64_t extent) {
  int64_t c = (int64_t)floor(((double)v - (double)origin) / h);
  if (c < 0) c = 0;
  if (c >= extent) c = extent - 1;
  return c;
}

static int grid_build(Grid* g, const float* coords, int64_t n, int dim, float eps, int minpts) {
  float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
  for (int64_t i = 0; i < n; ++i) /* compute_bounds (REF geometry.hpp:95-101) */
    for (int k = 0; k < dim; ++k) {
      float v = coords[i * dim + k];
      if (v < lo[k]) lo[k] = v;
      if (v > hi[k]) hi[k] = v;
    }
  double h = (double)eps / sqrt((double)dim);
  int64_t extent[3];
  uint64_t total = 1;
  for (int k = 0; k < dim; ++k) {
    double width = (double)hi[k] - (double)lo[k];
    int64_t e = (int64_t)ceil(width / h);
    extent[k] = e < 1 ? 1 : e;
    if (total > (1ull << 62) / (uint64_t)extent[k]) return -1;
    total *= (uint64_t)extent[k];
  }
  KeyIdx* ki = (KeyIdx*)malloc(sizeof(KeyIdx) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t id = 0;
    for (int k = dim - 1; k >= 0; --k)
      id = id * (uint64_t)extent[k] + (uint64_t)cell_coord(coords[i * dim + k], lo[k], h, extent[k]);
    ki[i].code = id;
    ki[i].idx = (int32_t)i;
  }
  qsort(ki, (size_t)n, sizeof(KeyIdx), cmp_key_idx);
  g->perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  g->cell_of_point = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  g->cells = (Cell*)malloc(sizeof(Cell) * (size_t)n);
  g->num_cells = 0;
  for (int64_t i = 0; i < n; ++i) g->perm[i] = ki[i].idx;
  for (int64_t i = 0; i < n;) {
    int64_t j = i;
    while (j < n && ki[j].code == ki[i].code) ++j;
    Cell* c = &g->cells[g->num_cells];
    c->id = ki[i].code;
    c->begin = (int32_t)i;
    c->end = (int32_t)j;
    c->dense = (j - i) >= minpts;
    for (int64_t k = i; k < j; ++k) g->cell_of_point[g->perm[k]] = (int32_t)g->num_cells;
    g->num_cells++;
    i = j;
  }
  free(ki);
  return 0;
}

static void grid_free(Grid* g) {
  free(g->perm);
  free(g->cell_of_point);
  free(g->cells);
}

int64_t oracle_build_grid(const float* coords, int64_t n, int dim, float eps, int minpts,
                          int32_t* perm, int32_t* cell_of_point, uint64_t* cell_id,
                          int32_t* cell_begin, int32_t* cell_end, uint8_t* cell_dense,
                          int64_t cap) {
  Grid g;
  if (grid_build(&g, coords, n, dim, eps, minpts)) return -1;
  memcpy(perm, g.perm, sizeof(int32_t) * (size_t)n);
  memcpy(cell_of_point, g.cell_of_point, sizeof(int32_t) * (size_t)n);
  if (g.num_cells <= cap)
    for (int64_t c = 0; c < g.num_cells; ++c) {
      cell_id[c] = g.cells[c].id;
      cell_begin[c] = g.cells[c].begin;
      cell_end[c] = g.cells[c].end;
      cell_dense[c] = (uint8_t)g.cells[c].dense;
    }
  int64_t m = g.num_cells;
  grid_free(&g);
  return m;
}

/* make_mixed_primitives (REF dense_grid.cpp:79-98) */
static Prim* mixed_prims(const Grid* g, const float* coords, int dim, int32_t* count) {
  Prim* prims = (Prim*)malloc(sizeof(Prim) * (size_t)(g->num_cells > 0 ? g->cells[g->num_cells - 1].end : 1));
  int32_t m = 0;
  for (int64_t c = 0; c < g->num_cells; ++c) {
    const Cell* cell = &g->cells[c];
    if (cell->dense) {
      Prim* p = &prims[m++];
      p->kind = KIND_DENSE;
      p->id = (int32_t)c;
      memset(&p->b, 0, sizeof(Box));
      const float* first = coords + (int64_t)g->perm[cell->begin] * dim;
      for (int k = 0; k < dim; ++k) p->b.lo[k] = p->b.hi[k] = first[k];
      for (int32_t k = cell->begin + 1; k < cell->end; ++k) {
        const float* q = coords + (int64_t)g->perm[k] * dim;
        for (int a = 0; a < dim; ++a) {
          if (q[a] < p->b.lo[a]) p->b.lo[a] = q[a];
          if (q[a] > p->b.hi[a]) p->b.hi[a] = q[a];
        }
      }
    } else {
      for (int32_t k = cell->begin; k < cell->end; ++k) {
        Prim* p = &prims[m++];
        int32_t i = g->perm[k];
        p->kind = KIND_POINT;
        p->id = i;
        memset(&p->b, 0, sizeof(Box));
        for (int a = 0; a < dim; ++a) p->b.lo[a] = p->b.hi[a] = coords[(int64_t)i * dim + a];
      }
    }
  }
  *count = m;
  return prims;
}

/* ---- union-find, sequential (REF union_find.hpp:36-86) ---- */

static int32_t uf_find(int32_t* parent, int32_t i) {
  int32_t cur = parent[i];
  if (cur != i) {
    int32_t prev = i, next = parent[cur];
    while (cur != next) {
      parent[prev] = next;
      prev = cur;
      cur = next;
      next = parent[cur];
    }
  }
  return cur;
}

static void uf_unite(int32_t* parent, int32_t i, int32_t j) {
  i = uf_find(parent, i);
  j = uf_find(parent, j);
  if (i == j) return;
  if (i > j) {
    int32_t t = i;
    i = j;
    j = t;
  }
  parent[j] = i;
}

/* resolve_pair (REF dbscan.hpp:82-99) */
static void resolve(int32_t i, int32_t j, uint8_t* core, int32_t* parent, int force) {
  int ci, cj;
  if (force) {
    core[i] = core[j] = 1;
    ci = cj = 1;
  } else {
    ci = core[i];
    cj = core[j];
  }
  if (ci && cj)
    uf_unite(parent, i, j);
  else if (ci && parent[j] == j)
    parent[j] = uf_find(parent, i);
  else if (cj && parent[i] == i)
    parent[i] = uf_find(parent, j);
}

/* ---- visitors ---- */

typedef struct {
  const float* coords;
  int dim;
  const float* p;
  double eps2;
  int minpts;
  int count;
  int32_t self_rank;
  int32_t i;
  uint8_t* core;
  int32_t* parent;
  int force;
  const Grid* grid;
  int64_t dists, pairs;
} Ctx;

static int visit_fd_core(void* vc, int32_t rank, const Prim* prim) { /* REF dbscan.cpp:46-53 */
  (void)rank;
  Ctx* c = (Ctx*)vc;
  c->dists++;
  if (dist2(c->p, c->coords + (int64_t)prim->id * c->dim, c->dim) <= c->eps2)
    if (++c->count >= c->minpts) return 0;
  return 1;
}

static int visit_fd_main(void* vc, int32_t rank, const Prim* prim) { /* REF dbscan.cpp:76-84 */
  Ctx* c = (Ctx*)vc;
  if (rank == c->self_rank) return 1;
  c->dists++;
  if (dist2(c->p, c->coords + (int64_t)prim->id * c->dim, c->dim) <= c->eps2) {
    c->pairs++;
    resolve(c->i, prim->id, c->core, c->parent, c->force);
  }
  return 1;
}

static int visit_db_core(void* vc, int32_t rank, const Prim* prim) { /* REF dbscan.cpp:121-133 */
  (void)rank;
  Ctx* c = (Ctx*)vc;
  if (prim->kind == KIND_POINT) {
    c->dists++;
    if (dist2(c->p, c->coords + (int64_t)prim->id * c->dim, c->dim) <= c->eps2) c->count++;
  } else {
    const Cell* cell = &c->grid->cells[prim->id];
    for (int32_t k = cell->begin; k < cell->end; ++k) {
      c->dists++;
      if (dist2(c->p, c->coords + (int64_t)c->grid->perm[k] * c->dim, c->dim) <= c->eps2)
        if (++c->count >= c->minpts) break;
    }
  }
  return c->count < c->minpts;
}

static int visit_db_main(void* vc, int32_t rank, const Prim* prim) { /* REF dbscan.cpp:170-195 */
  Ctx* c = (Ctx*)vc;
  if (rank == c->self_rank) return 1;
  if (prim->kind == KIND_POINT) {
    c->dists++;
    if (dist2(c->p, c->coords + (int64_t)prim->id * c->dim, c->dim) <= c->eps2) {
      c->pairs++;
      resolve(c->i, prim->id, c->core, c->parent, c->force);
    }
  } else {
    const Cell* cell = &c->grid->cells[prim->id];
    for (int32_t k = cell->begin; k < cell->end; ++k) {
      int32_t j = c->grid->perm[k];
      c->dists++;
      if (dist2(c->p, c->coords + (int64_t)j * c->dim, c->dim) <= c->eps2) {
        c->pairs++;
        resolve(c->i, j, c->core, c->parent, c->force);
        break;
      }
    }
  }
  return 1;
}

static int valid_points(const float* coords, int64_t n, int dim) {
  if ((dim != 2 && dim != 3) || n < 1) return 0;
  for (int64_t i = 0; i < n * dim; ++i)
    if (!isfinite(coords[i])) return 0;
  return 1;
}

/* dbscan_bruteforce (REF oracle.cpp:10-60): BFS in index order. */
static void bruteforce(const float* coords, int64_t n, int dim, double eps2, int minpts,
                       int32_t* labels, uint8_t* core) {
  uint8_t* visited = (uint8_t*)calloc((size_t)n, 1);
  int64_t qcap = 4 * n + 16;
  int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * (size_t)qcap);
  int64_t* nb = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    labels[i] = -1;
    core[i] = 0;
  }
  for (int64_t x = 0; x < n; ++x) {
    if (visited[x]) continue;
    visited[x] = 1;
    int64_t cnt = 0;
    for (int64_t j = 0; j < n; ++j)
      if (dist2(coords + x * dim, coords + j * dim, dim) <= eps2) nb[cnt++] = j;
    if (cnt < minpts) continue;
    core[x] = 1;
    int32_t cid = (int32_t)x;
    labels[x] = cid;
    int64_t head = 0, tail = 0;
#define PUSH(v)                                                              \
  do {                                                                       \
    if (tail == qcap) {                                                      \
      qcap *= 2;                                                             \
      queue = (int64_t*)realloc(queue, sizeof(int64_t) * (size_t)qcap);      \
    }                                                                        \
    queue[tail++] = (v);                                                     \
  } while (0)
    for (int64_t k = 0; k < cnt; ++k) PUSH(nb[k]);
    while (head < tail) {
      int64_t y = queue[head++];
      if (!visited[y]) {
        visited[y] = 1;
        int64_t c2 = 0;
        for (int64_t j = 0; j < n; ++j)
          if (dist2(coords + y * dim, coords + j * dim, dim) <= eps2) nb[c2++] = j;
        if (c2 >= minpts) {
          core[y] = 1;
          for (int64_t k = 0; k < c2; ++k) PUSH(nb[k]);
        }
      }
      if (labels[y] == -1) labels[y] = cid;
    }
#undef PUSH
  }
  free(visited);
  free(queue);
  free(nb);
}

int oracle_dbscan(const float* coords, int64_t n, int dim, float eps, int minpts, int algo,
                  int32_t* labels, uint8_t* core, int64_t* counters) {
  if (!valid_points(coords, n, dim)) return 1;
  if (!(eps > 0.f) || !isfinite(eps) || minpts < 2) return 1; /* REF dbscan.cpp:21-25 */
  const double eps2 = (double)eps * eps;
  for (int k = 0; k < 7; ++k) counters[k] = 0;
  if (algo == 2) {
    bruteforce(coords, n, dim, eps2, minpts, labels, core);
  } else {
    int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      parent[i] = (int32_t)i;
      core[i] = 0;
    }
    Ctx c;
    memset(&c, 0, sizeof c);
    c.coords = coords;
    c.dim = dim;
    c.eps2 = eps2;
    c.minpts = minpts;
    c.core = core;
    c.parent = parent;
    c.force = minpts == 2;
    Tree t;
    Grid g;
    memset(&g, 0, sizeof g);
    if (algo == 0) {
      Prim* prims = point_prims(coords, n, dim);
      tree_build(&t, prims, (int32_t)n, dim);
      free(prims);
      if (minpts > 2) /* REF dbscan.cpp:36-58 */
        for (int32_t r = 0; r < t.m; ++r) {
          int32_t i = t.leaves[r].id;
          c.p = coords + (int64_t)i * dim;
          c.count = 0;
          tree_query(&t, c.p, (double)eps, 0, visit_fd_core, &c);
          if (c.count >= minpts) core[i] = 1;
        }
      for (int32_t r = 0; r < t.m; ++r) { /* REF dbscan.cpp:60-88 */
        c.i = t.leaves[r].id;
        c.p = coords + (int64_t)c.i * dim;
        c.self_rank = r;
        tree_query(&t, c.p, (double)eps, r, visit_fd_main, &c);
      }
    } else {
      if (grid_build(&g, coords, n, dim, eps, minpts)) {
        free(parent);
        return 1; /* cell id overflow -> invalid_argument */
      }
      int32_t m;
      Prim* prims = mixed_prims(&g, coords, dim, &m);
      tree_build(&t, prims, m, dim);
      free(prims);
      c.grid = &g;
      int64_t dense_pts = 0;
      for (int64_t k = 0; k < g.num_cells; ++k)
        if (g.cells[k].dense) dense_pts += g.cells[k].end - g.cells[k].begin;
      counters[6] = dense_pts;
      if (minpts > 2) /* REF dbscan.cpp:110-139 */
        for (int64_t i = 0; i < n; ++i) {
          if (g.cells[g.cell_of_point[i]].dense) continue;
          c.p = coords + i * dim;
          c.count = 0;
          tree_query(&t, c.p, (double)eps, 0, visit_db_core, &c);
          if (c.count >= minpts) core[i] = 1;
        }
      for (int64_t k = 0; k < g.num_cells; ++k) { /* union_dense_cells REF dbscan.cpp:90-108 */
        const Cell* cell = &g.cells[k];
        if (!cell->dense) continue;
        int32_t first = g.perm[cell->begin];
        core[first] = 1;
        for (int32_t q = cell->begin + 1; q < cell->end; ++q) {
          core[g.perm[q]] = 1;
          uf_unite(parent, first, g.perm[q]);
        }
      }
      int32_t* own = (int32_t*)malloc(sizeof(int32_t) * (size_t)n); /* REF dbscan.cpp:152-162 */
      for (int32_t s = 0; s < t.m; ++s) {
        const Prim* pr = &t.leaves[s];
        if (pr->kind == KIND_POINT)
          own[pr->id] = s;
        else
          for (int32_t q = g.cells[pr->id].begin; q < g.cells[pr->id].end; ++q) own[g.perm[q]] = s;
      }
      for (int64_t i = 0; i < n; ++i) { /* REF dbscan.cpp:164-197 */
        c.i = (int32_t)i;
        c.p = coords + i * dim;
        c.self_rank = own[i];
        tree_query(&t, c.p, (double)eps, own[i], visit_db_main, &c);
      }
      free(own);
    }
    for (int64_t i = 0; i < n; ++i) { /* flatten + finalize (REF dbscan.cpp:202-219) */
      int32_t p = parent[i];
      while (p != parent[p]) p = parent[p];
      parent[i] = p;
    }
    for (int64_t i = 0; i < n; ++i)
      labels[i] = (core[i] || parent[i] != (int32_t)i) ? parent[i] : -1;
    counters[0] = minpts == 2;
    counters[1] = c.pairs;
    counters[2] = c.dists;
    tree_free(&t);
    if (algo == 1) grid_free(&g);
    free(parent);
  }
  for (int64_t i = 0; i < n; ++i) { /* REF dbscan.cpp:276-282 */
    if (labels[i] == -1)
      counters[5]++;
    else if (labels[i] == (int32_t)i)
      counters[3]++;
    counters[4] += core[i];
  }
  return 0;
}

/* ---- check_equivalence (REF oracle.cpp:72-163), O(n^2) border rule ---- */

static int64_t bad_border(const float* coords, int64_t n, int dim, double eps2,
                          const int32_t* l, const uint8_t* c) {
  for (int64_t i = 0; i < n; ++i) {
    if (c[i] || l[i] == -1) continue;
    int ok = 0;
    for (int64_t j = 0; j < n && !ok; ++j)
      ok = c[j] && l[j] == l[i] && dist2(coords + i * dim, coords + j * dim, dim) <= eps2;
    if (!ok) return i;
  }
  return -1;
}

static const int32_t* g_sort_labels; /* qsort context (single-threaded oracle) */
static int cmp_label_index(const void* x, const void* y) {
  const int64_t i = *(const int64_t*)x, j = *(const int64_t*)y;
  const int32_t a = g_sort_labels[i], b = g_sort_labels[j];
  if (a != b) return a < b ? -1 : 1;
  return i < j ? -1 : (i > j);
}

int oracle_check_equivalence(const float* coords, int64_t n, int dim, float eps,
                             const int32_t* la, const uint8_t* ca, const int32_t* lb,
                             const uint8_t* cb, char* msg, int64_t msg_len) {
  char buf[256];
  int pass = 0;
  int64_t at = -1;
  const char* what = NULL;
  for (int64_t i = 0; i < n && !what; ++i)
    if (ca[i] != cb[i]) what = "core flags differ", at = i;
  for (int64_t i = 0; i < n && !what; ++i)
    if ((la[i] == -1) != (lb[i] == -1)) what = "noise sets differ", at = i;
  if (!what) { /* bijection (REF oracle.cpp:144-152): the sequential emplace keeps,
                 per label, the FIRST core carrying it, and fails at the first core
                 whose other label differs from that core's; labels are arbitrary
                 int32, so the first core per label comes from a sort */
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i) m += ca[i] != 0;
    int64_t* ia = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
    int64_t* ib = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
    int64_t* fa = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t* fb = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i)
      if (ca[i]) ia[k] = ib[k] = i, ++k;
    g_sort_labels = la;
    qsort(ia, (size_t)m, sizeof(int64_t), cmp_label_index);
    g_sort_labels = lb;
    qsort(ib, (size_t)m, sizeof(int64_t), cmp_label_index);
    for (int64_t t = 0; t < m; ++t) { /* fa[i] = first core with i's a-label */
      fa[ia[t]] = (t > 0 && la[ia[t - 1]] == la[ia[t]]) ? fa[ia[t - 1]] : ia[t];
      fb[ib[t]] = (t > 0 && lb[ib[t - 1]] == lb[ib[t]]) ? fb[ib[t - 1]] : ib[t];
    }
    for (int64_t i = 0; i < n && !what; ++i)
      if (ca[i] && (lb[fa[i]] != lb[i] || la[fb[i]] != la[i])) what = "core partitions differ", at = i;
    free(ia);
    free(ib);
    free(fa);
    free(fb);
  }
  const double eps2 = (double)eps * eps;
  if (!what && (at = bad_border(coords, n, dim, eps2, la, ca)) >= 0)
    what = "first clustering has an invalid border label";
  if (!what && (at = bad_border(coords, n, dim, eps2, lb, cb)) >= 0)
    what = "second clustering has an invalid border label";
  if (!what) {
    pass = 1;
    snprintf(buf, sizeof buf, "PASS");
  } else {
    snprintf(buf, sizeof buf, "%s (first divergence at point %lld)", what, (long long)at);
  }
  if (msg && msg_len > 0) {
    strncpy(msg, buf, (size_t)msg_len - 1);
    msg[msg_len - 1] = '\0';
  }
  return pass;
}

/* ---- benchmark inputs -------------------------------------
 * Test/bench infrastructure: the reference arm of bench.py and the full-size
 * parity tests generate their inputs here, so they never load the product
 * library. SplitMix64 follows REF rng.hpp:11-47; the HACC-like and taxi-like
 * recipes are the SURVEY §8d specifications (the reference ships neither).
 * Output must be byte-identical to the product's tcg_generate_* (checked by
 * tests/test_oracle.py against the sha256 in tests/golden/generators.json). */

typedef struct {
  uint64_t state;
  int have_spare;
  double spare;
} Rng;

static uint64_t rng_next(Rng* r) { /* REF rng.hpp:15-20 */
  uint64_t z = (r->state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static double rng_unit(Rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; } /* :23 */
static double rng_range(Rng* r, double lo, double hi) { return lo + (hi - lo) * rng_unit(r); }
static double rng_gauss(Rng* r) { /* REF rng.hpp:28-41 (Box-Muller, cached half) */
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = rng_unit(r), u2 = rng_unit(r);
  while (u1 == 0.0) u1 = rng_unit(r);
  const double mag = sqrt(-2.0 * log(u1)), ang = 2.0 * 3.141592653589793 * u2;
  r->spare = mag * sin(ang);
  r->have_spare = 1;
  return mag * cos(ang);
}

int oracle_gen_hacc_like(int64_t n, double box_len, double halo_frac, uint64_t seed,
                         float* out) {
  if (n < 1 || !(box_len > 0.0) || !(halo_frac >= 0.0 && halo_frac <= 1.0)) return 1;
  Rng r = {seed, 0, 0.0};
  const int64_t n_halo = (int64_t)(halo_frac * (double)n);
  float* w = out;
  for (int64_t i = 0; i < (n - n_halo) * 3; ++i) *w++ = (float)rng_range(&r, 0.0, box_len);
  for (int64_t made = 0; made < n_halo;) {
    int64_t m = (int64_t)(20.0 / pow(1.0 - rng_unit(&r), 1.0 / 0.9));
    if (m > 200000) m = 200000;
    if (m > n_halo - made) m = n_halo - made;
    if (m < 1) m = 1;
    const double a = 0.010 * cbrt((double)m / 20.0);
    double c[3];
    for (int k = 0; k < 3; ++k) c[k] = rng_range(&r, a, box_len - a);
    for (int64_t p = 0; p < m; ++p) {
      double rad;
      do { /* Plummer radius, redrawn beyond 10a */
        double uu;
        do uu = rng_unit(&r); while (uu == 0.0);
        rad = a / sqrt(pow(uu, -2.0 / 3.0) - 1.0);
      } while (!(rad <= 10.0 * a));
      const double z = rng_range(&r, -1.0, 1.0);
      const double phi = rng_range(&r, 0.0, 2.0 * 3.141592653589793);
      const double s = sqrt(1.0 - z * z);
      *w++ = (float)(c[0] + rad * s * cos(phi));
      *w++ = (float)(c[1] + rad * s * sin(phi));
      *w++ = (float)(c[2] + rad * z);
    }
    made += m;
  }
  return 0;
}

int oracle_gen_taxi_like(int64_t n, uint64_t seed, float* out) {
  enum { CITIES = 8, SEGMENTS = 300 };
  if (n < 1) return 1;
  Rng r = {seed, 0, 0.0};
  double city[CITIES][2], seg[SEGMENTS][4], cdf[SEGMENTS], total = 0.0;
  for (int c = 0; c < CITIES; ++c)
    for (int k = 0; k < 2; ++k) city[c][k] = rng_range(&r, 0.2, 0.8);
  for (int s = 0; s < SEGMENTS; ++s) {
    const int c = (int)(rng_next(&r) % CITIES);
    const double ax = city[c][0] + 0.08 * rng_gauss(&r);
    const double ay = city[c][1] + 0.08 * rng_gauss(&r);
    const double ang = rng_range(&r, 0.0, 3.141592653589793);
    const double len = -0.02 * log(1.0 - rng_unit(&r));
    seg[s][0] = ax;
    seg[s][1] = ay;
    seg[s][2] = len * cos(ang);
    seg[s][3] = len * sin(ang);
    total += pow((double)(s + 1), -0.8); /* Zipf(0.8) weights */
    cdf[s] = total;
  }
  for (int64_t i = 0; i < n; ++i) {
    double x, y;
    if (rng_unit(&r) < 0.98) {
      const double pick = rng_unit(&r) * total;
      int lo = 0, hi = SEGMENTS; /* first cdf entry > pick */
      while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (cdf[mid] > pick) hi = mid; else lo = mid + 1;
      }
      const double* g = seg[lo < SEGMENTS ? lo : SEGMENTS - 1];
      const double t = rng_unit(&r);
      x = g[0] + t * g[2] + 1e-4 * rng_gauss(&r);
      y = g[1] + t * g[3] + 1e-4 * rng_gauss(&r);
    } else {
      x = rng_unit(&r);
      y = rng_unit(&r);
    }
    out[2 * i] = (float)(x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x));
    out[2 * i + 1] = (float)(y < 0.0 ? 0.0 : (y > 1.0 ? 1.0 : y));
  }
  return 0;
}
