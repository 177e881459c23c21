/* tree.c — ORACLE (test infrastructure only; see oracle.h).
 *
 * Root cube, Morton keys, stable key sort and the adaptive octree, written out plainly:
 *   SURVEY.md §8(c) c2 (root cube of power-of-two side centred on the bounding box, integer keys,
 *   x bit most significant in each triple), c3 (split any cell with count > ncrit and level < 21
 *   into its non-empty octant children; PAPER.md:47 and :168 adaptive tree with N_crit;
 *   S:96-104), c4 (cell radius = cube half-width).
 * Every floating-point step here is an IEEE-exact or correctly-rounded FP64 operation, so the
 * keys are a pure function of the float32 inputs (reading R9).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* c2: returns 0, or -1 if any coordinate is not finite. */
int orc_root_cube(const float *xyz, int64_t n, double origin[3], double *L) {
  double mn[3] = {0, 0, 0}, mx[3] = {0, 0, 0};
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      const float v = xyz[3 * i + a];
      if (!isfinite(v)) return -1;
      if (i == 0 || v < mn[a]) mn[a] = v;
      if (i == 0 || v > mx[a]) mx[a] = v;
    }
  double extent = 0.0;
  for (int a = 0; a < 3; ++a)
    if (mx[a] - mn[a] > extent) extent = mx[a] - mn[a];
  double side = 1.0; /* L = 2^ceil(log2 extent); 1 when the extent is 0 */
  if (extent > 0.0) {
    while (side < extent) side *= 2.0;
    while (side * 0.5 >= extent) side *= 0.5;
  }
  for (int a = 0; a < 3; ++a) origin[a] = 0.5 * (mn[a] + mx[a]) - 0.5 * side;
  *L = side;
  return 0;
}

/* c2: ix = clamp(floor((x - origin) * 2^21 / L), 0, 2^21 - 1); key interleaves bit b of
 * (ix, iy, iz) at bits (3b+2, 3b+1, 3b). */
void orc_morton_keys(const float *xyz, int64_t n, const double origin[3], double L,
                     uint64_t *keys) {
  const double scale = 2097152.0 / L; /* 2^21 / L: a power of two */
  for (int64_t i = 0; i < n; ++i) {
    int64_t g[3];
    for (int a = 0; a < 3; ++a) {
      double t = floor(((double)xyz[3 * i + a] - origin[a]) * scale);
      if (t < 0.0) t = 0.0;
      if (t > 2097151.0) t = 2097151.0;
      g[a] = (int64_t)t;
    }
    uint64_t k = 0;
    for (int b = 0; b < ORC_LEVELS; ++b) {
      k |= (uint64_t)((g[0] >> b) & 1) << (3 * b + 2);
      k |= (uint64_t)((g[1] >> b) & 1) << (3 * b + 1);
      k |= (uint64_t)((g[2] >> b) & 1) << (3 * b + 0);
    }
    keys[i] = k;
  }
}

static const uint64_t *g_sort_keys;
static int cmp_key_idx(const void *pa, const void *pb) {
  const int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
  if (g_sort_keys[a] != g_sort_keys[b]) return g_sort_keys[a] < g_sort_keys[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}

/* c2: perm[i] = original index of the i-th particle in (key, original index) order. */
void orc_sort_keys(const uint64_t *keys, int64_t n, int64_t *perm) {
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  g_sort_keys = keys;
  qsort(perm, (size_t)n, sizeof(int64_t), cmp_key_idx);
  g_sort_keys = NULL;
}

typedef struct {
  orc_cell *v;
  int64_t n, cap;
} cellvec;

static int64_t new_cell(cellvec *cv) {
  if (cv->n == cv->cap) {
    cv->cap = cv->cap ? 2 * cv->cap : 64;
    cv->v = (orc_cell *)realloc(cv->v, sizeof(orc_cell) * (size_t)cv->cap);
  }
  memset(&cv->v[cv->n], 0, sizeof(orc_cell));
  return cv->n++;
}

/* c3, recursive: the cell (level, prefix) owns sorted particles [begin, begin+count). */
static int64_t build(cellvec *cv, const uint64_t *keys, int64_t begin, int64_t count, int level,
                     uint64_t prefix, int64_t parent, int ncrit) {
  const int64_t id = new_cell(cv);
  cv->v[id].level = level;
  cv->v[id].prefix = prefix;
  cv->v[id].begin = begin;
  cv->v[id].count = count;
  cv->v[id].parent = parent;
  cv->v[id].nchild = 0;
  if (count > ncrit && level < ORC_LEVELS) {
    const int shift = 3 * (ORC_LEVELS - (level + 1));
    int64_t i = begin;
    for (int oct = 0; oct < 8; ++oct) {
      const uint64_t cp = prefix * 8 + (uint64_t)oct;
      const int64_t b = i;
      while (i < begin + count && (keys[i] >> shift) == cp) ++i;
      if (i > b) {
        const int64_t c = build(cv, keys, b, i - b, level + 1, cp, id, ncrit);
        cv->v[id].child[cv->v[id].nchild++] = c;
      }
    }
  }
  return id;
}

/* Builds the tree over sorted keys; returns the number of cells (root = cell 0, DFS order). */
int64_t orc_build_tree(const uint64_t *sorted_keys, int64_t n, int ncrit, orc_cell **cells_out) {
  cellvec cv = {0, 0, 0};
  build(&cv, sorted_keys, 0, n, 0, 0, -1, ncrit);
  *cells_out = cv.v;
  return cv.n;
}

/* c4: centre = origin + (cell grid coordinate + 1/2) * L / 2^level; radius = L / 2^(level+1). */
void orc_cell_geometry(const orc_cell *c, const double origin[3], double L, double centre[3],
                       double *radius) {
  uint64_t g[3] = {0, 0, 0};
  for (int b = 0; b < c->level; ++b) {
    g[0] |= ((c->prefix >> (3 * b + 2)) & 1) << b;
    g[1] |= ((c->prefix >> (3 * b + 1)) & 1) << b;
    g[2] |= ((c->prefix >> (3 * b + 0)) & 1) << b;
  }
  const double w = L / ldexp(1.0, c->level);
  for (int a = 0; a < 3; ++a) centre[a] = origin[a] + ((double)g[a] + 0.5) * w;
  *radius = 0.5 * w;
}
