/* traversal.c — ORACLE (test infrastructure only; see oracle.h).
 *
 * The dual tree traversal exactly as PAPER.md:148-153 describes it: a "last in, first out" stack
 * of (target cell, source cell) pairs, initialised with the pair of roots; pop a pair, subdivide
 * the larger cell, match its offspring with the other cell, and for each new pair either
 * compute the interaction at once (MAC accepted; the kind chosen to optimise performance,
 * PAPER.md:153, :169) or push the pair back on the stack.
 *
 * Readings (restated in DESIGN.md §3):
 *   R4  cell radius = cube half-width;  R5  accept iff (r_t + r_s) <= theta * R;
 *   R6  the MAC is tested before the leaf rule; a rejected leaf-leaf pair is a P2P;
 *   R7  ties in size split the SOURCE (the illustrated case); a leaf is never split;
 *   R8  kind = argmin of the linear cost model {t_ml, t_mp*n_t, t_pp*n_t*n_s}, ties M2L > M2P > P2P.
 * The MAC is evaluated in integer "doubled grid" units (c4): centre c~ = (2*g + 1) * 2^(21-level),
 * radius r~ = 2^(21-level); R~^2 is an exact int64, and the comparison is one fixed FP64
 * expression (compiled with -ffp-contract=off), so the decision is bit-reproducible.
 */
#include <math.h>
#include <stdlib.h>

#include "oracle.h"

static void grid_centre(const orc_cell *c, int64_t g2[3]) {
  int64_t g[3] = {0, 0, 0};
  for (int b = 0; b < c->level; ++b) {
    g[0] |= (int64_t)((c->prefix >> (3 * b + 2)) & 1) << b;
    g[1] |= (int64_t)((c->prefix >> (3 * b + 1)) & 1) << b;
    g[2] |= (int64_t)((c->prefix >> (3 * b + 0)) & 1) << b;
  }
  const int64_t unit = (int64_t)1 << (ORC_LEVELS - c->level);
  for (int a = 0; a < 3; ++a) g2[a] = (2 * g[a] + 1) * unit;
}

/* theta = (r_t + r_s)/R; accepted ("far/small enough", :153) iff <= theta. */
int orc_mac_accept(const orc_cell *t, const orc_cell *s, double theta) {
  int64_t ct[3], cs[3];
  grid_centre(t, ct);
  grid_centre(s, cs);
  int64_t R2 = 0;
  for (int a = 0; a < 3; ++a) R2 += (ct[a] - cs[a]) * (ct[a] - cs[a]);
  const int64_t rsum = ((int64_t)1 << (ORC_LEVELS - t->level)) + ((int64_t)1 << (ORC_LEVELS - s->level));
  const double lhs = (double)rsum;
  const double rhs = theta * sqrt((double)R2);
  return lhs <= rhs;
}

/* PAPER.md:130 kernel pre-calculation -> per-unit costs; S:335 linear model; S:345 tie order.
 * cost[0] = t_pp (s per particle pair), cost[1] = t_mp (s per target particle), cost[2] = t_ml
 * (s per translation). */
int orc_select_kind(int mode, const double cost[3], int64_t nt, int64_t ns) {
  if (mode == ORC_FMM) return ORC_K_M2L;      /* PAPER.md:169 "FMM always performs cell-cell" */
  if (mode == ORC_TREECODE) return ORC_K_M2P; /* PAPER.md:169 "treecode always cell-particle" */
  const double c_pp = (cost[0] * (double)nt) * (double)ns;
  const double c_mp = cost[1] * (double)nt;
  const double c_ml = cost[2];
  if (c_ml <= c_mp && c_ml <= c_pp) return ORC_K_M2L;
  if (c_mp <= c_pp) return ORC_K_M2P;
  return ORC_K_P2P;
}

typedef struct {
  orc_task *v;
  int64_t n, cap;
} taskvec;

static void emit(taskvec *tv, int kind, int64_t t, int64_t s) {
  if (tv->n == tv->cap) {
    tv->cap = tv->cap ? 2 * tv->cap : 1024;
    tv->v = (orc_task *)realloc(tv->v, sizeof(orc_task) * (size_t)tv->cap);
  }
  tv->v[tv->n].kind = kind;
  tv->v[tv->n].t = t;
  tv->v[tv->n].s = s;
  tv->n++;
}

/* target_mask (may be NULL): sampled-target pruning — a pair whose target cell
 * holds no sampled particle is dropped; the surviving tasks are exactly those of the full run
 * whose target contains a sampled particle. */
int64_t orc_traverse(const orc_cell *cells, int64_t ncells, double theta, int mode,
                     const double cost[3], const unsigned char *target_mask, orc_task **tasks_out) {
  taskvec tv = {0, 0, 0};
  (void)ncells;
  int64_t cap = 1024, top = 0;
  int64_t *stack = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)cap);
  if (!target_mask || target_mask[0]) {
    stack[0] = 0;
    stack[1] = 0;
    top = 1;
  }
  while (top > 0) {
    --top;
    const int64_t A = stack[2 * top], B = stack[2 * top + 1];
    const orc_cell *a = &cells[A], *b = &cells[B];
    if (a->nchild == 0 && b->nchild == 0) { /* only the single-leaf root pair reaches here */
      emit(&tv, ORC_K_P2P, A, B);
      continue;
    }
    int split_source;
    if (a->nchild == 0)
      split_source = 1;
    else if (b->nchild == 0)
      split_source = 0;
    else
      split_source = (b->level <= a->level); /* larger cell = smaller level; tie -> source */
    const orc_cell *sp = split_source ? b : a;
    for (int c = 0; c < sp->nchild; ++c) {
      const int64_t t = split_source ? A : sp->child[c];
      const int64_t s = split_source ? sp->child[c] : B;
      if (target_mask && !target_mask[t]) continue;
      const orc_cell *ct = &cells[t], *cs = &cells[s];
      if (orc_mac_accept(ct, cs, theta)) {
        emit(&tv, orc_select_kind(mode, cost, ct->count, cs->count), t, s);
      } else if (ct->nchild == 0 && cs->nchild == 0) {
        emit(&tv, ORC_K_P2P, t, s);
      } else {
        if (top == cap) {
          cap *= 2;
          stack = (int64_t *)realloc(stack, sizeof(int64_t) * 2 * (size_t)cap);
        }
        stack[2 * top] = t;
        stack[2 * top + 1] = s;
        ++top;
      }
    }
  }
  free(stack);
  *tasks_out = tv.v;
  return tv.n;
}
