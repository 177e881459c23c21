/* evaluate.c — ORACLE (test infrastructure only; see oracle.h).
 *
 * The whole hybrid treecode/FMM of PAPER.md:145-169 in FP64, step by step (SURVEY.md §3 item 4,
 * S:274-277):  root cube + keys + sort -> adaptive tree -> P2M at leaves, M2M upward ->
 * LIFO dual traversal emitting M2L / M2P / P2P tasks -> execute tasks -> L2L downward, L2P ->
 * phi_i = sum_{j != i} q_j / r_ij and grad_i = -sum_j q_j (x_i - x_j)/r_ij^3,
 * returned in the caller's original particle order.
 *
 * OpenMP is used only over independent targets (each output is written by exactly one thread),
 * so the arithmetic is that of the plain sequential algorithm.
 *
 * Sampled-target mode (SURVEY §8(d) "oracle timing"): when `sample` is given, the traversal
 * drops pairs whose target holds no sampled particle and only the sampled particles are
 * evaluated; their values are exactly those of the full run.
 */
#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

struct orc_fmm {
  int64_t n;
  double origin[3], L;
  uint64_t *skeys;
  int64_t *perm;
  orc_cell *cells;
  int64_t ncells;
  orc_task *tasks;
  int64_t ntasks;
};

static double now(void) { return omp_get_wtime(); }

/* direct O(N^2) sum in FP64, ascending source order, r = 0 pairs skipped. */
void orc_direct(const float *xyz, const float *q, int64_t n, const int64_t *targets,
                int64_t ntargets, double *phi, double *grad) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t k = 0; k < ntargets; ++k) {
    const int64_t i = targets ? targets[k] : k;
    const double xi[3] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
    double ph = 0, g[3] = {0, 0, 0};
    for (int64_t j = 0; j < n; ++j) {
      const double d[3] = {xi[0] - (double)xyz[3 * j], xi[1] - (double)xyz[3 * j + 1],
                           xi[2] - (double)xyz[3 * j + 2]};
      const double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
      if (r2 == 0.0) continue;
      const double r = sqrt(r2);
      ph += (double)q[j] / r;
      for (int a = 0; a < 3; ++a) g[a] -= (double)q[j] * d[a] / (r2 * r);
    }
    phi[k] = ph;
    for (int a = 0; a < 3; ++a) grad[3 * k + a] = g[a];
  }
}

/* CSR of task indices grouped by target cell, for one kind. */
static void group_by_target(const orc_task *tasks, int64_t ntasks, int64_t ncells, int kind,
                            int64_t **off_out, int64_t **idx_out) {
  int64_t *off = (int64_t *)calloc((size_t)ncells + 1, sizeof(int64_t));
  for (int64_t k = 0; k < ntasks; ++k)
    if (tasks[k].kind == kind) off[tasks[k].t + 1]++;
  for (int64_t c = 0; c < ncells; ++c) off[c + 1] += off[c];
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * ((size_t)ncells + 1));
  memcpy(fill, off, sizeof(int64_t) * ((size_t)ncells + 1));
  int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(off[ncells] + 1));
  for (int64_t k = 0; k < ntasks; ++k)
    if (tasks[k].kind == kind) idx[fill[tasks[k].t]++] = k;
  free(fill);
  *off_out = off;
  *idx_out = idx;
}

orc_fmm *orc_fmm_run(const float *xyz, const float *q, int64_t n, int p, double theta, int ncrit,
                     int mode, const double cost[3], const int64_t *sample, int64_t nsample,
                     double *phi, double *grad, double *phase_seconds) {
  return orc_fmm_run_basis(xyz, q, n, p, theta, ncrit, mode, cost, sample, nsample, phi, grad,
                           phase_seconds, ORC_SPHERICAL);
}

/* basis: ORC_SPHERICAL (harmonics.c) or ORC_CARTESIAN (cartesian.c, Taylor of total order p);
 * tree, traversal, kind selection and P2P are the same for both. */
orc_fmm *orc_fmm_run_basis(const float *xyz, const float *q, int64_t n, int p, double theta,
                           int ncrit, int mode, const double cost[3], const int64_t *sample,
                           int64_t nsample, double *phi, double *grad, double *phase_seconds,
                           int basis) {
  const int cart = basis == ORC_CARTESIAN;
  double ph_t[5] = {0, 0, 0, 0, 0};
  orc_fmm *f = (orc_fmm *)calloc(1, sizeof(orc_fmm));
  f->n = n;
  const int64_t nout = sample ? nsample : n;
  for (int64_t k = 0; k < nout; ++k) {
    phi[k] = 0;
    grad[3 * k] = grad[3 * k + 1] = grad[3 * k + 2] = 0;
  }
  if (n == 0) return f;
  double t0 = now();

  /* (1) root cube, keys, stable sort */
  if (orc_root_cube(xyz, n, f->origin, &f->L) != 0) {
    free(f);
    return NULL;
  }
  uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
  orc_morton_keys(xyz, n, f->origin, f->L, keys);
  f->perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  orc_sort_keys(keys, n, f->perm);
  f->skeys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
  double *xs = (double *)malloc(sizeof(double) * 3 * (size_t)n);
  double *qs = (double *)malloc(sizeof(double) * (size_t)n);
  int64_t *inv = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t o = f->perm[i];
    f->skeys[i] = keys[o];
    for (int a = 0; a < 3; ++a) xs[3 * i + a] = xyz[3 * o + a];
    qs[i] = q[o];
    inv[o] = i;
  }
  free(keys);

  /* output slot of each sorted particle (-1 = not evaluated in sampled mode) */
  int64_t *slot = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) slot[i] = sample ? -1 : f->perm[i];
  if (sample)
    for (int64_t k = 0; k < nsample; ++k) slot[inv[sample[k]]] = k;
  free(inv);

  if (mode == ORC_DIRECT) { /* no tree: one all-pairs P2P (SURVEY §8(b) FMM_DIRECT) */
    ph_t[0] = now() - t0;
    double t3 = now();
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < n; ++i) {
      if (slot[i] < 0) continue;
      double ph = 0, g[3] = {0, 0, 0};
      orc_p2p(1, &xs[3 * i], n, xs, qs, &ph, g);
      phi[slot[i]] = ph;
      for (int a = 0; a < 3; ++a) grad[3 * slot[i] + a] = g[a];
    }
    ph_t[3] = now() - t3;
    free(xs);
    free(qs);
    free(slot);
    if (phase_seconds) memcpy(phase_seconds, ph_t, sizeof ph_t);
    return f;
  }

  /* (2) adaptive tree */
  f->ncells = orc_build_tree(f->skeys, n, ncrit, &f->cells);
  const int64_t nc = f->ncells;
  orc_cell *cells = f->cells;
  double *centre = (double *)malloc(sizeof(double) * 3 * (size_t)nc);
  int maxlev = 0;
  for (int64_t c = 0; c < nc; ++c) {
    double r;
    orc_cell_geometry(&cells[c], f->origin, f->L, &centre[3 * c], &r);
    if (cells[c].level > maxlev) maxlev = cells[c].level;
  }
  /* cells grouped by level (cells at one level are independent) */
  int64_t *lev_off = (int64_t *)calloc((size_t)maxlev + 2, sizeof(int64_t));
  int64_t *by_lev = (int64_t *)malloc(sizeof(int64_t) * (size_t)nc);
  for (int64_t c = 0; c < nc; ++c) lev_off[cells[c].level + 1]++;
  for (int l = 0; l <= maxlev; ++l) lev_off[l + 1] += lev_off[l];
  {
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * ((size_t)maxlev + 2));
    memcpy(fill, lev_off, sizeof(int64_t) * ((size_t)maxlev + 2));
    for (int64_t c = 0; c < nc; ++c) by_lev[fill[cells[c].level]++] = c;
    free(fill);
  }
  unsigned char *mask = NULL;
  if (sample) {
    mask = (unsigned char *)calloc((size_t)nc, 1);
    for (int64_t c = 0; c < nc; ++c) {
      if (cells[c].nchild) continue;
      int any = 0;
      for (int64_t i = cells[c].begin; i < cells[c].begin + cells[c].count; ++i) any |= slot[i] >= 0;
      if (!any) continue;
      for (int64_t a = c; a >= 0; a = cells[a].parent) mask[a] = 1;
    }
  }
  ph_t[0] = now() - t0;

  /* (3) upward sweep: P2M at leaves, M2M child -> parent, deepest level first */
  double t1 = now();
  const int64_t NT = (int64_t)(p + 1) * (p + 1);
  cplx *M = (cplx *)calloc((size_t)(nc * NT), sizeof(cplx));
  cplx *Lx = (cplx *)calloc((size_t)(nc * NT), sizeof(cplx));
  const int64_t NK = orc_cart_count(p);
  double *MC = cart ? (double *)calloc((size_t)(nc * NK), sizeof(double)) : NULL;
  double *LC = cart ? (double *)calloc((size_t)(nc * NK), sizeof(double)) : NULL;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t c = 0; c < nc; ++c)
    if (cells[c].nchild == 0) {
      if (cart)
        orc_cart_p2m(p, &centre[3 * c], cells[c].count, &xs[3 * cells[c].begin],
                     &qs[cells[c].begin], &MC[c * NK]);
      else
        orc_p2m(p, &centre[3 * c], cells[c].count, &xs[3 * cells[c].begin], &qs[cells[c].begin],
                &M[c * NT]);
    }
  for (int l = maxlev - 1; l >= 0; --l) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t k = lev_off[l]; k < lev_off[l + 1]; ++k) {
      const int64_t P = by_lev[k];
      for (int ch = 0; ch < cells[P].nchild; ++ch) {
        const int64_t C = cells[P].child[ch];
        const double b[3] = {centre[3 * C] - centre[3 * P], centre[3 * C + 1] - centre[3 * P + 1],
                             centre[3 * C + 2] - centre[3 * P + 2]};
        if (cart) orc_cart_m2m(p, &MC[C * NK], b, &MC[P * NK]);
        else orc_m2m(p, &M[C * NT], b, &M[P * NT]);
      }
    }
  }
  ph_t[1] = now() - t1;

  /* (4) dual tree traversal */
  double t2 = now();
  f->ntasks = orc_traverse(cells, nc, theta, mode, cost, mask, &f->tasks);
  ph_t[2] = now() - t2;

  /* (5) execute the tasks: M2L into the target's local expansion; M2P and P2P into the target
   * particles (done per leaf below, walking the leaf's ancestors, so each particle has one
   * writer). */
  double t3 = now();
  int64_t *off[3], *idx[3];
  for (int k = 0; k < 3; ++k) group_by_target(f->tasks, f->ntasks, nc, k, &off[k], &idx[k]);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < nc; ++t)
    for (int64_t e = off[ORC_K_M2L][t]; e < off[ORC_K_M2L][t + 1]; ++e) {
      const int64_t s = f->tasks[idx[ORC_K_M2L][e]].s;
      const double d[3] = {centre[3 * t] - centre[3 * s], centre[3 * t + 1] - centre[3 * s + 1],
                           centre[3 * t + 2] - centre[3 * s + 2]};
      if (cart) orc_cart_m2l(p, &MC[s * NK], d, &LC[t * NK]);
      else orc_m2l(p, &M[s * NT], d, &Lx[t * NT]);
    }
  double *acc_phi = (double *)calloc((size_t)n, sizeof(double));
  double *acc_grad = (double *)calloc(3 * (size_t)n, sizeof(double));
#pragma omp parallel
  {
#pragma omp for schedule(dynamic, 4)
    for (int64_t leaf = 0; leaf < nc; ++leaf) {
      if (cells[leaf].nchild != 0) continue;
      if (mask && !mask[leaf]) continue;
      const int64_t b = cells[leaf].begin, cnt = cells[leaf].count;
      for (int64_t a = leaf; a >= 0; a = cells[a].parent) {
        for (int64_t e = off[ORC_K_M2P][a]; e < off[ORC_K_M2P][a + 1]; ++e) {
          const int64_t s = f->tasks[idx[ORC_K_M2P][e]].s;
          for (int64_t i = b; i < b + cnt; ++i)
            if (slot[i] >= 0)
            {
              if (cart)
                orc_cart_m2p(p, &MC[s * NK], &centre[3 * s], 1, &xs[3 * i], &acc_phi[i],
                             &acc_grad[3 * i]);
              else
                orc_m2p(p, &M[s * NT], &centre[3 * s], 1, &xs[3 * i], &acc_phi[i], &acc_grad[3 * i]);
            }
        }
        for (int64_t e = off[ORC_K_P2P][a]; e < off[ORC_K_P2P][a + 1]; ++e) {
          const int64_t s = f->tasks[idx[ORC_K_P2P][e]].s;
          for (int64_t i = b; i < b + cnt; ++i)
            if (slot[i] >= 0)
              orc_p2p(1, &xs[3 * i], cells[s].count, &xs[3 * cells[s].begin], &qs[cells[s].begin],
                      &acc_phi[i], &acc_grad[3 * i]);
        }
      }
    }
  }
  ph_t[3] = now() - t3;

  /* (6) downward sweep: L2L parent -> child, shallowest level first; L2P at leaves */
  double t4 = now();
  for (int l = 1; l <= maxlev; ++l) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t k = lev_off[l]; k < lev_off[l + 1]; ++k) {
      const int64_t C = by_lev[k], P = cells[C].parent;
      if (mask && !mask[C]) continue;
      const double e[3] = {centre[3 * C] - centre[3 * P], centre[3 * C + 1] - centre[3 * P + 1],
                           centre[3 * C + 2] - centre[3 * P + 2]};
      if (cart) orc_cart_l2l(p, &LC[P * NK], e, &LC[C * NK]);
      else orc_l2l(p, &Lx[P * NT], e, &Lx[C * NT]);
    }
  }
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t leaf = 0; leaf < nc; ++leaf) {
    if (cells[leaf].nchild != 0) continue;
    for (int64_t i = cells[leaf].begin; i < cells[leaf].begin + cells[leaf].count; ++i)
      if (slot[i] >= 0)
      {
        if (cart)
          orc_cart_l2p(p, &LC[leaf * NK], &centre[3 * leaf], 1, &xs[3 * i], &acc_phi[i],
                       &acc_grad[3 * i]);
        else
          orc_l2p(p, &Lx[leaf * NT], &centre[3 * leaf], 1, &xs[3 * i], &acc_phi[i], &acc_grad[3 * i]);
      }
  }
  ph_t[4] = now() - t4;

  /* (7) back to the caller's order */
  for (int64_t i = 0; i < n; ++i) {
    if (slot[i] < 0) continue;
    phi[slot[i]] = acc_phi[i];
    for (int a = 0; a < 3; ++a) grad[3 * slot[i] + a] = acc_grad[3 * i + a];
  }
  for (int k = 0; k < 3; ++k) {
    free(off[k]);
    free(idx[k]);
  }
  free(acc_phi);
  free(acc_grad);
  free(M);
  free(Lx);
  free(MC);
  free(LC);
  free(centre);
  free(lev_off);
  free(by_lev);
  free(mask);
  free(xs);
  free(qs);
  free(slot);
  if (phase_seconds) memcpy(phase_seconds, ph_t, sizeof ph_t);
  return f;
}

int64_t orc_fmm_ncells(const orc_fmm *f) { return f->ncells; }
int64_t orc_fmm_ntasks(const orc_fmm *f) { return f->ntasks; }

static const orc_cell *g_cells;
static int cmp_cell(const void *pa, const void *pb) {
  const orc_cell *a = &g_cells[*(const int64_t *)pa], *b = &g_cells[*(const int64_t *)pb];
  if (a->level != b->level) return a->level < b->level ? -1 : 1;
  return a->prefix < b->prefix ? -1 : (a->prefix > b->prefix);
}

/* Canonical tree dump: (level, prefix, begin, count) sorted by (level, prefix). */
void orc_fmm_tree(const orc_fmm *f, int32_t *level, uint64_t *prefix, int64_t *begin,
                  int64_t *count) {
  int64_t *order = (int64_t *)malloc(sizeof(int64_t) * ((size_t)f->ncells + 1));
  for (int64_t c = 0; c < f->ncells; ++c) order[c] = c;
  g_cells = f->cells;
  qsort(order, (size_t)f->ncells, sizeof(int64_t), cmp_cell);
  for (int64_t k = 0; k < f->ncells; ++k) {
    const orc_cell *c = &f->cells[order[k]];
    level[k] = c->level;
    prefix[k] = c->prefix;
    begin[k] = c->begin;
    count[k] = c->count;
  }
  free(order);
}

/* Task dump (unsorted; the Python side sorts canonically). */
void orc_fmm_tasks(const orc_fmm *f, int32_t *kind, int32_t *tlevel, uint64_t *tprefix,
                   int32_t *slevel, uint64_t *sprefix) {
  for (int64_t k = 0; k < f->ntasks; ++k) {
    const orc_cell *t = &f->cells[f->tasks[k].t], *s = &f->cells[f->tasks[k].s];
    kind[k] = f->tasks[k].kind;
    tlevel[k] = t->level;
    tprefix[k] = t->prefix;
    slevel[k] = s->level;
    sprefix[k] = s->prefix;
  }
}

void orc_fmm_perm(const orc_fmm *f, int64_t *perm, uint64_t *sorted_keys) {
  if (f->n == 0) return;
  memcpy(perm, f->perm, sizeof(int64_t) * (size_t)f->n);
  memcpy(sorted_keys, f->skeys, sizeof(uint64_t) * (size_t)f->n);
}

void orc_fmm_root(const orc_fmm *f, double origin[3], double *L) {
  for (int a = 0; a < 3; ++a) origin[a] = f->origin[a];
  *L = f->L;
}

void orc_fmm_free(orc_fmm *f) {
  if (!f) return;
  free(f->skeys);
  free(f->perm);
  free(f->cells);
  free(f->tasks);
  free(f);
}
