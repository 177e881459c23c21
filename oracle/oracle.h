/* oracle.h — CPU FP64 ORACLE of the hybrid treecode/FMM (Yokota & Barba, arxiv 1108.5815).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. It shares no source, header, table or helper with
 * the CUDA path (paper_1108_5815_b200/csrc); neither side includes or links the other.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n; SURVEY §8(c) cN = the
 * oracle readings c1..c7 listed in SURVEY.md §8(c) and restated in DESIGN.md §3.
 *
 * Storage convention (plain, not optimised): an expansion of order p holds (p+1)^2 complex
 * coefficients, every degree n = 0..p and every SIGNED order m = -n..n, at index n*n + n + m.
 * Expansions are the classical unscaled ones: R_n^m = r^n P_n^m(cos t) e^{im f}/(n+m)!,
 * I_n^m = (n-m)! P_n^m(cos t) e^{im f} / r^{n+1}, Condon-Shortley phase.
 */
#ifndef FMM_ORACLE_H
#define FMM_ORACLE_H
#include <complex.h>
#include <stdint.h>

typedef double complex cplx;

#define ORC_IDX(n, m) ((n) * (n) + (n) + (m))
#define ORC_LEVELS 21 /* 21 key bits per axis, 63-bit Morton keys */

enum { ORC_HYBRID = 0, ORC_FMM = 1, ORC_TREECODE = 2, ORC_DIRECT = 3 };
enum { ORC_K_M2L = 0, ORC_K_M2P = 1, ORC_K_P2P = 2 };
enum { ORC_SPHERICAL = 0, ORC_CARTESIAN = 1 };

/* ---- harmonics.c: solid harmonics and the seven operators ---- */
void orc_harm_R(const double x[3], int P, cplx *R);
void orc_harm_I(const double x[3], int P, cplx *Iv);
void orc_p2m(int p, const double c[3], int64_t n, const double *y, const double *q, cplx *M);
void orc_m2m(int p, const cplx *Mc, const double b[3], cplx *Mp);
void orc_m2l(int p, const cplx *Ms, const double d[3], cplx *Lt);
void orc_l2l(int p, const cplx *Lp, const double e[3], cplx *Lc);
void orc_l2p(int p, const cplx *L, const double c[3], int64_t n, const double *x, double *phi,
             double *grad);
void orc_m2p(int p, const cplx *M, const double c[3], int64_t n, const double *x, double *phi,
             double *grad);
void orc_p2p(int64_t nt, const double *xt, int64_t ns, const double *ys, const double *qs,
             double *phi, double *grad);

/* ---- cartesian.c: Cartesian Taylor expansions of total order p (NEXT-2; DESIGN reading R17) ----
 * Real coefficients, one per multi-index k with |k| <= p, indexed by orc_cart_index. */
int orc_cart_count(int P);
int orc_cart_index(int kx, int ky, int kz);
void orc_cart_multi(int P, int *k3);
void orc_cart_derivs(const double d[3], int P, double *a);
void orc_cart_p2m(int p, const double c[3], int64_t n, const double *y, const double *q, double *M);
void orc_cart_m2m(int p, const double *Mc, const double b[3], double *Mp);
void orc_cart_m2l(int p, const double *Ms, const double d[3], double *Lt);
void orc_cart_l2l(int p, const double *Lp, const double e[3], double *Lc);
void orc_cart_l2p(int p, const double *L, const double c[3], int64_t n, const double *x,
                  double *phi, double *grad);
void orc_cart_m2p(int p, const double *M, const double c[3], int64_t n, const double *x,
                  double *phi, double *grad);

/* ---- tree.c: root cube, Morton keys, sort, adaptive octree ---- */
typedef struct {
  int level;
  uint64_t prefix;   /* key >> 3*(21-level) */
  int64_t begin;     /* first particle (sorted order) */
  int64_t count;     /* particles in the cell */
  int64_t parent;    /* -1 for the root */
  int64_t child[8];  /* non-empty children in Morton order */
  int nchild;        /* 0 => leaf */
} orc_cell;

int orc_root_cube(const float *xyz, int64_t n, double origin[3], double *L);
void orc_morton_keys(const float *xyz, int64_t n, const double origin[3], double L,
                     uint64_t *keys);
void orc_sort_keys(const uint64_t *keys, int64_t n, int64_t *perm);
int64_t orc_build_tree(const uint64_t *sorted_keys, int64_t n, int ncrit, orc_cell **cells_out);
void orc_cell_geometry(const orc_cell *c, const double origin[3], double L, double centre[3],
                       double *radius);

/* ---- traversal.c: MAC, kind selection and the LIFO dual-tree traversal ---- */
typedef struct {
  int kind;
  int64_t t, s; /* cell ids */
} orc_task;

int orc_mac_accept(const orc_cell *t, const orc_cell *s, double theta);
int orc_select_kind(int mode, const double cost[3], int64_t nt, int64_t ns);
int64_t orc_traverse(const orc_cell *cells, int64_t ncells, double theta, int mode,
                     const double cost[3], const unsigned char *target_mask, orc_task **tasks_out);

/* ---- evaluate.c: the whole method + direct sum ---- */
typedef struct orc_fmm orc_fmm;
orc_fmm *orc_fmm_run(const float *xyz, const float *q, int64_t n, int p, double theta, int ncrit,
                     int mode, const double cost[3], const int64_t *sample, int64_t nsample,
                     double *phi, double *grad, double *phase_seconds);
orc_fmm *orc_fmm_run_basis(const float *xyz, const float *q, int64_t n, int p, double theta,
                           int ncrit, int mode, const double cost[3], const int64_t *sample,
                           int64_t nsample, double *phi, double *grad, double *phase_seconds,
                           int basis);
int64_t orc_fmm_ncells(const orc_fmm *f);
void orc_fmm_tree(const orc_fmm *f, int32_t *level, uint64_t *prefix, int64_t *begin,
                  int64_t *count);
int64_t orc_fmm_ntasks(const orc_fmm *f);
void orc_fmm_tasks(const orc_fmm *f, int32_t *kind, int32_t *tlevel, uint64_t *tprefix,
                   int32_t *slevel, uint64_t *sprefix);
void orc_fmm_perm(const orc_fmm *f, int64_t *perm, uint64_t *sorted_keys);
void orc_fmm_root(const orc_fmm *f, double origin[3], double *L);
void orc_fmm_free(orc_fmm *f);
void orc_direct(const float *xyz, const float *q, int64_t n, const int64_t *targets,
                int64_t ntargets, double *phi, double *grad);

#endif
