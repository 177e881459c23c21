/* fmm.h — C ABI of libfmm.so: the B200-native (sm_100a) hybrid treecode/FMM of
 * Yokota & Barba, "Hierarchical N-body simulations with auto-tuning for heterogeneous systems"
 * (arxiv 1108.5815). Citations: P:n = PAPER.md line n, S:n = SPEC.md line n (both under the
 * upstream reference); SURVEY §8 = /root/repo/SURVEY.md §8 (hot-path scope), DESIGN.md = this repo.
 *
 * What is computed ("Laplace kernel potential and force"):
 *   phi_i      = sum_{j != i, r_ij > 0} q_j / r_ij
 *   grad_phi_i = -sum_{j, r_ij > 0} q_j (x_i - x_j) / r_ij^3        (= -force of S:30)
 * approximated by the hybrid treecode/FMM of P:145-169: Morton-keyed adaptive octree with at most
 * ncrit particles per leaf, P2M/M2M upward sweep, dual tree traversal with the MAC
 * theta = (r_t + r_s)/R, per-pair choice among M2L / M2P / P2P from kernel timings
 * measured on the device, L2L/L2P downward sweep. Spherical-harmonic expansions of
 * order p, single precision on the device.
 *
 * Conventions (all entry points):
 *   - Return 0 (FMM_OK) or a negative fmm_status; nothing throws across the ABI. The message of the
 *     last failure on a handle is available from fmm_last_error().
 *   - Pointers named d_* are DEVICE pointers (cudaMalloc / torch CUDA tensors) on the handle's
 *     device; pointers named h_* are HOST pointers. The caller owns every buffer it passes; the
 *     handle owns all scratch (grow-only, reused across calls).
 *   - One handle = one CUDA device (the device current at fmm_create) and one stream; a handle is
 *     not thread-safe. Evaluations are stream-ordered and synchronous on return.
 *   - Results are written in the caller's particle order and overwrite the output buffers.
 *   - Precision: the device arithmetic is FP32. Expansion centres and particle offsets
 *     from them are formed in FP32, so a cloud whose distance from the origin is large compared
 *     with its extent loses relative accuracy (e.g. a unit-sized cloud placed at 1e4); callers
 *     should pass coordinates of the order of the cloud's own size (translate it first).
 */
#ifndef FMM_B200_H
#define FMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fmm_ctx *fmm_t;

/* Evaluation modes ("the treecode always performs cell-particle interactions, and the FMM
 * always performs cell-cell interactions, while the hybrid can choose between cell-cell,
 * cell-particle, and particle-particle interactions"). FMM_DIRECT = one all-pairs P2P. */
enum fmm_mode { FMM_HYBRID = 0, FMM_FMM = 1, FMM_TREECODE = 2, FMM_DIRECT = 3 };

/* Interaction kinds in exported lists. */
enum fmm_kind { FMM_KIND_M2L = 0, FMM_KIND_M2P = 1, FMM_KIND_P2P = 2 };
/* expansion basis (fmm_set_basis): spherical harmonics (default), Cartesian Taylor of total order
 * p (p <= 4), or the automatic switch between them */
enum fmm_basis { FMM_BASIS_SPHERICAL = 0, FMM_BASIS_CARTESIAN = 1, FMM_BASIS_AUTO = 2 };
/* M2L translation scheme (fmm_set_m2l_scheme) */
enum fmm_m2l_scheme { FMM_M2L_AUTO = 0, FMM_M2L_TC = 1, FMM_M2L_GEMM = 2, FMM_M2L_ROTATION = 3,
                      FMM_M2L_PAIRS = 4 };

enum fmm_status {
  FMM_OK = 0,
  FMM_E_INVALID = -1,    /* p not in [1, FMM_P_MAX], theta not in (0,1), ncrit < 1, n < 0, NULL */
  FMM_E_NOT_DEVICE = -2, /* a d_* pointer is not device memory of the handle's device */
  FMM_E_NONFINITE = -3,  /* a coordinate or charge is not finite; outputs untouched */
  FMM_E_CUDA = -4,       /* CUDA runtime / kernel failure */
  FMM_E_OOM = -5,        /* device allocation failed */
  FMM_E_NCCL = -6,       /* NCCL (or in-process group) collective failure, multi-GPU handles */
  FMM_E_STATE = -7       /* export called before any evaluation */
};

#define FMM_P_MAX 16 /* P:205 goes to p = 15; FP32 scaled I_n^m up to degree 2p stays finite */

/* Kernel pre-calculation result ("All kernels are evaluated using artificial coordinates,
 * mass/charges, multipole coefficients, and their execution time is measured"). Linear per-unit
 * cost model: P2P = t_pp * n_t * n_s, M2P = t_mp * n_t, M2L = t_ml; argmin with ties
 * M2L > M2P > P2P. */
typedef struct {
  double t_pp;  /* seconds per particle pair (P2P) */
  double t_mp;  /* seconds per target particle per source cell (M2P) */
  double t_ml;  /* seconds per cell-cell translation (M2L) */
  int p;        /* expansion order the timings belong to */
  int measured; /* 1 = measured on this device by fmm_create/fmm_tune, 0 = set by the caller */
} fmm_cost_t;

/* Counters and per-phase device times of the last evaluation (S:141-144 KernelCounters; SURVEY
 * §5 tracing). Times are CUDA-event milliseconds on the handle's stream, filled only when timing
 * is enabled with fmm_set_timing(h, 1). */
typedef struct {
  int64_t n, ncells, nleaves;
  int32_t depth, p;
  int64_t n_m2l, n_m2p, n_p2p;      /* cell pairs per kind */
  int64_t p2p_pairs, m2p_evals;     /* particle pairs in P2P; target-particle x source-cell in M2P */
  int64_t traversal_pairs;          /* MAC tests performed */
  double ms_total, ms_tree, ms_upward, ms_traverse, ms_m2l, ms_p2p, ms_m2p, ms_downward;
  int64_t launches;                 /* libfmm kernels launched by the evaluation (CUB's excluded) */
  int64_t cub_calls;                /* CUB radix-sort / scan calls (library kernels) */
  /* multi-GPU handles (fmm_create_dist / fmm_create_in_group); zero otherwise */
  int64_t n_global;                 /* particles over all ranks */
  int64_t rank_lo, rank_hi;         /* this rank's targets: global Morton-order range [lo, hi) */
  int64_t n_straddle;               /* cells whose particles span ranks (multipoles allreduced) */
  int64_t let_cells, let_particles; /* remote multipoles / particles received (local essential tree) */
  int64_t bytes_sent;               /* bytes this rank sent in all exchanges of the evaluation */
  double ms_comm;                   /* host wall time inside collectives (includes waiting) */
  /* sender-side local essential tree (default on distributed handles; timing enabled): device
   * time of the exchange on its own stream, and how far it ran past the end of the traversal it
   * overlaps (0 = hidden; the near field and M2L wait for it) */
  double ms_let, ms_let_exposed;
  /* the P2P kernel alone (ms_p2p also covers its per-leaf descriptor and range-merge passes) */
  double ms_p2p_kernel;
} fmm_stats_t;

/* Create a handle on the current CUDA device. p = expansion order (coefficients n = 0..p,
 * SURVEY §8(c) reading 2), theta = MAC, ncrit = max particles per leaf.
 * Runs the kernel pre-calculation unless FMM_NO_TUNE is set in the environment.
 * Errors: FMM_E_INVALID, FMM_E_CUDA, FMM_E_OOM. */
int fmm_create(fmm_t *out, int p, double theta, int ncrit);

/* Release the handle and all device scratch. NULL-safe. */
int fmm_destroy(fmm_t h);

/* Evaluate potential and gradient for n particles.
 *   d_xyz  [3n] float, AoS (x0,y0,z0,x1,...)     d_q [n] float
 *   d_phi  [n]  float (out)                       d_grad [3n] float, AoS (out)
 * Ordering: the work runs on the handle's internal streams, after everything already queued on
 * the handle's stream (fmm_set_stream), and that stream waits for the results; the call also
 * returns only when they are complete. n = 0 is a successful no-op (on a distributed handle it
 * still takes part in the collective). Errors: FMM_E_INVALID, FMM_E_NOT_DEVICE, FMM_E_NONFINITE
 * (outputs untouched), FMM_E_CUDA, FMM_E_OOM, FMM_E_NCCL. */
int fmm_evaluate(fmm_t h, const float *d_xyz, const float *d_q, int64_t n, float *d_phi,
                 float *d_grad);

/* Distinct target and source sets (the dual tree traversal pairs target cells with
 * source cells): phi / grad at the n_t target points d_xyz_t [3 n_t] due to the n_s charges
 * d_q_s [n_s] at d_xyz_s [3 n_s] (all device, AoS as in fmm_evaluate). One octree is built over
 * the union (targets carry zero charge, so they are not sources); only cells holding targets are
 * traversed as targets and only leaves holding targets are evaluated. A target coincident with a
 * source gets no contribution from it (r = 0 rule). Outputs are written for the n_t targets in
 * their order. n_s = 0 gives zero fields. Not available on distributed handles or in FMM_DIRECT
 * mode. Errors: as fmm_evaluate. */
int fmm_evaluate_ts(fmm_t h, const float *d_xyz_t, int64_t n_t, const float *d_xyz_s,
                    const float *d_q_s, int64_t n_s, float *d_phi_t, float *d_grad_t);

/* Same with HOST buffers (pinned or pageable): copies in, evaluates, copies out (end-to-end path). */
int fmm_evaluate_host(fmm_t h, const float *h_xyz, const float *h_q, int64_t n, float *h_phi,
                      float *h_grad);

/* The stream the evaluations are ordered with (a cudaStream_t passed as void*); NULL restores the
 * handle's own. See fmm_evaluate for the ordering guarantees. */
int fmm_set_stream(fmm_t h, void *stream);
int fmm_set_mode(fmm_t h, int mode);
/* 1 = record per-phase CUDA events (small overhead), 0 = off (default). */
int fmm_set_timing(fmm_t h, int enable);
/* 1 (default) = bit-reproducible results: every target's M2L results are summed in its
 * interaction-list order (per-pair slots in HBM + one reduction pass). 0 = the tensor-core M2L adds
 * each pair's local expansion straight into its target with vector reductions in L2: faster, but
 * the summation order then varies from run to run (differences at FP32 rounding level). */
int fmm_set_deterministic(fmm_t h, int enable);

/* M2L translation scheme, spherical basis (PAPER.md:122, P:153, P:169 name
 * the choice of translation scheme, P:205 the O(p^4) kernel). Every scheme computes the same
 * operator (up to rounding):
 *   FMM_M2L_TC        class-batched dense translation matrices on the tcgen05 tensor cores
 *                     (3xTF32), p <= 10;
 *   FMM_M2L_GEMM      the same class GEMM on CUDA cores, p <= 12;
 *   FMM_M2L_ROTATION  rotation-based O(p^3): per class, rotate the multipole onto the z axis,
 *                     translate along z, rotate back (m2l_rot.cu), any p;
 *   FMM_M2L_PAIRS     the direct per-pair double loop, any p.
 * FMM_M2L_AUTO (default): fmm_tune / fmm_create's kernel pre-calculation times the M2L phase of
 * one FMM-mode evaluation of the synthetic set with every scheme available at this p and keeps
 * the fastest (before it: TC, else GEMM, else ROTATION). Errors: FMM_E_INVALID (not available at
 * this p). */
int fmm_set_m2l_scheme(fmm_t h, int scheme);
/* The scheme evaluations use; tuned_ms[FMM_M2L_*] (5 doubles, may be NULL) = the M2L times the
 * last tuning measured (0 = not run). */
int fmm_get_m2l_scheme(fmm_t h, int *scheme, double *tuned_ms);

/* Expansion basis ("capability to switch to Cartesian expansions
 * ... key to achieving high performance for low-accuracy").
 *   FMM_BASIS_SPHERICAL  solid harmonics of order p (the default; every p).
 *   FMM_BASIS_CARTESIAN  Cartesian Taylor expansions of total order p (reading R17:
 *                        multipole moments sum q (y-c)^k, |k| <= p; M2L truncated at
 *                        |k| + |n| <= p), for 1 <= p <= 4 on single-GPU handles; the cell-cell
 *                        M2L runs on CUDA cores, one warp per target cell.
 *   FMM_BASIS_AUTO       the automatic switch: for p <= 4 each basis gets its kernel
 *                        pre-calculation and one hybrid evaluation of 2^20 synthetic particles is
 *                        timed; the faster basis is kept (spherical for p > 4 or distributed
 *                        handles). Synchronous; takes about a second.
 * Switching basis re-runs the kernel pre-calculation when the cost model was measured.
 * Errors: FMM_E_INVALID (unknown basis, Cartesian with p > 4 or on a distributed handle). */
int fmm_set_basis(fmm_t h, int basis);
/* The basis in use; after FMM_BASIS_AUTO the two measured evaluation times (ms, else 0). */
int fmm_get_basis(fmm_t h, int *basis, double *ms_spherical, double *ms_cartesian);

/* Re-run the kernel pre-calculation on this device (a single-GPU run on synthetic data).
 * On a distributed handle it is collective and every rank then holds rank 0's table. */
int fmm_tune(fmm_t h);
int fmm_get_cost_model(fmm_t h, fmm_cost_t *out);
/* Pin the cost model (reproducible lists; the oracle imports the same numbers). in->p must equal
 * the handle's p. On distributed handles every rank must pin the same table. */
int fmm_set_cost_model(fmm_t h, const fmm_cost_t *in);
int fmm_get_stats(fmm_t h, fmm_stats_t *out);

/* Canonical exports of the last evaluation (host buffers, caller-allocated with `cap` entries;
 * the required count is always written to *count_out, and FMM_E_INVALID is returned when cap is
 * too small). Tree: cells in (level, prefix) order. Lists: one row per interaction pair, grouped
 * by target cell. Perm: h_perm[i] = caller index of the i-th particle in Morton order; h_keys[i]
 * its 63-bit key. Errors: FMM_E_STATE before the first tree evaluation. */
int fmm_export_tree(fmm_t h, int64_t cap, int32_t *h_level, uint64_t *h_prefix, int64_t *h_begin,
                    int64_t *h_count, int64_t *count_out);
int fmm_export_lists(fmm_t h, int64_t cap, int32_t *h_kind, int32_t *h_tlevel, uint64_t *h_tprefix,
                     int32_t *h_slevel, uint64_t *h_sprefix, int64_t *count_out);
int fmm_export_perm(fmm_t h, int64_t cap, int64_t *h_perm, uint64_t *h_keys, double *h_origin3,
                    double *h_L);

/* Multi-GPU building block (PAPER.md:89 spatial domain decomposition). With a
 * partition set, fmm_evaluate builds the tree and the upward sweep over all n particles it is
 * given but evaluates only the targets of Morton part `part` of `nparts`: the leaves whose first
 * sorted particle index b satisfies floor(b * nparts / n) == part. Only those particles' entries of
 * d_phi / d_grad are written. fmm_get_partition returns that part's sorted-order particle range
 * [lo, hi) of the last evaluation; fmm_partition_indices writes the caller indices of those
 * particles (int64, DEVICE buffer d_out of cap entries) so results can be routed to their owners.
 * nparts = 1 (default) restores whole evaluation. Errors: FMM_E_INVALID, FMM_E_STATE. */
int fmm_set_partition(fmm_t h, int nparts, int part);
int fmm_get_partition(fmm_t h, int64_t *lo, int64_t *hi);
int fmm_partition_indices(fmm_t h, int64_t *d_out, int64_t cap, int64_t *count_out);

/* ---- Multi-GPU: one handle per rank, one rank per GPU ----
 * A distributed handle takes the rank's own particle shard in fmm_evaluate (any size, any subset;
 * n may be 0 on some ranks) and returns phi / grad for exactly those particles in the caller's
 * order. fmm_evaluate is then COLLECTIVE: every rank of the group must call it (same mode and
 * cost model; the cost model measured by rank 0 is broadcast at creation so that the per-pair
 * kind choice, and hence the union of the lists, equals a single-GPU evaluation of the union).
 * The method inside: global bbox (allreduce) -> local keys + sort -> the global
 * adaptive octree built level by level from allreduced split bounds (no particle moves) -> ranks
 * own contiguous Morton runs of whole leaves, balanced by count -> particle alltoallv -> P2M/M2M,
 * allreduce of the multipoles of cells that straddle ranks -> traversal of the own targets ->
 * receiver-driven local essential tree: the remote multipoles and particle ranges the lists name
 * are requested and received (alltoallv) -> M2L / P2P / M2P / L2L / L2P -> results sent back to
 * the ranks that own the particles. FMM_DIRECT is not available on distributed handles.
 * Global particle count < 2^30. Errors: FMM_E_INVALID, FMM_E_NCCL, plus those of fmm_create.
 *
 * fmm_comm_unique_id: NCCL unique id (rank 0 creates it, the caller broadcasts the 128 bytes,
 *   e.g. with torch.distributed). NCCL is loaded at run time (dlopen libnccl.so.2).
 * fmm_create_dist: handle on the current CUDA device joined to an NCCL communicator of nranks.
 * fmm_group_create / fmm_create_in_group: an IN-PROCESS group of nranks handles (one host thread
 *   per handle; the handles may share one GPU). Collectives are device copies between barriers;
 *   the distributed algorithm is the same as over NCCL (used to test it on one GPU). The group
 *   must outlive its handles; at most 16 ranks. */
typedef struct fmm_group *fmm_group_t;
int fmm_comm_unique_id(unsigned char h_id[128]);
int fmm_create_dist(fmm_t *out, int p, double theta, int ncrit, int nranks, int rank,
                    const unsigned char h_id[128]);
int fmm_group_create(fmm_group_t *out, int nranks);
int fmm_group_destroy(fmm_group_t g);
int fmm_create_in_group(fmm_t *out, int p, double theta, int ncrit, fmm_group_t g, int rank);

const char *fmm_strerror(int code);
const char *fmm_last_error(fmm_t h);

#ifdef __cplusplus
}
#endif
#endif
