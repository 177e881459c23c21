// kernels.cuh — host-side launcher declarations of the sm_100a kernels (internal to libfmm.so).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

// ---- tree.cu ----
void launch_bbox(const float *xyz, const float *q, int64_t n, unsigned *mm, RootInfo *root,
                 cudaStream_t st);
void launch_keys(const float *xyz, int64_t n, const RootInfo *root, uint64_t *keys, unsigned *idx,
                 cudaStream_t st);
void launch_gather(const float *xyz, const float *q, const unsigned *perm, int64_t n, float4 *pos,
                   cudaStream_t st);
int sort_runs_cap(int64_t n);  // entries of the long-run scratch sort_keys_short needs
cudaError_t sort_keys_short(void *tmp, size_t &tmp_bytes, const uint64_t *kin, uint64_t *kout,
                            const unsigned *vin, unsigned *vout, int64_t n, int *flag, int2 *runs,
                            int low_bits, cudaStream_t st);
int tree_coop_grid();
cudaError_t launch_tree_coop(const uint64_t *keys, int n, int ncrit, const RootInfo *root,
                             CellsView C, uint64_t *prefix, int cap, int *bnd, int *nch,
                             int2 *crange, int *blk, int *st_dev, int *leaves, int grid,
                             cudaStream_t st);
cudaError_t sort_keys(void *tmp, size_t &tmp_bytes, const uint64_t *kin, uint64_t *kout,
                      const unsigned *vin, unsigned *vout, int64_t n, cudaStream_t st);
cudaError_t exclusive_scan(void *tmp, size_t &tmp_bytes, const int *in, int *out, int n,
                           cudaStream_t st);
void launch_root_cell(int64_t n, const RootInfo *root, CellsView C, uint64_t *prefix,
                      cudaStream_t st);
void launch_split(int c0, int nl, int level, int ncrit, const uint64_t *keys, CellsView C,
                  const uint64_t *prefix, int *nch, int2 *crange, int *bnd, cudaStream_t st);
void launch_split_bounds(int c0, int nl, int level, int ncrit, const uint64_t *keys, int nloc,
                         CellsView C, const uint64_t *prefix, int *bnd, cudaStream_t st);
void launch_split_ranges(int c0, int nl, int level, int ncrit, CellsView C, const int *bnd,
                         int *nch, int2 *crange, cudaStream_t st);
void launch_bbox_local(const float *xyz, const float *q, int64_t n, unsigned *mm, RootInfo *root,
                       cudaStream_t st);
void launch_root_from_mm(const unsigned *mm, RootInfo *root, cudaStream_t st);
void launch_emit(int c0, int nl, int next0, int level, const int *nch, const int *excl,
                 const int2 *crange, const RootInfo *root, CellsView C, uint64_t *prefix,
                 cudaStream_t st);
void launch_level_total(const int *nch, const int *excl, int nl, int *total, cudaStream_t st);
void launch_leaf_flags(int ncells, const int *nchild, int *flag, cudaStream_t st);
void launch_part_flags(int ncells, CellsView C, int64_t n, int nparts, int part, int *flag,
                       int *lohi, cudaStream_t st);
void launch_part_indices(int lo, int cnt, const unsigned *perm, int64_t *out, cudaStream_t st);
void launch_leaf_scatter(int ncells, const int *flag, const int *excl, int *leaves,
                         cudaStream_t st);
// distinct target / source sets: flag[i] = (perm[i] < nt) over sorted particles; per cell target
// counts from the exclusive scan of the flags; leaf flags of the leaves holding targets
void launch_target_flags(const unsigned *perm, int n, int nt, int *flag, cudaStream_t st);
void launch_cell_targets(int ncells, CellsView C, const int *excl, const int *flag, int n,
                         int *ntgt, int *leafflag, cudaStream_t st);

// ---- traverse.cu ----
// the four list counters of the traversal, one per 128-byte line (every target does one atomic
// on each: on a shared line they would serialise in one L2 slice)
#define TRAV_CNT(c) (32 + 32 * (c))
#define TRAV_BK_INTS 160
struct TravArgs {
  CellsView C;
  const int4 *pk;  // packed cell records (k_pack_cells): [2c] = grid, [2c+1] = beg, cnt, child0, nchild
  int t0, nt, level, mode, stack_cap, grid_blocks;
  int tlo, thi;  // targets restricted to cells intersecting sorted particle range [tlo, thi)
  const int *tmask;  // or null: per cell, number of target particles (0: not a target cell)
  double theta, t_pp, t_mp, t_ml;
  const unsigned *in_src;
  const int *in_off, *in_cnt;
  unsigned *scratch, *overflow;  // per-warp stack; overflow bits: 1 stack, 2 list scratch
  unsigned *oscratch;            // per-warp [4][ocap] lists of the current target
  int2 *rscratch;                // per-warp [ocap] P2P source ranges
  int ocap;
  // device-resident bookkeeping (no host round trip per level): [8..11] capacities of the three
  // lists and of the deferred-pair buffer, [12] overflow flag, [TRAV_CNT(0..2)] running list
  // sizes, [TRAV_CNT(3)] this level's deferred pairs (reset per level)
  int *bk;
  unsigned *lsrc[3];
  int *loff[3], *lcnt[3];
  unsigned *out_src;
  int *out_off, *out_cnt;
  int2 *p2p_rng;  // (begin, count) of each P2P source cell, parallel to lsrc[2]
  unsigned long long *stats;  // [0] P2P particle pairs, [1] M2P target evaluations
};
void launch_traverse(const TravArgs &A, cudaStream_t st);
void launch_pack_cells(int ncells, CellsView C, int4 *pk, cudaStream_t st);

// ---- expansions.cu ----
struct M2LTiles {
  int ntiles;
  int tile[64];  // j | k0 << 8 | K << 16
};
void launch_p2m(int p, const int *leaves, int nleaves, CellsView C, const float4 *pos, float2 *M,
                cudaStream_t st);
void launch_m2m(int p, int c0, int nl, CellsView C, float2 *M, cudaStream_t st);
void launch_l2l(int p, int c0, int nl, CellsView C, float2 *L, cudaStream_t st);
void launch_m2p(int p, const int *leaves, int nleaves, CellsView C, ListsView Ls,
                const float4 *pos, const float2 *M, float4 *acc, int *counter, cudaStream_t st);
void launch_l2p(int p, const int *leaves, int nleaves, CellsView C, const float4 *pos,
                const float2 *L, const float4 *acc, const unsigned *perm, float *phi, float *grad,
                int use_local, cudaStream_t st);
M2LTiles make_m2l_tiles(int p);

// ---- m2l.cu ----
struct M2LWork {
  CellsView C;
  const int *off, *cnt;     // per target cell: M2L list segment
  const unsigned *src;      // source cell of each pair
  int *pair_t;              // target cell of each pair
  uint2 *pst;               // (source, target) of each pair, list order
  uint2 *spst;              // accumulate mode: the same records in class-sorted order (else null;
                            // class_rep and the direct-path list then hold sorted positions)
  unsigned *keys_in, *keys;  // 24-bit class keys
  unsigned *idx_in, *sidx;  // pair indices sorted by class key
  unsigned *ssrc;           // source cell of each class-sorted pair
  unsigned *stgt;           // target cell of each class-sorted pair (accumulate mode), or null
  int *flag, *cid, *cstart, *counters;
  int4 *items;              // GEMM work items (first sorted position, count, representative pair)
  unsigned *small;          // pairs on the direct path
  unsigned *class_rep;      // representative pair of every GEMM class
  float *Tg;                // translation matrices of the GEMM classes [ngclass][m2l_T_floats(p)]
  float *Y;                 // per-pair results [npairs][m2l_y_stride(p)]
  void *tmp;
  size_t tmp_bytes;
  int direct_all;           // 1: every pair on the direct path (p > 12)
  // block-major execution order (m2l_sort_items): runs of a class split at target blocks
  int blk_level;            // Morton level of the spatial blocks (0: one block)
  int compact_key;          // 21-bit class keys (counters[6] reports pairs they cannot hold)
  int *rflag, *rid, *rstart, *gid_of;
  int4 *items_raw;          // items as emitted (unordered); `items` = block-major order
  unsigned *ikeys_in, *ikeys, *iidx_in, *iidx;
};
size_t m2l_gemm_smem(int p);
bool m2l_gemm_supported(int p);
int m2l_y_stride(int p);
size_t m2l_temp_bytes(int npairs);
cudaError_t m2l_prepare(const M2LWork &W, int npairs, int ncells, cudaStream_t st);
cudaError_t m2l_sort_items(const M2LWork &W, int nitems, cudaStream_t st);
size_t m2l_T_floats(int p);
cudaError_t m2l_build_T(int p, const M2LWork &W, int ngclass, cudaStream_t st);
cudaError_t m2l_execute(int p, const M2LWork &W, int npairs, int ncells, const float2 *M,
                        float2 *L, cudaStream_t st, bool gemm_done = false, bool accum = false,
                        int ydof = -1);  // Y rows in dof order (-1: when gemm_done)

// ---- m2l_rot.cu (rotation-based O(p^3) M2L, NEXT-1) ----
bool m2l_rot_supported(int p);
size_t m2l_rot_class_floats(int p);
cudaError_t m2l_rot_build(int p, const M2LWork &W, int ngclass, float *R, cudaStream_t st);
cudaError_t m2l_rot_apply(int p, const M2LWork &W, const float *R, const float2 *M,
                          cudaStream_t st, float2 *Lacc);

// ---- m2l_tc.cu (tcgen05 3xTF32 class GEMM) ----
bool m2l_tc_supported(int p);
// K-tiled tcgen05 class GEMM for 10 < p <= 15 (float-order rows, Y in float order)
bool m2l_tck_supported(int p);
size_t m2l_tck_T_words(int p);
cudaError_t m2l_tck_build_T(int p, const M2LWork &W, int ngclass, unsigned *Timg, cudaStream_t st);
cudaError_t m2l_tck_gemm(int p, const M2LWork &W, const unsigned *Timg, const float2 *M,
                         cudaStream_t st, float2 *Lacc);
size_t m2l_tc_T_words(int p);
cudaError_t m2l_tc_build_T(int p, const M2LWork &W, int ngclass, unsigned *Timg, cudaStream_t st);
cudaError_t m2l_tc_gemm(int p, const M2LWork &W, const unsigned *Timg, const float2 *M,
                        cudaStream_t st, float2 *Lacc = nullptr);

struct TcShiftWork {
  unsigned *keys_in, *keys, *vals_in, *cells;  // (level<<3 | octant) sort of all non-root cells
  unsigned *src_l2l;                           // per sorted position: L2L source (the parent)
  int4 *items;                                 // [level][items_per_level]
  int *lvl_counters;                           // [level][8]: [1] = #items, [4] = queue
  int items_per_level;
  unsigned *Tm2m, *Tl2l;                       // 8 octant operators each (tf32 hi/lo images)
  void *tmp;
  size_t tmp_bytes;
};
cudaError_t tc_class_gemm(int p, const int4 *items, const int *counters, int *queue,
                          const unsigned *sidx, const unsigned *ssrc, const unsigned *Timg,
                          const float2 *M, float *Y, int grid, cudaStream_t st,
                          float *Lacc = nullptr);
cudaError_t tc_shift_build_ops(int p, unsigned *Tm2m, unsigned *Tl2l, cudaStream_t st);
int tc_shift_items_per_level(int ncells);  // work-item capacity per level of the shift GEMMs
size_t tc_shift_sort_bytes(int ncells);
cudaError_t tc_shift_prepare(int ncells, int depth, const TcShiftWork &S, CellsView C,
                             cudaStream_t st);
cudaError_t tc_shift_m2m_level(int p, int level, int c0, int nl, CellsView C,
                               const TcShiftWork &S, float2 *M, float *Y, cudaStream_t st);
cudaError_t tc_shift_l2l_level(int p, int level, int c0, int nl, const TcShiftWork &S, float2 *L,
                               float *Y, cudaStream_t st);

// ---- cart.cu (Cartesian Taylor expansions, NEXT-2) ----
#define CART_PMAX 4
bool cart_supported(int p);
int cart_stride(int p);
int cart_count(int p);
void launch_cart_p2m(int p, const int *leaves, int nleaves, CellsView C, const float4 *pos,
                     float *M, cudaStream_t st);
void launch_cart_m2m(int p, int c0, int nl, CellsView C, float *M, cudaStream_t st);
void launch_cart_m2l(int p, int ncells, CellsView C, ListsView Ls, const float *M, float *L,
                     cudaStream_t st);
void launch_cart_l2l(int p, int c0, int nl, CellsView C, float *L, cudaStream_t st);
void launch_cart_l2p(int p, const int *leaves, int nleaves, CellsView C, const float4 *pos,
                     const float *L, const float4 *acc, const unsigned *perm, float *phi,
                     float *grad, int use_local, cudaStream_t st);
void launch_cart_m2p(int p, const int *leaves, int nleaves, CellsView C, ListsView Ls,
                     const float4 *pos, const float *M, float4 *acc, int *counter,
                     cudaStream_t st);

// ---- p2p.cu ----
// desc: scratch of nleaves int4 (per-leaf work descriptors built by the launch); mrg: scratch
// parallel to the P2P lists (their capacity) for the merged per-leaf source ranges
void launch_p2p_leaves(const int *leaves, int nleaves, CellsView C, ListsView Ls,
                       const float4 *pos, float4 *acc, int *counter, int4 *desc, int2 *mrg,
                       cudaStream_t st, cudaEvent_t ev_main = nullptr);
void launch_p2p_direct(int64_t n, const float4 *pos, float *phi, float *grad, cudaStream_t st);

// ---- synthetic batches for the kernel pre-calculation (autotune.cu) ----
void launch_fill_random(float *dst, int64_t n, unsigned seed, float lo, float hi,
                        cudaStream_t st);

// ---- dist.cu (multi-GPU evaluation) ----
void launch_iota(unsigned *a, int n, cudaStream_t st);
void launch_gather4(const float4 *src, const unsigned *perm, int n, float4 *dst, cudaStream_t st);
void launch_partition(const int *leaves, int nleaves, CellsView C, const uint64_t *prefix, int N,
                      int R, int *off, uint64_t *K, cudaStream_t st);
void launch_key_bounds(const uint64_t *keys, int n, const uint64_t *K, int R, int *lb,
                       cudaStream_t st);
void launch_range_leaf_flags(int ncells, CellsView C, int lo, int hi, int *flag, cudaStream_t st);
void launch_straddle_flags(int ncells, CellsView C, const int *off, int R, int *flag,
                           cudaStream_t st);
void launch_rows(const float2 *src, float2 *dst, int stride, const unsigned *ids, int n,
                 bool to_ids, cudaStream_t st);
void launch_need_flags(ListsView Ls, int n_m2l, int n_m2p, int n_p2p, CellsView C,
                       const int *strad, int lo, int hi, int *needM, int *needP, cudaStream_t st);
void launch_owner_of_cells(const unsigned *ids, int n, CellsView C, const int *off, int R,
                           unsigned *owner, cudaStream_t st);
void launch_piece_count(const unsigned *ids, int n, CellsView C, const int *off, int R, int me,
                        int *cnt, cudaStream_t st);
void launch_piece_write(const unsigned *ids, int n, CellsView C, const int *off, int R, int me,
                        const int *excl, unsigned *owner, unsigned *pidx, int2 *rng,
                        cudaStream_t st);
void launch_gather_int2(const int2 *src, const unsigned *idx, int n, int2 *dst, int *size,
                        cudaStream_t st);
void launch_range_sizes(const int2 *rng, int n, int *size, cudaStream_t st);
void launch_owner_hist(const unsigned *owner, int n, int *counts, cudaStream_t st);
void launch_range_copy(float4 *pos, const int2 *rng, const int *roff, int n, float4 *buf,
                       bool to_pos, cudaStream_t st);
void launch_scatter_results(const float *rphi, const float *rgrad, const unsigned *perm, int n,
                            float *phi, float *grad, cudaStream_t st);
// sender-side local essential tree (dist.cu)
int let_box_ints(int R);
void launch_let_boxes(const int *leaves, int nleaves, int ncells, CellsView C, const int *off,
                      int R, int kmax, int *box, cudaStream_t st);
void launch_let_flags(int ncells, CellsView C, const int *box, const int *off, int R, int me,
                      double theta, double t_pp, double t_mp, double t_ml, unsigned *open,
                      unsigned *near, int *flags, cudaStream_t st);
void launch_seg_counts(const int *flags, const int *excl, int nseg, int nc, int *cnt,
                       cudaStream_t st);
void launch_seg_scatter(const int *flags, const int *excl, int64_t n, int nc, unsigned *ids,
                        cudaStream_t st);
void launch_let_prange(const unsigned *ids, int n, CellsView C, int lo, int hi, int2 *rng,
                       int *size, cudaStream_t st);
void launch_let_precords(const int2 *rng, const int *excl, int n, const int *seg0, int R,
                         int4 *rec, cudaStream_t st);
void launch_let_punpack(const int4 *rec, int n, const float4 *data, float4 *pos, int *have,
                        cudaStream_t st);
void launch_let_mark(const unsigned *ids, int n, int *have, cudaStream_t st);
void launch_let_verify(ListsView Ls, int n_m2l, int n_m2p, int n_p2p, CellsView C,
                       const int *strad, int lo, int hi, const int *haveM, const int *haveP,
                       int *missing, cudaStream_t st);
cudaError_t sort_owner_pairs(void *tmp, size_t &tmp_bytes, const unsigned *kin, unsigned *kout,
                             const unsigned *vin, unsigned *vout, int n, int bits,
                             cudaStream_t st);
