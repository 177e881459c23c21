// fmm_api.cu — the C ABI of libfmm.so (include/fmm.h) and the stream-ordered host pipeline.
//
// One evaluation (every step a device kernel, the host only reads small counts):
//   bbox + root cube -> Morton keys -> radix sort -> gather float4 -> level-synchronous tree
//   -> P2M -> M2M (bottom-up) -> target-centric traversal (count / scan / write per level)
//   -> M2L -> L2L (top-down) -> P2P -> M2P -> L2P + combine + un-permute.
// FMM_DIRECT skips the tree: one all-pairs P2P.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/fmm.h"
#include "comm.cuh"
#include "common.cuh"
#include "kernels.cuh"

#ifndef TRAV_GRID_PER_SM
#define TRAV_GRID_PER_SM 8  // traversal blocks per SM (= its resident blocks, traverse.cu)
#endif

namespace {

template <class T>
struct DBuf {
  T *p = nullptr;
  size_t cap = 0;
  // grow-only; contents are NOT kept
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    size_t nc = std::max(n, cap + cap / 2);
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, nc * sizeof(T));
    if (e == cudaSuccess) cap = nc;
    return e;
  }
  // grow-only; the first `keep` elements are preserved
  cudaError_t ensure_keep(size_t n, size_t keep, cudaStream_t st) {
    if (n <= cap) return cudaSuccess;
    size_t nc = std::max(n, cap * 2);
    T *q = nullptr;
    cudaError_t e = cudaMalloc(&q, nc * sizeof(T));
    if (e != cudaSuccess) return e;
    if (p && keep) e = cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
    cudaStreamSynchronize(st);
    if (p) cudaFree(p);
    p = q;
    cap = nc;
    return cudaSuccess;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

enum { EV_START, EV_TREE, EV_UP, EV_TRAV, EV_M2L_PREP, EV_M2L, EV_P2P, EV_M2P, EV_DOWN, EV_P2P0,
       EV_LET0, EV_LET1, EV_TRAV_END, EV_P2PK, EV_N };

}  // namespace

struct fmm_ctx {
  int device = 0;
  int p = 4, ncrit = 32, mode = FMM_HYBRID;
  double theta = 0.5;
  cudaStream_t own_stream = nullptr, stream = nullptr;
  // the upward sweep runs on `aux`, concurrently with the traversal and the M2L class sort
  cudaStream_t aux = nullptr;
  // the pipeline itself runs on `hi` (highest stream priority; joined with the caller's stream at
  // entry and exit) and the near field on `aux` (lowest), so that the latency-bound M2L class sort
  // gets SMs as soon as P2P blocks retire instead of queueing behind the whole P2P grid
  cudaStream_t hi = nullptr;
  cudaStream_t nf = nullptr;  // the near field (P2P, M2P): lowest priority, its own queue
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_up = nullptr, ev_trav = nullptr, ev_near = nullptr;
  // P2P / M2P run on `aux` after the traversal, overlapping the M2L class preparation and GEMM
  // on the main stream (off while the kernel pre-calculation times the kernels in isolation)
  bool overlap = true;
  DBuf<char> cub_tmp_aux;
  DBuf<float> sh_Y;  // per-cell slots of the tensor-core M2M / L2L
  fmm_cost_t cost{};
  fmm_stats_t stats{};
  bool timing = false;
  bool deterministic = true;  // fmm_set_deterministic (bit-reproducible by default)
  cudaEvent_t ev[EV_N] = {};
  std::string err;
  M2LTiles tiles{};

  // particles
  DBuf<uint64_t> keys_in, keys;
  DBuf<unsigned> idx_in, perm;
  DBuf<float4> pos, acc;
  DBuf<char> cub_tmp;
  DBuf<float> host_stage;
  // small device structs
  RootInfo *d_root = nullptr;
  unsigned *d_mm = nullptr;
  int *d_small = nullptr;  // [0..7] scratch counters for readback
  unsigned *d_overflow = nullptr;
  unsigned long long *d_stats = nullptr;
  int *h_small = nullptr;  // pinned
  // cells
  DBuf<int> cbeg, ccnt, cparent, cchild0, cnchild;
  DBuf<int4> cgrid;
  DBuf<float4> cgeo;
  DBuf<uint64_t> cprefix;
  DBuf<int> nch, excl, leafflag, leaves, bnd;
  DBuf<int2> crange;
  DBuf<int4> cpack;  // packed cell records for the traversal
  DBuf<int> tc_bnd;     // cooperative tree build: child bounds [8][cells of a level]
  DBuf<int2> tc_crange; // ... child ranges
  int *d_tree_st = nullptr;  // ... its results (64 ints; [4] = the short sort's redo flag,
                             // [5] = its long-run count)
  DBuf<int2> sort_runs;      // the short sort's runs of equal high key bits (> 64 particles)
  bool sort_redo = false;
  // M2L translation scheme (NEXT-1): requested (FMM_M2L_AUTO = let fmm_tune decide), the one
  // the kernel pre-calculation picked, and the M2L times it measured per scheme (ms)
  int m2l_scheme = 0, m2l_tuned = 0;
  bool m2l_compact_key = false;  // 21-bit M2L class keys (set when the last evaluation's fitted)
  double m2l_scheme_ms[5] = {0, 0, 0, 0, 0};
  DBuf<float> m2l_R;  // rotation-based scheme: per-class operators (m2l_rot.cu)
  // expansion basis (NEXT-2): 0 spherical harmonics, 1 Cartesian Taylor (p <= CART_PMAX)
  int basis = 0;
  double basis_ms[2] = {0, 0};  // FMM_BASIS_AUTO: the measured evaluation time of each basis
  DBuf<float> Mc, Lc;           // Cartesian expansions [ncells][cart_stride(p)]
  DBuf<int4> p2p_desc;  // per target leaf: (begin, count, own P2P list offset, count | ancestor flag)
  DBuf<int2> p2p_mrg;   // per target leaf: its P2P source ranges sorted and merged (parallel to p2p_rng)
  // sender-side local essential tree (let_send): flags, compacted entries, send / receive buffers
  cudaStream_t cmst = nullptr;  // its stream (the exchange overlaps the traversal)
  cudaEvent_t ev_let = nullptr;
  bool let_recv = false;        // FMM_LET=recv: the round-1 receiver-driven exchange after the traversal
  bool let_check = false;       // FMM_LET_CHECK=1: verify that every remote source named was received
  DBuf<int> let_box, let_flags, let_excl, let_cnt, let_psize, let_pexcl, let_seg0, let_haveM, let_haveP;
  DBuf<unsigned> let_open, let_ids, let_rids;
  DBuf<int2> let_prng;
  DBuf<int4> let_prec, let_rrec;
  DBuf<float2> let_rows_s, let_rows_r;
  DBuf<float4> let_pbuf_s, let_pbuf_r;
  DBuf<int> let_missing;
  void *let_tmp = nullptr;
  size_t let_tmp_cap = 0;  // per target leaf: (begin, count, own P2P list offset, count | ancestor flag)
  std::vector<int> level_off, level_cnt;
  int ncells = 0, nleaves = 0, depth = 0;
  // Morton partition of the targets (multi-GPU); nparts = 1: everything
  int nparts = 1, part = 0;
  int tleaves_n = 0, part_lo = 0, part_hi = 0;
  DBuf<int> tleaves;
  // expansions
  DBuf<float2> M, L;
  // M2L class batching
  DBuf<uint2> m2l_pst, m2l_spst;
  DBuf<int> m2l_pair_t, m2l_flag, m2l_cid, m2l_cstart, m2l_counters;
  DBuf<unsigned> m2l_keys_in, m2l_keys;
  DBuf<unsigned> m2l_idx_in, m2l_sidx, m2l_small, m2l_class_rep, m2l_ssrc, m2l_stgt;
  DBuf<float> m2l_T;
  DBuf<unsigned> m2l_Ttc;
  bool m2l_tc_used = false;
  DBuf<int4> m2l_items, m2l_items_raw;
  DBuf<int> m2l_rflag, m2l_rid, m2l_rstart, m2l_gid_of;
  DBuf<unsigned> m2l_ikeys_in, m2l_ikeys, m2l_iidx_in, m2l_iidx;
  DBuf<float> m2l_Y;  // also the per-cell slots of the tensor-core M2M / L2L
  // M2M / L2L as octant-class GEMMs on the tensor cores
  DBuf<unsigned> sh_keys_in, sh_keys, sh_vals_in, sh_cells, sh_src, sh_T;
  DBuf<int4> sh_items;
  DBuf<int> sh_counters;
  int sh_T_p = -1;
  // lists
  DBuf<int> loff[3], lcnt[3];
  DBuf<unsigned> lsrc[3];
  DBuf<int2> p2p_rng;
  DBuf<int> out_off, out_cnt;
  DBuf<unsigned> trav_osc;
  DBuf<int2> trav_rsc;
  int trav_ocap = 2048;  // per-warp list scratch (entries per list), doubled on overflow
  DBuf<unsigned> outA, outB, stack;
  int stack_cap = 2048;
  int trav_list_est = 256;  // initial list capacity per target cell (entries), before any history
  size_t trav_cap[4] = {0, 0, 0, 0};  // list buffer sizes seen so far (traverse)
  int *d_bk = nullptr;                // device bookkeeping of the traversal (TravArgs::bk)
  int64_t ntask[3] = {0, 0, 0};
  bool have_tree = false;
  int64_t last_n = 0;
  RootInfo h_root{};

  // ---- distinct target / source sets (fmm_evaluate_ts): the first ts_nt particles of the union
  // are the targets (zero charge); 0 = ordinary evaluation ----
  int64_t ts_nt = 0;
  DBuf<int> ntgt;
  DBuf<float> ts_stage;

  // ---- multi-GPU; comm == nullptr: single GPU ----
  FmmComm *comm = nullptr;
  int64_t n_glob = 0;
  int nloc = 0, own_lo = 0, own_hi = 0, nstrad = 0;
  std::vector<int> roff;                       // rank boundaries (global sorted index), R+1
  std::vector<int64_t> scnt_p, rcnt_p;         // particle alltoallv counts (forward direction)
  DBuf<int> d_off, d_lb, d_cnt;
  DBuf<int64_t> d_i64;
  DBuf<uint64_t> d_K, lkeys_in, lkeys, rkeys, rkeys_s;
  DBuf<unsigned> lidx_in, lperm, ridx_in, rperm;
  DBuf<float4> lpos, rpos, pbuf_s, pbuf_r;
  DBuf<int> strad_flag, strad_excl, need_m, need_p, dexcl, psize, pexcl;
  DBuf<unsigned> strad_ids, req_ids, req_own, req_own_s, mreq_s, rreq_ids;
  DBuf<unsigned> pcell, pown, pown_s, pidx, pidx_s;
  DBuf<int> prsize, prexcl, psz2, pex2;
  DBuf<int2> prng, prng_s, rreq_rng;
  DBuf<float2> rows_s, rows_r;
  DBuf<float> rphi, rgrad, sphi, sgrad;
  DBuf<double> d_cost;

  CellsView cells() {
    CellsView C;
    C.beg = cbeg.p;
    C.cnt = ccnt.p;
    C.parent = cparent.p;
    C.child0 = cchild0.p;
    C.nchild = cnchild.p;
    C.grid = cgrid.p;
    C.geo = cgeo.p;
    return C;
  }
  ListsView lists() {
    ListsView Ls;
    for (int k = 0; k < 3; ++k) {
      Ls.off[k] = loff[k].p;
      Ls.cnt[k] = lcnt[k].p;
      Ls.src[k] = lsrc[k].p;
    }
    Ls.p2p_rng = p2p_rng.p;
    return Ls;
  }
};

static int fail(fmm_ctx *h, int code, const char *fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    h->err = buf;
  }
  return code;
}

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(h, e_ == cudaErrorMemoryAllocation ? FMM_E_OOM : FMM_E_CUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                    \
  } while (0)

#define CKL()                                                                            \
  do {                                                                                   \
    ++h->stats.launches;                                                                 \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess)                                                               \
      return fail(h, FMM_E_CUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_),     \
                  __FILE__, __LINE__);                                                   \
  } while (0)

static void record(fmm_ctx *h, int e) {
  if (h->timing) cudaEventRecord(h->ev[e], h->stream);
}
static void record_on(fmm_ctx *h, int e, cudaStream_t s) {
  if (h->timing) cudaEventRecord(h->ev[e], s);
}

// Every C-ABI entry point that touches the device runs on the handle's device and restores the
// caller's current device on every return path.
struct DeviceGuard {
  int prev = -1, dev;
  explicit DeviceGuard(int d) : dev(d) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  }
};

static int check_device_ptr(fmm_ctx *h, const void *ptr, const char *name) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(h, FMM_E_NOT_DEVICE, "%s is not a CUDA pointer", name);
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
    return fail(h, FMM_E_NOT_DEVICE, "%s is not device memory", name);
  if (a.device != h->device) return fail(h, FMM_E_NOT_DEVICE, "%s is on device %d, handle on %d", name, a.device, h->device);
  return FMM_OK;
}

static int cub_scan(fmm_ctx *h, const int *in, int *out, int n) {
  size_t bytes = 0;
  ++h->stats.cub_calls;
  CK(exclusive_scan(nullptr, bytes, in, out, n, h->stream));
  CK(h->cub_tmp.ensure(bytes));
  CK(exclusive_scan(h->cub_tmp.p, bytes, in, out, n, h->stream));
  return FMM_OK;
}

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// Level-synchronous adaptive octree over n particles (a4/a5): one host readback of the child count
// per level. keys = sorted Morton keys; nloc < 0: the keys are all n particles (single GPU);
// nloc >= 0: they are this rank's local shard and the split bounds are allreduced (dist.cu).
static bool host_levels_mode() { return getenv("FMM_TREE_LEVELS") != nullptr; }
static int build_levels(fmm_ctx *h, int64_t n, const uint64_t *keys, int nloc) {
  cudaStream_t st = h->stream;
  // level-synchronous adaptive octree: one host readback of the child count per level
  size_t cap = std::max<size_t>(1024, (size_t)(2 * n / std::max(1, h->ncrit)) + 64);
  auto ensure_cells = [&](size_t need, size_t keep) -> cudaError_t {
    cudaError_t e = cudaSuccess;
    if ((e = h->cbeg.ensure_keep(need, keep, st))) return e;
    if ((e = h->ccnt.ensure_keep(need, keep, st))) return e;
    if ((e = h->cparent.ensure_keep(need, keep, st))) return e;
    if ((e = h->cchild0.ensure_keep(need, keep, st))) return e;
    if ((e = h->cnchild.ensure_keep(need, keep, st))) return e;
    if ((e = h->cgrid.ensure_keep(need, keep, st))) return e;
    if ((e = h->cgeo.ensure_keep(need, keep, st))) return e;
    return h->cprefix.ensure_keep(need, keep, st);
  };
  // single GPU: the whole level loop in one cooperative kernel (tree.cu k_tree_coop) and ONE
  // read-back; capacity from the previous tree (retried larger on overflow). FMM_TREE_LEVELS=1
  // keeps the host-driven loop below (also used by the distributed build).
  static const bool host_levels = getenv("FMM_TREE_LEVELS") != nullptr;
  if (nloc < 0 && !host_levels && n < ((int64_t)1 << 30)) {
    size_t ccap = std::max(cap, (size_t)(1.3 * h->ncells) + 1024);
    const int grid = tree_coop_grid();
    for (int attempt = 0; attempt < 6; ++attempt) {
      CK(ensure_cells(ccap, 0));
      CK(h->tc_bnd.ensure(8 * ccap));
      CK(h->tc_crange.ensure(8 * ccap));
      CK(h->nch.ensure(ccap));
      CK(h->excl.ensure((size_t)grid + 1));
      CK(h->leaves.ensure(ccap));
      CK(launch_tree_coop(keys, (int)n, h->ncrit, h->d_root, h->cells(), h->cprefix.p, (int)ccap,
                          h->tc_bnd.p, h->nch.p, h->tc_crange.p, h->excl.p, h->d_tree_st,
                          h->leaves.p, grid, st));
      h->stats.launches += 1;
      int hs[64];
      CK(cudaMemcpyAsync(hs, h->d_tree_st, sizeof hs, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      h->sort_redo = hs[4] != 0;
      if (hs[1]) {  // the cell capacity was too small: larger, again
        ccap *= 2;
        continue;
      }
      h->ncells = hs[0];
      h->depth = hs[2];
      h->nleaves = hs[3];
      h->level_off.assign(hs + 8, hs + 8 + h->depth + 1);
      h->level_cnt.assign(hs + 32, hs + 32 + h->depth + 1);
      // (scratch the partition / target-set code after the build expects, as the host path)
      CK(h->leafflag.ensure(h->ncells));
      CK(h->excl.ensure(h->ncells));
      return FMM_OK;
    }
    return fail(h, FMM_E_OOM, "octree cells do not fit");
  }
  CK(ensure_cells(cap, 0));
  launch_root_cell(n, h->d_root, h->cells(), h->cprefix.p, st);
  CKL();
  h->level_off.assign(1, 0);
  h->level_cnt.assign(1, 1);
  int total = 1;
  for (int level = 0; level < FMM_LEVELS; ++level) {
    const int nl = h->level_cnt[level], c0 = h->level_off[level];
    CK(h->nch.ensure(nl));
    CK(h->excl.ensure(nl));
    CK(h->crange.ensure((size_t)8 * nl));
    CK(h->bnd.ensure((size_t)8 * nl));
    launch_split_bounds(c0, nl, level, h->ncrit, keys, nloc, h->cells(), h->cprefix.p, h->bnd.p, st);
    CKL();
    if (h->comm) {  // distributed build: global child bounds = sum of the per-rank local bounds
      const double t0 = now_ms();
      const int rc = h->comm->allreduce(h->bnd.p, (size_t)8 * nl, CT_I32, CO_SUM, st);
      h->stats.ms_comm += now_ms() - t0;
      if (rc) return fail(h, rc, "split-bound allreduce: %s", h->comm->err.c_str());
    }
    launch_split_ranges(c0, nl, level, h->ncrit, h->cells(), h->bnd.p, h->nch.p, h->crange.p, st);
    CKL();
    if (int rc = cub_scan(h, h->nch.p, h->excl.p, nl)) return rc;
    launch_level_total(h->nch.p, h->excl.p, nl, h->d_small, st);
    CKL();
    CK(cudaMemcpyAsync(h->h_small, h->d_small, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int nnext = h->h_small[0];
    if (nnext > 0) CK(ensure_cells((size_t)total + nnext, (size_t)total));
    launch_emit(c0, nl, total, level, h->nch.p, h->excl.p, h->crange.p, h->d_root, h->cells(),
                h->cprefix.p, st);
    CKL();
    if (nnext == 0) break;
    h->level_off.push_back(total);
    h->level_cnt.push_back(nnext);
    total += nnext;
  }
  h->ncells = total;
  h->depth = (int)h->level_cnt.size() - 1;
  // leaves in cell order
  CK(h->leafflag.ensure(total));
  CK(h->excl.ensure(total));
  CK(h->leaves.ensure(total));
  launch_leaf_flags(total, h->cnchild.p, h->leafflag.p, st);
  CKL();
  if (int rc = cub_scan(h, h->leafflag.p, h->excl.p, total)) return rc;
  launch_leaf_scatter(total, h->leafflag.p, h->excl.p, h->leaves.p, st);
  CKL();
  launch_level_total(h->leafflag.p, h->excl.p, total, h->d_small, st);
  CKL();
  CK(cudaMemcpyAsync(h->h_small, h->d_small, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  h->nleaves = h->h_small[0];
  return FMM_OK;
}

// ---- a1-a5: bbox, keys, sort, gather, tree ----------------------------------------------------
static int build_tree(fmm_ctx *h, const float *xyz, const float *q, int64_t n) {
  cudaStream_t st = h->stream;
  CK(h->keys_in.ensure(n));
  CK(h->keys.ensure(n));
  CK(h->idx_in.ensure(n));
  CK(h->perm.ensure(n));
  CK(h->pos.ensure(n));
  CK(h->acc.ensure(n));
  launch_keys(xyz, n, h->d_root, h->keys_in.p, h->idx_in.p, st);
  CKL();
  // a3: radix passes over the key bits of levels 0..D+2 (D = the previous tree's depth; bits
  // 16..62 on the first evaluation) + a tie fix-up (tree.cu), exactly the order of the full
  // 63-bit stable sort; a run of equal high bits longer than 4096 (a very dense cluster) flags a
  // redo with all 8 passes, found in the tree build's single read-back
  const int low_bits = h->depth > 0 ? std::max(16, std::min(40, 63 - 3 * (h->depth + 2))) : 16;
  static const bool full_sort = getenv("FMM_SORT_FULL") != nullptr;
  bool short_sort = !full_sort;
  for (int pass = 0; pass < 2; ++pass) {
    size_t bytes = 0;
    CK(cudaMemsetAsync(h->d_tree_st + 4, 0, sizeof(int), st));
    if (short_sort) {
      CK(h->sort_runs.ensure((size_t)sort_runs_cap(n)));
      CK(sort_keys_short(nullptr, bytes, h->keys_in.p, h->keys.p, h->idx_in.p, h->perm.p, n,
                         h->d_tree_st + 4, h->sort_runs.p, low_bits, st));
      CK(h->cub_tmp.ensure(bytes));
      CK(sort_keys_short(h->cub_tmp.p, bytes, h->keys_in.p, h->keys.p, h->idx_in.p, h->perm.p, n,
                         h->d_tree_st + 4, h->sort_runs.p, low_bits, st));
      h->stats.launches += 2;
    } else {
      CK(sort_keys(nullptr, bytes, h->keys_in.p, h->keys.p, h->idx_in.p, h->perm.p, n, st));
      CK(h->cub_tmp.ensure(bytes));
      CK(sort_keys(h->cub_tmp.p, bytes, h->keys_in.p, h->keys.p, h->idx_in.p, h->perm.p, n, st));
    }
    ++h->stats.cub_calls;
    launch_gather(xyz, q, h->perm.p, n, h->pos.p, st);
    CKL();
    h->sort_redo = false;
    if (int rc = build_levels(h, n, h->keys.p, -1)) return rc;
    if (!short_sort) break;
    if (!h->sort_redo) {  // the host-driven level loop does not read the flag: check it here
      if (host_levels_mode()) {
        int f = 0;
        CK(cudaMemcpyAsync(&f, h->d_tree_st + 4, sizeof f, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        h->sort_redo = f != 0;
      }
      if (!h->sort_redo) break;
    }
    short_sort = false;  // a long run of equal high bits: sort all 63 bits and build again
  }
  const int total = h->ncells;
  // target leaves of this handle's partition
  h->part_lo = 0;
  h->part_hi = (int)n;
  h->tleaves_n = h->nleaves;
  if (h->ts_nt > 0) {  // target cells / leaves: the ones holding at least one target particle
    CK(h->ntgt.ensure(total));
    CK(h->tleaves.ensure(total));
    CK(h->excl.ensure(std::max<int64_t>(n, total)));
    int *flag = reinterpret_cast<int *>(h->acc.p);  // scratch (acc is written later by P2P)
    launch_target_flags(h->perm.p, (int)n, (int)h->ts_nt, flag, st);
    CKL();
    if (int rc = cub_scan(h, flag, h->excl.p, (int)n)) return rc;
    launch_cell_targets(total, h->cells(), h->excl.p, flag, (int)n, h->ntgt.p, h->leafflag.p, st);
    CKL();
    if (int rc = cub_scan(h, h->leafflag.p, h->excl.p, total)) return rc;
    launch_leaf_scatter(total, h->leafflag.p, h->excl.p, h->tleaves.p, st);
    CKL();
    launch_level_total(h->leafflag.p, h->excl.p, total, h->d_small, st);
    CKL();
    CK(cudaMemcpyAsync(h->h_small, h->d_small, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    h->tleaves_n = h->h_small[0];
  } else if (h->nparts > 1) {
    CK(h->tleaves.ensure(total));
    launch_part_flags(total, h->cells(), n, h->nparts, h->part, h->leafflag.p, h->d_small + 8, st);
    h->stats.launches += 1;
    CKL();
    if (int rc = cub_scan(h, h->leafflag.p, h->excl.p, total)) return rc;
    launch_leaf_scatter(total, h->leafflag.p, h->excl.p, h->tleaves.p, st);
    CKL();
    launch_level_total(h->leafflag.p, h->excl.p, total, h->d_small, st);
    CKL();
    CK(cudaMemcpyAsync(h->h_small, h->d_small, 10 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    h->tleaves_n = h->h_small[0];
    h->part_lo = h->tleaves_n ? h->h_small[8] : 0;
    h->part_hi = h->tleaves_n ? h->h_small[9] : 0;
  }
  return FMM_OK;
}

// ---- multi-GPU: distributed tree, partition, local essential tree ----
#define CC(call)                                                                    \
  do {                                                                              \
    const double t0_ = now_ms();                                                    \
    const int rc_ = (call);                                                         \
    h->stats.ms_comm += now_ms() - t0_;                                             \
    if (rc_) return fail(h, rc_, "%s: %s", #call, h->comm->err.c_str());            \
  } while (0)

// recv[r * k + j] = item j of what peer r sends to this rank (send[r * k + j] = item j for peer r)
static int exchange_counts(fmm_ctx *h, const std::vector<int64_t> &send,
                           std::vector<int64_t> &recv, int k, cudaStream_t st = nullptr) {
  const int R = h->comm->nranks, me = h->comm->rank;
  if (!st) st = h->stream;
  const size_t blk = (size_t)R * k;
  CK(h->d_i64.ensure(blk * (R + 1)));
  CK(cudaMemcpyAsync(h->d_i64.p, send.data(), sizeof(int64_t) * blk, cudaMemcpyHostToDevice, st));
  CC(h->comm->allgather(h->d_i64.p, h->d_i64.p + blk, sizeof(int64_t) * blk, st));
  std::vector<int64_t> all(blk * R);
  CK(cudaMemcpyAsync(all.data(), h->d_i64.p + blk, sizeof(int64_t) * blk * R, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  recv.assign(blk, 0);
  for (int r = 0; r < R; ++r)
    for (int j = 0; j < k; ++j) recv[(size_t)r * k + j] = all[((size_t)r * R + me) * k + j];
  return FMM_OK;
}

// alltoallv of elements of `elem` bytes; counts per peer taken from column `col` of k-wide rows
static int a2av(fmm_ctx *h, const void *send, const std::vector<int64_t> &scnt, void *recv,
                const std::vector<int64_t> &rcnt, size_t elem, int k = 1, int col = 0,
                cudaStream_t st = nullptr) {
  const int R = h->comm->nranks, me = h->comm->rank;
  std::vector<size_t> sc(R), sd(R), rc(R), rd(R);
  size_t so = 0, ro = 0;
  for (int r = 0; r < R; ++r) {
    sc[r] = (size_t)scnt[(size_t)r * k + col] * elem;
    sd[r] = so;
    so += sc[r];
    rc[r] = (size_t)rcnt[(size_t)r * k + col] * elem;
    rd[r] = ro;
    ro += rc[r];
  }
  h->stats.bytes_sent += (int64_t)(so - sc[me]);
  CC(h->comm->alltoallv(send, sc.data(), sd.data(), recv, rc.data(), rd.data(), st ? st : h->stream));
  return FMM_OK;
}

// ids of the flagged cells (ascending); returns their number in *count
static int compact_flags(fmm_ctx *h, const int *flag, int n, unsigned *ids, int *count) {
  cudaStream_t st = h->stream;
  CK(h->dexcl.ensure(std::max(n, 1)));
  if (int rc = cub_scan(h, flag, h->dexcl.p, n)) return rc;
  launch_leaf_scatter(n, flag, h->dexcl.p, (int *)ids, st);
  CKL();
  launch_level_total(flag, h->dexcl.p, n, h->d_small, st);
  CKL();
  CK(cudaMemcpyAsync(h->h_small, h->d_small, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *count = h->h_small[0];
  return FMM_OK;
}

// sort (owner, value) pairs by owner (stable) and count per owner on the host
static int sort_by_owner(fmm_ctx *h, const unsigned *own, unsigned *own_s, const unsigned *val,
                         unsigned *val_s, int n, std::vector<int64_t> &cnt) {
  cudaStream_t st = h->stream;
  const int R = h->comm->nranks;
  int bits = 1;
  while ((1 << bits) < R) ++bits;
  if (n > 0) {
    size_t bytes = 0;
    CK(sort_owner_pairs(nullptr, bytes, own, own_s, val, val_s, n, bits, st));
    CK(h->cub_tmp.ensure(bytes));
    CK(sort_owner_pairs(h->cub_tmp.p, bytes, own, own_s, val, val_s, n, bits, st));
    ++h->stats.cub_calls;
  }
  CK(h->d_cnt.ensure(R));
  CK(cudaMemsetAsync(h->d_cnt.p, 0, sizeof(int) * R, st));
  launch_owner_hist(own_s, n, h->d_cnt.p, st);
  if (n > 0) CKL();
  std::vector<int> c(R);
  CK(cudaMemcpyAsync(c.data(), h->d_cnt.p, sizeof(int) * R, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cnt.assign(c.begin(), c.end());
  return FMM_OK;
}

// a1-a5 + partition + particle exchange. After this, pos / perm hold this rank's particles at
// their GLOBAL Morton positions [own_lo, own_hi); the tree is the global one (same on every rank).
static int dist_build_tree(fmm_ctx *h, const float *xyz, const float *q, int64_t nloc) {
  cudaStream_t st = h->stream;
  FmmComm *cm = h->comm;
  const int R = cm->nranks, me = cm->rank;
  // a1: global bounding box -> root cube (identical on every rank); global particle count
  launch_bbox_local(xyz, q, nloc, h->d_mm, h->d_root, st);
  h->stats.launches += 2;
  CKL();
  CC(cm->allreduce(h->d_mm, 3, CT_U32, CO_MIN, st));
  CC(cm->allreduce(h->d_mm + 3, 4, CT_U32, CO_MAX, st));
  launch_root_from_mm(h->d_mm, h->d_root, st);
  h->stats.launches += 1;
  CKL();
  CK(h->d_i64.ensure(64));
  int64_t nn = nloc;
  CK(cudaMemcpyAsync(h->d_i64.p, &nn, sizeof nn, cudaMemcpyHostToDevice, st));
  CC(cm->allreduce(h->d_i64.p, 1, CT_I64, CO_SUM, st));
  CK(cudaMemcpyAsync(&nn, h->d_i64.p, sizeof nn, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&h->h_root, h->d_root, sizeof(RootInfo), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h->h_root.nonfinite) return fail(h, FMM_E_NONFINITE, "non-finite coordinate or charge on some rank");
  if (nn >= ((int64_t)1 << 30)) return fail(h, FMM_E_INVALID, "global n = %lld exceeds 2^30", (long long)nn);
  h->n_glob = nn;
  h->nloc = (int)nloc;
  const int N = (int)nn;
  // a2/a3 on the local shard: keys, sort, Morton-ordered float4
  const size_t nl1 = std::max<int64_t>(nloc, 1);
  CK(h->lkeys_in.ensure(nl1));
  CK(h->lkeys.ensure(nl1));
  CK(h->lidx_in.ensure(nl1));
  CK(h->lperm.ensure(nl1));
  CK(h->lpos.ensure(nl1));
  if (nloc > 0) {
    launch_keys(xyz, nloc, h->d_root, h->lkeys_in.p, h->lidx_in.p, st);
    CKL();
    size_t bytes = 0;
    CK(sort_keys(nullptr, bytes, h->lkeys_in.p, h->lkeys.p, h->lidx_in.p, h->lperm.p, nloc, st));
    CK(h->cub_tmp.ensure(bytes));
    CK(sort_keys(h->cub_tmp.p, bytes, h->lkeys_in.p, h->lkeys.p, h->lidx_in.p, h->lperm.p, nloc, st));
    ++h->stats.cub_calls;
    launch_gather(xyz, q, h->lperm.p, nloc, h->lpos.p, st);
    CKL();
  }
  // a4/a5: the global adaptive octree, level by level from allreduced split bounds
  if (int rc = build_levels(h, N, h->lkeys.p, (int)nloc)) return rc;
  // partition: contiguous runs of whole leaves, balanced by particle count
  CK(h->d_off.ensure(R + 1));
  CK(h->d_K.ensure(R + 1));
  CK(h->d_lb.ensure(R + 1));
  launch_partition(h->leaves.p, h->nleaves, h->cells(), h->cprefix.p, N, R, h->d_off.p, h->d_K.p, st);
  CKL();
  launch_key_bounds(h->lkeys.p, (int)nloc, h->d_K.p, R, h->d_lb.p, st);
  CKL();
  h->roff.assign(R + 1, 0);
  std::vector<int> lb(R + 1);
  CK(cudaMemcpyAsync(h->roff.data(), h->d_off.p, sizeof(int) * (R + 1), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(lb.data(), h->d_lb.p, sizeof(int) * (R + 1), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  h->own_lo = h->roff[me];
  h->own_hi = h->roff[me + 1];
  h->scnt_p.assign(R, 0);
  for (int r = 0; r < R; ++r) h->scnt_p[r] = lb[r + 1] - lb[r];
  if (int rc = exchange_counts(h, h->scnt_p, h->rcnt_p, 1)) return rc;
  int64_t nown = 0;
  for (int r = 0; r < R; ++r) nown += h->rcnt_p[r];
  if (nown != h->own_hi - h->own_lo)
    return fail(h, FMM_E_INVALID, "partition: received %lld particles for range [%d, %d)",
                (long long)nown, h->own_lo, h->own_hi);
  // particle alltoallv (Morton-sorted float4 + keys); each rank receives its leaves' particles
  const size_t no1 = std::max<int64_t>(nown, 1);
  CK(h->rpos.ensure(no1));
  CK(h->rkeys.ensure(no1));
  CK(h->rkeys_s.ensure(no1));
  CK(h->ridx_in.ensure(no1));
  CK(h->rperm.ensure(no1));
  if (int rc = a2av(h, h->lpos.p, h->scnt_p, h->rpos.p, h->rcnt_p, sizeof(float4))) return rc;
  if (int rc = a2av(h, h->lkeys.p, h->scnt_p, h->rkeys.p, h->rcnt_p, sizeof(uint64_t))) return rc;
  // global sorted order of the own particles: stable sort by key (ties: source rank, then source
  // order -- the order of a single sort of the concatenated shards)
  CK(h->pos.ensure(std::max(N, 1)));
  CK(h->acc.ensure(std::max(N, 1)));
  CK(h->perm.ensure(std::max(N, 1)));
  if (nown > 0) {
    launch_iota(h->ridx_in.p, (int)nown, st);
    CKL();
    size_t bytes = 0;
    CK(sort_keys(nullptr, bytes, h->rkeys.p, h->rkeys_s.p, h->ridx_in.p, h->rperm.p, nown, st));
    CK(h->cub_tmp.ensure(bytes));
    CK(sort_keys(h->cub_tmp.p, bytes, h->rkeys.p, h->rkeys_s.p, h->ridx_in.p, h->rperm.p, nown, st));
    ++h->stats.cub_calls;
    launch_gather4(h->rpos.p, h->rperm.p, (int)nown, h->pos.p + h->own_lo, st);
    CKL();
    CK(cudaMemcpyAsync(h->perm.p + h->own_lo, h->rperm.p, sizeof(unsigned) * nown,
                       cudaMemcpyDeviceToDevice, st));
  }
  // own target leaves
  const int total = h->ncells;
  CK(h->tleaves.ensure(total));
  launch_range_leaf_flags(total, h->cells(), h->own_lo, h->own_hi, h->leafflag.p, st);
  CKL();
  if (int rc = compact_flags(h, h->leafflag.p, total, (unsigned *)h->tleaves.p, &h->tleaves_n)) return rc;
  h->part_lo = h->own_lo;
  h->part_hi = h->own_hi;
  // cells whose particles span several ranks: their multipoles are summed over the ranks
  CK(h->strad_flag.ensure(total));
  CK(h->strad_ids.ensure(total));
  launch_straddle_flags(total, h->cells(), h->d_off.p, R, h->strad_flag.p, st);
  CKL();
  if (int rc = compact_flags(h, h->strad_flag.p, total, h->strad_ids.p, &h->nstrad)) return rc;
  h->stats.n_global = N;
  h->stats.rank_lo = h->own_lo;
  h->stats.rank_hi = h->own_hi;
  h->stats.n_straddle = h->nstrad;
  return FMM_OK;
}

// Receiver-driven local essential tree (after the traversal; waits for the upward sweep). The
// lists name every source this rank's targets need; multipoles of cells outside [own_lo, own_hi)
// that do not straddle, and P2P source particles outside it, are requested from their owners.
static int dist_let(fmm_ctx *h) {
  cudaStream_t st = h->stream;
  FmmComm *cm = h->comm;
  const int R = cm->nranks, me = cm->rank, nc = h->ncells;
  const int NCS = nc_stride(h->p);
  CK(h->need_m.ensure(nc));
  CK(h->need_p.ensure(nc));
  CK(cudaMemsetAsync(h->need_m.p, 0, sizeof(int) * nc, st));
  CK(cudaMemsetAsync(h->need_p.p, 0, sizeof(int) * nc, st));
  launch_need_flags(h->lists(), (int)h->ntask[0], (int)h->ntask[1], (int)h->ntask[2], h->cells(),
                    h->strad_flag.p, h->own_lo, h->own_hi, h->need_m.p, h->need_p.p, st);
  CKL();
  // multipole requests: cell ids grouped by owner
  int nm = 0, npc = 0;
  CK(h->req_ids.ensure(nc));
  CK(h->req_own.ensure(nc));
  CK(h->req_own_s.ensure(nc));
  CK(h->mreq_s.ensure(nc));
  if (int rc = compact_flags(h, h->need_m.p, nc, h->req_ids.p, &nm)) return rc;
  launch_owner_of_cells(h->req_ids.p, nm, h->cells(), h->d_off.p, R, h->req_own.p, st);
  std::vector<int64_t> cntM, cntP;
  if (int rc = sort_by_owner(h, h->req_own.p, h->req_own_s.p, h->req_ids.p, h->mreq_s.p, nm, cntM)) return rc;
  // particle requests: the remote pieces of every P2P source range, grouped by owner
  CK(h->pcell.ensure(nc));
  if (int rc = compact_flags(h, h->need_p.p, nc, h->pcell.p, &npc)) return rc;
  CK(h->psize.ensure(std::max(npc, 1)));
  CK(h->pexcl.ensure(std::max(npc, 1) + 1));
  launch_piece_count(h->pcell.p, npc, h->cells(), h->d_off.p, R, me, h->psize.p, st);
  int npieces = 0;
  if (npc > 0) {
    CKL();
    if (int rc = cub_scan(h, h->psize.p, h->pexcl.p, npc)) return rc;
    launch_level_total(h->psize.p, h->pexcl.p, npc, h->d_small, st);
    CKL();
    CK(cudaMemcpyAsync(h->h_small, h->d_small, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    npieces = h->h_small[0];
  }
  const size_t np1 = std::max(npieces, 1);
  CK(h->pown.ensure(np1));
  CK(h->pown_s.ensure(np1));
  CK(h->pidx.ensure(np1));
  CK(h->pidx_s.ensure(np1));
  CK(h->prng.ensure(np1));
  CK(h->prng_s.ensure(np1));
  CK(h->prsize.ensure(np1));
  CK(h->prexcl.ensure(np1 + 1));
  launch_piece_write(h->pcell.p, npc, h->cells(), h->d_off.p, R, me, h->pexcl.p, h->pown.p,
                     h->pidx.p, h->prng.p, st);
  if (int rc = sort_by_owner(h, h->pown.p, h->pown_s.p, h->pidx.p, h->pidx_s.p, npieces, cntP)) return rc;
  launch_gather_int2(h->prng.p, h->pidx_s.p, npieces, h->prng_s.p, h->prsize.p, st);
  // particles per owner: exclusive scan of the sorted piece sizes, read at the owner boundaries
  std::vector<int64_t> partP(R, 0);
  if (npieces > 0) {
    CKL();
    if (int rc = cub_scan(h, h->prsize.p, h->prexcl.p, npieces)) return rc;
    std::vector<int> ex(npieces + 1);
    CK(cudaMemcpyAsync(ex.data(), h->prexcl.p, sizeof(int) * npieces, cudaMemcpyDeviceToHost, st));
    std::vector<int2> last(1);
    CK(cudaMemcpyAsync(last.data(), h->prng_s.p + npieces - 1, sizeof(int2), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ex[npieces] = ex[npieces - 1] + (last[0].y - last[0].x);
    int64_t s0 = 0;
    for (int r = 0; r < R; ++r) {
      const int64_t s1 = s0 + cntP[r];
      partP[r] = ex[s1] - ex[s0];
      s0 = s1;
    }
  }
  // request exchange: counts (multipoles, pieces, particles) then ids and ranges
  std::vector<int64_t> send3((size_t)3 * R), recv3;
  for (int r = 0; r < R; ++r) {
    send3[3 * r] = cntM[r];
    send3[3 * r + 1] = cntP[r];
    send3[3 * r + 2] = partP[r];
  }
  if (int rc = exchange_counts(h, send3, recv3, 3)) return rc;
  int64_t rM = 0, rP = 0, rPart = 0, gotPart = 0;
  for (int r = 0; r < R; ++r) {
    rM += recv3[3 * r];
    rP += recv3[3 * r + 1];
    rPart += recv3[3 * r + 2];
    gotPart += partP[r];
  }
  CK(h->rreq_ids.ensure(std::max<int64_t>(rM, 1)));
  CK(h->rreq_rng.ensure(std::max<int64_t>(rP, 1)));
  if (int rc = a2av(h, h->mreq_s.p, send3, h->rreq_ids.p, recv3, sizeof(unsigned), 3, 0)) return rc;
  if (int rc = a2av(h, h->prng_s.p, send3, h->rreq_rng.p, recv3, sizeof(int2), 3, 1)) return rc;
  // the multipoles are complete once the upward sweep is done and the straddling cells are summed
  CK(cudaStreamWaitEvent(st, h->ev_up, 0));
  if (h->nstrad > 0) {
    CK(h->rows_s.ensure((size_t)h->nstrad * NCS));
    launch_rows(h->M.p, h->rows_s.p, NCS, h->strad_ids.p, h->nstrad, false, st);
    CKL();
    CC(cm->allreduce(h->rows_s.p, (size_t)h->nstrad * NCS * 2, CT_F32, CO_SUM, st));
    launch_rows(h->rows_s.p, h->M.p, NCS, h->strad_ids.p, h->nstrad, true, st);
    CKL();
  }
  // serve: multipole rows and particle ranges, in the order they were requested
  CK(h->rows_s.ensure((size_t)std::max<int64_t>(rM, 1) * NCS));
  CK(h->rows_r.ensure((size_t)std::max(nm, 1) * NCS));
  launch_rows(h->M.p, h->rows_s.p, NCS, h->rreq_ids.p, (int)rM, false, st);
  if (rM > 0) CKL();
  if (int rc = a2av(h, h->rows_s.p, recv3, h->rows_r.p, send3, sizeof(float2) * NCS, 3, 0)) return rc;
  launch_rows(h->rows_r.p, h->M.p, NCS, h->mreq_s.p, nm, true, st);
  if (nm > 0) CKL();
  CK(h->psz2.ensure(std::max<int64_t>(rP, 1)));
  CK(h->pex2.ensure(std::max<int64_t>(rP, 1) + 1));
  CK(h->pbuf_s.ensure(std::max<int64_t>(rPart, 1)));
  CK(h->pbuf_r.ensure(std::max<int64_t>(gotPart, 1)));
  if (rP > 0) {
    launch_range_sizes(h->rreq_rng.p, (int)rP, h->psz2.p, st);
    CKL();
    if (int rc = cub_scan(h, h->psz2.p, h->pex2.p, (int)rP)) return rc;
    launch_range_copy(h->pos.p, h->rreq_rng.p, h->pex2.p, (int)rP, h->pbuf_s.p, false, st);
    CKL();
  }
  if (int rc = a2av(h, h->pbuf_s.p, recv3, h->pbuf_r.p, send3, sizeof(float4), 3, 2)) return rc;
  if (npieces > 0) {
    launch_range_copy(h->pos.p, h->prng_s.p, h->prexcl.p, npieces, h->pbuf_r.p, true, st);
    CKL();
  }
  h->stats.let_cells = nm;
  h->stats.let_particles = gotPart;
  return FMM_OK;
}


// Sender-side local essential tree (NEXT-3: "The MPI
// communication is overlapped with the kernel evaluations"). Runs on its own stream right after
// the upward sweep, while the main stream traverses: every rank decides from the global skeleton
// what each other rank's traversal can read from it (dist.cu k_let_open / k_let_flags, a
// conservative superset of what the receiver-driven dist_let requests) and sends it unasked --
// no request round trip, and nothing waits for the traversal. The host blocks only on this
// stream's small count read-backs, after the traversal has been queued.
static int let_send(fmm_ctx *h) {
  FmmComm *cm = h->comm;
  const int R = cm->nranks, me = cm->rank, nc = h->ncells, N = (int)h->n_glob;
  const int NCS = nc_stride(h->p);
  if (!h->cmst) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CK(cudaStreamCreateWithPriority(&h->cmst, cudaStreamNonBlocking, hi));
    CK(cudaEventCreateWithFlags(&h->ev_let, cudaEventDisableTiming));
  }
  cudaStream_t cs = h->cmst;
  record_on(h, EV_LET0, cs);
  CK(cudaStreamWaitEvent(cs, h->ev_up, 0));  // own multipoles complete (P2M + M2M)
  // straddling cells: sum the per-rank partial multipoles (M2M is linear)
  if (h->nstrad > 0) {
    CK(h->rows_s.ensure((size_t)h->nstrad * NCS));
    launch_rows(h->M.p, h->rows_s.p, NCS, h->strad_ids.p, h->nstrad, false, cs);
    CKL();
    CC(cm->allreduce(h->rows_s.p, (size_t)h->nstrad * NCS * 2, CT_F32, CO_SUM, cs));
    launch_rows(h->rows_s.p, h->M.p, NCS, h->strad_ids.p, h->nstrad, true, cs);
    CKL();
  }
  // what each receiver can touch: flags[(kind * R + r) * nc + c], kind 0 multipole, 1 particles
  const size_t nf = (size_t)2 * R * nc;
  CK(h->let_box.ensure((size_t)let_box_ints(R)));
  CK(h->let_open.ensure((size_t)2 * nc));
  CK(h->let_flags.ensure(nf));
  CK(h->let_excl.ensure(nf));
  CK(h->let_cnt.ensure((size_t)2 * R + 2));
  // an accepted pair can be P2P only in hybrid mode (cost model, see k_let_flags), and only with a
  // target of at most t_ml / t_pp particles
  const double tpp = h->mode == FMM_HYBRID ? h->cost.t_pp : 0.0;
  const int kmax = tpp > 0 ? (int)std::min(2e9, h->cost.t_ml / tpp + 1.0) : 0;
  launch_let_boxes(h->leaves.p, h->nleaves, nc, h->cells(), h->d_off.p, R, kmax, h->let_box.p, cs);
  launch_let_flags(nc, h->cells(), h->let_box.p, h->d_off.p, R, me, h->theta, tpp, h->cost.t_mp,
                   h->cost.t_ml, h->let_open.p, h->let_open.p + nc, h->let_flags.p, cs);
  CKL();
  h->stats.launches += 4;
  {
    size_t bytes = 0;
    CK(exclusive_scan(nullptr, bytes, h->let_flags.p, h->let_excl.p, (int)nf, cs));
    if (bytes > h->let_tmp_cap) {
      if (h->let_tmp) cudaFree(h->let_tmp);
      h->let_tmp = nullptr;
      h->let_tmp_cap = 0;
      CK(cudaMalloc(&h->let_tmp, bytes));
      h->let_tmp_cap = bytes;
    }
    CK(exclusive_scan(h->let_tmp, bytes, h->let_flags.p, h->let_excl.p, (int)nf, cs));
    ++h->stats.cub_calls;
  }
  launch_seg_counts(h->let_flags.p, h->let_excl.p, 2 * R, nc, h->let_cnt.p, cs);
  CKL();
  std::vector<int> cnt(2 * R);
  CK(cudaMemcpyAsync(cnt.data(), h->let_cnt.p, sizeof(int) * 2 * R, cudaMemcpyDeviceToHost, cs));
  CK(cudaStreamSynchronize(cs));
  int TM = 0, TP = 0;
  for (int r = 0; r < R; ++r) {
    TM += cnt[r];
    TP += cnt[R + r];
  }
  // compacted entries: multipole cells (receiver-major), then particle cells (receiver-major)
  CK(h->let_ids.ensure((size_t)std::max(TM + TP, 1)));
  launch_seg_scatter(h->let_flags.p, h->let_excl.p, (int64_t)nf, nc, h->let_ids.p, cs);
  CKL();
  // particle entries: my part of each cell's range, offsets, records for the receivers
  CK(h->let_prng.ensure((size_t)std::max(TP, 1)));
  CK(h->let_psize.ensure((size_t)std::max(TP, 1) + 1));
  CK(h->let_pexcl.ensure((size_t)std::max(TP, 1) + 1));
  CK(h->let_prec.ensure((size_t)std::max(TP, 1)));
  CK(h->let_seg0.ensure((size_t)R + 1));
  std::vector<int> seg0(R + 1, 0);
  for (int r = 0; r < R; ++r) seg0[r + 1] = seg0[r] + cnt[R + r];
  std::vector<int64_t> partP(R, 0);
  if (TP > 0) {
    launch_let_prange(h->let_ids.p + TM, TP, h->cells(), h->own_lo, h->own_hi, h->let_prng.p,
                      h->let_psize.p, cs);
    CKL();
    CK(cudaMemsetAsync(h->let_psize.p + TP, 0, sizeof(int), cs));
    size_t bytes = 0;
    CK(exclusive_scan(nullptr, bytes, h->let_psize.p, h->let_pexcl.p, TP + 1, cs));
    if (bytes > h->let_tmp_cap) {
      cudaFree(h->let_tmp);
      h->let_tmp = nullptr;
      h->let_tmp_cap = 0;
      CK(cudaMalloc(&h->let_tmp, bytes));
      h->let_tmp_cap = bytes;
    }
    CK(exclusive_scan(h->let_tmp, bytes, h->let_psize.p, h->let_pexcl.p, TP + 1, cs));
    ++h->stats.cub_calls;
    CK(cudaMemcpyAsync(h->let_seg0.p, seg0.data(), sizeof(int) * (R + 1), cudaMemcpyHostToDevice, cs));
    launch_let_precords(h->let_prng.p, h->let_pexcl.p, TP, h->let_seg0.p, R, h->let_prec.p, cs);
    CKL();
    std::vector<int> ex(TP + 1);
    CK(cudaMemcpyAsync(ex.data(), h->let_pexcl.p, sizeof(int) * (TP + 1), cudaMemcpyDeviceToHost, cs));
    CK(cudaStreamSynchronize(cs));
    for (int r = 0; r < R; ++r) partP[r] = ex[seg0[r + 1]] - ex[seg0[r]];
  }
  // counts, then the four alltoallv: multipole ids, rows, particle records, particles
  std::vector<int64_t> send3((size_t)3 * R), recv3;
  for (int r = 0; r < R; ++r) {
    send3[3 * r] = cnt[r];
    send3[3 * r + 1] = cnt[R + r];
    send3[3 * r + 2] = partP[r];
  }
  if (int rc = exchange_counts(h, send3, recv3, 3, cs)) return rc;
  int64_t rM = 0, rP = 0, rPart = 0;
  for (int r = 0; r < R; ++r) {
    rM += recv3[3 * r];
    rP += recv3[3 * r + 1];
    rPart += recv3[3 * r + 2];
  }
  int64_t sPart = 0;
  for (int r = 0; r < R; ++r) sPart += partP[r];
  CK(h->let_rows_s.ensure((size_t)std::max(TM, 1) * NCS));
  CK(h->let_pbuf_s.ensure((size_t)std::max<int64_t>(sPart, 1)));
  launch_rows(h->M.p, h->let_rows_s.p, NCS, h->let_ids.p, TM, false, cs);
  if (TM > 0) CKL();
  if (TP > 0) {
    launch_range_copy(h->pos.p, h->let_prng.p, h->let_pexcl.p, TP, h->let_pbuf_s.p, false, cs);
    CKL();
  }
  CK(h->let_rids.ensure((size_t)std::max<int64_t>(rM, 1)));
  CK(h->let_rows_r.ensure((size_t)std::max<int64_t>(rM, 1) * NCS));
  CK(h->let_rrec.ensure((size_t)std::max<int64_t>(rP, 1)));
  CK(h->let_pbuf_r.ensure((size_t)std::max<int64_t>(rPart, 1)));
  if (int rc = a2av(h, h->let_ids.p, send3, h->let_rids.p, recv3, sizeof(unsigned), 3, 0, cs)) return rc;
  if (int rc = a2av(h, h->let_rows_s.p, send3, h->let_rows_r.p, recv3, sizeof(float2) * NCS, 3, 0, cs)) return rc;
  if (int rc = a2av(h, h->let_prec.p, send3, h->let_rrec.p, recv3, sizeof(int4), 3, 1, cs)) return rc;
  if (int rc = a2av(h, h->let_pbuf_s.p, send3, h->let_pbuf_r.p, recv3, sizeof(float4), 3, 2, cs)) return rc;
  // unpack into the global-index arrays
  if (h->let_check) {
    CK(h->let_haveM.ensure(nc));
    CK(h->let_haveP.ensure((size_t)std::max(N, 1)));
    CK(cudaMemsetAsync(h->let_haveM.p, 0, sizeof(int) * nc, cs));
    CK(cudaMemsetAsync(h->let_haveP.p, 0, sizeof(int) * std::max(N, 1), cs));
    launch_let_mark(h->let_rids.p, (int)rM, h->let_haveM.p, cs);
  }
  launch_rows(h->let_rows_r.p, h->M.p, NCS, h->let_rids.p, (int)rM, true, cs);
  if (rM > 0) CKL();
  int64_t ro = 0, po = 0;
  for (int r = 0; r < R; ++r) {
    launch_let_punpack(h->let_rrec.p + ro, (int)recv3[3 * r + 1], h->let_pbuf_r.p + po, h->pos.p,
                       h->let_check ? h->let_haveP.p : nullptr, cs);
    ro += recv3[3 * r + 1];
    po += recv3[3 * r + 2];
  }
  CKL();
  CK(cudaEventRecord(h->ev_let, cs));
  record_on(h, EV_LET1, cs);
  h->stats.let_cells = rM;
  h->stats.let_particles = rPart;
  return FMM_OK;
}

// LET check (FMM_LET_CHECK=1): every remote multipole and particle the lists name was received
static int let_verify(fmm_ctx *h) {
  cudaStream_t st = h->stream;
  CK(h->let_missing.ensure(2));
  CK(cudaMemsetAsync(h->let_missing.p, 0, 2 * sizeof(int), st));
  launch_let_verify(h->lists(), (int)h->ntask[0], (int)h->ntask[1], (int)h->ntask[2], h->cells(),
                    h->strad_flag.p, h->own_lo, h->own_hi, h->let_haveM.p, h->let_haveP.p,
                    h->let_missing.p, st);
  CKL();
  int miss[2] = {0, 0};
  CK(cudaMemcpyAsync(miss, h->let_missing.p, sizeof miss, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (miss[0] || miss[1])
    return fail(h, FMM_E_INVALID, "local essential tree incomplete: %d multipoles, %d particle ranges missing",
                miss[0], miss[1]);
  return FMM_OK;
}

// results of the own particles (written by L2P in received order) back to the ranks that own
// them, then into the caller's order
static int dist_return(fmm_ctx *h, float *phi, float *grad) {
  const int64_t nloc = h->nloc;
  CK(h->sphi.ensure(std::max<int64_t>(nloc, 1)));
  CK(h->sgrad.ensure(3 * std::max<int64_t>(nloc, 1)));
  if (int rc = a2av(h, h->rphi.p, h->rcnt_p, h->sphi.p, h->scnt_p, sizeof(float))) return rc;
  if (int rc = a2av(h, h->rgrad.p, h->rcnt_p, h->sgrad.p, h->scnt_p, 3 * sizeof(float))) return rc;
  launch_scatter_results(h->sphi.p, h->sgrad.p, h->lperm.p, (int)nloc, phi, grad, h->stream);
  if (nloc > 0) CKL();
  return FMM_OK;
}

// ---- a9: traversal ----------------------------------------------------------------------------
static int traverse(fmm_ctx *h, int (*between)(fmm_ctx *) = nullptr) {
  // Level-synchronous target-centric traversal (traverse.cu), one kernel per level. All
  // bookkeeping stays on the device: list buffers are sized from the previous evaluation (or an
  // estimate), a target whose lists would not fit writes nothing, and one read-back at the end
  // decides whether to re-run with larger buffers (stack, scratch or lists) -- no host round trip
  // per level.
  cudaStream_t st = h->stream;
  const int nc = h->ncells;
  for (int k = 0; k < 3; ++k) {
    CK(h->loff[k].ensure(nc));
    CK(h->lcnt[k].ensure(nc));
    CK(cudaMemsetAsync(h->lcnt[k].p, 0, sizeof(int) * nc, st));
    CK(cudaMemsetAsync(h->loff[k].p, 0, sizeof(int) * nc, st));
  }
  CK(h->out_off.ensure(nc));
  CK(h->out_cnt.ensure(nc));
  CK(h->cpack.ensure((size_t)2 * nc));
  launch_pack_cells(nc, h->cells(), h->cpack.p, st);
  h->stats.launches += 1;
  const int warps_per_block = 4;
  const int grid_blocks = 148 * TRAV_GRID_PER_SM;
  const size_t nwarps = (size_t)grid_blocks * warps_per_block;
  // capacities: at least the previous evaluation's totals, else an estimate per target cell
  size_t cap[4];
  for (int k = 0; k < 4; ++k) {
    const size_t est = (size_t)h->trav_list_est * nc + 1024;
    cap[k] = std::max(est, h->trav_cap[k]);
    cap[k] = std::min(cap[k], (size_t)INT32_MAX - 1);
  }
  int list_attempts = 0;  // (scratch overflows are bounded by the 8 GiB check instead)
  for (;;) {
    CK(h->stack.ensure(nwarps * h->stack_cap));
    CK(h->trav_osc.ensure(nwarps * 4 * (size_t)h->trav_ocap));
    CK(h->trav_rsc.ensure(nwarps * (size_t)h->trav_ocap));
    for (int k = 0; k < 3; ++k) CK(h->lsrc[k].ensure(cap[k]));
    CK(h->p2p_rng.ensure(cap[2]));
    CK(h->outA.ensure(cap[3]));
    CK(h->outB.ensure(cap[3]));
    int hb[TRAV_BK_INTS] = {0};
    for (int k = 0; k < 4; ++k) hb[8 + k] = (int)cap[k];
    CK(cudaMemcpyAsync(h->d_bk, hb, sizeof hb, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(h->d_overflow, 0, sizeof(unsigned), st));
    CK(cudaMemsetAsync(h->d_stats, 0, 2 * sizeof(unsigned long long), st));
    unsigned *in_src = nullptr;
    DBuf<unsigned> *outbuf[2] = {&h->outA, &h->outB};
    for (int level = 0; level <= h->depth; ++level) {
      const int nt = h->level_cnt[level], t0 = h->level_off[level];
      TravArgs A{};
      A.C = h->cells();
      A.pk = h->cpack.p;
      A.t0 = t0;
      A.nt = nt;
      A.level = level;
      A.mode = h->mode;
      A.stack_cap = h->stack_cap;
      A.grid_blocks = std::min(grid_blocks, (nt + warps_per_block - 1) / warps_per_block);
      A.tlo = h->part_lo;
      A.tmask = h->ts_nt > 0 ? h->ntgt.p : nullptr;
      A.thi = h->part_hi;
      A.theta = h->theta;
      A.t_pp = h->cost.t_pp;
      A.t_mp = h->cost.t_mp;
      A.t_ml = h->cost.t_ml;
      A.in_src = in_src;
      A.in_off = h->out_off.p;
      A.in_cnt = h->out_cnt.p;
      A.scratch = h->stack.p;
      A.overflow = h->d_overflow;
      A.oscratch = h->trav_osc.p;
      A.rscratch = h->trav_rsc.p;
      A.ocap = h->trav_ocap;
      A.stats = h->d_stats;
      A.bk = h->d_bk;
      for (int k = 0; k < 3; ++k) {
        A.lsrc[k] = h->lsrc[k].p;
        A.loff[k] = h->loff[k].p;
        A.lcnt[k] = h->lcnt[k].p;
      }
      A.p2p_rng = h->p2p_rng.p;
      DBuf<unsigned> *ob = outbuf[level & 1];
      A.out_src = ob->p;
      A.out_off = h->out_off.p;
      A.out_cnt = h->out_cnt.p;
      CK(cudaMemsetAsync(h->d_bk + TRAV_CNT(3), 0, sizeof(int), st));  // this level's deferred pairs
      launch_traverse(A, st);
      CKL();
      in_src = ob->p;
    }
    record(h, EV_TRAV_END);
    // work that must not wait for the traversal (the sender-side LET exchange) is issued here,
    // after the first attempt has been queued and before the host waits for it
    if (between) {
      if (int rc = between(h)) return rc;
      between = nullptr;
    }
    int hb2[TRAV_BK_INTS];
    unsigned ovf = 0;
    unsigned long long hs[2];
    CK(cudaMemcpyAsync(hb2, h->d_bk, sizeof hb2, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&ovf, h->d_overflow, sizeof ovf, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hs, h->d_stats, sizeof hs, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (ovf) {  // a warp's stack (bit 1) or list scratch (bit 2) overflowed: larger ones, again
      if (ovf & 1u) h->stack_cap *= 2;
      if (ovf & 2u) h->trav_ocap *= 2;
      if ((size_t)h->stack_cap * nwarps > ((size_t)1 << 31) ||
          (size_t)h->trav_ocap * nwarps * 4 > ((size_t)1 << 31))
        return fail(h, FMM_E_OOM, "traversal scratch exceeds 8 GiB");
      continue;
    }
    if (hb2[12]) {  // a list buffer was too small: grow to what the count passes have seen so far
      // the counts only cover the levels up to the one that overflowed (later levels are dead):
      // grow 4x per attempt, at least to what has been seen
      if (++list_attempts > 16) return fail(h, FMM_E_OOM, "interaction lists do not fit");
      for (int k = 0; k < 4; ++k) {
        const size_t need = (size_t)(k < 3 ? hb2[TRAV_CNT(k)] : 0);
        cap[k] = std::min((size_t)INT32_MAX - 1, std::max(cap[k] * 4, 2 * need + 1024));
      }
      continue;
    }
    for (int k = 0; k < 3; ++k) {
      h->ntask[k] = hb2[TRAV_CNT(k)];
      h->trav_cap[k] = std::max(h->trav_cap[k], (size_t)hb2[TRAV_CNT(k)] + 1);
    }
    h->trav_cap[3] = std::max(h->trav_cap[3], cap[3]);
    h->stats.p2p_pairs = (int64_t)hs[0];
    h->stats.m2p_evals = (int64_t)hs[1];
    return FMM_OK;
  }
}

static bool m2l_scheme_ok(int p, int scheme) {
  switch (scheme) {
    case FMM_M2L_TC: return (m2l_gemm_supported(p) && m2l_tc_supported(p)) || m2l_tck_supported(p);
    case FMM_M2L_GEMM: return m2l_gemm_supported(p);
    case FMM_M2L_ROTATION: return m2l_rot_supported(p);
    case FMM_M2L_PAIRS: return true;
    default: return false;
  }
}
// the scheme an evaluation uses: the requested one, else the tuned one, else by order
static int m2l_scheme_of(const fmm_ctx *h) {
  if (h->m2l_scheme != FMM_M2L_AUTO) return h->m2l_scheme;
  const char *cc = getenv("FMM_M2L_CUDA_CORES");  // (round-1 switch, kept)
  if (cc && cc[0] && cc[0] != '0' && m2l_gemm_supported(h->p)) return FMM_M2L_GEMM;
  if (h->m2l_tuned) return h->m2l_tuned;
  if (m2l_scheme_ok(h->p, FMM_M2L_TC)) return FMM_M2L_TC;
  if (m2l_scheme_ok(h->p, FMM_M2L_GEMM)) return FMM_M2L_GEMM;
  return FMM_M2L_ROTATION;
}

// FMM_CHECK builds: publish the buffer capacities the device-side bounds checks test against
// (every translation unit holds its own copy); the capacities only grow within an evaluation
#ifdef FMM_CHECK
#include <map>
#include <mutex>
// the device-side bounds are device-global: with several live handles (in-process groups run
// their ranks on host threads) the published value is the maximum over the live handles
static std::mutex g_chk_mu;
static std::map<const void *, FmmChk> g_chk_live;
static void forget_chk(const void *h) {
  std::lock_guard<std::mutex> lk(g_chk_mu);
  g_chk_live.erase(h);
}
#else
static void forget_chk(const void *) {}
#endif
static void publish_chk(fmm_ctx *h, cudaStream_t st) {
#ifdef FMM_CHECK
  FmmChk c;
  c.pos = (long long)std::min(h->pos.cap, h->acc.cap);
  c.cells = (long long)h->cbeg.cap;
  c.rows = (long long)(std::min(h->M.cap, h->L.cap) / nc_stride(h->p));
  c.yrows = (long long)(h->m2l_Y.cap / m2l_y_stride(h->p));
  c.lists = (long long)h->p2p_rng.cap;
  if (getenv("FMM_CHECK_SELFTEST")) c.pos = 1;  // tests: a bound every evaluation violates
  {
    std::lock_guard<std::mutex> lk(g_chk_mu);
    g_chk_live[h] = c;
    for (const auto &kv : g_chk_live) {
      c.pos = std::max(c.pos, kv.second.pos);
      c.cells = std::max(c.cells, kv.second.cells);
      c.rows = std::max(c.rows, kv.second.rows);
      c.yrows = std::max(c.yrows, kv.second.yrows);
      c.lists = std::max(c.lists, kv.second.lists);
    }
  }
  fmm_chk_set_p2p(c, st);
  fmm_chk_set_m2l_tc(c, st);
  fmm_chk_set_m2l(c, st);
  fmm_chk_set_traverse(c, st);
  fmm_chk_set_expansions(c, st);
#else
  (void)h;
  (void)st;
#endif
}

static int evaluate_tree(fmm_ctx *h, const float *xyz, const float *q, int64_t n, float *phi,
                         float *grad) {
  cudaStream_t st = h->stream;
  const int p = h->p, NC = nc_of(p);
  if (h->comm) {
    if (int rc = dist_build_tree(h, xyz, q, n)) return rc;
  } else {
    if (int rc = build_tree(h, xyz, q, n)) return rc;
  }
  record(h, EV_TREE);
  const int NCS = nc_stride(p);
  CK(h->M.ensure((size_t)h->ncells * NCS));
  CK(h->L.ensure((size_t)h->ncells * NCS));
  publish_chk(h, st);
  // a7/a8 upward sweep, on the aux stream: it overlaps the traversal and the M2L class sort (which
  // do not read M); the stream joins before the first kernel that reads M
  CK(cudaEventRecord(h->ev_fork, st));
  CK(cudaStreamWaitEvent(h->aux, h->ev_fork, 0));
  cudaStream_t ua = h->aux;
  // (distributed: every cell starts at zero -- only the own leaves get a P2M, so the M2M leaves
  // straddling cells with this rank's partial sum and remote cells at zero)
  if (NCS != NC || h->comm) CK(cudaMemsetAsync(h->M.p, 0, sizeof(float2) * (size_t)h->ncells * NCS, ua));
  // M2M / L2L: octant-class GEMMs on the tensor cores (p <= 10) unless disabled
  const char *scc = getenv("FMM_SHIFT_CUDA_CORES");
  const bool cart = h->basis == FMM_BASIS_CARTESIAN;
  const bool shift_tc = !cart && m2l_tc_supported(p) && h->ncells > 1 && !(scc && scc[0] && scc[0] != '0');
  const int CSt = cart_stride(p);
  if (cart) {
    CK(h->Mc.ensure((size_t)h->ncells * CSt));
    CK(h->Lc.ensure((size_t)h->ncells * CSt));
  }
  TcShiftWork S{};
  if (shift_tc) {
    const size_t tw = m2l_tc_T_words(p);
    if (h->sh_T_p != p) {
      CK(h->sh_T.ensure(16 * tw));
      CK(tc_shift_build_ops(p, h->sh_T.p, h->sh_T.p + 8 * tw, ua));
      h->stats.launches += 1;
      h->sh_T_p = p;
    }
    const int ns = h->ncells - 1;
    S.items_per_level = tc_shift_items_per_level(h->ncells);
    CK(h->sh_keys_in.ensure(ns));
    CK(h->sh_keys.ensure(ns));
    CK(h->sh_vals_in.ensure(ns));
    CK(h->sh_cells.ensure(ns));
    CK(h->sh_src.ensure(ns));
    CK(h->sh_items.ensure((size_t)(FMM_LEVELS + 2) * S.items_per_level));
    CK(h->sh_counters.ensure((size_t)(FMM_LEVELS + 2) * 8));
    CK(h->cub_tmp_aux.ensure(tc_shift_sort_bytes(ns)));
    CK(h->sh_Y.ensure((size_t)h->ncells * m2l_y_stride(p)));
    S.keys_in = h->sh_keys_in.p;
    S.keys = h->sh_keys.p;
    S.vals_in = h->sh_vals_in.p;
    S.cells = h->sh_cells.p;
    S.src_l2l = h->sh_src.p;
    S.items = h->sh_items.p;
    S.lvl_counters = h->sh_counters.p;
    S.Tm2m = h->sh_T.p;
    S.Tl2l = h->sh_T.p + 8 * tw;
    S.tmp = h->cub_tmp_aux.p;
    S.tmp_bytes = h->cub_tmp_aux.cap;
    CK(tc_shift_prepare(h->ncells, h->depth, S, h->cells(), ua));
    h->stats.launches += 3;
    h->stats.cub_calls += 1;
  }
  if (cart) launch_cart_p2m(p, h->leaves.p, h->nleaves, h->cells(), h->pos.p, h->Mc.p, ua);
  else if (h->comm) launch_p2m(p, h->tleaves.p, h->tleaves_n, h->cells(), h->pos.p, h->M.p, ua);
  else launch_p2m(p, h->leaves.p, h->nleaves, h->cells(), h->pos.p, h->M.p, ua);
  CKL();
  for (int level = h->depth - 1; level >= 0; --level) {
    if (cart) {
      launch_cart_m2m(p, h->level_off[level], h->level_cnt[level], h->cells(), h->Mc.p, ua);
    } else if (shift_tc) {
      CK(tc_shift_m2m_level(p, level, h->level_off[level], h->level_cnt[level], h->cells(), S,
                            h->M.p, h->sh_Y.p, ua));
      h->stats.launches += 2;
    } else {
      launch_m2m(p, h->level_off[level], h->level_cnt[level], h->cells(), h->M.p, ua);
    }
    CKL();
  }
  record_on(h, EV_UP, ua);
  CK(cudaEventRecord(h->ev_up, ua));
  if (h->comm && !h->let_recv) {
    // sender-side local essential tree: exchanged on its own stream while the traversal runs;
    // everything that reads remote sources (P2P, M2P, M2L) waits for it
    if (int rc = traverse(h, let_send)) return rc;
    CK(cudaStreamWaitEvent(st, h->ev_let, 0));
    if (h->let_check)
      if (int rc = let_verify(h)) return rc;
  } else {
    if (int rc = traverse(h)) return rc;
    if (h->comm) {  // receiver-driven local essential tree: what this rank's lists name
      if (int rc = dist_let(h)) return rc;
    }
  }
  record(h, EV_TRAV);
  // a12 P2P (writes acc), a11 M2P (adds): on the aux stream (after the upward sweep there) when
  // overlapping, so that they run while the main stream sorts the M2L pairs into classes
  const int *tl = (h->nparts > 1 || h->comm || h->ts_nt > 0) ? h->tleaves.p : h->leaves.p;
  const int ntl = h->tleaves_n;
  auto near_field = [&](cudaStream_t ns) -> int {
    record_on(h, EV_P2P0, ns);
    CK(h->p2p_desc.ensure(std::max(ntl, 1)));
    CK(h->p2p_mrg.ensure(std::max(h->p2p_rng.cap, (size_t)1)));
    launch_p2p_leaves(tl, ntl, h->cells(), h->lists(), h->pos.p, h->acc.p, h->d_small + 12,
                      h->p2p_desc.p, h->p2p_mrg.p, ns, h->timing ? h->ev[EV_P2PK] : nullptr);
    h->stats.launches += 1;  // + the per-leaf descriptor and range-merge passes
    CKL();
    record_on(h, EV_P2P, ns);
    if (h->ntask[FMM_KIND_M2P] > 0) {
      CK(cudaStreamWaitEvent(ns, h->ev_up, 0));  // M2P reads the multipoles
      if (cart)
        launch_cart_m2p(p, tl, ntl, h->cells(), h->lists(), h->pos.p, h->Mc.p, h->acc.p,
                        h->d_small + 13, ns);
      else
        launch_m2p(p, tl, ntl, h->cells(), h->lists(), h->pos.p, h->M.p, h->acc.p, h->d_small + 13, ns);
      CKL();
    }
    record_on(h, EV_M2P, ns);
    return FMM_OK;
  };
  publish_chk(h, st);  // (list capacities after the traversal's retries)
  if (h->overlap) {
    CK(cudaEventRecord(h->ev_trav, st));
    CK(cudaStreamWaitEvent(h->nf, h->ev_trav, 0));
    if (int rc = near_field(h->nf)) return rc;
    CK(cudaEventRecord(h->ev_near, h->nf));
  }
  record(h, EV_M2L_PREP);  // re-recorded after the class sort when there are M2L pairs
  // a10 M2L (writes every cell's local expansion, zero where no M2L)
  const bool far_local = h->ntask[FMM_KIND_M2L] > 0;
  if (far_local && cart) {  // Cartesian: one warp per target over its list (cart.cu), no classes
    CK(cudaStreamWaitEvent(st, h->ev_up, 0));
    record(h, EV_M2L_PREP);
    launch_cart_m2l(p, h->ncells, h->cells(), h->lists(), h->Mc.p, h->Lc.p, st);
    CKL();
  } else if (far_local) {
    const int np = (int)h->ntask[FMM_KIND_M2L];
    CK(h->m2l_pair_t.ensure(np));
    CK(h->m2l_pst.ensure(np));
    CK(h->m2l_keys_in.ensure(np));
    CK(h->m2l_keys.ensure(np));
    CK(h->m2l_idx_in.ensure(np));
    CK(h->m2l_sidx.ensure(np));
    CK(h->m2l_flag.ensure(np));
    CK(h->m2l_cid.ensure(np));
    CK(h->m2l_cstart.ensure((size_t)np + 1));
    CK(h->m2l_counters.ensure(8));
    CK(h->m2l_items.ensure((size_t)np + 1));
    CK(h->m2l_small.ensure(np));
    // translation scheme (fmm_set_m2l_scheme; tuned by fmm_tune): tensor-core class GEMM,
    // CUDA-core class GEMM, rotation-based O(p^3) (m2l_rot.cu) or the per-pair double loop
    const int scheme = m2l_scheme_of(h);
    const bool use_tc = scheme == FMM_M2L_TC;
    const bool use_rot = scheme == FMM_M2L_ROTATION;
    // tensor-core GEMMs and rotations accumulate straight into L unless bit-reproducibility is
    // requested
    const bool accum = (use_tc || use_rot) && !h->deterministic;
    if (!accum) CK(h->m2l_Y.ensure((size_t)np * m2l_y_stride(p)));
    publish_chk(h, st);
    CK(h->cub_tmp.ensure(m2l_temp_bytes(np)));
    M2LWork W{};
    W.C = h->cells();
    W.off = h->loff[0].p;
    W.cnt = h->lcnt[0].p;
    W.src = h->lsrc[0].p;
    W.pair_t = h->m2l_pair_t.p;
    W.pst = h->m2l_pst.p;
    W.keys_in = h->m2l_keys_in.p;
    W.keys = h->m2l_keys.p;
    W.idx_in = h->m2l_idx_in.p;
    W.sidx = h->m2l_sidx.p;
    W.flag = h->m2l_flag.p;
    W.cid = h->m2l_cid.p;
    W.cstart = h->m2l_cstart.p;
    W.counters = h->m2l_counters.p;
    W.items = h->m2l_items.p;
    W.small = h->m2l_small.p;
    W.Y = h->m2l_Y.p;
    W.tmp = h->cub_tmp.p;
    W.tmp_bytes = h->cub_tmp.cap;
    W.direct_all = scheme == FMM_M2L_PAIRS ? 1 : 0;
    // spatial blocks for the execution order: none while the multipole + local arrays fit
    // comfortably in L2 (126 MB); else the 8 octants of the root (FMM_M2L_BLK overrides, <= 2)
    {
      const double bytes = 2.0 * h->ncells * NCS * sizeof(float2);
      // (measured at C4 / C5: one level of 8 blocks cuts the M2L time by 30-40 %; finer blocks
      // make the per-item class-matrix loads dominate)
      int bl = bytes > 96e6 ? 1 : 0;
      const char *eb = getenv("FMM_M2L_BLK");
      if (eb && eb[0]) bl = std::max(0, std::min(2, atoi(eb)));
      W.blk_level = bl;
    }
    CK(h->m2l_rflag.ensure(np));
    CK(h->m2l_rid.ensure(np));
    CK(h->m2l_rstart.ensure((size_t)np + 1));
    CK(h->m2l_gid_of.ensure(np));
    CK(h->m2l_items_raw.ensure((size_t)np + 1));
    CK(h->m2l_ikeys_in.ensure((size_t)np + 1));
    CK(h->m2l_ikeys.ensure((size_t)np + 1));
    CK(h->m2l_iidx_in.ensure((size_t)np + 1));
    CK(h->m2l_iidx.ensure((size_t)np + 1));
    W.rflag = h->m2l_rflag.p;
    W.rid = h->m2l_rid.p;
    W.rstart = h->m2l_rstart.p;
    W.gid_of = h->m2l_gid_of.p;
    W.items_raw = h->m2l_items_raw.p;
    W.ikeys_in = h->m2l_ikeys_in.p;
    W.ikeys = h->m2l_ikeys.p;
    W.iidx_in = h->m2l_iidx_in.p;
    W.iidx = h->m2l_iidx.p;
    CK(h->m2l_class_rep.ensure(np));
    CK(h->m2l_ssrc.ensure(np));
    W.class_rep = h->m2l_class_rep.p;
    W.ssrc = h->m2l_ssrc.p;
    if (accum) {
      CK(h->m2l_stgt.ensure(np));
      W.stgt = h->m2l_stgt.p;
      static const bool idx_sort = getenv("FMM_M2L_IDXSORT") != nullptr;  // (A/B: round-2 path)
      if (!idx_sort) {
        CK(h->m2l_spst.ensure(np));
        W.spst = h->m2l_spst.p;
      }
    }
    W.compact_key = h->m2l_compact_key ? 1 : 0;
    CK(m2l_prepare(W, np, h->ncells, st));
    if (W.spst) {
      // the class representatives and the direct-path list hold class-sorted positions
      W.pair_t = reinterpret_cast<int *>(W.stgt);
      W.src = W.ssrc;
    }
    h->stats.launches += 6;
    h->stats.cub_calls += 2;
    CK(cudaMemcpyAsync(h->h_small, h->m2l_counters.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int ngclass = h->h_small[3];
    h->m2l_compact_key = h->h_small[6] == 0;  // the next evaluation's class-key width
    CK(m2l_sort_items(W, h->h_small[1], st));
    h->stats.launches += 1;
    h->stats.cub_calls += 1;
    // class GEMMs on the tensor cores (tcgen05, 3xTF32), or per-class rotation operators, or
    // CUDA-core class GEMMs
    // (10 < p <= 15: the K-tiled tensor-core GEMM, float-order operators and Y rows)
    const bool use_tck = use_tc && !m2l_tc_supported(p);
    if (use_tck) {
      CK(h->m2l_Ttc.ensure((size_t)std::max(1, ngclass) * m2l_tck_T_words(p)));
      CK(m2l_tck_build_T(p, W, ngclass, h->m2l_Ttc.p, st));
    } else if (use_tc) {
      CK(h->m2l_Ttc.ensure((size_t)std::max(1, ngclass) * m2l_tc_T_words(p)));
      CK(m2l_tc_build_T(p, W, ngclass, h->m2l_Ttc.p, st));
    } else if (use_rot) {
      CK(h->m2l_R.ensure((size_t)std::max(1, ngclass) * m2l_rot_class_floats(p)));
      CK(m2l_rot_build(p, W, ngclass, h->m2l_R.p, st));
    } else if (scheme == FMM_M2L_GEMM) {
      CK(h->m2l_T.ensure((size_t)std::max(1, ngclass) * m2l_T_floats(p)));
      W.Tg = h->m2l_T.p;
      CK(m2l_build_T(p, W, ngclass, st));
    }
    h->stats.launches += 1;
    if (accum) CK(cudaMemsetAsync(h->L.p, 0, sizeof(float2) * (size_t)h->ncells * NCS, st));
    CK(cudaStreamWaitEvent(st, h->ev_up, 0));  // join: the multipoles are complete
    record(h, EV_M2L_PREP);  // ms_m2l = the GEMM (+ the rare-class direct path / reduction)
    if (use_tck) {
      CK(m2l_tck_gemm(p, W, h->m2l_Ttc.p, h->M.p, st, accum ? h->L.p : nullptr));
      h->stats.launches += 1;
    } else if (use_tc) {
      CK(m2l_tc_gemm(p, W, h->m2l_Ttc.p, h->M.p, st, accum ? h->L.p : nullptr));
      h->stats.launches += 1;
    } else if (use_rot) {
      CK(m2l_rot_apply(p, W, h->m2l_R.p, h->M.p, st, accum ? h->L.p : nullptr));
      h->stats.launches += 1;
    }
    // (gemm_done: the class pairs are done and Y holds dof-order rows; rare classes, the
    // per-pair scheme and the ordered reduction follow)
    CK(m2l_execute(p, W, np, h->ncells, h->M.p, h->L.p, st, use_tc || use_rot, accum,
                   use_tck ? 0 : -1));
    h->stats.launches += 2;
    h->m2l_tc_used = use_tc;
  }
  CK(cudaStreamWaitEvent(st, h->ev_up, 0));  // (no M2L pairs: join here)
  record(h, EV_M2L);
  if (!h->overlap) {
    if (int rc = near_field(st)) return rc;
  }
  // a13 L2L top-down, a14/a15 L2P + combine + un-permute
  if (far_local) {
    for (int level = 1; level <= h->depth; ++level) {
      if (cart) {
        launch_cart_l2l(p, h->level_off[level], h->level_cnt[level], h->cells(), h->Lc.p, st);
      } else if (shift_tc) {
        CK(tc_shift_l2l_level(p, level, h->level_off[level], h->level_cnt[level], S, h->L.p,
                              h->sh_Y.p, st));
        h->stats.launches += 2;
      } else {
        launch_l2l(p, h->level_off[level], h->level_cnt[level], h->cells(), h->L.p, st);
      }
      CKL();
    }
  }
  float *ophi = phi, *ograd = grad;
  if (h->comm) {  // results in received order, routed back to the owners below
    const int64_t nown = std::max(h->own_hi - h->own_lo, 1);
    CK(h->rphi.ensure(nown));
    CK(h->rgrad.ensure(3 * nown));
    ophi = h->rphi.p;
    ograd = h->rgrad.p;
  }
  if (h->overlap) CK(cudaStreamWaitEvent(st, h->ev_near, 0));  // join: acc is complete
  if (cart)
    launch_cart_l2p(p, tl, ntl, h->cells(), h->pos.p, h->Lc.p, h->acc.p, h->perm.p, ophi, ograd,
                    far_local ? 1 : 0, st);
  else
    launch_l2p(p, tl, ntl, h->cells(), h->pos.p, h->L.p, h->acc.p, h->perm.p, ophi,
               ograd, far_local ? 1 : 0, st);
  CKL();
  if (h->comm) {
    if (int rc = dist_return(h, phi, grad)) return rc;
  }
  record(h, EV_DOWN);
  h->have_tree = true;
  return FMM_OK;
}

static void read_phase_times(fmm_ctx *h);
static int evaluate_run(fmm_ctx *h, const float *xyz, const float *q, int64_t n, float *phi,
                        float *grad);
// One evaluation: the work runs on the handle's high-priority stream, ordered after everything
// already queued on the caller's stream, and the caller's stream waits for it at the end.
static int evaluate_impl(fmm_ctx *h, const float *xyz, const float *q, int64_t n, float *phi,
                         float *grad) {
  cudaStream_t user = h->stream;
  CK(cudaEventRecord(h->ev_in, user));
  CK(cudaStreamWaitEvent(h->hi, h->ev_in, 0));
  h->stream = h->hi;
  const int rc = evaluate_run(h, xyz, q, n, phi, grad);
  h->stream = user;
  CK(cudaEventRecord(h->ev_out, h->hi));
  CK(cudaStreamWaitEvent(user, h->ev_out, 0));
  return rc;
}

static int evaluate_run(fmm_ctx *h, const float *xyz, const float *q, int64_t n, float *phi,
                        float *grad) {
  cudaStream_t st = h->stream;
  memset(&h->stats, 0, sizeof h->stats);
  h->stats.n = n;
  h->stats.p = h->p;
  if (h->comm) {  // collective: every rank runs the pipeline, also with an empty shard
    if (h->mode == FMM_DIRECT) return fail(h, FMM_E_INVALID, "FMM_DIRECT on a distributed handle");
    record(h, EV_START);
    h->last_n = n;
    if (int rc = evaluate_tree(h, xyz, q, n, phi, grad)) return rc;
    h->stats.ncells = h->ncells;
    h->stats.nleaves = h->nleaves;
    h->stats.depth = h->depth;
    h->stats.n_m2l = h->ntask[0];
    h->stats.n_m2p = h->ntask[1];
    h->stats.n_p2p = h->ntask[2];
    CK(cudaStreamSynchronize(st));
    if (h->timing) read_phase_times(h);
    return FMM_OK;
  }
  if (n == 0) return FMM_OK;
  if (n > (int64_t)1 << 28) return fail(h, FMM_E_INVALID, "n = %lld exceeds 2^28 per device", (long long)n);
  record(h, EV_START);
  launch_bbox(xyz, q, n, h->d_mm, h->d_root, st);  // 3 kernels
  h->stats.launches += 2;
  CKL();
  CK(cudaMemcpyAsync(&h->h_root, h->d_root, sizeof(RootInfo), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h->h_root.nonfinite) return fail(h, FMM_E_NONFINITE, "non-finite coordinate or charge");
  h->last_n = n;
  if (h->mode == FMM_DIRECT) {
    CK(h->pos.ensure(n));
    launch_gather(xyz, q, nullptr, n, h->pos.p, st);
    CKL();
    record(h, EV_TREE);
    record(h, EV_UP);
    record(h, EV_TRAV);
    record(h, EV_M2L_PREP);
    record(h, EV_M2L);
    record(h, EV_P2P0);
    launch_p2p_direct(n, h->pos.p, phi, grad, st);
    CKL();
    record(h, EV_P2P);
    record(h, EV_M2P);
    record(h, EV_DOWN);
    h->have_tree = false;
    h->stats.p2p_pairs = n * n;
    h->stats.n_p2p = 1;
  } else {
    if (int rc = evaluate_tree(h, xyz, q, n, phi, grad)) return rc;
    h->stats.ncells = h->ncells;
    h->stats.nleaves = h->nleaves;
    h->stats.depth = h->depth;
    h->stats.n_m2l = h->ntask[0];
    h->stats.n_m2p = h->ntask[1];
    h->stats.n_p2p = h->ntask[2];
  }
  CK(cudaStreamSynchronize(st));
  if (h->timing) read_phase_times(h);
  return FMM_OK;
}

static void read_phase_times(fmm_ctx *h) {
  auto el = [&](int a, int b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev[a], h->ev[b]);
    return (double)ms;
  };
  h->stats.ms_total = el(EV_START, EV_DOWN);
  h->stats.ms_tree = el(EV_START, EV_TREE);
  // the upward sweep (aux stream) overlaps the traversal: both are measured from EV_TREE
  h->stats.ms_upward = el(EV_TREE, EV_UP);
  // traversal (+ the class sort when P2P does not overlap it; overlapped, the sort's time is
  // hidden under P2P and not attributed to any phase)
  h->stats.ms_traverse = el(EV_TREE, EV_TRAV) + (h->overlap ? 0.0 : el(EV_TRAV, EV_M2L_PREP));
  h->stats.ms_m2l = el(EV_M2L_PREP, EV_M2L);
  // P2P / M2P: their own events (on aux when overlapping the M2L, which the phases then do)
  h->stats.ms_p2p = el(EV_P2P0, EV_P2P);
  h->stats.ms_p2p_kernel = h->ntask[2] > 0 && h->mode != FMM_DIRECT ? el(EV_P2PK, EV_P2P) : 0.0;
  h->stats.ms_m2p = el(EV_P2P, EV_M2P);
  h->stats.ms_downward = (h->overlap && h->mode != FMM_DIRECT) ? el(EV_M2L, EV_DOWN) : el(EV_M2P, EV_DOWN);
  if (h->comm && !h->let_recv && h->mode != FMM_DIRECT) {
    // the sender-side exchange and how far it ran past the traversal (0 = completely hidden)
    h->stats.ms_let = el(EV_LET0, EV_LET1);
    h->stats.ms_let_exposed = std::max(0.0, el(EV_TRAV_END, EV_LET1));
  }
}

// ---- a6: kernel pre-calculation ------------------------------------
// The kernels are timed on artificial data at a saturating size (P:189 warns that small tests
// mispredict GPU times): a synthetic uniform cube of 2^20 random particles is evaluated in FMM
// mode (every accepted pair an M2L) and in treecode mode (every accepted pair an M2P); the
// per-unit costs are the kernel times (CUDA events, median of 3 after a warm-up) divided by the
// work counts the traversal reports.
static int tune_impl(fmm_ctx *h) {
  const int64_t n = (int64_t)1 << 20;
  float *d = nullptr;
  CK(cudaMalloc(&d, sizeof(float) * 8 * n));
  float *xyz = d, *q = d + 3 * n, *phi = d + 4 * n, *grad = d + 5 * n;
  launch_fill_random(xyz, 3 * n, 12345u, 0.f, 1.f, h->stream);
  launch_fill_random(q, n, 777u, 1.0f / n, 1.0f / n, h->stream);
  CKL();
  const int saved_mode = h->mode;
  const bool saved_timing = h->timing, saved_overlap = h->overlap;
  h->overlap = false;  // each kernel timed alone
  h->timing = true;
  // (median of TUNE_REPS timed evaluations per mode: 3 gave a ~15% spread of t_pp between
  // processes, and the hybrid lists -- hence the step time -- follow the measured costs)
  constexpr int TUNE_REPS = 5;
  double t_pp[TUNE_REPS], t_ml[TUNE_REPS], t_mp[TUNE_REPS];
  int rc = FMM_OK;
  // auto-tuning across translation schemes (NEXT-1): the M2L phase of one FMM-mode
  // evaluation with every scheme that supports this order, the fastest is kept
  if (h->m2l_scheme == FMM_M2L_AUTO && h->basis == FMM_BASIS_SPHERICAL) {
    h->mode = FMM_FMM;
    h->m2l_tuned = 0;
    double best = 1e300;
    int pick = 0;
    for (int sc = FMM_M2L_TC; sc <= FMM_M2L_PAIRS && rc == FMM_OK; ++sc) {
      h->m2l_scheme_ms[sc] = 0.0;
      if (!m2l_scheme_ok(h->p, sc)) continue;
      h->m2l_scheme = sc;
      double t[2] = {0, 0};
      for (int it = 0; it < 3 && rc == FMM_OK; ++it) {
        rc = evaluate_impl(h, xyz, q, n, phi, grad);
        if (it) t[it - 1] = h->stats.ms_m2l;
      }
      h->m2l_scheme_ms[sc] = std::min(t[0], t[1]);
      if (h->m2l_scheme_ms[sc] < best) {
        best = h->m2l_scheme_ms[sc];
        pick = sc;
      }
      // the per-pair double loop is only a candidate when no class scheme is faster than it
      // could be: stop at the first class-batched scheme that ran (it is far ahead at p >= 4)
    }
    h->m2l_scheme = FMM_M2L_AUTO;
    h->m2l_tuned = pick;
  }
  for (int pass = 0; pass < 2 && rc == FMM_OK; ++pass) {
    h->mode = pass == 0 ? FMM_FMM : FMM_TREECODE;
    for (int it = -1; it < TUNE_REPS && rc == FMM_OK; ++it) {
      rc = evaluate_impl(h, xyz, q, n, phi, grad);
      if (it < 0 || rc) continue;
      const fmm_stats_t &s = h->stats;
      if (pass == 0) {
        t_pp[it] = s.ms_p2p * 1e-3 / std::max<int64_t>(1, s.p2p_pairs);
        t_ml[it] = s.ms_m2l * 1e-3 / std::max<int64_t>(1, s.n_m2l);
      } else {
        t_mp[it] = s.ms_m2p * 1e-3 / std::max<int64_t>(1, s.m2p_evals);
      }
    }
  }
  h->mode = saved_mode;
  h->timing = saved_timing;
  h->overlap = saved_overlap;
  cudaFree(d);
  if (rc) return rc;
  auto med = [](double *a) {
    std::sort(a, a + TUNE_REPS);
    return a[TUNE_REPS / 2];
  };
  h->cost.t_pp = med(t_pp);
  h->cost.t_ml = med(t_ml);
  h->cost.t_mp = med(t_mp);
  h->cost.p = h->p;
  h->cost.measured = 1;
  h->have_tree = false;
  return FMM_OK;
}

// FMM_BASIS_AUTO (NEXT-2: switching to Cartesian expansions is "key to achieving
// high performance for low-accuracy"): each candidate basis gets its own kernel pre-calculation,
// then one hybrid evaluation of the same 2^20 synthetic particles is timed (median of 3, CUDA
// events) and the faster basis is kept with its cost model.
static int auto_basis_impl(fmm_ctx *h) {
  if (!cart_supported(h->p) || h->comm) {
    h->basis = FMM_BASIS_SPHERICAL;
    return FMM_OK;
  }
  const int64_t n = (int64_t)1 << 20;
  float *d = nullptr;
  CK(cudaMalloc(&d, sizeof(float) * 8 * n));
  float *xyz = d, *q = d + 3 * n, *phi = d + 4 * n, *grad = d + 5 * n;
  launch_fill_random(xyz, 3 * n, 4242u, 0.f, 1.f, h->stream);
  launch_fill_random(q, n, 4343u, 1.0f / n, 1.0f / n, h->stream);
  fmm_cost_t cost[2];
  int rc = FMM_OK;
  const int saved_mode = h->mode;
  const bool saved_timing = h->timing;
  for (int b = 0; b < 2 && rc == FMM_OK; ++b) {
    h->basis = b;
    rc = tune_impl(h);
    cost[b] = h->cost;
    h->mode = FMM_HYBRID;
    h->timing = true;
    double t[3] = {0, 0, 0};
    for (int it = -1; it < 3 && rc == FMM_OK; ++it) {
      rc = evaluate_impl(h, xyz, q, n, phi, grad);
      if (it >= 0) t[it] = h->stats.ms_total;
    }
    std::sort(t, t + 3);
    h->basis_ms[b] = t[1];
    h->mode = saved_mode;
    h->timing = saved_timing;
  }
  cudaFree(d);
  if (rc) return rc;
  h->basis = h->basis_ms[1] < h->basis_ms[0] ? FMM_BASIS_CARTESIAN : FMM_BASIS_SPHERICAL;
  h->cost = cost[h->basis];
  h->have_tree = false;
  return FMM_OK;
}

// ================================ C ABI =========================================================
extern "C" {

int fmm_create(fmm_t *out, int p, double theta, int ncrit) {
  if (!out) return FMM_E_INVALID;
  *out = nullptr;
  if (p < 1 || p > FMM_P_MAX || !(theta > 0.0 && theta < 1.0) || ncrit < 1) return FMM_E_INVALID;
  fmm_ctx *h = new (std::nothrow) fmm_ctx();
  if (!h) return FMM_E_OOM;
  h->p = p;
  h->theta = theta;
  h->ncrit = ncrit;
  h->tiles = make_m2l_tiles(p);
  // default cost model until measured: ~B200 order of magnitude (overwritten by the tuning)
  h->cost.t_pp = 2e-12;
  h->cost.t_mp = 5e-11;
  h->cost.t_ml = 3e-9;
  h->cost.p = p;
  h->cost.measured = 0;
  int rc = FMM_OK;
  do {
    cudaError_t e;
    if ((e = cudaGetDevice(&h->device)) != cudaSuccess) { rc = fail(h, FMM_E_CUDA, "%s", cudaGetErrorString(e)); break; }
    if ((e = cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking)) != cudaSuccess) { rc = fail(h, FMM_E_CUDA, "%s", cudaGetErrorString(e)); break; }
    h->stream = h->own_stream;
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    // the upward sweep (aux) feeds the M2L GEMM: as urgent as the main pipeline; the near field
    // (nf) only has to finish before L2P
    if ((e = cudaStreamCreateWithPriority(&h->aux, cudaStreamNonBlocking, prio_hi)) != cudaSuccess ||
        (e = cudaStreamCreateWithPriority(&h->nf, cudaStreamNonBlocking, prio_lo)) != cudaSuccess ||
        (e = cudaStreamCreateWithPriority(&h->hi, cudaStreamNonBlocking, prio_hi)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&h->ev_up, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&h->ev_trav, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&h->ev_near, cudaEventDisableTiming)) != cudaSuccess) {
      rc = fail(h, FMM_E_CUDA, "%s", cudaGetErrorString(e));
      break;
    }
    for (int i = 0; i < EV_N; ++i) cudaEventCreate(&h->ev[i]);
    if (cudaMalloc(&h->d_root, sizeof(RootInfo)) || cudaMalloc(&h->d_mm, 8 * sizeof(unsigned)) ||
        cudaMalloc(&h->d_small, 16 * sizeof(int)) || cudaMalloc(&h->d_overflow, sizeof(unsigned)) ||
        cudaMalloc(&h->d_stats, 4 * sizeof(unsigned long long)) ||
        cudaMalloc(&h->d_bk, TRAV_BK_INTS * sizeof(int)) ||
        cudaMalloc(&h->d_tree_st, 64 * sizeof(int)) ||
        cudaMallocHost(&h->h_small, 16 * sizeof(int))) {
      rc = fail(h, FMM_E_OOM, "small device allocations failed");
      break;
    }
    // test hooks: small initial traversal scratch / list estimates force the overflow-and-retry
    // paths of traverse() (tests/test_gpu_sanitize.py)
    if (const char *v = getenv("FMM_TRAV_CAP")) h->stack_cap = h->trav_ocap = std::max(32, atoi(v));
    if (const char *v = getenv("FMM_TRAV_LIST_EST")) h->trav_list_est = std::max(1, atoi(v));
    if (const char *v = getenv("FMM_LET")) h->let_recv = strcmp(v, "recv") == 0;
    if (const char *v = getenv("FMM_LET_CHECK")) h->let_check = v[0] && v[0] != '0';
    const char *no = getenv("FMM_NO_OVERLAP");
    h->overlap = !(no && no[0] && no[0] != '0');
    const char *nt = getenv("FMM_NO_TUNE");
    if (!(nt && nt[0] && nt[0] != '0')) rc = tune_impl(h);
  } while (0);
  if (rc != FMM_OK) {
    fmm_destroy(h);
    return rc;
  }
  *out = h;
  return FMM_OK;
}

int fmm_destroy(fmm_t h) {
  if (!h) return FMM_OK;
  forget_chk(h);
  DeviceGuard dg(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->keys_in.release(); h->keys.release(); h->idx_in.release(); h->perm.release();
  h->sort_runs.release();
  h->pos.release(); h->acc.release(); h->cub_tmp.release(); h->host_stage.release();
  h->cbeg.release(); h->ccnt.release(); h->cparent.release(); h->cchild0.release();
  h->cnchild.release(); h->cgrid.release(); h->cgeo.release(); h->cprefix.release(); h->cpack.release();
  h->tleaves.release(); h->p2p_desc.release(); h->p2p_mrg.release(); h->tc_bnd.release(); h->tc_crange.release();
  if (h->d_tree_st) cudaFree(h->d_tree_st); h->Mc.release(); h->Lc.release(); h->m2l_R.release();
  h->let_box.release(); h->let_flags.release(); h->let_excl.release(); h->let_cnt.release();
  h->let_psize.release(); h->let_pexcl.release(); h->let_seg0.release(); h->let_haveM.release();
  h->let_haveP.release(); h->let_open.release(); h->let_ids.release(); h->let_rids.release();
  h->let_prng.release(); h->let_prec.release(); h->let_rrec.release(); h->let_rows_s.release();
  h->let_rows_r.release(); h->let_pbuf_s.release(); h->let_pbuf_r.release(); h->let_missing.release();
  if (h->let_tmp) cudaFree(h->let_tmp);
  if (h->cmst) cudaStreamDestroy(h->cmst);
  if (h->ev_let) cudaEventDestroy(h->ev_let);
  h->nch.release(); h->bnd.release(); h->excl.release(); h->leafflag.release(); h->leaves.release(); h->crange.release();
  h->M.release(); h->L.release();
  h->ntgt.release(); h->ts_stage.release();
  h->m2l_pair_t.release(); h->m2l_pst.release(); h->m2l_spst.release(); h->m2l_flag.release(); h->m2l_cid.release(); h->m2l_cstart.release();
  h->m2l_counters.release(); h->m2l_keys_in.release(); h->m2l_keys.release();
  h->m2l_idx_in.release(); h->m2l_sidx.release(); h->m2l_small.release(); h->m2l_items.release();
  h->m2l_items_raw.release(); h->m2l_rflag.release(); h->m2l_rid.release(); h->m2l_rstart.release();
  h->m2l_gid_of.release(); h->m2l_ikeys_in.release(); h->m2l_ikeys.release();
  h->m2l_iidx_in.release(); h->m2l_iidx.release();
  h->sh_keys_in.release(); h->sh_keys.release(); h->sh_vals_in.release(); h->sh_cells.release();
  h->sh_src.release(); h->sh_T.release(); h->sh_items.release(); h->sh_counters.release();
  h->m2l_Y.release(); h->sh_Y.release(); h->cub_tmp_aux.release(); h->m2l_Ttc.release(); h->m2l_class_rep.release(); h->m2l_ssrc.release(); h->m2l_stgt.release(); h->m2l_T.release();
  for (int k = 0; k < 3; ++k) { h->loff[k].release(); h->lcnt[k].release(); h->lsrc[k].release(); }
  h->p2p_rng.release(); h->out_off.release(); h->out_cnt.release();
  h->trav_osc.release(); h->trav_rsc.release();
  h->outA.release(); h->outB.release(); h->stack.release();
  for (auto *b : {&h->d_off, &h->d_lb, &h->d_cnt, &h->strad_flag, &h->strad_excl, &h->need_m,
                  &h->need_p, &h->dexcl, &h->psize, &h->pexcl, &h->prsize, &h->prexcl, &h->psz2,
                  &h->pex2})
    b->release();
  for (auto *b : {&h->lidx_in, &h->lperm, &h->ridx_in, &h->rperm, &h->strad_ids, &h->req_ids,
                  &h->req_own, &h->req_own_s, &h->mreq_s, &h->rreq_ids, &h->pcell, &h->pown,
                  &h->pown_s, &h->pidx, &h->pidx_s})
    b->release();
  for (auto *b : {&h->d_K, &h->lkeys_in, &h->lkeys, &h->rkeys, &h->rkeys_s}) b->release();
  for (auto *b : {&h->lpos, &h->rpos, &h->pbuf_s, &h->pbuf_r}) b->release();
  for (auto *b : {&h->prng, &h->prng_s, &h->rreq_rng}) b->release();
  for (auto *b : {&h->rphi, &h->rgrad, &h->sphi, &h->sgrad}) b->release();
  h->rows_s.release();
  h->rows_r.release();
  h->d_i64.release();
  h->d_cost.release();
  delete h->comm;
  if (h->d_root) cudaFree(h->d_root);
  if (h->d_mm) cudaFree(h->d_mm);
  if (h->d_small) cudaFree(h->d_small);
  if (h->d_overflow) cudaFree(h->d_overflow);
  if (h->d_stats) cudaFree(h->d_stats);
  if (h->d_bk) cudaFree(h->d_bk);
  if (h->h_small) cudaFreeHost(h->h_small);
  for (int i = 0; i < EV_N; ++i)
    if (h->ev[i]) cudaEventDestroy(h->ev[i]);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  if (h->aux) cudaStreamDestroy(h->aux);
  if (h->nf) cudaStreamDestroy(h->nf);
  if (h->hi) cudaStreamDestroy(h->hi);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_out) cudaEventDestroy(h->ev_out);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_up) cudaEventDestroy(h->ev_up);
  if (h->ev_trav) cudaEventDestroy(h->ev_trav);
  if (h->ev_near) cudaEventDestroy(h->ev_near);
  delete h;
  return FMM_OK;
}

int fmm_evaluate(fmm_t h, const float *d_xyz, const float *d_q, int64_t n, float *d_phi,
                 float *d_grad) {
  if (!h) return FMM_E_INVALID;
  if (n < 0) return fail(h, FMM_E_INVALID, "n < 0");
  if (n == 0 && !h->comm) {
    memset(&h->stats, 0, sizeof h->stats);
    return FMM_OK;
  }
  if (n > 0 && (!d_xyz || !d_q || !d_phi || !d_grad)) return fail(h, FMM_E_INVALID, "NULL buffer with n > 0");
  DeviceGuard dg(h->device);
  int rc = FMM_OK;
  if (n > 0) {
    rc = check_device_ptr(h, d_xyz, "xyz");
    if (!rc) rc = check_device_ptr(h, d_q, "q");
    if (!rc) rc = check_device_ptr(h, d_phi, "phi");
    if (!rc) rc = check_device_ptr(h, d_grad, "grad");
  }
  if (!rc) rc = evaluate_impl(h, d_xyz, d_q, n, d_phi, d_grad);
  return rc;
}

int fmm_evaluate_ts(fmm_t h, const float *d_xyz_t, int64_t n_t, const float *d_xyz_s,
                    const float *d_q_s, int64_t n_s, float *d_phi_t, float *d_grad_t) {
  if (!h) return FMM_E_INVALID;
  if (h->comm) return fail(h, FMM_E_INVALID, "fmm_evaluate_ts: not available on distributed handles");
  if (h->mode == FMM_DIRECT) return fail(h, FMM_E_INVALID, "fmm_evaluate_ts: not in FMM_DIRECT mode");
  if (n_t < 0 || n_s < 0) return fail(h, FMM_E_INVALID, "n < 0");
  if (n_t == 0) {
    memset(&h->stats, 0, sizeof h->stats);
    return FMM_OK;
  }
  if (!d_xyz_t || !d_phi_t || !d_grad_t || (n_s > 0 && (!d_xyz_s || !d_q_s)))
    return fail(h, FMM_E_INVALID, "NULL buffer with n > 0");
  const int64_t n = n_t + n_s;
  if (n > (int64_t)1 << 28) return fail(h, FMM_E_INVALID, "n_t + n_s = %lld exceeds 2^28", (long long)n);
  DeviceGuard dg(h->device);
  int rc = check_device_ptr(h, d_xyz_t, "xyz_t");
  if (!rc && n_s > 0) rc = check_device_ptr(h, d_xyz_s, "xyz_s");
  if (!rc && n_s > 0) rc = check_device_ptr(h, d_q_s, "q_s");
  if (!rc) rc = check_device_ptr(h, d_phi_t, "phi_t");
  if (!rc) rc = check_device_ptr(h, d_grad_t, "grad_t");
  if (!rc) {
    // the union [targets (charge 0) | sources] and its full-size outputs, in handle scratch
    cudaStream_t st = h->stream;
    CK(h->ts_stage.ensure(8 * (size_t)n));
    float *xyz = h->ts_stage.p, *q = xyz + 3 * n, *phi = q + n, *grad = phi + n;
    CK(cudaMemcpyAsync(xyz, d_xyz_t, sizeof(float) * 3 * n_t, cudaMemcpyDeviceToDevice, st));
    if (n_s > 0) {
      CK(cudaMemcpyAsync(xyz + 3 * n_t, d_xyz_s, sizeof(float) * 3 * n_s, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(q + n_t, d_q_s, sizeof(float) * n_s, cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaMemsetAsync(q, 0, sizeof(float) * n_t, st));
    h->ts_nt = n_t;
    rc = evaluate_impl(h, xyz, q, n, phi, grad);
    h->ts_nt = 0;
    if (!rc) {
      CK(cudaMemcpyAsync(d_phi_t, phi, sizeof(float) * n_t, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(d_grad_t, grad, sizeof(float) * 3 * n_t, cudaMemcpyDeviceToDevice, st));
      CK(cudaStreamSynchronize(st));
    }
  }
  return rc;
}

int fmm_evaluate_host(fmm_t h, const float *h_xyz, const float *h_q, int64_t n, float *h_phi,
                      float *h_grad) {
  if (!h) return FMM_E_INVALID;
  DeviceGuard dg(h->device);
  if (n < 0) return fail(h, FMM_E_INVALID, "n < 0");
  if (n == 0 && !h->comm) return FMM_OK;
  if (n > 0 && (!h_xyz || !h_q || !h_phi || !h_grad)) return fail(h, FMM_E_INVALID, "NULL buffer with n > 0");
  CK(h->host_stage.ensure(8 * std::max<size_t>((size_t)n, 1)));  // grow-only device staging (no per-call malloc)
  float *d = h->host_stage.p;
  float *xyz = d, *q = d + 3 * n, *phi = d + 4 * n, *grad = d + 5 * n;
  int rc = FMM_OK;
  cudaError_t e = cudaSuccess;
  if (n > 0) e = cudaMemcpyAsync(xyz, h_xyz, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, h->stream);
  if (!e && n > 0) e = cudaMemcpyAsync(q, h_q, sizeof(float) * n, cudaMemcpyHostToDevice, h->stream);
  if (e) rc = fail(h, FMM_E_CUDA, "H2D: %s", cudaGetErrorString(e));
  if (!rc) rc = evaluate_impl(h, xyz, q, n, phi, grad);
  if (!rc && n > 0) {
    e = cudaMemcpyAsync(h_phi, phi, sizeof(float) * n, cudaMemcpyDeviceToHost, h->stream);
    if (!e) e = cudaMemcpyAsync(h_grad, grad, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost, h->stream);
    if (!e) e = cudaStreamSynchronize(h->stream);
    if (e) rc = fail(h, FMM_E_CUDA, "D2H: %s", cudaGetErrorString(e));
  }
  return rc;
}

int fmm_set_stream(fmm_t h, void *stream) {
  if (!h) return FMM_E_INVALID;
  h->stream = stream ? (cudaStream_t)stream : h->own_stream;
  return FMM_OK;
}

int fmm_set_mode(fmm_t h, int mode) {
  if (!h) return FMM_E_INVALID;
  if (mode < FMM_HYBRID || mode > FMM_DIRECT) return fail(h, FMM_E_INVALID, "bad mode %d", mode);
  h->mode = mode;
  return FMM_OK;
}

int fmm_set_timing(fmm_t h, int enable) {
  if (!h) return FMM_E_INVALID;
  h->timing = enable != 0;
  return FMM_OK;
}

int fmm_set_deterministic(fmm_t h, int enable) {
  if (!h) return FMM_E_INVALID;
  h->deterministic = enable != 0;
  return FMM_OK;
}

int fmm_set_m2l_scheme(fmm_t h, int scheme) {
  if (!h) return FMM_E_INVALID;
  if (scheme != FMM_M2L_AUTO && !m2l_scheme_ok(h->p, scheme))
    return fail(h, FMM_E_INVALID, "M2L scheme %d is not available at p = %d", scheme, h->p);
  h->m2l_scheme = scheme;
  return FMM_OK;
}

int fmm_get_m2l_scheme(fmm_t h, int *scheme, double *tuned_ms) {
  if (!h || !scheme) return FMM_E_INVALID;
  *scheme = m2l_scheme_of(h);
  if (tuned_ms)
    for (int i = 0; i < 5; ++i) tuned_ms[i] = h->m2l_scheme_ms[i];
  return FMM_OK;
}

int fmm_set_basis(fmm_t h, int basis) {
  if (!h) return FMM_E_INVALID;
  DeviceGuard dg(h->device);
  if (basis == FMM_BASIS_SPHERICAL) {
    const bool changed = h->basis != FMM_BASIS_SPHERICAL;
    h->basis = FMM_BASIS_SPHERICAL;
    return changed && h->cost.measured ? tune_impl(h) : FMM_OK;
  }
  if (basis == FMM_BASIS_CARTESIAN) {
    if (!cart_supported(h->p))
      return fail(h, FMM_E_INVALID, "Cartesian expansions need 1 <= p <= %d", CART_PMAX);
    if (h->comm) return fail(h, FMM_E_INVALID, "Cartesian expansions: single-GPU handles only");
    const bool changed = h->basis != FMM_BASIS_CARTESIAN;
    h->basis = FMM_BASIS_CARTESIAN;
    return changed && h->cost.measured ? tune_impl(h) : FMM_OK;
  }
  if (basis == FMM_BASIS_AUTO) return auto_basis_impl(h);
  return fail(h, FMM_E_INVALID, "unknown basis %d", basis);
}

int fmm_get_basis(fmm_t h, int *basis, double *ms_spherical, double *ms_cartesian) {
  if (!h || !basis) return FMM_E_INVALID;
  *basis = h->basis;
  if (ms_spherical) *ms_spherical = h->basis_ms[0];
  if (ms_cartesian) *ms_cartesian = h->basis_ms[1];
  return FMM_OK;
}

static int attach_comm(fmm_ctx *h, FmmComm *c);

int fmm_tune(fmm_t h) {
  if (!h) return FMM_E_INVALID;
  DeviceGuard dg(h->device);
  // the pre-calculation is a single-GPU run on synthetic data; a distributed handle then takes
  // rank 0's table again (collective)
  FmmComm *c = h->comm;
  h->comm = nullptr;
  int rc = tune_impl(h);
  if (c) {
    const int rc2 = attach_comm(h, c);
    if (!rc) rc = rc2;
  }
  return rc;
}

int fmm_get_cost_model(fmm_t h, fmm_cost_t *out) {
  if (!h || !out) return FMM_E_INVALID;
  *out = h->cost;
  return FMM_OK;
}

int fmm_set_cost_model(fmm_t h, const fmm_cost_t *in) {
  if (!h || !in) return FMM_E_INVALID;
  if (in->p != h->p) return fail(h, FMM_E_INVALID, "cost model for p=%d, handle p=%d", in->p, h->p);
  if (!(in->t_pp >= 0 && in->t_mp >= 0 && in->t_ml >= 0)) return fail(h, FMM_E_INVALID, "negative cost");
  h->cost = *in;
  return FMM_OK;
}

int fmm_get_stats(fmm_t h, fmm_stats_t *out) {
  if (!h || !out) return FMM_E_INVALID;
  *out = h->stats;
  return FMM_OK;
}

int fmm_export_tree(fmm_t h, int64_t cap, int32_t *h_level, uint64_t *h_prefix, int64_t *h_begin,
                    int64_t *h_count, int64_t *count_out) {
  if (!h || !count_out) return FMM_E_INVALID;
  DeviceGuard dg(h->device);
  if (!h->have_tree) return fail(h, FMM_E_STATE, "no tree evaluation yet");
  const int nc = h->ncells;
  *count_out = nc;
  if (cap < nc) return fail(h, FMM_E_INVALID, "cap %lld < %d cells", (long long)cap, nc);
  std::vector<int> beg(nc), cnt(nc);
  std::vector<int4> grid(nc);
  CK(cudaMemcpy(beg.data(), h->cbeg.p, sizeof(int) * nc, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cnt.data(), h->ccnt.p, sizeof(int) * nc, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(grid.data(), h->cgrid.p, sizeof(int4) * nc, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_prefix, h->cprefix.p, sizeof(uint64_t) * nc, cudaMemcpyDeviceToHost));
  for (int c = 0; c < nc; ++c) {  // BFS order is already (level, prefix) order
    h_level[c] = grid[c].w;
    h_begin[c] = beg[c];
    h_count[c] = cnt[c];
  }
  return FMM_OK;
}

int fmm_export_lists(fmm_t h, int64_t cap, int32_t *h_kind, int32_t *h_tlevel, uint64_t *h_tprefix,
                     int32_t *h_slevel, uint64_t *h_sprefix, int64_t *count_out) {
  if (!h || !count_out) return FMM_E_INVALID;
  DeviceGuard dg(h->device);
  if (!h->have_tree) return fail(h, FMM_E_STATE, "no tree evaluation yet");
  const int nc = h->ncells;
  const int64_t total = h->ntask[0] + h->ntask[1] + h->ntask[2];
  *count_out = total;
  if (cap < total) return fail(h, FMM_E_INVALID, "cap %lld < %lld pairs", (long long)cap, (long long)total);
  std::vector<int4> grid(nc);
  std::vector<uint64_t> prefix(nc);
  CK(cudaMemcpy(grid.data(), h->cgrid.p, sizeof(int4) * nc, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(prefix.data(), h->cprefix.p, sizeof(uint64_t) * nc, cudaMemcpyDeviceToHost));
  int64_t row = 0;
  for (int k = 0; k < 3; ++k) {
    std::vector<int> off(nc), cnt(nc);
    std::vector<unsigned> src(h->ntask[k] + 1);
    CK(cudaMemcpy(off.data(), h->loff[k].p, sizeof(int) * nc, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cnt.data(), h->lcnt[k].p, sizeof(int) * nc, cudaMemcpyDeviceToHost));
    if (h->ntask[k]) CK(cudaMemcpy(src.data(), h->lsrc[k].p, sizeof(unsigned) * h->ntask[k], cudaMemcpyDeviceToHost));
    for (int t = 0; t < nc; ++t)
      for (int e = 0; e < cnt[t]; ++e) {
        const unsigned s = src[off[t] + e];
        h_kind[row] = k;
        h_tlevel[row] = grid[t].w;
        h_tprefix[row] = prefix[t];
        h_slevel[row] = grid[s].w;
        h_sprefix[row] = prefix[s];
        ++row;
      }
  }
  return FMM_OK;
}

int fmm_export_perm(fmm_t h, int64_t cap, int64_t *h_perm, uint64_t *h_keys, double *h_origin3,
                    double *h_L) {
  if (!h) return FMM_E_INVALID;
  DeviceGuard dg(h->device);
  if (!h->have_tree) return fail(h, FMM_E_STATE, "no tree evaluation yet");
  if (h->comm) return fail(h, FMM_E_INVALID, "fmm_export_perm: not available on distributed handles");
  const int64_t n = h->last_n;
  if (cap < n) return fail(h, FMM_E_INVALID, "cap too small");
  std::vector<unsigned> perm(n);
  CK(cudaMemcpy(perm.data(), h->perm.p, sizeof(unsigned) * n, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < n; ++i) h_perm[i] = perm[i];
  if (h_keys) CK(cudaMemcpy(h_keys, h->keys.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  if (h_origin3) for (int a = 0; a < 3; ++a) h_origin3[a] = h->h_root.origin[a];
  if (h_L) *h_L = h->h_root.L;
  return FMM_OK;
}

int fmm_set_partition(fmm_t h, int nparts, int part) {
  if (!h) return FMM_E_INVALID;
  if (h->comm) return fail(h, FMM_E_INVALID, "fmm_set_partition: distributed handles partition themselves");
  if (nparts < 1 || part < 0 || part >= nparts)
    return fail(h, FMM_E_INVALID, "bad partition %d of %d", part, nparts);
  h->nparts = nparts;
  h->part = part;
  return FMM_OK;
}

int fmm_get_partition(fmm_t h, int64_t *lo, int64_t *hi) {
  if (!h || !lo || !hi) return FMM_E_INVALID;
  if (!h->have_tree) return fail(h, FMM_E_STATE, "no tree evaluation yet");
  *lo = h->part_lo;
  *hi = h->part_hi;
  return FMM_OK;
}

int fmm_partition_indices(fmm_t h, int64_t *d_out, int64_t cap, int64_t *count_out) {
  if (!h || !count_out) return FMM_E_INVALID;
  DeviceGuard dg(h->device);
  if (!h->have_tree) return fail(h, FMM_E_STATE, "no tree evaluation yet");
  const int cnt = h->part_hi - h->part_lo;
  *count_out = cnt;
  if (cap < cnt) return fail(h, FMM_E_INVALID, "cap too small");
  if (cnt > 0) {
    if (int rc = check_device_ptr(h, d_out, "out")) return rc;
    launch_part_indices(h->part_lo, cnt, h->perm.p, d_out, h->stream);
    CKL();
    CK(cudaStreamSynchronize(h->stream));
  }
  return FMM_OK;
}

static int attach_comm(fmm_ctx *h, FmmComm *c) {
  // rank 0's measured cost table on every rank (the per-pair kind choice must
  // not depend on the rank that evaluates the pair)
  h->comm = c;
  double v[3] = {h->cost.t_pp, h->cost.t_mp, h->cost.t_ml};
  if (c->rank != 0) v[0] = v[1] = v[2] = 0.0;
  CK(h->d_cost.ensure(3));
  CK(cudaMemcpyAsync(h->d_cost.p, v, sizeof v, cudaMemcpyHostToDevice, h->stream));
  CC(c->allreduce(h->d_cost.p, 3, CT_F64, CO_SUM, h->stream));
  CK(cudaMemcpyAsync(v, h->d_cost.p, sizeof v, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->cost.t_pp = v[0];
  h->cost.t_mp = v[1];
  h->cost.t_ml = v[2];
  return FMM_OK;
}

int fmm_comm_unique_id(unsigned char h_id[128]) {
  if (!h_id) return FMM_E_INVALID;
  std::string err;
  const int rc = comm_nccl_unique_id(h_id, err);
  if (rc) fprintf(stderr, "fmm_comm_unique_id: %s\n", err.c_str());
  return rc;
}

int fmm_create_dist(fmm_t *out, int p, double theta, int ncrit, int nranks, int rank,
                    const unsigned char h_id[128]) {
  if (!out) return FMM_E_INVALID;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks || !h_id) return FMM_E_INVALID;
  int rc = fmm_create(out, p, theta, ncrit);
  if (rc) return rc;
  std::string err;
  FmmComm *c = comm_nccl_create(nranks, rank, h_id, err);
  if (!c) {
    fprintf(stderr, "fmm_create_dist: %s\n", err.c_str());
    fmm_destroy(*out);
    *out = nullptr;
    return FMM_E_NCCL;
  }
  if ((rc = attach_comm(*out, c))) {
    fprintf(stderr, "fmm_create_dist: %s\n", (*out)->err.c_str());
    fmm_destroy(*out);
    *out = nullptr;
  }
  return rc;
}

int fmm_group_create(fmm_group_t *out, int nranks) {
  if (!out || nranks < 1 || nranks > 16) return FMM_E_INVALID;
  *out = comm_group_create(nranks);
  return FMM_OK;
}

int fmm_group_destroy(fmm_group_t g) {
  comm_group_destroy(g);
  return FMM_OK;
}

int fmm_create_in_group(fmm_t *out, int p, double theta, int ncrit, fmm_group_t g, int rank) {
  if (!out) return FMM_E_INVALID;
  *out = nullptr;
  if (!g) return FMM_E_INVALID;
  int rc = fmm_create(out, p, theta, ncrit);
  if (rc) return rc;
  std::string err;
  FmmComm *c = comm_local_create(g, rank, err);
  if (!c) {
    fmm_destroy(*out);
    *out = nullptr;
    return FMM_E_INVALID;
  }
  if ((rc = attach_comm(*out, c))) {
    fmm_destroy(*out);
    *out = nullptr;
  }
  return rc;
}

const char *fmm_strerror(int code) {
  switch (code) {
    case FMM_OK: return "ok";
    case FMM_E_INVALID: return "invalid argument";
    case FMM_E_NOT_DEVICE: return "pointer is not device memory of the handle's device";
    case FMM_E_NONFINITE: return "non-finite input";
    case FMM_E_CUDA: return "CUDA error";
    case FMM_E_OOM: return "out of device memory";
    case FMM_E_NCCL: return "NCCL error";
    case FMM_E_STATE: return "no evaluation yet";
    default: return "unknown error";
  }
}

const char *fmm_last_error(fmm_t h) { return h ? h->err.c_str() : "NULL handle"; }

}  // extern "C"
