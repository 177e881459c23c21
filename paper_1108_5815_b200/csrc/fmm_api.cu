// fmm_api.cu — the C ABI of libfmm.so (include/fmm.h) and the stream-ordered host pipeline.
//
// One evaluation (every step a device kernel, the host only reads small counts):
//   bbox + root cube -> Morton keys -> radix sort -> gather float4 -> level-synchronous tree
//   -> P2M -> M2M (bottom-up) -> target-centric traversal (count / scan / write per level)
//   -> M2L -> L2L (top-down) -> P2P -> M2P -> L2P + combine + un-permute.
// FMM_DIRECT skips the tree: one all-pairs P2P.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/fmm.h"
#include "common.cuh"
#include "kernels.cuh"

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

enum { EV_START, EV_TREE, EV_UP, EV_TRAV, EV_M2L_PREP, EV_M2L, EV_P2P, EV_M2P, EV_DOWN, EV_N };

}  // namespace

struct fmm_ctx {
  int device = 0;
  int p = 4, ncrit = 32, mode = FMM_HYBRID;
  double theta = 0.5;
  cudaStream_t own_stream = nullptr, stream = nullptr;
  // the upward sweep runs on `aux`, concurrently with the traversal and the M2L class sort
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_up = nullptr;
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
  std::vector<int> level_off, level_cnt;
  int ncells = 0, nleaves = 0, depth = 0;
  // Morton partition of the targets (multi-GPU); nparts = 1: everything
  int nparts = 1, part = 0;
  int tleaves_n = 0, part_lo = 0, part_hi = 0;
  DBuf<int> tleaves;
  // expansions
  DBuf<float2> M, L;
  // M2L class batching
  DBuf<int> m2l_pair_t, m2l_flag, m2l_cid, m2l_cstart, m2l_counters;
  DBuf<unsigned> m2l_keys_in, m2l_keys;
  DBuf<unsigned> m2l_idx_in, m2l_sidx, m2l_small, m2l_class_rep, m2l_ssrc, m2l_stgt;
  DBuf<float> m2l_T;
  DBuf<unsigned> m2l_Ttc;
  bool m2l_tc_used = false;
  DBuf<int4> m2l_items;
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
  DBuf<int> out_off, out_cnt, cnt4, excl4;
  DBuf<unsigned> outA, outB, stack;
  int stack_cap = 2048;
  size_t trav_cap[4] = {0, 0, 0, 0};  // list buffer sizes seen so far (traverse)
  int *d_bk = nullptr;                // device bookkeeping of the traversal (TravArgs::bk)
  int64_t ntask[3] = {0, 0, 0};
  bool have_tree = false;
  int64_t last_n = 0;
  RootInfo h_root{};

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
  size_t bytes = 0;
  CK(sort_keys(nullptr, bytes, h->keys_in.p, h->keys.p, h->idx_in.p, h->perm.p, n, st));
  CK(h->cub_tmp.ensure(bytes));
  CK(sort_keys(h->cub_tmp.p, bytes, h->keys_in.p, h->keys.p, h->idx_in.p, h->perm.p, n, st));
  ++h->stats.cub_calls;
  launch_gather(xyz, q, h->perm.p, n, h->pos.p, st);
  CKL();

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
    launch_split(c0, nl, level, h->ncrit, h->keys.p, h->cells(), h->cprefix.p, h->nch.p,
                 h->crange.p, h->bnd.p, st);
    h->stats.launches += 1;
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
  // target leaves of this handle's partition
  h->part_lo = 0;
  h->part_hi = (int)n;
  h->tleaves_n = h->nleaves;
  if (h->nparts > 1) {
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

// ---- a9: traversal ----------------------------------------------------------------------------
static int traverse(fmm_ctx *h) {
  // Level-synchronous target-centric traversal (traverse.cu). All bookkeeping stays on the
  // device: list buffers are sized from the previous evaluation (or an estimate), the write pass
  // of a level whose lists would not fit does nothing, and one read-back at the end decides
  // whether to re-run with larger buffers (stack or lists) -- no host round trip per level.
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
  const int grid_blocks = 148 * 8;
  const size_t nwarps = (size_t)grid_blocks * warps_per_block;
  int maxnt = 1;
  for (int level = 0; level <= h->depth; ++level) maxnt = std::max(maxnt, h->level_cnt[level]);
  CK(h->cnt4.ensure((size_t)4 * maxnt));
  CK(h->excl4.ensure((size_t)4 * maxnt));
  // capacities: at least the previous evaluation's totals, else an estimate per target cell
  size_t cap[4];
  for (int k = 0; k < 4; ++k) {
    const size_t est = (size_t)256 * nc + 1024;
    cap[k] = std::max(est, h->trav_cap[k]);
    cap[k] = std::min(cap[k], (size_t)INT32_MAX - 1);
  }
  for (int attempt = 0;; ++attempt) {
    CK(h->stack.ensure(nwarps * h->stack_cap));
    for (int k = 0; k < 3; ++k) CK(h->lsrc[k].ensure(cap[k]));
    CK(h->p2p_rng.ensure(cap[2]));
    CK(h->outA.ensure(cap[3]));
    CK(h->outB.ensure(cap[3]));
    int hb[20] = {0};
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
      A.cnt4 = h->cnt4.p;
      A.excl = h->excl4.p;
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
      launch_traverse(A, false, st);
      CKL();
      if (int rc = cub_scan(h, h->cnt4.p, h->excl4.p, 4 * nt)) return rc;
      launch_trav_totals(h->excl4.p, h->cnt4.p, nt, h->d_bk, st);
      CKL();
      launch_traverse(A, true, st);
      CKL();
      in_src = ob->p;
    }
    int hb2[20];
    unsigned ovf = 0;
    unsigned long long hs[2];
    CK(cudaMemcpyAsync(hb2, h->d_bk, sizeof hb2, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&ovf, h->d_overflow, sizeof ovf, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hs, h->d_stats, sizeof hs, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (ovf) {  // a warp's traversal stack overflowed: larger stacks, again
      h->stack_cap *= 2;
      if ((size_t)h->stack_cap * nwarps > ((size_t)1 << 31))
        return fail(h, FMM_E_OOM, "traversal stack exceeds 8 GiB");
      continue;
    }
    if (hb2[12]) {  // a list buffer was too small: grow to what the count passes have seen so far
      if (attempt > 8) return fail(h, FMM_E_OOM, "interaction lists do not fit");
      for (int k = 0; k < 4; ++k) {
        const size_t need = (size_t)(k < 3 ? hb2[16 + k] : 0);
        cap[k] = std::min((size_t)INT32_MAX - 1, std::max(cap[k] * 2, need + need / 4 + 1024));
      }
      continue;
    }
    for (int k = 0; k < 3; ++k) {
      h->ntask[k] = hb2[16 + k];
      h->trav_cap[k] = std::max(h->trav_cap[k], (size_t)hb2[16 + k] + 1);
    }
    h->trav_cap[3] = std::max(h->trav_cap[3], cap[3]);
    h->stats.p2p_pairs = (int64_t)hs[0];
    h->stats.m2p_evals = (int64_t)hs[1];
    return FMM_OK;
  }
}

static int evaluate_tree(fmm_ctx *h, const float *xyz, const float *q, int64_t n, float *phi,
                         float *grad) {
  cudaStream_t st = h->stream;
  const int p = h->p, NC = nc_of(p);
  if (int rc = build_tree(h, xyz, q, n)) return rc;
  record(h, EV_TREE);
  // a7/a8 upward sweep, on the aux stream: it overlaps the traversal and the M2L class sort (which
  // do not read M); the stream joins before the first kernel that reads M
  CK(cudaEventRecord(h->ev_fork, st));
  CK(cudaStreamWaitEvent(h->aux, h->ev_fork, 0));
  cudaStream_t ua = h->aux;
  const int NCS = nc_stride(p);
  CK(h->M.ensure((size_t)h->ncells * NCS));
  CK(h->L.ensure((size_t)h->ncells * NCS));
  if (NCS != NC) CK(cudaMemsetAsync(h->M.p, 0, sizeof(float2) * (size_t)h->ncells * NCS, ua));
  // M2M / L2L: octant-class GEMMs on the tensor cores (p <= 10) unless disabled
  const char *scc = getenv("FMM_SHIFT_CUDA_CORES");
  const bool shift_tc = m2l_tc_supported(p) && h->ncells > 1 && !(scc && scc[0] && scc[0] != '0');
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
    S.items_per_level = 16 + h->ncells / 2048;
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
  launch_p2m(p, h->leaves.p, h->nleaves, h->cells(), h->pos.p, h->M.p, ua);
  CKL();
  for (int level = h->depth - 1; level >= 0; --level) {
    if (shift_tc) {
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
  if (int rc = traverse(h)) return rc;
  record(h, EV_TRAV);
  record(h, EV_M2L_PREP);  // re-recorded after the class sort when there are M2L pairs
  // a10 M2L (writes every cell's local expansion, zero where no M2L)
  const bool far_local = h->ntask[FMM_KIND_M2L] > 0;
  if (far_local) {
    const int np = (int)h->ntask[FMM_KIND_M2L];
    CK(h->m2l_pair_t.ensure(np));
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
    // tensor-core GEMMs accumulate straight into L unless bit-reproducibility is requested
    const char *cc = getenv("FMM_M2L_CUDA_CORES");
    const bool use_tc = m2l_gemm_supported(p) && m2l_tc_supported(p) && !(cc && cc[0] && cc[0] != '0');
    const bool accum = use_tc && !h->deterministic;
    if (!accum) CK(h->m2l_Y.ensure((size_t)np * m2l_y_stride(p)));
    CK(h->cub_tmp.ensure(m2l_temp_bytes(np)));
    M2LWork W{};
    W.C = h->cells();
    W.off = h->loff[0].p;
    W.cnt = h->lcnt[0].p;
    W.src = h->lsrc[0].p;
    W.pair_t = h->m2l_pair_t.p;
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
    W.direct_all = m2l_gemm_supported(p) ? 0 : 1;
    CK(h->m2l_class_rep.ensure(np));
    CK(h->m2l_ssrc.ensure(np));
    W.class_rep = h->m2l_class_rep.p;
    W.ssrc = h->m2l_ssrc.p;
    if (accum) {
      CK(h->m2l_stgt.ensure(np));
      W.stgt = h->m2l_stgt.p;
    }
    CK(m2l_prepare(W, np, h->ncells, st));
    h->stats.launches += 6;
    h->stats.cub_calls += 2;
    CK(cudaMemcpyAsync(h->h_small, h->m2l_counters.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int ngclass = h->h_small[3];
    // class GEMMs on the tensor cores (tcgen05, 3xTF32) unless disabled / unsupported
    if (use_tc) {
      CK(h->m2l_Ttc.ensure((size_t)std::max(1, ngclass) * m2l_tc_T_words(p)));
      CK(m2l_tc_build_T(p, W, ngclass, h->m2l_Ttc.p, st));
    } else {
      CK(h->m2l_T.ensure((size_t)std::max(1, ngclass) * m2l_T_floats(p)));
      W.Tg = h->m2l_T.p;
      CK(m2l_build_T(p, W, ngclass, st));
    }
    h->stats.launches += 1;
    if (accum) CK(cudaMemsetAsync(h->L.p, 0, sizeof(float2) * (size_t)h->ncells * NCS, st));
    CK(cudaStreamWaitEvent(st, h->ev_up, 0));  // join: the multipoles are complete
    record(h, EV_M2L_PREP);  // ms_m2l = the GEMM (+ the rare-class direct path / reduction)
    if (use_tc) {
      CK(m2l_tc_gemm(p, W, h->m2l_Ttc.p, h->M.p, st, accum ? h->L.p : nullptr));
      h->stats.launches += 1;
    }
    CK(m2l_execute(p, W, np, h->ncells, h->M.p, h->L.p, st, use_tc, accum));
    h->stats.launches += 2;
    h->m2l_tc_used = use_tc;
  }
  CK(cudaStreamWaitEvent(st, h->ev_up, 0));  // (no M2L pairs: join here)
  record(h, EV_M2L);
  // a12 P2P (writes acc), a11 M2P (adds)
  const int *tl = h->nparts > 1 ? h->tleaves.p : h->leaves.p;
  const int ntl = h->tleaves_n;
  launch_p2p_leaves(tl, ntl, h->cells(), h->lists(), h->pos.p, h->acc.p,
                    h->d_small + 12, st);
  CKL();
  record(h, EV_P2P);
  if (h->ntask[FMM_KIND_M2P] > 0) {
    launch_m2p(p, tl, ntl, h->cells(), h->lists(), h->pos.p, h->M.p, h->acc.p, h->d_small + 13, st);
    CKL();
  }
  record(h, EV_M2P);
  // a13 L2L top-down, a14/a15 L2P + combine + un-permute
  if (far_local) {
    for (int level = 1; level <= h->depth; ++level) {
      if (shift_tc) {
        CK(tc_shift_l2l_level(p, level, h->level_off[level], h->level_cnt[level], S, h->L.p,
                              h->sh_Y.p, st));
        h->stats.launches += 2;
      } else {
        launch_l2l(p, h->level_off[level], h->level_cnt[level], h->cells(), h->L.p, st);
      }
      CKL();
    }
  }
  launch_l2p(p, tl, ntl, h->cells(), h->pos.p, h->L.p, h->acc.p, h->perm.p, phi,
             grad, far_local ? 1 : 0, st);
  CKL();
  record(h, EV_DOWN);
  h->have_tree = true;
  return FMM_OK;
}

static int evaluate_impl(fmm_ctx *h, const float *xyz, const float *q, int64_t n, float *phi,
                         float *grad) {
  cudaStream_t st = h->stream;
  memset(&h->stats, 0, sizeof h->stats);
  h->stats.n = n;
  h->stats.p = h->p;
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
  if (h->timing) {
    float ms[EV_N];
    for (int e = 1; e < EV_N; ++e) cudaEventElapsedTime(&ms[e], h->ev[e - 1], h->ev[e]);
    cudaEventElapsedTime(&ms[0], h->ev[EV_START], h->ev[EV_DOWN]);
    h->stats.ms_total = ms[0];
    h->stats.ms_tree = ms[EV_TREE];
    // the upward sweep (aux stream) overlaps the traversal: both are measured from EV_TREE
    float up = 0.f, trav = 0.f;
    cudaEventElapsedTime(&up, h->ev[EV_TREE], h->ev[EV_UP]);
    cudaEventElapsedTime(&trav, h->ev[EV_TREE], h->ev[EV_TRAV]);
    h->stats.ms_upward = up;
    h->stats.ms_traverse = trav + ms[EV_M2L_PREP];  // class sort counted as bookkeeping
    h->stats.ms_m2l = ms[EV_M2L];
    h->stats.ms_p2p = ms[EV_P2P];
    h->stats.ms_m2p = ms[EV_M2P];
    h->stats.ms_downward = ms[EV_DOWN];
  }
  return FMM_OK;
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
  const bool saved_timing = h->timing;
  h->timing = true;
  double t_pp[3], t_ml[3], t_mp[3];
  int rc = FMM_OK;
  for (int pass = 0; pass < 2 && rc == FMM_OK; ++pass) {
    h->mode = pass == 0 ? FMM_FMM : FMM_TREECODE;
    for (int it = -1; it < 3 && rc == FMM_OK; ++it) {
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
  cudaFree(d);
  if (rc) return rc;
  auto med3 = [](double *a) { std::sort(a, a + 3); return a[1]; };
  h->cost.t_pp = med3(t_pp);
  h->cost.t_ml = med3(t_ml);
  h->cost.t_mp = med3(t_mp);
  h->cost.p = h->p;
  h->cost.measured = 1;
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
    if ((e = cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&h->ev_up, cudaEventDisableTiming)) != cudaSuccess) {
      rc = fail(h, FMM_E_CUDA, "%s", cudaGetErrorString(e));
      break;
    }
    for (int i = 0; i < EV_N; ++i) cudaEventCreate(&h->ev[i]);
    if (cudaMalloc(&h->d_root, sizeof(RootInfo)) || cudaMalloc(&h->d_mm, 8 * sizeof(unsigned)) ||
        cudaMalloc(&h->d_small, 16 * sizeof(int)) || cudaMalloc(&h->d_overflow, sizeof(unsigned)) ||
        cudaMalloc(&h->d_stats, 4 * sizeof(unsigned long long)) ||
        cudaMalloc(&h->d_bk, 32 * sizeof(int)) ||
        cudaMallocHost(&h->h_small, 16 * sizeof(int))) {
      rc = fail(h, FMM_E_OOM, "small device allocations failed");
      break;
    }
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
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->keys_in.release(); h->keys.release(); h->idx_in.release(); h->perm.release();
  h->pos.release(); h->acc.release(); h->cub_tmp.release(); h->host_stage.release();
  h->cbeg.release(); h->ccnt.release(); h->cparent.release(); h->cchild0.release();
  h->cnchild.release(); h->cgrid.release(); h->cgeo.release(); h->cprefix.release(); h->cpack.release();
  h->tleaves.release();
  h->nch.release(); h->bnd.release(); h->excl.release(); h->leafflag.release(); h->leaves.release(); h->crange.release();
  h->M.release(); h->L.release();
  h->m2l_pair_t.release(); h->m2l_flag.release(); h->m2l_cid.release(); h->m2l_cstart.release();
  h->m2l_counters.release(); h->m2l_keys_in.release(); h->m2l_keys.release();
  h->m2l_idx_in.release(); h->m2l_sidx.release(); h->m2l_small.release(); h->m2l_items.release();
  h->sh_keys_in.release(); h->sh_keys.release(); h->sh_vals_in.release(); h->sh_cells.release();
  h->sh_src.release(); h->sh_T.release(); h->sh_items.release(); h->sh_counters.release();
  h->m2l_Y.release(); h->sh_Y.release(); h->cub_tmp_aux.release(); h->m2l_Ttc.release(); h->m2l_class_rep.release(); h->m2l_ssrc.release(); h->m2l_stgt.release(); h->m2l_T.release();
  for (int k = 0; k < 3; ++k) { h->loff[k].release(); h->lcnt[k].release(); h->lsrc[k].release(); }
  h->p2p_rng.release(); h->out_off.release(); h->out_cnt.release(); h->cnt4.release(); h->excl4.release();
  h->outA.release(); h->outB.release(); h->stack.release();
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
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_up) cudaEventDestroy(h->ev_up);
  delete h;
  return FMM_OK;
}

int fmm_evaluate(fmm_t h, const float *d_xyz, const float *d_q, int64_t n, float *d_phi,
                 float *d_grad) {
  if (!h) return FMM_E_INVALID;
  if (n < 0) return fail(h, FMM_E_INVALID, "n < 0");
  if (n == 0) {
    memset(&h->stats, 0, sizeof h->stats);
    return FMM_OK;
  }
  if (!d_xyz || !d_q || !d_phi || !d_grad) return fail(h, FMM_E_INVALID, "NULL buffer with n > 0");
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != h->device) cudaSetDevice(h->device);
  int rc = check_device_ptr(h, d_xyz, "xyz");
  if (!rc) rc = check_device_ptr(h, d_q, "q");
  if (!rc) rc = check_device_ptr(h, d_phi, "phi");
  if (!rc) rc = check_device_ptr(h, d_grad, "grad");
  if (!rc) rc = evaluate_impl(h, d_xyz, d_q, n, d_phi, d_grad);
  if (cur != h->device && cur >= 0) cudaSetDevice(cur);
  return rc;
}

int fmm_evaluate_host(fmm_t h, const float *h_xyz, const float *h_q, int64_t n, float *h_phi,
                      float *h_grad) {
  if (!h) return FMM_E_INVALID;
  if (n < 0) return fail(h, FMM_E_INVALID, "n < 0");
  if (n == 0) return FMM_OK;
  if (!h_xyz || !h_q || !h_phi || !h_grad) return fail(h, FMM_E_INVALID, "NULL buffer with n > 0");
  CK(h->host_stage.ensure(8 * (size_t)n));  // grow-only device staging (no per-call malloc)
  float *d = h->host_stage.p;
  float *xyz = d, *q = d + 3 * n, *phi = d + 4 * n, *grad = d + 5 * n;
  int rc = FMM_OK;
  cudaError_t e = cudaMemcpyAsync(xyz, h_xyz, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, h->stream);
  if (!e) e = cudaMemcpyAsync(q, h_q, sizeof(float) * n, cudaMemcpyHostToDevice, h->stream);
  if (e) rc = fail(h, FMM_E_CUDA, "H2D: %s", cudaGetErrorString(e));
  if (!rc) rc = evaluate_impl(h, xyz, q, n, phi, grad);
  if (!rc) {
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

int fmm_tune(fmm_t h) {
  if (!h) return FMM_E_INVALID;
  return tune_impl(h);
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
  if (!h->have_tree) return fail(h, FMM_E_STATE, "no tree evaluation yet");
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
