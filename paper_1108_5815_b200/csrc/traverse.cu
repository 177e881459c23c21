// traverse.cu — dual tree traversal on the device.
//
// The paper's traversal pops (target, source) pairs from a LIFO stack, splits the larger cell and
// either evaluates each offspring pair at once (MAC accepted) or pushes it. The
// emitted multiset does not depend on the processing order (each pair's fate is a pure function
// of the pair), so the device runs it TARGET-CENTRIC and level-synchronous: one warp owns one
// target cell t of the current level and runs the paper's stack for all pairs (t, s); a pair
// whose target must be split is deferred to Out(t), which every child of t inherits as its
// starting list at the next level ("target cells inherit a unique stack of source cells from
// their parents"). Each target's interaction lists therefore come out contiguous and in
// a deterministic order, with no global sort.
//
// Two passes per level: COUNT (sizes per target) -> one exclusive scan -> WRITE (same logic,
// writing at the scanned offsets). The MAC is the exact integer/FP64 test of DESIGN.md §3 (R4, R5)
// and the kind choice the linear cost model with ties M2L > M2P > P2P (R8).
#include "common.cuh"
#include "kernels.cuh"

enum { CAT_M2L = 0, CAT_M2P = 1, CAT_P2P = 2, CAT_OUT = 3, CAT_PUSH = 4, CAT_NONE = 5 };

__device__ __forceinline__ bool mac_accept(int4 gt, int4 gs, double theta) {
  const long long dx = gt.x - gs.x, dy = gt.y - gs.y, dz = gt.z - gs.z;
  const long long R2 = dx * dx + dy * dy + dz * dz;
  const long long rsum = (1LL << (FMM_LEVELS - gt.w)) + (1LL << (FMM_LEVELS - gs.w));
  const double rhs = __dmul_rn(theta, __dsqrt_rn(__ll2double_rn(R2)));
  return __ll2double_rn(rsum) <= rhs;
}

__device__ __forceinline__ int select_kind(const TravArgs &A, int nt, int ns) {
  if (A.mode == 1) return CAT_M2L;  // FMM_FMM
  if (A.mode == 2) return CAT_M2P;  // FMM_TREECODE
  const double cpp = __dmul_rn(__dmul_rn(A.t_pp, (double)nt), (double)ns);
  const double cmp = __dmul_rn(A.t_mp, (double)nt);
  const double cml = A.t_ml;
  if (cml <= cmp && cml <= cpp) return CAT_M2L;
  if (cmp <= cpp) return CAT_M2P;
  return CAT_P2P;
}

// packed cell record (built once per tree by k_pack_cells): one 32-byte sector per cell instead
// of four scattered loads on the traversal's latency-bound path
struct CellRec {
  int4 g;  // doubled-grid centre, level
  int4 b;  // beg, cnt, child0, nchild
};
__device__ __forceinline__ CellRec load_rec(const int4 *pk, unsigned c) {
  CellRec r;
  r.g = __ldg(pk + 2 * (size_t)c);
  r.b = __ldg(pk + 2 * (size_t)c + 1);
  return r;
}

__global__ void k_pack_cells(int ncells, CellsView C, int4 *pk) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  pk[2 * c] = C.grid[c];
  pk[2 * c + 1] = make_int4(C.beg[c], C.cnt[c], C.child0[c], C.nchild[c]);
}
void launch_pack_cells(int ncells, CellsView C, int4 *pk, cudaStream_t st) {
  if (ncells > 0) k_pack_cells<<<(ncells + 255) / 256, 256, 0, st>>>(ncells, C, pk);
}

template <bool WRITE>
__global__ void __launch_bounds__(128) k_traverse(TravArgs A) {
  const CellsView C = A.C;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  unsigned *stack = A.scratch + (size_t)gw * A.stack_cap;

  int bk_excl[4] = {0, 0, 0, 0}, bk_base[4] = {0, 0, 0, 0};
  if (WRITE) {
    if (A.bk[12]) return;  // a list would overflow its buffer: the host re-runs with larger ones
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      bk_excl[c] = A.bk[c];
      bk_base[c] = A.bk[4 + c];
    }
  }
  unsigned long long warp_pp = 0, warp_mp = 0;
  for (int k = gw; k < A.nt; k += nw) {
    const int t = A.t0 + k;
    const CellRec rt = load_rec(A.pk, t);
    const int4 gt = rt.g;
    const int tcnt = rt.b.y;
    // outside this rank's target partition, or (distinct target / source sets) no target inside
    if (!(rt.b.x < A.thi && rt.b.x + tcnt > A.tlo) || (A.tmask && A.tmask[t] == 0)) {
      if (lane == 0) {
        if (WRITE) {
          for (int c = 0; c < 3; ++c) {
            A.loff[c][t] = 0;
            A.lcnt[c][t] = 0;
          }
          A.out_off[t] = 0;
          A.out_cnt[t] = 0;
        } else {
          for (int c = 0; c < 4; ++c) A.cnt4[c * A.nt + k] = 0;
        }
      }
      continue;
    }
    const bool tleaf = rt.b.w == 0;
    int n[4] = {0, 0, 0, 0};
    unsigned *dst[4] = {nullptr, nullptr, nullptr, nullptr};
    if (WRITE) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int o = bk_base[c] + A.excl[c * A.nt + k] - bk_excl[c];
        dst[c] = (c < 3 ? A.lsrc[c] : A.out_src) + o;
        if (lane == 0) {
          if (c < 3) {
            A.loff[c][t] = o;
            A.lcnt[c][t] = A.cnt4[c * A.nt + k];
          } else {
            A.out_off[t] = o;
            A.out_cnt[t] = A.cnt4[c * A.nt + k];
          }
        }
      }
    }
    unsigned long long pp_pairs = 0, mp_evals = 0;  // this target's lane partials
    int top = 0;
    bool overflow = false;

    // classify (t, s) and append it to its category with ballots (deterministic order)
    auto consider_and_put = [&](bool valid, unsigned s, int forced_cat) {
      int cat = CAT_NONE;
      int scnt = 0, sbeg = 0;
      if (valid) {
        if (forced_cat >= 0) {
          cat = forced_cat;
        } else {
          const CellRec rs = load_rec(A.pk, s);
          scnt = rs.b.y;
          sbeg = rs.b.x;
          if (mac_accept(gt, rs.g, A.theta))
            cat = select_kind(A, tcnt, scnt);
          else if (tleaf && rs.b.w == 0)
            cat = CAT_P2P;
          else
            cat = CAT_PUSH;
        }
      }
      if (!WRITE) {
        if (cat == CAT_P2P) pp_pairs += (unsigned long long)tcnt * (unsigned long long)scnt;
        if (cat == CAT_M2P) mp_evals += (unsigned long long)tcnt;
      }
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const unsigned b = __ballot_sync(0xffffffffu, cat == c);
        if (!b) continue;
        const int pos = __popc(b & lt_mask);
        if (c == CAT_PUSH) {
          if (cat == c && top + pos < A.stack_cap) stack[top + pos] = s;
          top += __popc(b);
          if (top > A.stack_cap) overflow = true;
        } else {
          if (WRITE && cat == c) {
            dst[c][n[c] + pos] = s;
            if (c == CAT_P2P) A.p2p_rng[(dst[c] - A.lsrc[2]) + n[c] + pos] = make_int2(sbeg, scnt);
          }
          n[c] += __popc(b);
        }
      }
    };

    // 1) inherited pairs (parent(t), s) split on the target side: test (t, s)
    int in_off = 0, in_cnt = 1;
    if (A.level > 0) {
      const int p = C.parent[t];
      in_off = A.in_off[p];
      in_cnt = A.in_cnt[p];
    }
    for (int b0 = 0; b0 < in_cnt; b0 += 32) {
      const int e = b0 + lane;
      const bool valid = e < in_cnt;
      const unsigned s = valid ? (A.level > 0 ? A.in_src[in_off + e] : 0u) : 0u;
      consider_and_put(valid, s, -1);
    }
    __syncwarp();
    // 2) the paper's stack: pop, split the larger cell (ties and leaf targets split the source)
    while (top > 0 && !overflow) {
      const int nb = min(top, 32);
      top -= nb;
      const bool valid = lane < nb;
      const unsigned s = valid ? stack[top + lane] : 0u;
      __syncwarp();
      int snch = 0, sc0 = 0;
      bool split_src = false;
      if (valid) {
        const CellRec rs = load_rec(A.pk, s);
        snch = rs.b.w;
        sc0 = rs.b.z;
        split_src = tleaf || (snch > 0 && rs.g.w <= gt.w);
      }
      consider_and_put(valid && !split_src, s, CAT_OUT);  // target splits: defer to children
      const int c0 = split_src ? sc0 : 0;
      const int m = split_src ? snch : 0;
      int mmax = m;
      for (int o = 16; o > 0; o >>= 1) mmax = max(mmax, __shfl_xor_sync(0xffffffffu, mmax, o));
      for (int j = 0; j < mmax; ++j) consider_and_put(j < m, (unsigned)(c0 + j), -1);
      __syncwarp();
    }
    if (overflow) {
      if (lane == 0) atomicOr(A.overflow, 1u);
      continue;
    }
    if (!WRITE) {
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) A.cnt4[c * A.nt + k] = n[c];
      }
      warp_pp += pp_pairs;  // one atomic per warp at the end, not two per target
      warp_mp += mp_evals;
    }
  }
  if (!WRITE) {
    for (int o = 16; o > 0; o >>= 1) {
      warp_pp += __shfl_xor_sync(0xffffffffu, warp_pp, o);
      warp_mp += __shfl_xor_sync(0xffffffffu, warp_mp, o);
    }
    if (lane == 0 && (warp_pp | warp_mp)) {
      atomicAdd(&A.stats[0], warp_pp);
      atomicAdd(&A.stats[1], warp_mp);
    }
  }
}

// level totals from the one exclusive scan over the four categories: where each category's
// scan starts, where this level's lists go (running sizes) and an overflow flag when a buffer
// is too small (the write pass then does nothing and the host re-runs the traversal)
__global__ void k_trav_totals(const int *excl, const int *cnt4, int nt, int *bk) {
  for (int c = 0; c < 4; ++c) {
    const int e0 = excl[c * nt];
    const int last = (c + 1) * nt - 1;
    const long long tot = (long long)excl[last] + cnt4[last] - e0;
    bk[c] = e0;
    const long long start = c < 3 ? bk[16 + c] : 0;
    bk[4 + c] = (int)start;
    if (start + tot + 1 > bk[8 + c]) bk[12] = 1;
    if (c < 3) bk[16 + c] = (int)min(start + tot, (long long)INT32_MAX);
  }
}

void launch_traverse(const TravArgs &A, bool write, cudaStream_t st) {
  const int blocks = A.grid_blocks;
  if (write)
    k_traverse<true><<<blocks, 128, 0, st>>>(A);
  else
    k_traverse<false><<<blocks, 128, 0, st>>>(A);
}
void launch_trav_totals(const int *excl, const int *cnt4, int nt, int *bk, cudaStream_t st) {
  k_trav_totals<<<1, 1, 0, st>>>(excl, cnt4, nt, bk);
}
