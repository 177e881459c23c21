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
// One pass per level: a warp collects its target's four lists (M2L, M2P, P2P, deferred) in its own
// scratch, then claims their final space with one atomic per list and copies them there. Each
// target's lists are contiguous and in a deterministic order (ballot order); only where a target's
// segment lands in the global arrays depends on the schedule, and every consumer addresses the
// lists through the per-target (offset, count). The MAC is the exact integer/FP64 test of
// DESIGN.md §3 (R4, R5) and the kind choice the linear cost model with ties M2L > M2P > P2P (R8).
#include "common.cuh"
#include "kernels.cuh"

enum { CAT_M2L = 0, CAT_M2P = 1, CAT_P2P = 2, CAT_OUT = 3, CAT_PUSH = 4, CAT_NONE = 5 };

// The MAC's decision is the FP64 expression rsum <= theta * sqrt(R2) (R4/R5, the
// oracle's). Away from the boundary it equals the exact comparison rsum^2 <= theta^2 R2, which
// needs no square root: rsum and R2 are integers below 2^45 (exact in FP64, rsum^2 too), and
// theta2 * R2 is within 3e-16 relative of theta^2 R2 while the FP64 expression's rounding moves the
// boundary by at most 3e-16 relative; a pair within 1e-14 of it takes the exact FP64 path.
__device__ __forceinline__ bool mac_accept(int4 gt, int4 gs, double theta, double theta2) {
  const long long dx = gt.x - gs.x, dy = gt.y - gs.y, dz = gt.z - gs.z;
  const long long R2 = dx * dx + dy * dy + dz * dz;
  const long long rsum = (1LL << (FMM_LEVELS - gt.w)) + (1LL << (FMM_LEVELS - gs.w));
  const double a = __ll2double_rn(rsum), a2 = __dmul_rn(a, a);
  const double t = __dmul_rn(theta2, __ll2double_rn(R2));
  if (a2 < __dmul_rn(t, 1.0 - 1e-14)) return true;
  if (a2 > __dmul_rn(t, 1.0 + 1e-14)) return false;
  const double rhs = __dmul_rn(theta, __dsqrt_rn(__ll2double_rn(R2)));
  return a <= rhs;
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

#ifndef TRAV_MINB
#define TRAV_MINB 8  // 64 registers: 8 resident blocks per SM (the traversal is latency-bound)
#endif
#ifndef TRAV_CP
#define TRAV_CP 4  // list entries per lane loaded ahead of their stores in the copy-out
#endif
#ifndef TRAV_PF
#define TRAV_PF 0  // children records prefetched per lane per round (0: load each on use; 4:
                   // C2 traversal 0.478 -> 0.501 ms, C4 6.36 -> 6.72, slower)
#endif
__device__ __forceinline__ void trav_cp16(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__global__ void __launch_bounds__(128, TRAV_MINB) k_traverse(TravArgs A) {
#if TRAV_PF
  __shared__ CellRec trec[4][TRAV_PF][32];
  const int wib = threadIdx.x >> 5;
#endif
  const CellsView C = A.C;
  const double theta2 = __dmul_rn(A.theta, A.theta);
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  unsigned *stack = A.scratch + (size_t)gw * A.stack_cap;
  unsigned *osc = A.oscratch + (size_t)gw * 4 * A.ocap;  // [4][ocap] this target's lists
  int2 *rsc = A.rscratch + (size_t)gw * A.ocap;          // P2P source ranges, parallel to [2]

  unsigned long long warp_pp = 0, warp_mp = 0;
  // An earlier level of this attempt overflowed a warp's scratch or a list buffer: its deferred
  // lists are incomplete (or were never copied), so this level must not read them. Every target
  // gets empty lists and the host re-runs the traversal with larger buffers.
  const bool dead = *(volatile unsigned *)A.overflow != 0u || *(volatile int *)&A.bk[12] != 0;
  for (int k = gw; k < A.nt; k += nw) {
    const int t = A.t0 + k;
    const CellRec rt = load_rec(A.pk, t);
    const int4 gt = rt.g;
    const int tcnt = rt.b.y;
    // outside this rank's target partition, or (distinct target / source sets) no target inside
    if (dead || !(rt.b.x < A.thi && rt.b.x + tcnt > A.tlo) || (A.tmask && A.tmask[t] == 0)) {
      if (lane == 0) {
        for (int c = 0; c < 3; ++c) {
          A.loff[c][t] = 0;
          A.lcnt[c][t] = 0;
        }
        A.out_off[t] = 0;
        A.out_cnt[t] = 0;
      }
      continue;
    }
    const bool tleaf = rt.b.w == 0;
    int n[4] = {0, 0, 0, 0};
    // this target's lane partials: source particles of its P2P pairs, number of M2P pairs
    // (32-bit adds per candidate; multiplied by the target's count once, at the end)
    unsigned pp_src = 0, mp_n = 0;
    int top = 0;
    bool overflow = false, ovf_out = false;

    // classify (t, s) and append it to its category with ballots (deterministic order); prec:
    // s's record already in shared memory (else it is loaded here)
    auto consider_and_put = [&](bool valid, unsigned s, int forced_cat, const CellRec *prec = nullptr) {
      int cat = CAT_NONE;
      int scnt = 0, sbeg = 0;
      if (valid) {
        if (forced_cat >= 0) {
          cat = forced_cat;
        } else {
          FMM_DCHECK(FMM_IN(s, g_fmm_chk.cells), "traversal source cell");
          const CellRec rs = prec ? *prec : load_rec(A.pk, s);
          scnt = rs.b.y;
          sbeg = rs.b.x;
          if (mac_accept(gt, rs.g, A.theta, theta2))
            cat = select_kind(A, tcnt, scnt);
          else if (tleaf && rs.b.w == 0)
            cat = CAT_P2P;
          else
            cat = CAT_PUSH;
        }
      }
      pp_src += cat == CAT_P2P ? (unsigned)scnt : 0u;
      mp_n += cat == CAT_M2P ? 1u : 0u;
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
          if (cat == c && n[c] + pos < A.ocap) {
            osc[(size_t)c * A.ocap + n[c] + pos] = s;
            if (c == CAT_P2P) rsc[n[c] + pos] = make_int2(sbeg, scnt);
          }
          n[c] += __popc(b);
          if (n[c] > A.ocap) ovf_out = true;
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
    // (the next batch's source ids are loaded one batch ahead)
    unsigned s_next = lane < in_cnt ? (A.level > 0 ? A.in_src[in_off + lane] : 0u) : 0u;
    for (int b0 = 0; b0 < in_cnt; b0 += 32) {
      const int e = b0 + lane;
      const bool valid = e < in_cnt;
      const unsigned s = s_next;
      s_next = e + 32 < in_cnt ? A.in_src[in_off + e + 32] : 0u;
      consider_and_put(valid, s, -1);
    }
    __syncwarp();
    // 2) the paper's stack: pop, split the larger cell (ties and leaf targets split the source)
    while (top > 0 && !overflow && !ovf_out) {
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
#if TRAV_PF
      // the children's records, TRAV_PF per lane at a time, fetched with cp.async into shared
      // memory before any is classified: one L2 round trip per TRAV_PF children instead of one
      // per child (the children loop is a chain of dependent loads otherwise)
      for (int j0 = 0; j0 < mmax; j0 += TRAV_PF) {
#pragma unroll
        for (int jj = 0; jj < TRAV_PF; ++jj)
          if (j0 + jj < m) {
            const int4 *src = A.pk + 2 * (size_t)(c0 + j0 + jj);
            CellRec *dst = &trec[wib][jj][lane];
            trav_cp16(&dst->g, src);
            trav_cp16(&dst->b, src + 1);
          }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int jj = 0; jj < TRAV_PF; ++jj)
          if (j0 + jj < mmax)
            consider_and_put(j0 + jj < m, (unsigned)(c0 + j0 + jj), -1, &trec[wib][jj][lane]);
        __syncwarp();
      }
#else
      for (int j = 0; j < mmax; ++j) consider_and_put(j < m, (unsigned)(c0 + j), -1);
#endif
      __syncwarp();
    }
    if (overflow || ovf_out) {  // the host re-runs the traversal with larger scratch
      if (lane == 0) {
        atomicOr(A.overflow, overflow ? 1u : 2u);
        for (int c = 0; c < 3; ++c) {
          A.loff[c][t] = 0;
          A.lcnt[c][t] = 0;
        }
        A.out_off[t] = 0;  // the children of t must not read a deferred list that was not written
        A.out_cnt[t] = 0;
      }
      continue;
    }
    // claim the final space of the four lists (running list sizes, this level's deferred pairs:
    // counters in separate 128-byte lines, see TRAV_CNT) and copy them there
    FMM_DCHECK(FMM_IN(t, g_fmm_chk.cells), "traversal target cell");
    int base[4];
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        base[c] = n[c] ? atomicAdd(&A.bk[TRAV_CNT(c)], n[c]) : 0;
        if ((long long)base[c] + n[c] + 1 > A.bk[8 + c]) A.bk[12] = 1;
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) base[c] = __shfl_sync(0xffffffffu, base[c], 0);
    const bool fits = *(volatile int *)&A.bk[12] == 0;
    if (lane == 0) {
      for (int c = 0; c < 3; ++c) {
        A.loff[c][t] = base[c];
        A.lcnt[c][t] = n[c];
      }
      A.out_off[t] = fits ? base[3] : 0;  // not copied: the next level is dead (see `dead`)
      A.out_cnt[t] = fits ? n[3] : 0;
    }
    if (fits) {
      // copy-out in batches of TRAV_CP loads per lane before their stores (the loop was a chain
      // of dependent load -> store round trips)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        unsigned *dst = (c < 3 ? A.lsrc[c] : A.out_src) + base[c];
        const unsigned *src = osc + (size_t)c * A.ocap;
        for (int e0 = 0; e0 < n[c]; e0 += 32 * TRAV_CP) {
          unsigned v[TRAV_CP];
#pragma unroll
          for (int k = 0; k < TRAV_CP; ++k) {
            const int e = e0 + lane + 32 * k;
            v[k] = e < n[c] ? src[e] : 0u;
          }
#pragma unroll
          for (int k = 0; k < TRAV_CP; ++k) {
            const int e = e0 + lane + 32 * k;
            if (e < n[c]) dst[e] = v[k];
          }
        }
      }
      for (int e0 = 0; e0 < n[2]; e0 += 32 * TRAV_CP) {
        int2 v[TRAV_CP];
#pragma unroll
        for (int k = 0; k < TRAV_CP; ++k) {
          const int e = e0 + lane + 32 * k;
          v[k] = e < n[2] ? rsc[e] : make_int2(0, 0);
        }
#pragma unroll
        for (int k = 0; k < TRAV_CP; ++k) {
          const int e = e0 + lane + 32 * k;
          if (e < n[2]) A.p2p_rng[base[2] + e] = v[k];
        }
      }
    }
    __syncwarp();
    warp_pp += (unsigned long long)tcnt * pp_src;  // one atomic per warp at the end
    warp_mp += (unsigned long long)tcnt * mp_n;
  }
  for (int o = 16; o > 0; o >>= 1) {
    warp_pp += __shfl_xor_sync(0xffffffffu, warp_pp, o);
    warp_mp += __shfl_xor_sync(0xffffffffu, warp_mp, o);
  }
  if (lane == 0 && (warp_pp | warp_mp)) {
    atomicAdd(&A.stats[0], warp_pp);
    atomicAdd(&A.stats[1], warp_mp);
  }
}

void launch_traverse(const TravArgs &A, cudaStream_t st) {
  k_traverse<<<A.grid_blocks, 128, 0, st>>>(A);
}

FMM_CHK_DEFINE_SETTER(fmm_chk_set_traverse)
