// m2l.cu — M2L ("O(p^4) cell-cell interaction kernel") as
// class-batched dense products on the FP32 CUDA cores.
//
// The translation of one pair is the linear map  Lhat_j^k(t) += (-1)^{j+k} sum_{n,m} Mhat_n^m(s)
// rho^n I_{n+j}^{m-k}(u),  u = (c_t - c_s)/r_t, rho = r_s/r_t  (expansions.cu header). It depends
// on the pair only through (level difference, integer offset) — its "class". Written over the
// real degrees of freedom of a real field (Re/Im of m >= 0 coefficients), it is a real matrix
// T_class of size 2NC x 2NC. Pairs are sorted by class key, and one CTA per work item (class,
// up to M2L_ITEM pairs) builds T_class in shared memory from the I table of the class and
// multiplies it with the gathered multipoles of the item's sources, 64 pairs per chunk, in a
// register-tiled FP32 product (packed FFMA2). Each pair's result goes to its own slot Y[pair];
// k_m2l_reduce then sums every target's slots in list order, so the result is deterministic and
// independent of how pairs were grouped. The arithmetic is the paper's translation operator
// unchanged; only the evaluation order differs from the direct double loop.
//
// Rare classes (< M2L_SMALL pairs) and orders p > 12 (T too large for shared memory) use
// k_m2l_pairs: one warp per pair evaluating the double loop directly.
#include <cub/cub.cuh>
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

#ifndef M2L_ITEM
#define M2L_ITEM 4096  // pairs per work item: fewer 128-KiB class-matrix loads; 8192 unbalances C2
#endif
#define M2L_PREF 12  // float4 per thread staged for the next chunk (= max over p <= 12 of ceil(Kpad/4*64/threads))
#define M2L_CHUNK 64
#define M2L_SMALL 16
#define M2L_XCH 32  // pair columns per chunk (double-buffered)

// coefficient index c = n(n+1)/2 + m  ->  (n, m)
__device__ __forceinline__ short2 nm_of(int c) {
  int n = (int)((sqrtf(8.f * c + 1.f) - 1.f) * 0.5f);
  while ((n + 1) * (n + 2) / 2 <= c) ++n;
  while (n * (n + 1) / 2 > c) --n;
  return make_short2((short)n, (short)(c - n * (n + 1) / 2));
}

__device__ __forceinline__ float2 cmul2(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// I_a^b(u) for a <= P2 and every signed b, into tab[a*a + a + b]; thread `col` owns column |b|.
__device__ void irregular_table(float ux, float uy, float uz, int P2, float2 *tab, int col,
                                int ncol_threads) {
  const float r2 = ux * ux + uy * uy + uz * uz;
  const float ir2 = 1.f / r2;
  for (int mm = col; mm <= P2; mm += ncol_threads) {
    float2 Imm = make_float2(rsqrtf(r2), 0.f);
    for (int k = 1; k <= mm; ++k) {
      const float2 t = cmul2(Imm, make_float2(ux, uy));
      const float s = -(2.f * k - 1.f) * ir2;
      Imm = make_float2(t.x * s, t.y * s);
    }
    float2 I2 = make_float2(0.f, 0.f), I1 = Imm;
    const float sg = (mm & 1) ? -1.f : 1.f;
    for (int a = mm; a <= P2; ++a) {
      float2 Ia;
      if (a == mm) Ia = Imm;
      else if (a == mm + 1) {
        const float s = (2.f * mm + 1.f) * uz * ir2;
        Ia = make_float2(Imm.x * s, Imm.y * s);
      } else {
        const float c1 = (2.f * a - 1.f) * uz, c2 = (float)(a + mm - 1) * (float)(a - mm - 1);
        Ia = make_float2((c1 * I1.x - c2 * I2.x) * ir2, (c1 * I1.y - c2 * I2.y) * ir2);
      }
      if (a > mm) {
        I2 = I1;
        I1 = Ia;
      }
      tab[a * a + a + mm] = Ia;
      tab[a * a + a - mm] = make_float2(sg * Ia.x, -sg * Ia.y);
    }
  }
}

// Geometry of a pair: target-units offset (u-form when rho <= 1, v = u/rho when rho > 1).
struct PairGeo {
  float ux, uy, uz;
  int dl;
  bool vform;
};
__device__ __forceinline__ PairGeo pair_geo(int4 gt, int4 gs) {
  PairGeo g;
  const float rt_inv = 1.f / (float)(1 << (FMM_LEVELS - gt.w));
  g.dl = gt.w - gs.w;  // rho = 2^dl
  g.ux = (gt.x - gs.x) * rt_inv;
  g.uy = (gt.y - gs.y) * rt_inv;
  g.uz = (gt.z - gs.z) * rt_inv;
  g.vform = g.dl > 0;
  if (g.vform) {
    const float ir = ldexpf(1.f, -g.dl);
    g.ux *= ir;
    g.uy *= ir;
    g.uz *= ir;
  }
  return g;
}

// ---- pair bookkeeping -------------------------------------------------------------------------
// Class key = (level difference, integer offset in units of the smaller cell); the source cell
// id fills the low bits so that, after the radix sort, each class lists its pairs in source
// order (consecutive source cells -> contiguous multipole rows -> one bulk copy per chunk).
// class key (24 bits, so the radix sort takes 3 passes): level difference and the integer offset
// of the two centres in units of the smaller cell. Pairs outside that range get the reserved key
// M2L_KEY_OWN and form classes of their own (evaluated by the direct per-pair path).
#define M2L_KEY_BITS 24
#define M2L_KEY_OWN 0xFFFFFFu
// compact class key (21 bits, so that with the 3 bits of spatial block the radix sort still takes 3
// passes): 6-bit offsets, |offset| <= 30; used when the previous evaluation had no pair outside
// that range (uniform trees), else the 24-bit key (k_m2l_keys reports any pair the compact key
// cannot hold; in compact mode such a pair takes the reserved key: its own class, direct path)
#define M2L_KEYC_BITS 21
#define M2L_KEYC_OWN 0x1FFFFFu
#define M2L_KEYC_LIM 30
__device__ __forceinline__ unsigned cell_block(int4 g, int bl);
__device__ __forceinline__ unsigned m2l_class_key(int4 gt, int4 gs, int bl, int compact,
                                                  bool &any_wide) {
  const int dl = gt.w - gs.w;
  const int sh = FMM_LEVELS - max(gt.w, gs.w);
  const int dx = (gt.x - gs.x) >> sh, dy = (gt.y - gs.y) >> sh, dz = (gt.z - gs.z) >> sh;
  const bool fits_c = abs(dx) <= M2L_KEYC_LIM && abs(dy) <= M2L_KEYC_LIM &&
                      abs(dz) <= M2L_KEYC_LIM && dl >= -4 && dl <= 3;
  any_wide |= !fits_c;
  unsigned key;
  if (compact) {
    key = M2L_KEYC_OWN;
    if (fits_c)  // fields in [2, 62]: never all ones
      key = ((unsigned)(dl + 4) << 18) | ((unsigned)(dx + 32) << 12) | ((unsigned)(dy + 32) << 6) |
            (unsigned)(dz + 32);
  } else {
    key = M2L_KEY_OWN;
    if (abs(dx) < 63 && abs(dy) < 63 && abs(dz) < 63 && dl >= -4 && dl <= 3)  // never all ones
      key = ((unsigned)(dl + 4) << 21) | ((unsigned)(dx + 64) << 14) | ((unsigned)(dy + 64) << 7) |
            (unsigned)(dz + 64);
  }
  // below the class: the spatial block of the target, so that each class is ordered by block
  // and a run (class, block) is contiguous whatever the target levels
  return (key << (3 * bl)) | cell_block(gt, bl);
}

// a warp per target cell over its list segment (the target's grid record read once): class keys,
// the (source, target) records, and -- for the index sort -- pair indices and per-pair targets
__global__ void k_m2l_keys(int ncells, const int *__restrict__ off, const int *__restrict__ cnt,
                          const unsigned *__restrict__ src, CellsView C, int bl,
                          unsigned *__restrict__ keys, unsigned *__restrict__ idx,
                          int *__restrict__ pair_t, uint2 *__restrict__ pst, int compact,
                          int *wide) {
  bool any_wide = false;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < ncells; t += nw) {
    const int o = off[t], c = cnt[t];
    if (c <= 0) continue;
    const int4 gt = C.grid[t];
    for (int k = lane; k < c; k += 32) {
      const int e = o + k;
      const unsigned s = src[e];
      pst[e] = make_uint2(s, (unsigned)t);  // one 8-byte record for the class sort / gather
      keys[e] = m2l_class_key(gt, C.grid[s], bl, compact, any_wide);
      if (idx) {  // (null: the sort carries the records instead)
        idx[e] = (unsigned)e;
        pair_t[e] = t;
      }
    }
  }
  if (__any_sync(0xffffffffu, any_wide) && lane == 0) atomicOr(wide, 1);
}

// Spatial block (Morton index at level bl) of a cell, from its doubled-grid centre. Work items are
// executed block-major (m2l_sort_items), so that at large N the multipole rows of one block's
// neighbourhood and the local rows of its targets stay in L2 while all classes touch them; in
// class-major order every class would stream the whole M and L arrays through L2.
__device__ __forceinline__ unsigned cell_block(int4 g, int bl) {
  if (bl <= 0) return 0u;
  const int sh = FMM_LEVELS + 1 - bl;
  const unsigned bx = (unsigned)g.x >> sh, by = (unsigned)g.y >> sh, bz = (unsigned)g.z >> sh;
  unsigned k = 0;
  for (int b = 0; b < bl; ++b)
    k |= (((bx >> b) & 1u) << (3 * b + 2)) | (((by >> b) & 1u) << (3 * b + 1)) | (((bz >> b) & 1u) << (3 * b));
  return k;
}

// flag = first pair of a class; rflag = first pair of a run (a class's pairs, in target order,
// split where the target's spatial block changes)
__global__ void k_m2l_class_flags(int npairs, const unsigned *__restrict__ skeys,
                                  const unsigned *__restrict__ sidx,
                                  const uint2 *__restrict__ pst, int *__restrict__ flag,
                                  unsigned *__restrict__ ssrc, unsigned *__restrict__ stgt, int bl,
                                  int *__restrict__ rflag, unsigned own) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += gridDim.x * blockDim.x) {
    const unsigned k = skeys[i], cls = k >> (3 * bl);
    const int f = (i == 0 || cls != (skeys[i - 1] >> (3 * bl)) || cls == own) ? 1 : 0;
    flag[i] = f;
    // source and target cell in class-sorted order (one random 8-byte load per pair; later
    // kernels read these arrays coalesced)
    const uint2 st = pst[sidx[i]];
    ssrc[i] = st.x;
    if (stgt) stgt[i] = st.y;
    rflag[i] = f || k != skeys[i - 1];
  }
}

// accumulate mode: the class sort carried the (source, target) records, so the flags pass reads
// them coalesced (the pair-index gather of k_m2l_class_flags was a random 8-byte load per pair)
__global__ void k_m2l_class_flags_sorted(int npairs, const unsigned *__restrict__ skeys,
                                         const uint2 *__restrict__ spst, int *__restrict__ flag,
                                         unsigned *__restrict__ ssrc, unsigned *__restrict__ stgt,
                                         int bl, int *__restrict__ rflag, unsigned own) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += gridDim.x * blockDim.x) {
    const unsigned k = skeys[i], cls = k >> (3 * bl);
    const int f = (i == 0 || cls != (skeys[i - 1] >> (3 * bl)) || cls == own) ? 1 : 0;
    flag[i] = f;
    const uint2 st = spst[i];
    ssrc[i] = st.x;
    stgt[i] = st.y;
    rflag[i] = f || k != skeys[i - 1];
  }
}

__global__ void k_m2l_run_start(int npairs, const int *__restrict__ rflag,
                                const int *__restrict__ rid, int *__restrict__ rstart) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += gridDim.x * blockDim.x) {
    if (rflag[i]) rstart[rid[i]] = i;
    if (i == npairs - 1) rstart[rid[i] + rflag[i]] = npairs;
  }
}

__global__ void k_m2l_class_start(int npairs, const int *__restrict__ flag,
                                  const int *__restrict__ cid, int *__restrict__ cstart,
                                  int *__restrict__ counters) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += gridDim.x * blockDim.x) {
    if (flag[i]) cstart[cid[i]] = i;
    if (i == npairs - 1) {
      const int ncls = cid[i] + flag[i];
      cstart[ncls] = npairs;
      counters[0] = ncls;
    }
  }
}

// counters: [0] classes, [1] GEMM work items, [2] pairs on the direct path, [3] GEMM classes.
// Per class (the GEMM / direct decision is taken on the class's total pair count): a GEMM class
// gets its T index gid, a rare class sends all its pairs to the direct path.
__global__ void k_m2l_class_gid(int npairs, int direct_all, const int *__restrict__ flag,
                                const int *__restrict__ cid, const int *__restrict__ cstart,
                                const unsigned *__restrict__ sidx, int *__restrict__ gid_of,
                                unsigned *__restrict__ small, unsigned *__restrict__ class_rep,
                                int *__restrict__ counters) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += gridDim.x * blockDim.x) {
    if (!flag[i]) continue;
    const int c = cid[i];
    const int n = cstart[c + 1] - i;
    if (!direct_all && n >= M2L_SMALL) {
      const int gid = atomicAdd(&counters[3], 1);
      class_rep[gid] = sidx ? sidx[i] : (unsigned)i;  // accumulate mode: the sorted position
      gid_of[c] = gid;
    } else {
      gid_of[c] = -1;
      const int base = atomicAdd(&counters[2], n);
      for (int b = 0; b < n; ++b) small[base + b] = sidx ? sidx[i + b] : (unsigned)(i + b);
    }
  }
}
// Per run of a GEMM class: work items of <= M2L_ITEM pairs, each with its execution-order key
// (spatial block of the run's targets, class)
__global__ void k_m2l_run_items(int npairs, const int *__restrict__ flag, const int *__restrict__ rflag,
                                const int *__restrict__ rid, const int *__restrict__ rstart,
                                const int *__restrict__ cid, const int *__restrict__ gid_of,
                                const unsigned *__restrict__ sidx, const unsigned *__restrict__ skeys,
                                int bl, int4 *__restrict__ items,
                                unsigned *__restrict__ ikeys, unsigned *__restrict__ iidx,
                                int *__restrict__ counters) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += gridDim.x * blockDim.x) {
    if (!rflag[i]) continue;
    // cid is an exclusive scan of the class flags: the class of position i is cid + flag - 1
    const int gid = gid_of[cid[i] + flag[i] - 1];
    if (gid < 0) continue;
    const int n = rstart[rid[i] + 1] - i;
    const int ni = (n + M2L_ITEM - 1) / M2L_ITEM;
    const int base = atomicAdd(&counters[1], ni);
    const unsigned key = ((skeys[i] & ((1u << (3 * bl)) - 1u)) << 20) | (unsigned)gid;
    for (int a = 0; a < ni; ++a) {
      items[base + a] = make_int4(i + a * M2L_ITEM, min(M2L_ITEM, n - a * M2L_ITEM), i, gid);
      ikeys[base + a] = key;
      iidx[base + a] = (unsigned)(base + a);
    }
  }
}
__global__ void k_m2l_gather_items(int n, const unsigned *__restrict__ order,
                                   const int4 *__restrict__ in, int4 *__restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = in[order[i]];
}

// ---- class translation matrices ---------------------------------------------------------------
// T_g[kcol][row] (Kpad x Rpad floats) for GEMM class g: row = output real index (2 c_out + re/im),
// kcol = input real index (2 c_in + re/im); derived from I(u) of the class representative.
__global__ void __launch_bounds__(256) k_m2l_build_T(int p, const int *__restrict__ counters,
                                                     const unsigned *__restrict__ class_rep,
                                                     const int *__restrict__ pair_t,
                                                     const unsigned *__restrict__ src,
                                                     CellsView C, float *__restrict__ Tg) {
  extern __shared__ float2 sh_itab[];
  const int NC = nc_of(p), KR = 2 * NC;
  const int Kpad = (KR + 3) & ~3, Rpad = ((KR + 11) / 12) * 12;
  const int ng = counters[3];
  for (int gid = blockIdx.x; gid < ng; gid += gridDim.x) {
    const int rep = class_rep[gid];
    const PairGeo g = pair_geo(C.grid[pair_t[rep]], C.grid[src[rep]]);
    __syncthreads();
    irregular_table(g.ux, g.uy, g.uz, 2 * p, sh_itab, threadIdx.x, blockDim.x);
    __syncthreads();
    float *T = Tg + (size_t)gid * Kpad * Rpad;
    for (int id = threadIdx.x; id < Kpad * Rpad; id += blockDim.x) {
      const int kcol = id / Rpad, row = id - kcol * Rpad;
      float v = 0.f;
      if (row < KR && kcol < KR) {
        const short2 jo = nm_of(row >> 1), ni = nm_of(kcol >> 1);
        const int j = jo.x, k = jo.y, n = ni.x, m = ni.y;
        const int rim = row & 1, cim = kcol & 1;
        if (!(k == 0 && rim) && !(m == 0 && cim)) {
          const float sgn = ((j + k) & 1) ? -1.f : 1.f;
          const float sc = sgn * (g.vform ? ldexpf(1.f, -g.dl * (j + 1)) : ldexpf(1.f, n * g.dl));
          const int a = n + j;
          const float2 Cp = sh_itab[a * a + a + (m - k)];
          if (m == 0) {
            v = sc * (rim ? Cp.y : Cp.x);
          } else {
            const float2 Cm = sh_itab[a * a + a + (-m - k)];
            const float sm = (m & 1) ? -1.f : 1.f;
            if (!cim)  // coefficient of Re M: Cp + (-1)^m Cm
              v = sc * (rim ? (Cp.y + sm * Cm.y) : (Cp.x + sm * Cm.x));
            else       // coefficient of Im M: i (Cp - (-1)^m Cm)
              v = sc * (rim ? (Cp.x - sm * Cm.x) : -(Cp.y - sm * Cm.y));
          }
        }
      }
      T[id] = v;
    }
  }
}

// ---- TMA bulk copies + mbarriers (sm_90+ PTX; SASS UBLKCP / SYNCS) ------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred P1;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n }" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- class GEMM -------------------------------------------------------------------------------
// Warp-specialised CTA per group of work items (class g, up to M2L_ITEM pairs each):
//   * producer warp: TMA bulk copy of T_g (one copy) and, per chunk of M2L_XCH pairs, one bulk
//     copy per source cell's multipole row into a double-buffered tile; full/empty mbarriers;
//   * consumer warps: thread (rg, cg) owns rows [12 rg, 12 rg + 12) and pair columns {cg, cg+16}
//     of the 2NC x M2L_XCH chunk product: 12 packed FFMA2 per 3 broadcast LDS.128 of T and
//     2 LDS.128 of X every 4 k. No CTA-wide barrier inside the item loop.
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int p>
__global__ void __launch_bounds__(288, 2) k_m2l_gemm(const int4 *__restrict__ items,
                                                     const int *__restrict__ counters,
                                                     const unsigned *__restrict__ sidx,
                                                     const unsigned *__restrict__ ssrc,
                                                     const float *__restrict__ Tg,
                                                     const float *__restrict__ M,
                                                     float *__restrict__ Y, int *queue) {
  extern __shared__ __align__(128) float sh_gemm[];
  constexpr int NC = nc_of(p), KR = 2 * NC;
  constexpr int Kpad = (KR + 3) & ~3, Rpad = ((KR + 11) / 12) * 12;
  constexpr int XKS = ((Kpad >> 2) & 1) ? Kpad : Kpad + 4;  // X row stride: odd # of 16-B slots
  constexpr int ncons = (Rpad / 12) * 16;                    // consumer threads
  constexpr int ncw = (ncons + 31) / 32;                     // consumer warps; the next produces
  float *Ts = sh_gemm;
  float *Xs0 = Ts + Kpad * Rpad;  // double buffer: Xs0 + b * M2L_XCH * XKS
  unsigned long long *bars = reinterpret_cast<unsigned long long *>(Xs0 + 2 * M2L_XCH * XKS);
  unsigned long long *t_full = &bars[0], *t_empty = &bars[1];
  unsigned long long *x_full = &bars[2], *x_empty = &bars[4];  // [2] each
  volatile int *item_slot = reinterpret_cast<volatile int *>(&bars[6]);  // [2]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned tbytes = (unsigned)(Kpad * Rpad * sizeof(float));
  const unsigned rbytes = (unsigned)(Kpad * sizeof(float));
  if (tid == 0) {
    mbar_init(t_full, 1);
    mbar_init(t_empty, ncw);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&x_full[b], 1);
      mbar_init(&x_empty[b], ncw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nitems = counters[1];

  if (warp == ncw) {  // ---------------- producer ----------------
    int g = 0, ii = 0;
    for (;; ++ii) {
      int it = 0;
      if (lane == 0) it = atomicAdd(&queue[0], 1);  // dynamic item queue
      it = __shfl_sync(0xffffffffu, it, 0);
      if (lane == 0) item_slot[ii & 1] = it;         // hand the item index to the consumers
      if (it >= nitems) {
        // release the consumers with a sentinel phase; first make sure the previous phase of
        // t_full has completed (the consumers finished the previous item), otherwise this arrival
        // would land in the still-pending phase
        if (ii > 0) mbar_wait(t_empty, (ii - 1) & 1);
        if (lane == 0) mbar_expect_tx(t_full, 0);
        break;
      }
      const int4 item = items[it];
      const int pos0 = item.x, cnt = item.y, gid = item.w;
      if (ii > 0) mbar_wait(t_empty, (ii - 1) & 1);
      if (lane == 0) {
        fence_proxy_async();
        mbar_expect_tx(t_full, tbytes);
        bulk_g2s(Ts, Tg + (size_t)gid * Kpad * Rpad, tbytes, t_full);
      }
      for (int c0 = 0; c0 < cnt; c0 += M2L_XCH, ++g) {
        const int b = g & 1, use = g >> 1;
        const int ncol = min(M2L_XCH, cnt - c0);
        // source ids are loaded before waiting for the buffer (the asm wait is a memory fence
        // for the compiler, so the load would otherwise sit on the critical path)
        const int s = lane < ncol ? (int)__ldg(&ssrc[pos0 + c0 + lane]) : 0;
        if (use > 0) mbar_wait(&x_empty[b], (use - 1) & 1);
        const int s0 = __shfl_sync(0xffffffffu, s, 0), sl = __shfl_sync(0xffffffffu, s, ncol - 1);
        const bool contiguous = (XKS == Kpad) && (sl - s0 == ncol - 1) &&
                                __all_sync(0xffffffffu, lane >= ncol || s == s0 + lane);
        if (lane == 0) mbar_expect_tx(&x_full[b], ncol * rbytes);
        __syncwarp();
        if (contiguous) {  // consecutive source cells: one copy of ncol rows
          if (lane == 0) {
            fence_proxy_async();
            bulk_g2s(Xs0 + b * M2L_XCH * XKS, M + (size_t)s0 * Kpad, ncol * rbytes, &x_full[b]);
          }
        } else if (lane < ncol) {
          fence_proxy_async();
          bulk_g2s(Xs0 + b * M2L_XCH * XKS + lane * XKS, M + (size_t)s * Kpad, rbytes, &x_full[b]);
        }
      }
    }
    return;
  }
  // ---------------- consumers ----------------
  const int rg = tid >> 4, cg = tid & 15;
  const bool active = tid < ncons;
  int g = 0, ii = 0;
  for (;; ++ii) {
    mbar_wait(t_full, ii & 1);
    const int it = item_slot[ii & 1];
    if (it >= nitems) break;
    const int4 item = items[it];
    const int pos0 = item.x, cnt = item.y;
    for (int c0 = 0; c0 < cnt; c0 += M2L_XCH, ++g) {
      const int b = g & 1, use = g >> 1;
      const int ncol = min(M2L_XCH, cnt - c0);
      // output rows of this thread's two pair columns, fetched before the product
      const unsigned y0 = cg < ncol ? sidx[pos0 + c0 + cg] : 0u;
      const unsigned y1 = cg + 16 < ncol ? sidx[pos0 + c0 + cg + 16] : 0u;
      mbar_wait(&x_full[b], use & 1);
      if (active) {
        float2 acc[6][2];
#pragma unroll
        for (int a = 0; a < 6; ++a) acc[a][0] = acc[a][1] = make_float2(0.f, 0.f);
        const float *Tp = Ts + rg * 12;
        const float *Xb = Xs0 + b * M2L_XCH * XKS;
        const float *x0p = Xb + cg * XKS, *x1p = Xb + (cg + 16) * XKS;
#pragma unroll 3
        for (int k = 0; k < Kpad; k += 4) {
          const float4 xa = *reinterpret_cast<const float4 *>(x0p + k);
          const float4 xb = *reinterpret_cast<const float4 *>(x1p + k);
          const float xav[4] = {xa.x, xa.y, xa.z, xa.w}, xbv[4] = {xb.x, xb.y, xb.z, xb.w};
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const float *tr = Tp + (k + kk) * Rpad;
            const float4 t0 = *reinterpret_cast<const float4 *>(tr);
            const float4 t1 = *reinterpret_cast<const float4 *>(tr + 4);
            const float4 t2 = *reinterpret_cast<const float4 *>(tr + 8);
            const float2 tv[6] = {make_float2(t0.x, t0.y), make_float2(t0.z, t0.w),
                                  make_float2(t1.x, t1.y), make_float2(t1.z, t1.w),
                                  make_float2(t2.x, t2.y), make_float2(t2.z, t2.w)};
            const float2 xs0 = make_float2(xav[kk], xav[kk]), xs1 = make_float2(xbv[kk], xbv[kk]);
#pragma unroll
            for (int a = 0; a < 6; ++a) {
              acc[a][0] = __ffma2_rn(tv[a], xs0, acc[a][0]);
              acc[a][1] = __ffma2_rn(tv[a], xs1, acc[a][1]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&x_empty[b]);  // this warp is done reading Xs[b]
        const int YS = Kpad;
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) {
          const int col = cg + 16 * bb;
          if (col >= ncol) continue;
          float *yr = Y + (size_t)(bb ? y1 : y0) * YS + rg * 12;
#pragma unroll
          for (int a = 0; a < 6; ++a) {
            const int r = rg * 12 + 2 * a;
            if (r + 1 < KR) *reinterpret_cast<float2 *>(yr + 2 * a) = acc[a][bb];
            else if (r < KR) yr[2 * a] = acc[a][bb].x;
          }
        }
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&x_empty[b]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(t_empty);  // this warp no longer reads Ts
  }
}

// ---- direct per-pair path (rare classes, p > 12) -------------------------------------------------
__global__ void __launch_bounds__(128) k_m2l_pairs(int p, const unsigned *__restrict__ list,
                                                   const int *__restrict__ counters,
                                                   const int *__restrict__ pair_t,
                                                   const unsigned *__restrict__ src, CellsView C,
                                                   const float2 *__restrict__ M,
                                                   float *__restrict__ Y, int ydof,
                                                   float *__restrict__ Lacc) {
  extern __shared__ float2 sh_pairs[];
  const int NC = nc_of(p), KR = 2 * NC, YS = (KR + 3) & ~3;
  const int P2 = 2 * p, nI = (P2 + 1) * (P2 + 1), nM = (p + 1) * (p + 1);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float2 *Mx = sh_pairs + wib * (nM + nI);
  float2 *Ix = Mx + nM;
  const int npairs = counters[2];
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int q = gw; q < npairs; q += nw) {
    const int e = list[q];
    const int s = src[e];
    const PairGeo g = pair_geo(C.grid[pair_t[e]], C.grid[s]);
    __syncwarp();
    for (int o = lane; o < nM; o += 32) {
      const int n = (int)sqrtf((float)o + 0.5f);
      const int m = o - n * n - n;
      const float2 v = sget(M + (size_t)s * nc_stride(p), n, m);
      const float sc = g.vform ? 1.f : ldexpf(1.f, n * g.dl);
      Mx[o] = make_float2(v.x * sc, v.y * sc);
    }
    irregular_table(g.ux, g.uy, g.uz, P2, Ix, lane, 32);
    __syncwarp();
    for (int o = lane; o < NC; o += 32) {
      const short2 jk = nm_of(o);
      const int j = jk.x, k = jk.y;
      float re = 0.f, im = 0.f;
      for (int n = 0; n <= p; ++n) {
        const float2 *Irow = Ix + (n + j) * (n + j) + (n + j);
        const float2 *Mrow = Mx + n * n + n;
        for (int m = -n; m <= n; ++m) {
          const float2 a = Mrow[m], b = Irow[m - k];
          re += a.x * b.x - a.y * b.y;
          im += a.x * b.y + a.y * b.x;
        }
      }
      const float sgn = ((j + k) & 1) ? -1.f : 1.f;
      const float sc = sgn * (g.vform ? ldexpf(1.f, -g.dl * (j + 1)) : 1.f);
      if (Lacc) {  // accumulate mode: straight into the target's expansion
        float *lr = Lacc + (size_t)pair_t[e] * 2 * nc_stride(p) + 2 * o;
        atomicAdd(lr, sc * re);
        if (k > 0) atomicAdd(lr + 1, sc * im);
      } else if (ydof) {  // tensor-core layout: dof order, stride dof_stride(p)
        const int d = j * j + (k == 0 ? 0 : 2 * k - 1);
        Y[(size_t)e * dof_stride(p) + d] = sc * re;
        if (k > 0) Y[(size_t)e * dof_stride(p) + d + 1] = sc * im;
      } else {
        Y[(size_t)e * YS + 2 * o] = sc * re;
        Y[(size_t)e * YS + 2 * o + 1] = (k == 0) ? 0.f : sc * im;
      }
    }
  }
}

// ---- per-target sum of the pair slots, in list order -------------------------------------------
// thread per (target, float4 column q): consecutive threads cover a target's row, so every load of
// a warp is a contiguous piece of one or two Y rows; each column is summed in list order.
// ydof: Y rows in dof order (tensor-core path), scattered into the float-order L row here.
__global__ void __launch_bounds__(256) k_m2l_reduce(int p, int ncells, const int *__restrict__ off,
                                                    const int *__restrict__ cnt,
                                                    const float *__restrict__ Y,
                                                    float *__restrict__ L, int ydof) {
  const int KR = 2 * nc_of(p), KD = dof_of(p);
  const int YSr = ydof ? dof_stride(p) : ((KR + 3) & ~3), NQ = YSr / 4;
  const int LS = 2 * nc_stride(p);  // L row stride (floats), multiple of 4
  const float4 *Y4 = reinterpret_cast<const float4 *>(Y);
  const long long total = (long long)ncells * NQ;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(i / NQ), q = (int)(i - (long long)t * NQ);
    const int o = off[t], c = cnt[t];
    FMM_DCHECK(o >= 0 && (long long)o + c <= g_fmm_chk.yrows && FMM_IN(t, g_fmm_chk.rows),
               "M2L per-pair slots of a target");
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 *y = Y4 + (size_t)o * NQ + q;
#pragma unroll 4
    for (int e = 0; e < c; ++e) {
      const float4 v = __ldcs(y + (size_t)e * NQ);
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    float *lr = L + (size_t)t * LS;
    if (ydof) {
      const float sv[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (4 * q + e < KD) lr[dof_to_float(4 * q + e)] = sv[e];
      if (q == 0)
        for (int n = 0; n <= p; ++n) lr[2 * cidx(n, 0) + 1] = 0.f;
    } else {
      lr += 4 * q;
      if (4 * q + 3 < KR) {
        *reinterpret_cast<float4 *>(lr) = s;
      } else {
        if (4 * q + 0 < KR) lr[0] = s.x;
        if (4 * q + 1 < KR) lr[1] = s.y;
        if (4 * q + 2 < KR) lr[2] = s.z;
      }
    }
  }
}

// ---- host orchestration -----------------------------------------------------------------------
size_t m2l_gemm_smem(int p) {
  const int KR = 2 * nc_of(p);
  const int Kpad = (KR + 3) & ~3, Rpad = ((KR + 11) / 12) * 12;
  const int XKS = ((Kpad >> 2) & 1) ? Kpad : Kpad + 4;
  return (size_t)(Kpad * Rpad + 2 * M2L_XCH * XKS) * sizeof(float) + 8 * sizeof(unsigned long long);
}
size_t m2l_T_floats(int p) {
  const int KR = 2 * nc_of(p);
  return (size_t)((KR + 3) & ~3) * (((KR + 11) / 12) * 12);
}
bool m2l_gemm_supported(int p) {
  const int KR = 2 * nc_of(p), nthr = (((KR + 11) / 12) * 16 + 31) / 32 * 32 + 32;
  return m2l_gemm_smem(p) <= 227 * 1024 && nthr <= 288;
}
int m2l_y_stride(int p) { return (2 * nc_of(p) + 3) & ~3; }

cudaError_t m2l_prepare(const M2LWork &W, int npairs, int ncells, cudaStream_t st) {
  const int b = (npairs + 255) / 256 < 148 * 16 ? (npairs + 255) / 256 : 148 * 16;
  cudaMemsetAsync(W.counters + 6, 0, sizeof(int), st);
  k_m2l_keys<<<148 * 8, 128, 0, st>>>(ncells, W.off, W.cnt, W.src, W.C, W.blk_level, W.keys_in,
                                      W.spst ? nullptr : W.idx_in, W.pair_t, W.pst, W.compact_key,
                                      W.counters + 6);
  const int kbits = (W.compact_key ? M2L_KEYC_BITS : M2L_KEY_BITS) + 3 * W.blk_level;
  size_t bytes = 0;
  cudaError_t e;
  const bool by_record = W.spst != nullptr;  // accumulate mode: sort the (source, target) records
  if (by_record) {
    unsigned long long *vin = reinterpret_cast<unsigned long long *>(W.pst);
    unsigned long long *vout = reinterpret_cast<unsigned long long *>(W.spst);
    e = cub::DeviceRadixSort::SortPairs(nullptr, bytes, W.keys_in, W.keys, vin, vout, npairs, 0,
                                        kbits, st);
    if (e) return e;
    if (bytes > W.tmp_bytes) return cudaErrorMemoryAllocation;
    e = cub::DeviceRadixSort::SortPairs(W.tmp, bytes, W.keys_in, W.keys, vin, vout, npairs, 0, kbits,
                                        st);
    if (e) return e;
    k_m2l_class_flags_sorted<<<b > 0 ? b : 1, 256, 0, st>>>(
        npairs, W.keys, W.spst, W.flag, W.ssrc, W.stgt, W.blk_level, W.rflag,
        W.compact_key ? M2L_KEYC_OWN : M2L_KEY_OWN);
  } else {
    e = cub::DeviceRadixSort::SortPairs(nullptr, bytes, W.keys_in, W.keys, W.idx_in, W.sidx, npairs,
                                        0, kbits, st);
    if (e) return e;
    if (bytes > W.tmp_bytes) return cudaErrorMemoryAllocation;
    e = cub::DeviceRadixSort::SortPairs(W.tmp, bytes, W.keys_in, W.keys, W.idx_in, W.sidx, npairs, 0,
                                        kbits, st);
    if (e) return e;
    k_m2l_class_flags<<<b > 0 ? b : 1, 256, 0, st>>>(npairs, W.keys, W.sidx, W.pst, W.flag, W.ssrc,
                                                      W.stgt, W.blk_level, W.rflag,
                                                      W.compact_key ? M2L_KEYC_OWN : M2L_KEY_OWN);
  }
  const unsigned *sidx = by_record ? nullptr : W.sidx;  // (pair indices exist only without records)
  bytes = 0;
  e = cub::DeviceScan::ExclusiveSum(nullptr, bytes, W.flag, W.cid, npairs, st);
  if (e) return e;
  if (bytes > W.tmp_bytes) return cudaErrorMemoryAllocation;
  e = cub::DeviceScan::ExclusiveSum(W.tmp, bytes, W.flag, W.cid, npairs, st);
  if (e) return e;
  e = cub::DeviceScan::ExclusiveSum(W.tmp, bytes, W.rflag, W.rid, npairs, st);
  if (e) return e;
  cudaMemsetAsync(W.counters, 0, 4 * sizeof(int), st);
  k_m2l_class_start<<<b > 0 ? b : 1, 256, 0, st>>>(npairs, W.flag, W.cid, W.cstart, W.counters);
  k_m2l_run_start<<<b > 0 ? b : 1, 256, 0, st>>>(npairs, W.rflag, W.rid, W.rstart);
  k_m2l_class_gid<<<b > 0 ? b : 1, 256, 0, st>>>(npairs, W.direct_all, W.flag, W.cid, W.cstart,
                                                 sidx, W.gid_of, W.small, W.class_rep, W.counters);
  k_m2l_run_items<<<b > 0 ? b : 1, 256, 0, st>>>(npairs, W.flag, W.rflag, W.rid, W.rstart, W.cid, W.gid_of,
                                                 sidx, W.keys, W.blk_level, W.items_raw,
                                                 W.ikeys_in, W.iidx_in, W.counters);
  return cudaGetLastError();
}

// block-major execution order of the nitems work items (counters[1], read back by the host)
cudaError_t m2l_sort_items(const M2LWork &W, int nitems, cudaStream_t st) {
  if (nitems <= 0) return cudaSuccess;
  size_t bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, bytes, W.ikeys_in, W.ikeys, W.iidx_in,
                                                  W.iidx, nitems, 0, 32, st);
  if (e) return e;
  if (bytes > W.tmp_bytes) return cudaErrorMemoryAllocation;
  e = cub::DeviceRadixSort::SortPairs(W.tmp, bytes, W.ikeys_in, W.ikeys, W.iidx_in, W.iidx, nitems,
                                      0, 32, st);
  if (e) return e;
  const int b = (nitems + 255) / 256 < 148 * 8 ? (nitems + 255) / 256 : 148 * 8;
  k_m2l_gather_items<<<b, 256, 0, st>>>(nitems, W.iidx, W.items_raw, W.items);
  return cudaGetLastError();
}

size_t m2l_temp_bytes(int npairs) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (unsigned *)nullptr, (unsigned *)nullptr,
                                  (unsigned *)nullptr, (unsigned *)nullptr, npairs, 0, 32);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int *)nullptr, (int *)nullptr, npairs);
  size_t c = 0;  // the work-item sort (at most npairs items, 32-bit keys)
  cub::DeviceRadixSort::SortPairs(nullptr, c, (unsigned *)nullptr, (unsigned *)nullptr,
                                  (unsigned *)nullptr, (unsigned *)nullptr, npairs, 0, 32);
  size_t d = 0;  // the accumulate mode's class sort carries the 8-byte (source, target) records
  cub::DeviceRadixSort::SortPairs(nullptr, d, (unsigned *)nullptr, (unsigned *)nullptr,
                                  (unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                  npairs, 0, 32);
  return std::max(std::max(a, d), std::max(b, c));
}

cudaError_t m2l_build_T(int p, const M2LWork &W, int ngclass, cudaStream_t st) {
  if (ngclass <= 0) return cudaSuccess;
  const size_t smem = (size_t)(2 * p + 1) * (2 * p + 1) * sizeof(float2);
  k_m2l_build_T<<<ngclass < 148 * 4 ? ngclass : 148 * 4, 256, smem, st>>>(
      p, W.counters, W.class_rep, W.pair_t, W.src, W.C, W.Tg);
  return cudaGetLastError();
}

cudaError_t m2l_execute(int p, const M2LWork &W, int npairs, int ncells, const float2 *M,
                        float2 *L, cudaStream_t st, bool gemm_done, bool accum, int ydof) {
  if (ydof < 0) ydof = gemm_done ? 1 : 0;
  if (!W.direct_all && !gemm_done) {
    const size_t smem = m2l_gemm_smem(p);
    const int KR = 2 * nc_of(p);
    const int nthr = (((KR + 11) / 12) * 16 + 31) / 32 * 32 + 32;  // consumer warps + producer
    const int per_sm = (int)((227 * 1024) / smem) < 2 ? 1 : 2;
    cudaMemsetAsync(W.counters + 4, 0, sizeof(int), st);
#define M2L_GEMM_CASE(PP)                                                                    \
  case PP: {                                                                               \
    fmm_smem_optin((const void *)k_m2l_gemm<PP>, smem);                                    \
    k_m2l_gemm<PP><<<148 * per_sm, nthr, smem, st>>>(W.items, W.counters, W.sidx, W.ssrc, W.Tg, \
                                                    reinterpret_cast<const float *>(M), W.Y, \
                                                    W.counters + 4);                     \
  } break;
    switch (p) {
      M2L_GEMM_CASE(1) M2L_GEMM_CASE(2) M2L_GEMM_CASE(3) M2L_GEMM_CASE(4) M2L_GEMM_CASE(5)
      M2L_GEMM_CASE(6) M2L_GEMM_CASE(7) M2L_GEMM_CASE(8) M2L_GEMM_CASE(9) M2L_GEMM_CASE(10)
      M2L_GEMM_CASE(11) M2L_GEMM_CASE(12)
      default: break;
    }
#undef M2L_GEMM_CASE
  }
  {
    const int nI = (2 * p + 1) * (2 * p + 1), nM = (p + 1) * (p + 1);
    const size_t smem = (size_t)4 * (nI + nM) * sizeof(float2);
    fmm_smem_optin((const void *)k_m2l_pairs, smem);
    k_m2l_pairs<<<148 * 4, 128, smem, st>>>(p, W.small, W.counters, W.pair_t, W.src, W.C, M, W.Y,
                                            ydof, accum ? reinterpret_cast<float *>(L) : nullptr);
  }
  if (!accum) {
    const long long nthr = (long long)ncells * ((ydof ? dof_stride(p) : m2l_y_stride(p)) / 4);
    int b = (int)std::min<long long>((nthr + 255) / 256, 148 * 16);
    b = b > 0 ? b : 1;
    k_m2l_reduce<<<b, 256, 0, st>>>(p, ncells, W.off, W.cnt, W.Y, reinterpret_cast<float *>(L),
                                    ydof);
  }
  return cudaGetLastError();
}

FMM_CHK_DEFINE_SETTER(fmm_chk_set_m2l)
