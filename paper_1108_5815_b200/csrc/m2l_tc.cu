// m2l_tc.cu — M2L class GEMMs on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// After class batching (m2l.cu) the translations of one class are a dense product
//     D[pair][out] = sum_k X[pair][k] * T[out][k]
// over the real degrees of freedom of a real field: d = 0..(p+1)^2-1 enumerates
// (n, m=0, Re), (n, m>0, Re), (n, m>0, Im) of every coefficient (the Im part of m = 0 is zero).
// At p = 10 that is 121 -> padded to K = N = 128 (multiples of 32: TMEM is moved in 32-column chunks). FP32 accuracy comes from 3xTF32 splitting:
//     X = Xh + Xl, T = Th + Tl (each part TF32), D = Xh Th + Xh Tl + Xl Th
// (the dropped Xl Tl term is ~2^-22 relative), accumulated in FP32 in TMEM.
//
// One CTA per SM (persistent, dynamic item queue), 4 warps = 128 threads:
//   * A operand (X tile, 128 pairs x K) lives in TMEM: thread i = TMEM lane i = pair i loads its
//     source multipole row, splits it and writes Xh, Xl with tcgen05.st;
//   * B operand (class matrix, N x K, hi and lo) is one TMA bulk copy of a pre-arranged K-major
//     core-matrix image into shared memory (built once per class by k_m2l_build_T_tc);
//   * one elected thread issues 3 * K/8 tcgen05.mma.kind::tf32 (M = 128, N = K, K = 8 each);
//     tcgen05.commit signals an mbarrier;
//   * D (128 lanes x N columns FP32) is read back with tcgen05.ld and written to the pair slots
//     Y[pair] in the same layout as the CUDA-core path, so k_m2l_reduce is shared.
#include <cub/cub.cuh>
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace {

// K = N is padded to at least 96 when the dofs exceed 32 (p = 5..7: 36..64 dofs): with K = N =
// 64 this kernel runs 3-4x slower than with the zero-padded 96 (C2 M2L at p = 5 / 6 / 7: 2.23 /
// 3.00 / 4.07 ms at 64, 0.67 / 0.76 / 0.92 ms at 96; measured, cause not identified), which made
// p = 5..7 slower than p = 8 (the "p = 6 outlier")
#ifndef TC_DIM_MIN
#define TC_DIM_MIN 96
#endif
__host__ __device__ constexpr int tc_dim(int p) {  // K = N, 32-column TMEM chunks
  return ((dof_of(p) + 31) & ~31) < TC_DIM_MIN && dof_of(p) > 32 ? TC_DIM_MIN : ((dof_of(p) + 31) & ~31);
}

__device__ __forceinline__ unsigned smem_addr(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init_tc(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx_tc(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_tc(unsigned long long *bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_TC:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE_TC;\n bra WAIT_TC;\n DONE_TC:\n }" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_tc(void *dst, const void *src, unsigned bytes,
                                            unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ unsigned f32_to_tf32(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// x = hi + lo for 3xTF32: hi = x rounded to the nearest TF32 (half an ulp of the 13 dropped bits
// added to the bit pattern, then truncated; the sign-magnitude format makes it round half away
// from zero), lo = x - hi (exact in FP32, |lo| <= 2^-12 |x|) rounded the same way, so the split
// loses <= 2^-24 |x| (a truncating split, hi = x & mask with the tensor core truncating lo: up to
// 2^-22 -- measured: a 3x larger phi error floor vs direct at p = 11..15). 4 integer ops + 1 FADD
// instead of two emulated cvt.rna.tf32.
__device__ __forceinline__ void tf32_split(float x, unsigned &hi, unsigned &lo) {
  hi = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
  lo = (__float_as_uint(x - __uint_as_float(hi)) + 0x1000u) & 0xFFFFE000u;
}

// tcgen05 wrappers -------------------------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_st32(unsigned taddr, const unsigned (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tc_ld32(unsigned taddr, unsigned (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]^T, kind::tf32, cta_group::1
__device__ __forceinline__ void tc_mma_ts(unsigned d_tmem, unsigned a_tmem, unsigned long long bdesc,
                                          unsigned idesc, unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit(unsigned long long *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_addr(bar))
               : "memory");
}

// K-major, no-swizzle ("interleaved") shared-memory operand: element (row, k) of an NR-row
// operand at byte (k/4)*(NR*16) + row*16 + (k%4)*4, i.e. 8x16-byte core matrices; the two
// 16-byte k-chunks of one K=8 MMA are LBO = NR*16 apart, 8-row groups SBO = 128 B apart.
__device__ __forceinline__ unsigned long long make_bdesc(unsigned saddr, int nrows) {
  unsigned long long d = 0;
  d |= (unsigned long long)((saddr >> 4) & 0x3fff);                  // start address
  d |= (unsigned long long)(((nrows * 16) >> 4) & 0x3fff) << 16;     // leading byte offset
  d |= (unsigned long long)((128 >> 4) & 0x3fff) << 32;              // stride byte offset
  d |= 1ull << 46;                                                   // version (sm_100)
  // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
  return d;
}

}  // namespace

// per class: Th | Tl images (N x K each, N = K = tc_dim(p)) in the core-matrix layout above,
// from the same translation formula as the CUDA-core k_m2l_build_T (m2l.cu header)
__global__ void __launch_bounds__(256) k_m2l_build_T_tc(int p, const int *__restrict__ counters,
                                                        const unsigned *__restrict__ class_rep,
                                                        const int *__restrict__ pair_t,
                                                        const unsigned *__restrict__ src,
                                                        CellsView C, unsigned *__restrict__ Timg) {
  extern __shared__ float2 itab_tc[];
  __shared__ int dec[512];  // dof -> n | m << 6 | part << 12
  const int KD = dof_of(p), NT = tc_dim(p);
  const int ng = counters[3];
  for (int d = threadIdx.x; d < KD; d += blockDim.x) {
    int n = 0;
    while ((n + 1) * (n + 1) <= d) ++n;
    const int r = d - n * n, m = (r + 1) / 2, part = r ? ((r + 1) & 1) : 0;
    dec[d] = n | (m << 6) | (part << 12);
  }
  for (int gid = blockIdx.x; gid < ng; gid += gridDim.x) {
    const int rep = class_rep[gid];
    const int4 gt = C.grid[pair_t[rep]], gs = C.grid[src[rep]];
    const float rt_inv = 1.f / (float)(1 << (FMM_LEVELS - gt.w));
    const int dl = gt.w - gs.w;
    float ux = (gt.x - gs.x) * rt_inv, uy = (gt.y - gs.y) * rt_inv, uz = (gt.z - gs.z) * rt_inv;
    const bool vform = dl > 0;
    if (vform) {
      const float ir = ldexpf(1.f, -dl);
      ux *= ir;
      uy *= ir;
      uz *= ir;
    }
    __syncthreads();
    // irregular harmonics I_a^b(u), a <= 2p, signed b (same recurrences as m2l.cu)
    {
      const float r2 = ux * ux + uy * uy + uz * uz, ir2 = 1.f / r2;
      for (int mm = threadIdx.x; mm <= 2 * p; mm += blockDim.x) {
        float2 Imm = make_float2(rsqrtf(r2), 0.f);
        for (int k = 1; k <= mm; ++k) {
          const float tx = Imm.x * ux - Imm.y * uy, ty = Imm.x * uy + Imm.y * ux;
          const float s = -(2.f * k - 1.f) * ir2;
          Imm = make_float2(tx * s, ty * s);
        }
        float2 I2 = make_float2(0.f, 0.f), I1 = Imm;
        const float sg = (mm & 1) ? -1.f : 1.f;
        for (int a = mm; a <= 2 * p; ++a) {
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
          itab_tc[a * a + a + mm] = Ia;
          itab_tc[a * a + a - mm] = make_float2(sg * Ia.x, -sg * Ia.y);
        }
      }
    }
    __syncthreads();
    unsigned *hi = Timg + (size_t)gid * 2 * NT * NT, *lo = hi + (size_t)NT * NT;
    // walk the image in memory order (coalesced stores); dof decodes come from the smem table
    for (int off = threadIdx.x; off < NT * NT; off += blockDim.x) {
      const int kq = off / (NT * 4), rem = off - kq * NT * 4;
      const int row = rem >> 2, kd = kq * 4 + (rem & 3);  // row = output dof, kd = input dof
      float v = 0.f;
      if (row < KD && kd < KD) {
        const int dr = dec[row], dk = dec[kd];  // (n, m, part) packed
        const int j = dr & 63, ko = (dr >> 6) & 63, rim = dr >> 12;
        const int n = dk & 63, m = (dk >> 6) & 63, cim = dk >> 12;
        const float sgn = ((j + ko) & 1) ? -1.f : 1.f;
        const float sc = sgn * (vform ? ldexpf(1.f, -dl * (j + 1)) : ldexpf(1.f, n * dl));
        const int a = n + j;
        const float2 Cp = itab_tc[a * a + a + (m - ko)];
        if (m == 0) {
          v = sc * (rim ? Cp.y : Cp.x);
        } else {
          const float2 Cm = itab_tc[a * a + a + (-m - ko)];
          const float sm = (m & 1) ? -1.f : 1.f;
          if (!cim)
            v = sc * (rim ? (Cp.y + sm * Cm.y) : (Cp.x + sm * Cm.x));
          else
            v = sc * (rim ? (Cp.x - sm * Cm.x) : -(Cp.y - sm * Cm.y));
        }
      }
      const unsigned vh = f32_to_tf32(v);
      hi[off] = vh;
      lo[off] = f32_to_tf32(v - __uint_as_float(vh));
    }
  }
}

__device__ __forceinline__ void cp_async16_tc(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit_tc() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all_tc() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Warp-specialised per CTA (160 threads):
//   warps 0-3 ("row warps", thread i = TMEM lane i = pair row i of a 128-pair tile): stage their
//     own X row by a TMA bulk copy, split it into TF32 hi/lo and store it as the A operand in
//     TMEM, then read the previous tile's accumulator back (tcgen05.ld) and write it to Y;
//   warp 4 (issuer): loads the class operator T (hi|lo) into shared memory by one TMA bulk copy
//     per item and issues the 3xTF32 MMAs of each tile as soon as its A operand is in TMEM.
// Barriers: x_full (128 arrivals + bytes: X rows staged), a_full (128: A stored), mma_done
// (tcgen05.commit), t_full (bytes: T loaded). The row warps never wait for the MMA issue and the
// issuer never waits for the epilogue, so MMA(i+1) overlaps the epilogue of tile i and the X
// gather of tile i+2.
// TMEM columns: Xh [0,NT) | Xl [NT,2NT) | D0 [2NT,3NT) | D1 [3NT,4NT)  (4 NT <= 512 -> p <= 10)
// The per-item hand-off between the issuer warp and the row warps: they reach it from their own
// code paths (and the issuer warp right after one lane's atomicAdd), so it is a named, non-aligned
// barrier with an explicit count (barrier.sync 1, 160) instead of __syncthreads (= the aligned
// bar.sync 0, which expects every warp converged on one barrier instruction).
__device__ __forceinline__ void item_bar() { asm volatile("barrier.sync 1, 160;" ::: "memory"); }

template <int p>
__global__ void __launch_bounds__(160, 1) k_m2l_tc(const int4 *__restrict__ items,
                                                   const int *__restrict__ counters,
                                                   const unsigned *__restrict__ sidx,
                                                   const unsigned *__restrict__ ssrc,
                                                   const unsigned *__restrict__ Timg,
                                                   const float *__restrict__ M,
                                                   float *__restrict__ Y, int *queue,
                                                   float *__restrict__ Lacc) {
  constexpr int KD = dof_of(p), NT = tc_dim(p);
  constexpr int YSD = dof_stride(p), MROW = 2 * nc_stride(p);
  constexpr unsigned TBYTES = 2u * NT * NT * 4u;
  constexpr int KH = (NT / 32 + 1) / 2;  // 32-column chunks of A's first K half
  static_assert(4 * NT <= 512, "TMEM budget");
  extern __shared__ __align__(1024) unsigned char sh_tc[];
  unsigned *Bimg = reinterpret_cast<unsigned *>(sh_tc);                      // Th | Tl
  float *Xst = reinterpret_cast<float *>(sh_tc + TBYTES);                     // [128][MROW]
  // the epilogue's transpose buffer exists only for the Y-slot epilogue: in accumulate mode the
  // CTA is 18 KB smaller, so that a P2P block fits on the same SM beside it
  float *Ep = Xst + 128 * MROW;                                                // [4][32][36]
  unsigned long long *bars = reinterpret_cast<unsigned long long *>(Ep + (Lacc ? 0 : 4 * 32 * 36));
  unsigned *tmem_base_slot = reinterpret_cast<unsigned *>(bars + 6);
  volatile int *item_sh = reinterpret_cast<volatile int *>(bars + 7);
  unsigned long long *t_full = &bars[0], *mma_done = &bars[1], *x_full = &bars[2];
  unsigned long long *a_full = &bars[3], *mma_h0 = &bars[5];  // a_full[2]: the two K halves of A
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool issuer = warp == 4;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(tmem_base_slot)),
                 "n"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init_tc(t_full, 1);
    mbar_init_tc(mma_done, 1);
    mbar_init_tc(x_full, 128);
    mbar_init_tc(a_full, 128);
    mbar_init_tc(a_full + 1, 128);
    mbar_init_tc(mma_h0, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = *tmem_base_slot;
  const unsigned tXh = tmem, tXl = tmem + NT;
  constexpr unsigned IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(NT >> 3) << 17) | (8u << 24);
  unsigned ph_x = 0, ph_m = 0, ph_a = 0, ph_t = 0;
  const int nitems = counters[1];

  if (issuer) {
    // ---------------------------------------------------------------- MMA issuer (one lane)
    const unsigned bh_addr = smem_addr(Bimg), bl_addr = bh_addr + (unsigned)(NT * NT * 4);
    for (;;) {
      if (tid == 128) item_sh[0] = atomicAdd(queue, 1);
      item_bar();
      const int it = item_sh[0];
      item_bar();  // item_sh is rewritten for the next item only after everyone read it
      if (it >= nitems) break;
      const int4 item = items[it];
      const int ntile = (item.y + 127) / 128;
      if (lane == 0) {
        // T of this item: every MMA of the previous item has completed (the row warps waited
        // for its last commit before the item barrier above)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx_tc(t_full, TBYTES);
        bulk_g2s_tc(Bimg, Timg + (size_t)item.w * 2 * NT * NT, TBYTES, t_full);
        mbar_wait_tc(t_full, ph_t);
        ph_t ^= 1;
        for (int i = 0; i < ntile; ++i) {
          const unsigned tD = tmem + (2 + (i & 1)) * NT;
          // two K halves: the row warps refill A's first half while the second half multiplies
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            mbar_wait_tc(a_full + h, ph_a);  // A(i) half h in TMEM (D(i & 1) drained)
            tc_fence_after();
#pragma unroll
            for (int ks = (h ? KH * 4 : 0); ks < (h ? NT / 8 : KH * 4); ++ks) {
              const unsigned long long bh = make_bdesc(bh_addr + ks * 2 * NT * 16, NT);
              const unsigned long long bl = make_bdesc(bl_addr + ks * 2 * NT * 16, NT);
              tc_mma_ts(tD, tXh + ks * 8, bh, IDESC, ks > 0 ? 1u : 0u);
              tc_mma_ts(tD, tXh + ks * 8, bl, IDESC, 1u);
              tc_mma_ts(tD, tXl + ks * 8, bh, IDESC, 1u);
            }
            tc_commit(h ? mma_done : mma_h0);
          }
          ph_a ^= 1;
        }
      }
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------------- row warps
    const unsigned lane_base = (unsigned)(warp * 32) << 16;
    float *myrow = Xst + tid * MROW;
    float *ep = Ep + warp * 32 * 36;
    // own row of the tile starting at c0 -> staging (every thread arrives on x_full, with its
    // row's bytes when it has one, so a phase completes only after all passed the previous one)
    auto stage = [&](int cnt, int c0, int s) {
      if (c0 + tid < cnt) {
        FMM_DCHECK(FMM_IN(s, g_fmm_chk.rows), "tcgen05 M2L / shift source row");
        mbar_expect_tx_tc(x_full, (unsigned)(MROW * 4));
        bulk_g2s_tc(myrow, M + (size_t)s * MROW, MROW * 4, x_full);
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(x_full)) : "memory");
      }
    };
    // D rows (dof order) -> Y rows (dof order, stride YSD), transposed through shared memory in
    // 32-column chunks: every store instruction writes four contiguous 128-byte row pieces
    // Lacc != nullptr ("accumulate" mode): `yslot` is the pair's target cell and the row is added
    // to its expansion (float order, row stride MROW) with 16-byte vector reductions in L2 --
    // no Y round trip through HBM, but the summation order is not fixed
    auto epilogue_acc = [&](unsigned tD, int cnt, int c0, unsigned trow) {
      constexpr int KR = 2 * nc_of(p);
      unsigned dv[NT];
#pragma unroll
      for (int cb = 0; cb < NT / 32; ++cb) {
        unsigned v[32];
        tc_ld32(tD + lane_base + cb * 32, v);
#pragma unroll
        for (int q = 0; q < 32; ++q) dv[cb * 32 + q] = v[q];
      }
      tc_wait_ld();
      if (c0 + tid < cnt) {
        FMM_DCHECK(FMM_IN(trow, g_fmm_chk.rows), "tcgen05 M2L target row");
        float *dst = Lacc + (size_t)trow * MROW;
#pragma unroll
        for (int q = 0; q < MROW / 4; ++q) {
          float o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int f = 4 * q + e;
            const int d = f < KR ? float_to_dof(f) : -1;
            o[e] = d >= 0 ? __uint_as_float(dv[d]) : 0.f;
          }
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * q), "f"(o[0]),
                       "f"(o[1]), "f"(o[2]), "f"(o[3])
                       : "memory");
        }
      }
    };
    auto epilogue = [&](unsigned tD, int cnt, int c0, unsigned yslot) {
      if (Lacc) {
        epilogue_acc(tD, cnt, c0, yslot);
        return;
      }
#pragma unroll
      for (int cb = 0; cb < NT / 32; ++cb) {
        unsigned v[32];
        tc_ld32(tD + lane_base + cb * 32, v);
        tc_wait_ld();
        float4 *dst = reinterpret_cast<float4 *>(ep + lane * 36);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          dst[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                               __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int r = 4 * k + (lane >> 3), c4 = lane & 7;
          const unsigned ys = __shfl_sync(0xffffffffu, yslot, r);
          const int col = cb * 32 + c4 * 4;
          if (c0 + warp * 32 + r < cnt && col < YSD)
            __stcs(reinterpret_cast<float4 *>(Y + (size_t)ys * YSD + col),
                   reinterpret_cast<const float4 *>(ep + r * 36)[c4]);  // streamed: keep M, T in L2
        }
        __syncwarp();
      }
    };
    for (;;) {
      item_bar();  // the issuer fetched the next item
      const int it = item_sh[0];
      item_bar();
      if (it >= nitems) break;
      const int4 item = items[it];
      const int pos0 = item.x, cnt = item.y;
      const int ntile = (cnt + 127) / 128;
      auto src_of = [&](int r) { return r < cnt ? (int)ssrc[pos0 + r] : 0; };
      int s_pf = src_of(128 + tid);  // source of the next tile's row (loaded a tile ahead)
      unsigned y_prev = 0u, y_cur = tid < cnt ? sidx[pos0 + tid] : 0u;
      stage(cnt, 0, src_of(tid));
      for (int i = 0; i < ntile; ++i) {
        const int r0 = i * 128 + tid;
        const int s_next = s_pf;
        s_pf = src_of(r0 + 256);
        const unsigned y_next = r0 + 128 < cnt ? sidx[pos0 + r0 + 128] : 0u;
        // X(i): own row -> registers; the staging row is refilled with X(i+1) at once
        mbar_wait_tc(x_full, ph_x);
        ph_x ^= 1;
        float xf[MROW];
#pragma unroll
        for (int q = 0; q < MROW / 4; ++q) {
          const float4 v4 = reinterpret_cast<const float4 *>(myrow)[q];
          xf[4 * q] = v4.x;
          xf[4 * q + 1] = v4.y;
          xf[4 * q + 2] = v4.z;
          xf[4 * q + 3] = v4.w;
        }
        if (i + 1 < ntile) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          stage(cnt, (i + 1) * 128, s_next);
        }
        const bool valid = r0 < cnt;
        // A(i) in two K halves: half 0 once MMA(i-1) has consumed its half 0 (mma_h0), half 1
        // once MMA(i-1) has completed (mma_done; D((i-1) & 1) is then ready as well)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (i > 0) {
            mbar_wait_tc(h ? mma_done : mma_h0, ph_m);
            tc_fence_after();
          }
#pragma unroll
          for (int cb = (h ? KH : 0); cb < (h ? NT / 32 : KH); ++cb) {
            unsigned vh[32], vl[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) {
              const int d = cb * 32 + q;
              const float x = (d < KD && valid) ? xf[dof_to_float(d < KD ? d : 0)] : 0.f;
              tf32_split(x, vh[q], vl[q]);
            }
            tc_st32(tXh + lane_base + cb * 32, vh);
            tc_st32(tXl + lane_base + cb * 32, vl);
          }
          tc_wait_st();
          tc_fence_before();
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(a_full + h))
                       : "memory");
        }
        if (i > 0) ph_m ^= 1;
        if (i > 0) epilogue(tmem + (2 + ((i - 1) & 1)) * NT, cnt, (i - 1) * 128, y_prev);
        y_prev = y_cur;
        y_cur = y_next;
      }
      // last tile
      mbar_wait_tc(mma_h0, ph_m);
      mbar_wait_tc(mma_done, ph_m);
      ph_m ^= 1;
      tc_fence_after();
      epilogue(tmem + (2 + ((ntile - 1) & 1)) * NT, cnt, (ntile - 1) * 128, y_prev);
      tc_fence_before();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512)
                 : "memory");
}

// ---- host side ----------------------------------------------------------------------------------
bool m2l_tc_supported(int p) { return p >= 1 && p <= 10; }
size_t m2l_tc_T_words(int p) { return (size_t)2 * tc_dim(p) * tc_dim(p); }

cudaError_t m2l_tc_build_T(int p, const M2LWork &W, int ngclass, unsigned *Timg, cudaStream_t st) {
  if (ngclass <= 0) return cudaSuccess;
  const size_t smem = (size_t)(2 * p + 1) * (2 * p + 1) * sizeof(float2);
  k_m2l_build_T_tc<<<ngclass < 148 * 4 ? ngclass : 148 * 4, 256, smem, st>>>(
      p, W.counters, W.class_rep, W.pair_t, W.src, W.C, Timg);
  return cudaGetLastError();
}

cudaError_t tc_class_gemm(int p, const int4 *items, const int *counters, int *queue,
                          const unsigned *sidx, const unsigned *ssrc, const unsigned *Timg,
                          const float2 *M, float *Y, int grid, cudaStream_t st, float *Lacc) {
  cudaMemsetAsync(queue, 0, sizeof(int), st);
#define M2L_TC_CASE(PP)                                                                        \
  case PP: {                                                                                 \
    const size_t ep_bytes = 4 * 32 * 36 * 4;                                                 \
    const size_t smem_full = (size_t)2 * tc_dim(PP) * tc_dim(PP) * 4 + (size_t)128 * 2 * nc_stride(PP) * 4 + ep_bytes + 128; \
    const size_t smem = Lacc ? smem_full - ep_bytes : smem_full;                             \
    fmm_smem_optin((const void *)k_m2l_tc<PP>, smem_full);                                   \
    k_m2l_tc<PP><<<grid, 160, smem, st>>>(items, counters, sidx, ssrc, Timg,                 \
                                         reinterpret_cast<const float *>(M), Y, queue, Lacc); \
  } break;
  switch (p) {
    M2L_TC_CASE(1) M2L_TC_CASE(2) M2L_TC_CASE(3) M2L_TC_CASE(4) M2L_TC_CASE(5) M2L_TC_CASE(6)
    M2L_TC_CASE(7) M2L_TC_CASE(8) M2L_TC_CASE(9) M2L_TC_CASE(10)
    default: break;
  }
#undef M2L_TC_CASE
  return cudaGetLastError();
}

cudaError_t m2l_tc_gemm(int p, const M2LWork &W, const unsigned *Timg, const float2 *M,
                        cudaStream_t st, float2 *Lacc) {
  // accumulate mode: the epilogue's per-row "slot" is the pair's target cell (W.stgt)
  return tc_class_gemm(p, W.items, W.counters, W.counters + 4, Lacc ? W.stgt : W.sidx, W.ssrc, Timg,
                       M, W.Y, 148, st, reinterpret_cast<float *>(Lacc));
}

// ================================================================================================
// M2M / L2L on the tensor cores. In the scaled form both shifts depend only on the octant of the
// child (b/r_P = (+-1/2, +-1/2, +-1/2)), so each level is a class GEMM with 8 classes:
//   M2M:  Y[child] = T^M2M_oct(child) Mhat[child];  Mhat[parent] = sum over its children of Y
//   L2L:  Y[child] = T^L2L_oct(child) Lhat[parent]; Lhat[child] += Y[child]
// The 16 operators are built once per handle by applying the shift formulas (expansions.cu
// header) to the unit vectors of the real degrees of freedom.
__device__ float2 sget_unit(int d, int n, int m) {  // unit vector e_d of the dofs, signed access
  int nd = 0;
  while ((nd + 1) * (nd + 1) <= d) ++nd;
  const int r = d - nd * nd, md = (r + 1) / 2, im = r ? ((r + 1) & 1) : 0;
  const int am = m < 0 ? -m : m;
  if (n != nd || am != md) return make_float2(0.f, 0.f);
  float2 v = im ? make_float2(0.f, 1.f) : make_float2(1.f, 0.f);
  if (m < 0) v = (am & 1) ? make_float2(-v.x, v.y) : make_float2(v.x, -v.y);  // (-1)^m conj
  return v;
}

// grid (8 octants, KD input dofs, 2 ops); block 128 threads over output coefficients
__global__ void k_shift_basis(int p, unsigned *__restrict__ Tm2m, unsigned *__restrict__ Tl2l) {
  const int o = blockIdx.x, d = blockIdx.y, op = blockIdx.z;
  const int NC = nc_of(p), KD = dof_of(p), NT = tc_dim(p);
  __shared__ float2 Rt[nc_of(FMM_PMAX)];
  const float bx = ((o >> 2) & 1) ? 0.5f : -0.5f, by = ((o >> 1) & 1) ? 0.5f : -0.5f,
              bz = (o & 1) ? 0.5f : -0.5f;
  // regular harmonics R_n^m(b), m >= 0 (same recurrences as expansions.cu)
  if (threadIdx.x <= p) {
    const int m = threadIdx.x;
    const float r2 = bx * bx + by * by + bz * bz;
    float2 Rmm = make_float2(1.f, 0.f);
    for (int k = 1; k <= m; ++k) {
      const float tx = Rmm.x * bx - Rmm.y * by, ty = Rmm.x * by + Rmm.y * bx;
      Rmm = make_float2(-tx / (2.f * k), -ty / (2.f * k));
    }
    Rt[cidx(m, m)] = Rmm;
    float2 R2 = make_float2(0.f, 0.f), R1 = Rmm;
    for (int n = m + 1; n <= p; ++n) {
      float2 Rn;
      if (n == m + 1) Rn = make_float2(Rmm.x * bz, Rmm.y * bz);
      else {
        const float inv = 1.f / ((float)(n - m) * (float)(n + m));
        Rn = make_float2(((2 * n - 1) * bz * R1.x - r2 * R2.x) * inv, ((2 * n - 1) * bz * R1.y - r2 * R2.y) * inv);
      }
      Rt[cidx(n, m)] = Rn;
      R2 = R1;
      R1 = Rn;
    }
  }
  __syncthreads();
  unsigned *img = (op == 0 ? Tm2m : Tl2l) + (size_t)o * 2 * NT * NT;
  for (int c = threadIdx.x; c < NC; c += blockDim.x) {
    int n = 0;
    while ((n + 1) * (n + 2) / 2 <= c) ++n;
    const int m = c - n * (n + 1) / 2;
    float2 a = make_float2(0.f, 0.f);
    if (op == 0) {  // M2M: sum_{j<=n,k} e_d(j,k) 2^-j conj(R_{n-j}^{m-k})
      float sc = 1.f;
      for (int j = 0; j <= n; ++j, sc *= 0.5f) {
        const int klo = max(-j, m - (n - j)), khi = min(j, m + (n - j));
        for (int k = klo; k <= khi; ++k) {
          const float2 e = sget_unit(d, j, k);
          if (e.x == 0.f && e.y == 0.f) continue;
          const float2 r = sget(Rt, n - j, m - k);
          const float2 rc = make_float2(r.x, -r.y);
          a.x += sc * (e.x * rc.x - e.y * rc.y);
          a.y += sc * (e.x * rc.y + e.y * rc.x);
        }
      }
    } else {  // L2L: 2^-(n+1) sum_{j>=n,k} e_d(j,k) R_{j-n}^{k-m}
      for (int j = n; j <= p; ++j) {
        const int klo = max(-j, m - (j - n)), khi = min(j, m + (j - n));
        for (int k = klo; k <= khi; ++k) {
          const float2 e = sget_unit(d, j, k);
          if (e.x == 0.f && e.y == 0.f) continue;
          const float2 r = sget(Rt, j - n, k - m);
          a.x += e.x * r.x - e.y * r.y;
          a.y += e.x * r.y + e.y * r.x;
        }
      }
      const float sc = ldexpf(1.f, -(n + 1));
      a.x *= sc;
      a.y *= sc;
    }
    // output dofs of coefficient (n, m): Re -> row n^2 (m = 0) or n^2 + 2m - 1, Im -> n^2 + 2m
    const int rows[2] = {m == 0 ? n * n : n * n + 2 * m - 1, m == 0 ? -1 : n * n + 2 * m};
    const float vals[2] = {a.x, a.y};
    for (int t = 0; t < 2; ++t) {
      if (rows[t] < 0) continue;
      const int off = (d >> 2) * (NT * 4) + rows[t] * 4 + (d & 3);
      const unsigned vh = f32_to_tf32(vals[t]);
      img[off] = vh;
      img[(size_t)NT * NT + off] = f32_to_tf32(vals[t] - __uint_as_float(vh));
    }
  }
  (void)KD;
}

// octant segments: the non-root cells sorted by (level << 3 | octant) give per level 8 contiguous
// segments; a level's items are chunks of TC_SHIFT_ITEM cells of one segment (class = octant).
// Output slots are the cell ids themselves (Y holds one row per cell).
#ifndef TC_SHIFT_ITEM
#define TC_SHIFT_ITEM 256  // children per M2M / L2L work item: enough items to spread a level over the SMs
#endif
int tc_shift_items_per_level(int ncells) { return 16 + ncells / TC_SHIFT_ITEM; }
__global__ void k_shift_keys(int ncells, CellsView C, unsigned *keys, unsigned *vals) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells - 1) return;
  const int cell = c + 1;  // the root has no parent
  const int4 g = C.grid[cell], gp = C.grid[C.parent[cell]];
  const unsigned oct = ((g.x > gp.x) << 2) | ((g.y > gp.y) << 1) | (g.z > gp.z);
  keys[c] = ((unsigned)g.w << 3) | oct;
  vals[c] = (unsigned)cell;
}
__global__ void k_shift_items(int nsorted, int depth, const unsigned *__restrict__ skeys,
                              const unsigned *__restrict__ scell, const int *__restrict__ parent,
                              int4 *__restrict__ items, int *__restrict__ lvl_counters,
                              unsigned *__restrict__ src_l2l, int items_per_level) {
  __shared__ int seg[(FMM_LEVELS + 2) * 8 + 1];
  // every block: the L2L source (parent) of each sorted child, grid-stride (a single block took
  // 0.7 ms at C4 on this chain of dependent loads)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nsorted; i += gridDim.x * blockDim.x)
    src_l2l[i] = (unsigned)parent[scell[i]];
  if (blockIdx.x != 0) return;
  // block 0: the per-level octant segments and their work items
  for (int k = threadIdx.x; k <= (FMM_LEVELS + 2) * 8; k += blockDim.x) {
    int l = 0, r = nsorted;  // first sorted position with key >= k
    while (l < r) {
      const int mid = (l + r) >> 1;
      if ((int)skeys[mid] < k) l = mid + 1;
      else r = mid;
    }
    seg[k] = l;
  }
  __syncthreads();
  for (int lv = threadIdx.x; lv <= depth; lv += blockDim.x) {
    int ni = 0;
    int4 *it = items + (size_t)lv * items_per_level;
    for (int o = 0; o < 8; ++o) {
      const int b = seg[lv * 8 + o], e = seg[lv * 8 + o + 1];
      for (int a = b; a < e; a += TC_SHIFT_ITEM) it[ni++] = make_int4(a, min(TC_SHIFT_ITEM, e - a), 0, o);
    }
    lvl_counters[lv * 8 + 1] = ni;
  }
}

// M2M: parent = sum of its children's slots (child order); L2L: child += its slot. Y rows are in
// dof order (stride dof_stride(p)); expansion rows in float order with Im(n, 0) = 0.
__global__ void __launch_bounds__(256) k_shift_m2m_reduce(int p, int c0, int nl, CellsView C,
                                                          const float *__restrict__ Y,
                                                          float *__restrict__ M) {
  const int KR = 2 * nc_of(p), YSD = dof_stride(p), LS = 2 * nc_stride(p);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nl * KR; i += gridDim.x * blockDim.x) {
    const int k = i / KR, f = i - k * KR;
    const int P = c0 + k, nch = C.nchild[P];
    if (nch == 0) continue;
    const int d = float_to_dof(f);
    float s = 0.f;
    if (d >= 0) {
      const int ch0 = C.child0[P];
      for (int c = 0; c < nch; ++c) s += Y[(size_t)(ch0 + c) * YSD + d];
    }
    M[(size_t)P * LS + f] = s;
  }
}
__global__ void __launch_bounds__(256) k_shift_l2l_add(int p, int c0, int nl,
                                                       const float *__restrict__ Y,
                                                       float *__restrict__ L) {
  const int KR = 2 * nc_of(p), YSD = dof_stride(p), LS = 2 * nc_stride(p);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nl * KR; i += gridDim.x * blockDim.x) {
    const int k = i / KR, f = i - k * KR;
    const int d = float_to_dof(f);
    if (d >= 0) L[(size_t)(c0 + k) * LS + f] += Y[(size_t)(c0 + k) * YSD + d];
  }
}

cudaError_t tc_shift_build_ops(int p, unsigned *Tm2m, unsigned *Tl2l, cudaStream_t st) {
  cudaMemsetAsync(Tm2m, 0, sizeof(unsigned) * 8 * m2l_tc_T_words(p), st);
  cudaMemsetAsync(Tl2l, 0, sizeof(unsigned) * 8 * m2l_tc_T_words(p), st);
  k_shift_basis<<<dim3(8, dof_of(p), 2), 128, 0, st>>>(p, Tm2m, Tl2l);
  return cudaGetLastError();
}

cudaError_t tc_shift_prepare(int ncells, int depth, const TcShiftWork &S, CellsView C,
                             cudaStream_t st) {
  const int ns = ncells - 1;
  cudaMemsetAsync(S.lvl_counters, 0, sizeof(int) * 8 * (FMM_LEVELS + 2), st);
  if (ns <= 0) return cudaGetLastError();
  k_shift_keys<<<(ns + 255) / 256, 256, 0, st>>>(ncells, C, S.keys_in, S.vals_in);
  size_t bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, bytes, S.keys_in, S.keys, S.vals_in,
                                                  S.cells, ns, 0, 8, st);
  if (e) return e;
  if (bytes > S.tmp_bytes) return cudaErrorMemoryAllocation;
  e = cub::DeviceRadixSort::SortPairs(S.tmp, bytes, S.keys_in, S.keys, S.vals_in, S.cells, ns, 0, 8,
                                      st);
  if (e) return e;
  const int nb = std::max(1, std::min(148 * 8, (ns + 1023) / 1024));
  k_shift_items<<<nb, 1024, 0, st>>>(ns, depth, S.keys, S.cells, C.parent, S.items, S.lvl_counters,
                                     S.src_l2l, S.items_per_level);
  return cudaGetLastError();
}

size_t tc_shift_sort_bytes(int ncells) {
  size_t a = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (unsigned *)nullptr, (unsigned *)nullptr,
                                  (unsigned *)nullptr, (unsigned *)nullptr, ncells, 0, 8);
  return a;
}

cudaError_t tc_shift_m2m_level(int p, int level, int c0, int nl, CellsView C,
                               const TcShiftWork &S, float2 *M, float *Y, cudaStream_t st) {
  // children of this level's parents live at level + 1
  const int lv = level + 1;
  cudaError_t e = tc_class_gemm(p, S.items + (size_t)lv * S.items_per_level, S.lvl_counters + lv * 8,
                                S.lvl_counters + lv * 8 + 4, S.cells, S.cells, S.Tm2m, M, Y, 148, st);
  if (e) return e;
  const int KR = 2 * nc_of(p);
  int b = (nl * KR + 255) / 256;
  b = b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16;
  k_shift_m2m_reduce<<<b, 256, 0, st>>>(p, c0, nl, C, Y, reinterpret_cast<float *>(M));
  return cudaGetLastError();
}

cudaError_t tc_shift_l2l_level(int p, int level, int c0, int nl, const TcShiftWork &S, float2 *L,
                               float *Y, cudaStream_t st) {
  cudaError_t e = tc_class_gemm(p, S.items + (size_t)level * S.items_per_level,
                                S.lvl_counters + level * 8, S.lvl_counters + level * 8 + 4, S.cells,
                                S.src_l2l, S.Tl2l, L, Y, 148, st);
  if (e) return e;
  const int KR = 2 * nc_of(p);
  int b = (nl * KR + 255) / 256;
  b = b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16;
  k_shift_l2l_add<<<b, 256, 0, st>>>(p, c0, nl, Y, reinterpret_cast<float *>(L));
  return cudaGetLastError();
}

// ================================================================================================
// k_m2l_tck -- the tcgen05 class GEMM for 10 < p <= 15 (a K-tiled variant; PAPER.md:205 runs
// p = 5..15). Above p = 10 neither the whole class operator (2 x N x K TF32 words: 205 KB at
// p = 11, 627 KB at p = 15) nor a TMEM-resident A operand plus a double-buffered D fits, so:
//   * rows and columns are in FLOAT order (the expansion row as stored: (n, m >= 0) complex, the
//     zero Im part of m = 0 included as a zero column / row of T), so a thread gathers its pair's
//     source row as contiguous float4s and the accumulator comes out as contiguous float4s;
//   * K is streamed in chunks of 32 floats through a 2-stage shared-memory ring: the A chunk
//     (128 pairs x 32, hi and lo, written by the row warps from registers) and the B chunk (the
//     class operator's 32 K-columns, hi and lo, one TMA bulk copy by the issuer);
//   * D (128 x N FP32, N = 2 nc padded to 16) accumulates in TMEM, double-buffered when 2N <= 512
//     (p <= 14), so the epilogue of tile i overlaps the MMAs of tile i+1; at p = 15 (N = 272 = 256
//     + 16, two MMAs per K step) it is single-buffered;
//   * 3xTF32 as in k_m2l_tc (hi.hi + hi.lo + lo.hi).
// Results: added into L with 16-byte vector reductions (accumulate mode) or written to per-pair
// slots Y in float order (deterministic mode; k_m2l_reduce with ydof = 0).
// ================================================================================================
__host__ __device__ constexpr int tck_nf(int p) { return 2 * nc_of(p); }            // floats per row
__host__ __device__ constexpr int tck_np(int p) { return (tck_nf(p) + 15) & ~15; }  // N
__host__ __device__ constexpr int tck_kp(int p) { return (tck_nf(p) + 31) & ~31; }  // K (chunks of 32)
#define TCK_KC 32

// per class: for every K chunk c, [hi: N x 32 | lo: N x 32] TF32 words in the K-major core-matrix
// layout (element (row, k) at word (k/4)*(N*4) + row*4 + k%4 of its half)
__global__ void __launch_bounds__(256) k_m2l_build_T_tck(int p, const int *__restrict__ counters,
                                                         const unsigned *__restrict__ class_rep,
                                                         const int *__restrict__ pair_t,
                                                         const unsigned *__restrict__ src,
                                                         CellsView C, unsigned *__restrict__ Timg) {
  extern __shared__ double2 itab_k[];  // FP64: the operator is built once per class
  __shared__ int dec[2 * nc_of(FMM_PMAX)];  // float index -> n | m << 6 | part << 12, or -1
  const int NF = tck_nf(p), NP = tck_np(p), KP = tck_kp(p);
  const int ng = counters[3];
  for (int f = threadIdx.x; f < NF; f += blockDim.x) {
    const int c = f >> 1, part = f & 1;
    int n = 0;
    while ((n + 1) * (n + 2) / 2 <= c) ++n;
    const int m = c - n * (n + 1) / 2;
    dec[f] = (m == 0 && part) ? -1 : (n | (m << 6) | (part << 12));
  }
  for (int gid = blockIdx.x; gid < ng; gid += gridDim.x) {
    const int rep = class_rep[gid];
    const int4 gt = C.grid[pair_t[rep]], gs = C.grid[src[rep]];
    const double rt_inv = 1.0 / (double)(1 << (FMM_LEVELS - gt.w));
    const int dl = gt.w - gs.w;
    double ux = (gt.x - gs.x) * rt_inv, uy = (gt.y - gs.y) * rt_inv, uz = (gt.z - gs.z) * rt_inv;
    const bool vform = dl > 0;
    if (vform) {
      const double ir = ldexp(1.0, -dl);
      ux *= ir;
      uy *= ir;
      uz *= ir;
    }
    __syncthreads();
    // irregular harmonics I_a^b(u), a <= 2p, signed b (the recurrences of k_m2l_build_T_tc)
    {
      const double r2 = ux * ux + uy * uy + uz * uz, ir2 = 1.0 / r2;
      for (int mm = threadIdx.x; mm <= 2 * p; mm += blockDim.x) {
        double2 Imm = make_double2(rsqrt(r2), 0.0);
        for (int k = 1; k <= mm; ++k) {
          const double tx = Imm.x * ux - Imm.y * uy, ty = Imm.x * uy + Imm.y * ux;
          const double s = -(2.0 * k - 1.0) * ir2;
          Imm = make_double2(tx * s, ty * s);
        }
        double2 I2 = make_double2(0.0, 0.0), I1 = Imm;
        const double sg = (mm & 1) ? -1.0 : 1.0;
        for (int a = mm; a <= 2 * p; ++a) {
          double2 Ia;
          if (a == mm) Ia = Imm;
          else if (a == mm + 1) {
            const double s = (2.0 * mm + 1.0) * uz * ir2;
            Ia = make_double2(Imm.x * s, Imm.y * s);
          } else {
            const double c1 = (2.0 * a - 1.0) * uz, c2 = (double)(a + mm - 1) * (double)(a - mm - 1);
            Ia = make_double2((c1 * I1.x - c2 * I2.x) * ir2, (c1 * I1.y - c2 * I2.y) * ir2);
          }
          if (a > mm) {
            I2 = I1;
            I1 = Ia;
          }
          itab_k[a * a + a + mm] = Ia;
          itab_k[a * a + a - mm] = make_double2(sg * Ia.x, -sg * Ia.y);
        }
      }
    }
    __syncthreads();
    unsigned *img = Timg + (size_t)gid * 2 * NP * KP;
    const int half = NP * TCK_KC;  // words per hi or lo half of a chunk
    for (int off = threadIdx.x; off < NP * KP; off += blockDim.x) {
      const int ch = off / half, w = off - ch * half;
      const int kq = w / (NP * 4), rem = w - kq * NP * 4;
      const int row = rem >> 2, kf = ch * TCK_KC + kq * 4 + (rem & 3);  // out float, in float
      double v = 0.0;
      if (row < NF && kf < NF && dec[row] >= 0 && dec[kf] >= 0) {
        const int dr = dec[row], dk = dec[kf];
        const int j = dr & 63, ko = (dr >> 6) & 63, rim = dr >> 12;
        const int n = dk & 63, m = (dk >> 6) & 63, cim = dk >> 12;
        const double sgn = ((j + ko) & 1) ? -1.0 : 1.0;
        const double sc = sgn * (vform ? ldexp(1.0, -dl * (j + 1)) : ldexp(1.0, n * dl));
        const int a = n + j;
        const double2 Cp = itab_k[a * a + a + (m - ko)];
        if (m == 0) {
          v = sc * (rim ? Cp.y : Cp.x);
        } else {
          const double2 Cm = itab_k[a * a + a + (-m - ko)];
          const double sm = (m & 1) ? -1.0 : 1.0;
          if (!cim)
            v = sc * (rim ? (Cp.y + sm * Cm.y) : (Cp.x + sm * Cm.x));
          else
            v = sc * (rim ? (Cp.x - sm * Cm.x) : -(Cp.y - sm * Cm.y));
        }
      }
      const unsigned vh = f32_to_tf32((float)v);
      unsigned *h = img + (size_t)ch * 2 * half;
      h[w] = vh;
      h[half + w] = f32_to_tf32((float)(v - (double)__uint_as_float(vh)));
    }
  }
}

namespace {
// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32, cta_group::1
__device__ __forceinline__ void tc_mma_ss(unsigned d_tmem, unsigned long long adesc,
                                          unsigned long long bdesc, unsigned idesc, unsigned acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__host__ __device__ constexpr unsigned tck_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(n >> 3) << 17) | (8u << 24);
}
}  // namespace

template <int p>
__global__ void __launch_bounds__(160, 1) k_m2l_tck(const int4 *__restrict__ items,
                                                    const int *__restrict__ counters,
                                                    const unsigned *__restrict__ sidx,
                                                    const unsigned *__restrict__ ssrc,
                                                    const unsigned *__restrict__ Timg,
                                                    const float *__restrict__ M,
                                                    float *__restrict__ Y, int *queue,
                                                    float *__restrict__ Lacc) {
  constexpr int NF = tck_nf(p), NP = tck_np(p), KP = tck_kp(p), NCH = KP / TCK_KC;
  constexpr int MROW = 2 * nc_stride(p);                   // M / L row stride (floats)
  constexpr int YS = (NF + 3) & ~3;                         // Y row stride (float order)
  constexpr int N0 = NP > 256 ? 256 : NP, N1 = NP - N0;     // the MMA N parts (N1 = 16 at p = 15)
  constexpr int DB = 2 * NP <= 512 ? 2 : 1;                 // D buffers in TMEM
  constexpr unsigned ABYTES = 128u * TCK_KC * 4u;           // one half (hi or lo) of an A chunk
  constexpr unsigned BBYTES = (unsigned)NP * TCK_KC * 4u;   // one half of a B chunk
  constexpr unsigned STAGE = 2 * ABYTES + 2 * BBYTES;
  static_assert(N1 == 0 || N1 % 16 == 0, "N parts");
  static_assert(DB * NP <= 512, "TMEM budget");
  extern __shared__ __align__(1024) unsigned char sh_tck[];
  unsigned long long *bars = reinterpret_cast<unsigned long long *>(sh_tck + 2 * STAGE);
  unsigned long long *a_full = bars, *b_full = bars + 2, *s_free = bars + 4, *d_full = bars + 6,
                     *d_free = bars + 8;
  unsigned *tmem_slot = reinterpret_cast<unsigned *>(bars + 10);
  volatile int *item_sh = reinterpret_cast<volatile int *>(bars + 11);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(tmem_slot)),
                 "n"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init_tc(&a_full[s], 128);
      mbar_init_tc(&b_full[s], 1);
      mbar_init_tc(&s_free[s], 1);
      mbar_init_tc(&d_full[s], 1);
      mbar_init_tc(&d_free[s], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = *tmem_slot;
  const int nitems = counters[1];
  auto a_base = [&](int s) { return sh_tck + (size_t)s * STAGE; };
  auto b_base = [&](int s) { return sh_tck + (size_t)s * STAGE + 2 * ABYTES; };
  unsigned g = 0, tt = 0;  // chunks / tiles consumed so far (identical in every role)

  if (warp == 4) {
    // ---------------------------------------------------------------- issuer (one lane)
    for (;;) {
      if (tid == 128) item_sh[0] = atomicAdd(queue, 1);
      item_bar();
      const int it = item_sh[0];
      item_bar();
      if (it >= nitems) break;
      const int4 item = items[it];
      const int ntile = (item.y + 127) / 128;
      const unsigned *Tcls = Timg + (size_t)item.w * 2 * NP * KP;
      if (lane == 0) {
        auto load_b = [&](unsigned gg, int ch) {  // the class operator's chunk ch -> stage gg & 1
          const int s = gg & 1;
          if (gg >= 2) mbar_wait_tc(&s_free[s], ((gg >> 1) - 1) & 1);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx_tc(&b_full[s], 2 * BBYTES);
          bulk_g2s_tc(b_base(s), Tcls + (size_t)ch * 2 * NP * TCK_KC, 2 * BBYTES, &b_full[s]);
        };
        load_b(g, 0);
        for (int i = 0; i < ntile; ++i, ++tt) {
          const int db = DB == 2 ? (tt & 1) : 0;
          const unsigned v = DB == 2 ? (tt >> 1) : tt;
          if (v >= 1) mbar_wait_tc(&d_free[db], (v - 1) & 1);  // the epilogue drained D(db)
          tc_fence_after();
          const unsigned tD = tmem + (unsigned)(db * NP);
          for (int c = 0; c < NCH; ++c, ++g) {
            const int s = g & 1;
            mbar_wait_tc(&b_full[s], (g >> 1) & 1);
            mbar_wait_tc(&a_full[s], (g >> 1) & 1);
            tc_fence_after();
            const unsigned ah = smem_addr(a_base(s)), al = ah + ABYTES;
            const unsigned bh = smem_addr(b_base(s)), bl = bh + BBYTES;
#pragma unroll
            for (int ks = 0; ks < TCK_KC / 8; ++ks) {
              const unsigned acc = (c > 0 || ks > 0) ? 1u : 0u;
              const unsigned long long dah = make_bdesc(ah + ks * 2 * 128 * 16, 128);
              const unsigned long long dal = make_bdesc(al + ks * 2 * 128 * 16, 128);
              const unsigned long long dbh = make_bdesc(bh + ks * 2 * NP * 16, NP);
              const unsigned long long dbl = make_bdesc(bl + ks * 2 * NP * 16, NP);
              tc_mma_ss(tD, dah, dbh, tck_idesc(N0), acc);
              tc_mma_ss(tD, dah, dbl, tck_idesc(N0), 1u);
              tc_mma_ss(tD, dal, dbh, tck_idesc(N0), 1u);
              if (N1 > 0) {  // rows N0.. of B: 16-byte core-matrix rows further
                const unsigned long long dbh1 = make_bdesc(bh + ks * 2 * NP * 16 + N0 * 16, NP);
                const unsigned long long dbl1 = make_bdesc(bl + ks * 2 * NP * 16 + N0 * 16, NP);
                tc_mma_ss(tD + N0, dah, dbh1, tck_idesc(N1 > 0 ? N1 : 16), acc);
                tc_mma_ss(tD + N0, dah, dbl1, tck_idesc(N1 > 0 ? N1 : 16), 1u);
                tc_mma_ss(tD + N0, dal, dbh1, tck_idesc(N1 > 0 ? N1 : 16), 1u);
              }
            }
            tc_commit(&s_free[s]);  // stage s is free once these MMAs completed
            // the next chunk's operator (this item's next chunk, or the next tile's first)
            if (c + 1 < NCH) load_b(g + 1, c + 1);
            else if (i + 1 < ntile) load_b(g + 1, 0);
          }
          tc_commit(&d_full[db]);
        }
      } else {
        g += (unsigned)(ntile * NCH);
        tt += (unsigned)ntile;
      }
      __syncwarp();
      g = __shfl_sync(0xffffffffu, g, 0);
      tt = __shfl_sync(0xffffffffu, tt, 0);
    }
  } else {
    // ---------------------------------------------------------------- row warps (thread = pair row)
    const unsigned lane_base = (unsigned)(warp * 32) << 16;
    auto epilogue = [&](unsigned ttile, int cnt, int r0, unsigned slot) {
      const int db = DB == 2 ? (ttile & 1) : 0;
      const unsigned v = DB == 2 ? (ttile >> 1) : ttile;
      mbar_wait_tc(&d_full[db], v & 1);
      tc_fence_after();
      const bool valid = r0 + tid < cnt;
      float *dst = Lacc ? Lacc + (size_t)slot * MROW : Y + (size_t)slot * YS;
#pragma unroll
      for (int cb = 0; cb < (NF + 31) / 32; ++cb) {
        unsigned vv[32];
        tc_ld32(tmem + (unsigned)(db * NP) + lane_base + cb * 32, vv);
        tc_wait_ld();
        if (valid) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int f = cb * 32 + 4 * q;
            if (f < (Lacc ? MROW : YS)) {
              const float o0 = __uint_as_float(vv[4 * q]), o1 = __uint_as_float(vv[4 * q + 1]);
              const float o2 = __uint_as_float(vv[4 * q + 2]), o3 = __uint_as_float(vv[4 * q + 3]);
              if (Lacc)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + f),
                             "f"(o0), "f"(o1), "f"(o2), "f"(o3)
                             : "memory");
              else
                __stcs(reinterpret_cast<float4 *>(dst + f), make_float4(o0, o1, o2, o3));
            }
          }
        }
      }
      tc_fence_before();
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&d_free[db])) : "memory");
    };
    for (;;) {
      item_bar();
      const int it = item_sh[0];
      item_bar();
      if (it >= nitems) break;
      const int4 item = items[it];
      const int pos0 = item.x, cnt = item.y;
      const int ntile = (cnt + 127) / 128;
      unsigned prev_slot = 0;
      // the row chunks are gathered two chunks ahead (a 2-deep register ring that crosses tile
      // boundaries): a chunk's MMAs take ~0.6 us at p = 12, an L2 gather ~1 us
      auto row_of = [&](int tile, bool &v) {
        const int r = tile * 128 + tid;
        v = r < cnt;
        return M + (size_t)(v ? ssrc[pos0 + r] : 0u) * MROW;
      };
      auto load_to = [&](float4(&x)[8], const float *row, bool valid, int c) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int f = c * TCK_KC + 4 * q;
          float4 v4 = (valid && f < MROW) ? __ldg(reinterpret_cast<const float4 *>(row + f))
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
          if (f + 3 >= NF) {  // the row's padding floats (never written) must not reach the MMA
            if (f + 0 >= NF) v4.x = 0.f;
            if (f + 1 >= NF) v4.y = 0.f;
            if (f + 2 >= NF) v4.z = 0.f;
            v4.w = 0.f;
          }
          x[q] = v4;
        }
      };
      float4 xa[8], xb[8];
      bool lvalid = false;
      const float *lrow = row_of(0, lvalid);
      load_to(xa, lrow, lvalid, 0);
      load_to(xb, lrow, lvalid, 1);  // (NCH >= 5)
      int lt = 0, lc = 2;            // the next chunk to gather: tile lt, chunk lc
      for (int i = 0; i < ntile; ++i, ++tt) {
        const int r = i * 128 + tid;
        const bool valid = r < cnt;
        const unsigned slot = valid ? sidx[pos0 + r] : 0u;
        FMM_DCHECK(!valid || (FMM_IN(ssrc[pos0 + r], g_fmm_chk.rows) &&
                              FMM_IN(slot, Lacc ? g_fmm_chk.rows : g_fmm_chk.yrows)),
                   "K-tiled M2L source row / result slot");
        for (int c = 0; c < NCH; ++c, ++g) {
          const int s = g & 1;
          if (g >= 2) {
            mbar_wait_tc(&s_free[s], ((g >> 1) - 1) & 1);  // the MMAs that read stage s are done
            tc_fence_after();
          }
          // A chunk: row tid, K-columns 4q..4q+3 of the chunk at (q * 128 + tid) * 16 bytes
          float4 *ah = reinterpret_cast<float4 *>(a_base(s)), *al = reinterpret_cast<float4 *>(a_base(s) + ABYTES);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 v4 = xa[q];
            const float vs[4] = {v4.x, v4.y, v4.z, v4.w};
            float hv[4], lv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              unsigned hb, lb;
              tf32_split(vs[e], hb, lb);
              hv[e] = __uint_as_float(hb);
              lv[e] = __uint_as_float(lb);
            }
            ah[q * 128 + tid] = make_float4(hv[0], hv[1], hv[2], hv[3]);
            al[q * 128 + tid] = make_float4(lv[0], lv[1], lv[2], lv[3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tc_fence_before();
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&a_full[s])) : "memory");
#pragma unroll
          for (int q = 0; q < 8; ++q) xa[q] = xb[q];
          if (lc == NCH) {
            lc = 0;
            if (++lt < ntile) lrow = row_of(lt, lvalid);
          }
          if (lt < ntile) load_to(xb, lrow, lvalid, lc);
          ++lc;
        }
        // the previous tile's epilogue overlaps this tile's MMAs (double-buffered D)
        if (DB == 2 && i > 0) epilogue(tt - 1, cnt, (i - 1) * 128, prev_slot);
        if (DB == 1) epilogue(tt, cnt, i * 128, slot);
        prev_slot = slot;
      }
      if (DB == 2 && ntile > 0) epilogue(tt - 1, cnt, (ntile - 1) * 128, prev_slot);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512)
                 : "memory");
}

bool m2l_tck_supported(int p) { return p >= 11 && p <= 15; }
size_t m2l_tck_T_words(int p) { return (size_t)2 * tck_np(p) * tck_kp(p); }

cudaError_t m2l_tck_build_T(int p, const M2LWork &W, int ngclass, unsigned *Timg, cudaStream_t st) {
  if (ngclass <= 0) return cudaSuccess;
  const size_t smem = (size_t)(2 * p + 1) * (2 * p + 1) * sizeof(double2);
  k_m2l_build_T_tck<<<ngclass < 148 * 4 ? ngclass : 148 * 4, 256, smem, st>>>(
      p, W.counters, W.class_rep, W.pair_t, W.src, W.C, Timg);
  return cudaGetLastError();
}

cudaError_t m2l_tck_gemm(int p, const M2LWork &W, const unsigned *Timg, const float2 *M,
                         cudaStream_t st, float2 *Lacc) {
  int *queue = W.counters + 4;
  cudaMemsetAsync(queue, 0, sizeof(int), st);
  const unsigned *slots = Lacc ? W.stgt : W.sidx;
#define M2L_TCK_CASE(PP)                                                                        \
  case PP: {                                                                                  \
    const size_t smem = (size_t)2 * (2u * 128u * TCK_KC * 4u + 2u * tck_np(PP) * TCK_KC * 4u) + 128; \
    fmm_smem_optin((const void *)k_m2l_tck<PP>, smem);                                        \
    k_m2l_tck<PP><<<148, 160, smem, st>>>(W.items, W.counters, slots, W.ssrc, Timg,           \
                                          reinterpret_cast<const float *>(M), W.Y, queue,      \
                                          reinterpret_cast<float *>(Lacc));                    \
  } break;
  switch (p) {
    M2L_TCK_CASE(11) M2L_TCK_CASE(12) M2L_TCK_CASE(13) M2L_TCK_CASE(14) M2L_TCK_CASE(15)
    default: break;
  }
#undef M2L_TCK_CASE
  return cudaGetLastError();
}

FMM_CHK_DEFINE_SETTER(fmm_chk_set_m2l_tc)
