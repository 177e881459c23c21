// p2p.cu — particle-particle direct summation ("a direct summation is performed
// between all particles in the cells"; P:67 target-parallel GPU N-body).
//
//   phi_i  += sum_j q_j / r_ij          grad_i += sum_j q_j (x_j - x_i) / r_ij^3
//
// Target-parallel, one warp per (target leaf, chunk of <= 32 targets). Every lane holds TWO
// targets in packed float2 registers, so each source costs 13 packed FP32 instructions
// (FADD2/FMUL2/FFMA2 with the source value as the broadcast operand) + 2 MUFU.RSQ for 2 pairs.
// Small leaves use a 2-D lane mapping: G target groups x S = 32/G source slices (slice h takes
// sources h, h+S, ...), reduced with shuffles at the end. The sources of the leaf's P2P list and
// of its ancestors' lists (a P2P pair with a non-leaf target applies to every particle under it)
// are concatenated into shared-memory tiles of P2P_TILE particles; the target leaf itself is
// processed in its own masked tiles (r = 0 pairs: the particle itself and coincident particles,
// which can only share a leaf). Accumulation is tile-blocked (per-tile partial sums added to the
// running total) to keep the FP32 error of long sums near 1e-7.
#include "common.cuh"
#include "kernels.cuh"

#ifndef P2P_TILE
#define P2P_TILE 256  // 16 KiB per warp double buffer; 256 beats 128 by ~2% at C2
#endif
#define P2P_WARPS 4
#ifndef P2P_SMAX
#define P2P_SMAX 32  // most source slices per warp (32 / G for G target pairs)
#endif
#ifndef P2P_MINB
#define P2P_MINB 4  // resident blocks per SM the register budget is sized for
#endif

__device__ __forceinline__ float rsqrt_approx(float x) {  // MUFU.RSQ, no denormal fix-up
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed f32x2 arithmetic on 64-bit registers (PTX add/mul/fma.rn.f32x2, sm_100+): keeping the
// pairs in .b64 values makes the register allocator hold them in aligned register pairs, so the
// compiler emits FADD2/FMUL2/FFMA2 without re-pairing MOVs.
typedef unsigned long long f2x;
__device__ __forceinline__ f2x pk(float a, float b) {
  f2x r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk(f2x v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ f2x add2(f2x a, f2x b) {
  f2x d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b) {
  f2x d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) {
  f2x d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// one source against the lane's two targets (tx = -x of the two targets)
__device__ __forceinline__ void ld_src(const float4 *sp, int j, f2x &xx, f2x &yy, f2x &zz,
                                       f2x &qq) {
  const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(sp + 2 * j);
  const ulonglong2 b = *reinterpret_cast<const ulonglong2 *>(sp + 2 * j + 1);
  xx = a.x;
  yy = a.y;
  zz = b.x;
  qq = b.y;
}
__device__ __forceinline__ void st_src(float4 *sp, int j, float4 v) {
  sp[2 * j] = make_float4(v.x, v.x, v.y, v.y);
  sp[2 * j + 1] = make_float4(v.z, v.z, v.w, v.w);
}

template <bool MASK>
__device__ __forceinline__ void p2p_pair2(const float4 *sp, int j, const f2x tx, const f2x ty,
                                          const f2x tz, f2x &ph, f2x &gx, f2x &gy, f2x &gz) {
  f2x sx, sy, sz, sq;
  ld_src(sp, j, sx, sy, sz, sq);
  const f2x dx = add2(sx, tx);
  const f2x dy = add2(sy, ty);
  const f2x dz = add2(sz, tz);
  f2x r2 = mul2(dx, dx);
  r2 = fma2(dy, dy, r2);
  r2 = fma2(dz, dz, r2);
  const float2 r2f = upk(r2);
  float rx = rsqrt_approx(r2f.x), ry = rsqrt_approx(r2f.y);
  if (MASK) {
    rx = r2f.x > 0.f ? rx : 0.f;
    ry = r2f.y > 0.f ? ry : 0.f;
  }
  const f2x ri = pk(rx, ry);
  const f2x qr = mul2(sq, ri);
  ph = add2(ph, qr);
  const f2x qr3 = mul2(qr, mul2(ri, ri));
  gx = fma2(dx, qr3, gx);
  gy = fma2(dy, qr3, gy);
  gz = fma2(dz, qr3, gz);
}

template <bool MASK>
__device__ __forceinline__ void p2p_tile2(const float4 *__restrict__ sp, int ns, int h, int S,
                                          f2x tx, f2x ty, f2x tz, f2x acc[4]) {
  f2x ph = 0ull, gx = 0ull, gy = 0ull, gz = 0ull;  // +0.0f pairs
  int j = h;
  for (; j + 3 * S < ns; j += 4 * S) {
    p2p_pair2<MASK>(sp, j, tx, ty, tz, ph, gx, gy, gz);
    p2p_pair2<MASK>(sp, j + S, tx, ty, tz, ph, gx, gy, gz);
    p2p_pair2<MASK>(sp, j + 2 * S, tx, ty, tz, ph, gx, gy, gz);
    p2p_pair2<MASK>(sp, j + 3 * S, tx, ty, tz, ph, gx, gy, gz);
  }
  for (; j < ns; j += S) p2p_pair2<MASK>(sp, j, tx, ty, tz, ph, gx, gy, gz);
  acc[0] = add2(acc[0], ph);
  acc[1] = add2(acc[1], gx);
  acc[2] = add2(acc[2], gy);
  acc[3] = add2(acc[3], gz);
}

// raw-float4 tile variant: source value as the broadcast operand of the packed ops
template <bool MASK>
__device__ __forceinline__ void p2p_raw(const float4 sv, const f2x tx, const f2x ty, const f2x tz,
                                        f2x &ph, f2x &gx, f2x &gy, f2x &gz) {
  const f2x dx = add2(pk(sv.x, sv.x), tx);
  const f2x dy = add2(pk(sv.y, sv.y), ty);
  const f2x dz = add2(pk(sv.z, sv.z), tz);
  f2x r2 = mul2(dx, dx);
  r2 = fma2(dy, dy, r2);
  r2 = fma2(dz, dz, r2);
  const float2 r2f = upk(r2);
  float rx = rsqrt_approx(r2f.x), ry = rsqrt_approx(r2f.y);
  if (MASK) {
    rx = r2f.x > 0.f ? rx : 0.f;
    ry = r2f.y > 0.f ? ry : 0.f;
  }
  const f2x ri = pk(rx, ry);
  const f2x qr = mul2(pk(sv.w, sv.w), ri);
  ph = add2(ph, qr);
  const f2x qr3 = mul2(qr, mul2(ri, ri));
  gx = fma2(dx, qr3, gx);
  gy = fma2(dy, qr3, gy);
  gz = fma2(dz, qr3, gz);
}

// S (source slices) is a compile-time constant so the four LDS.128 of an unrolled step use
// immediate offsets (no IMAD address arithmetic on the FMA pipe)
template <bool MASK, int S>
__device__ __forceinline__ void p2p_tile_rawS(const float4 *__restrict__ sp, int ns, int h,
                                              f2x tx, f2x ty, f2x tz, f2x acc[4]) {
  f2x ph = 0ull, gx = 0ull, gy = 0ull, gz = 0ull;
  const float4 *q = sp + h;
  // q + 3S < sp + ns; clamped so that the bound never lies below the buffer (as a 32-bit shared
  // address sp + ns - 3S would wrap around when the buffer starts near address 0)
  const float4 *end4 = ns > 3 * S ? sp + ns - 3 * S : sp;
  for (; q < end4; q += 4 * S) {
    const float4 s0 = q[0], s1 = q[S], s2 = q[2 * S], s3 = q[3 * S];
    p2p_raw<MASK>(s0, tx, ty, tz, ph, gx, gy, gz);
    p2p_raw<MASK>(s1, tx, ty, tz, ph, gx, gy, gz);
    p2p_raw<MASK>(s2, tx, ty, tz, ph, gx, gy, gz);
    p2p_raw<MASK>(s3, tx, ty, tz, ph, gx, gy, gz);
  }
  for (; q < sp + ns; q += S) p2p_raw<MASK>(q[0], tx, ty, tz, ph, gx, gy, gz);
  acc[0] = add2(acc[0], ph);
  acc[1] = add2(acc[1], gx);
  acc[2] = add2(acc[2], gy);
  acc[3] = add2(acc[3], gz);
}
template <bool MASK>
__device__ __forceinline__ void p2p_tile_raw(const float4 *__restrict__ sp, int ns, int h, int S,
                                             f2x tx, f2x ty, f2x tz, f2x acc[4]) {
  switch (S) {
    case 1: p2p_tile_rawS<MASK, 1>(sp, ns, h, tx, ty, tz, acc); break;
    case 2: p2p_tile_rawS<MASK, 2>(sp, ns, h, tx, ty, tz, acc); break;
    case 3: p2p_tile_rawS<MASK, 3>(sp, ns, h, tx, ty, tz, acc); break;
    case 4: p2p_tile_rawS<MASK, 4>(sp, ns, h, tx, ty, tz, acc); break;
    case 5: p2p_tile_rawS<MASK, 5>(sp, ns, h, tx, ty, tz, acc); break;
    case 6: p2p_tile_rawS<MASK, 6>(sp, ns, h, tx, ty, tz, acc); break;
    case 7: p2p_tile_rawS<MASK, 7>(sp, ns, h, tx, ty, tz, acc); break;
    case 8: p2p_tile_rawS<MASK, 8>(sp, ns, h, tx, ty, tz, acc); break;
    case 10: p2p_tile_rawS<MASK, 10>(sp, ns, h, tx, ty, tz, acc); break;
    case 16: p2p_tile_rawS<MASK, 16>(sp, ns, h, tx, ty, tz, acc); break;
    default: p2p_tile_rawS<MASK, 32>(sp, ns, h, tx, ty, tz, acc); break;
  }
}

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

#ifndef P2P_RANGES
#define P2P_RANGES 256  // per-warp list of source particle ranges (processed in batches)
#endif

__global__ void __launch_bounds__(P2P_WARPS * 32, P2P_MINB) k_p2p_leaves(const int *__restrict__ leaves,
                                                               int nleaves, CellsView C,
                                                               ListsView Ls,
                                                               const float4 *__restrict__ pos,
                                                               float4 *__restrict__ acc_out,
                                                               float m1, int *next_leaf) {
  __shared__ __align__(16) float4 sh[P2P_WARPS][2][P2P_TILE];
  __shared__ __align__(16) float4 shq[P2P_WARPS][64];  // 2 float4 per lane (target pairs)
  __shared__ int2 shr[P2P_WARPS][P2P_RANGES];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float4 *tq = shq[wib];
  int2 *rng = shr[wib];
  for (;;) {
    int li = 0;
    if (lane == 0) li = atomicAdd(next_leaf, 1);  // dynamic leaf queue (load balance)
    li = __shfl_sync(0xffffffffu, li, 0);
    if (li >= nleaves) break;
    const int leaf = leaves[li];
    const int tb = C.beg[leaf], tn = C.cnt[leaf];
    // ancestors of the leaf (each may carry a P2P list)
    int anc[FMM_LEVELS + 1], na = 0;
    for (int a = leaf; a >= 0 && na <= FMM_LEVELS; a = C.parent[a]) anc[na++] = a;
    for (int c0 = 0; c0 < tn; c0 += 32) {
      // G = ceil(nt / 2) target pairs x S = 32 / G source slices (lanes with h >= S idle): no
      // padding of the target count to a power of two (a 17-target leaf keeps 27 of 32 lanes
      // busy instead of 17 of 32 target slots), and the 1-10 targets left over by a 33-42
      // target leaf still spread the sources over all 32 lanes (S up to 32)
      const int nt = min(32, tn - c0);
      const int G = (nt + 1) >> 1;
      const int S = P2P_SMAX < 32 / G ? P2P_SMAX : 32 / G;
      const int grp = lane % G, h = lane / G;
      const bool active = h < S;
      const int i0 = c0 + 2 * grp, i1 = i0 + 1;
      const float4 t0 = i0 < tn ? pos[tb + i0] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 t1 = i1 < tn ? pos[tb + i1] : t0;
      __syncwarp();
      tq[2 * lane] = make_float4(m1 * t0.x, m1 * t1.x, m1 * t0.y, m1 * t1.y);
      tq[2 * lane + 1] = make_float4(m1 * t0.z, m1 * t1.z, 0.f, 0.f);
      __syncwarp();
      const ulonglong2 ta = *reinterpret_cast<const ulonglong2 *>(&tq[2 * lane]);
      const ulonglong2 tb2 = *reinterpret_cast<const ulonglong2 *>(&tq[2 * lane + 1]);
      const f2x tx = ta.x, ty = ta.y, tz = tb2.x;
      f2x acc[4] = {0ull, 0ull, 0ull, 0ull};
      // (1) the leaf itself, masked (r = 0 pairs)
      for (int j0 = 0; j0 < tn; j0 += P2P_TILE) {
        const int n = min(P2P_TILE, tn - j0);
        __syncwarp();
        for (int j = lane; j < n; j += 32) sh[wib][0][j] = pos[tb + j0 + j];
        __syncwarp();
        p2p_tile_raw<true>(sh[wib][0], active ? n : 0, h, S, tx, ty, tz, acc);
      }
      // (2) all other source cells of the P2P lists of the leaf and its ancestors, as particle
      // ranges collected into shared memory (batches of P2P_RANGES), streamed by cp.async into a
      // double-buffered tile: tile k+1 is in flight while tile k is computed
      int ai = 0, ae = 0;  // resume point: ancestor index, list position
      while (ai < na) {
        int nr = 0;
        while (ai < na && nr + 32 <= P2P_RANGES) {
          const int a = anc[ai];
          const int off = Ls.off[2][a], ncell = Ls.cnt[2][a];
          if (ae >= ncell) {
            ++ai;
            ae = 0;
            continue;
          }
          const int e = ae + lane;
          int2 r = make_int2(0, 0);
          if (e < ncell) {
            r = Ls.p2p_rng[off + e];   // (begin, count) stored by the traversal: one load
            if (r.x == tb) r.y = 0;     // the leaf itself is done separately (masked)
          }
          const unsigned bal = __ballot_sync(0xffffffffu, r.y > 0);
          if (r.y > 0) rng[nr + __popc(bal & ((1u << lane) - 1u))] = r;
          nr += __popc(bal);
          ae += 32;
        }
        __syncwarp();
        // stream the ranges through the two tile buffers
        int ri = 0, roff = 0, buf = 0;
        auto issue = [&](int b) -> int {  // fill tile b from the range cursor; returns its size
          int fill = 0;
          while (ri < nr && fill < P2P_TILE) {
            const int2 r = rng[ri];
            const int take = min(r.y - roff, P2P_TILE - fill);
            for (int j = lane; j < take; j += 32) cp_async16(&sh[wib][b][fill + j], &pos[r.x + roff + j]);
            fill += take;
            roff += take;
            if (roff == r.y) {
              ++ri;
              roff = 0;
            }
          }
          cp_async_commit();
          return fill;
        };
        int cur = issue(0);
        while (cur > 0) {
          const int nxt = issue(buf ^ 1);
          cp_async_wait1();  // tile `buf` has landed
          __syncwarp();
          p2p_tile_raw<false>(sh[wib][buf], active ? cur : 0, h, S, tx, ty, tz, acc);
          __syncwarp();
          buf ^= 1;
          cur = nxt;
        }
        cp_async_wait0();
        __syncwarp();
      }
      // reduce the S source slices (lanes grp, grp + G, ...) in slice order
      float2 r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) r[k] = upk(acc[k]);
      float2 tot[4] = {r[0], r[1], r[2], r[3]};
      for (int sl = 1; sl < S; ++sl) {  // slice order: deterministic
        const int from = grp + sl * G;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          tot[k].x += __shfl_sync(0xffffffffu, r[k].x, from);
          tot[k].y += __shfl_sync(0xffffffffu, r[k].y, from);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) r[k] = tot[k];
      if (h == 0) {
        if (i0 < tn) acc_out[tb + i0] = make_float4(r[0].x, r[1].x, r[2].x, r[3].x);
        if (i1 < tn) acc_out[tb + i1] = make_float4(r[0].y, r[1].y, r[2].y, r[3].y);
      }
      __syncwarp();
    }
  }
}

// FMM_DIRECT: all N targets against all N sources in caller order (no tree). Block of 256
// threads = 512 targets (2 per thread), source tiles of 512 staged by the whole block.
__global__ void __launch_bounds__(256) k_p2p_direct(int64_t n, const float4 *__restrict__ pos,
                                                    float *__restrict__ phi_out,
                                                    float *__restrict__ grad_out, float m1) {
  __shared__ float4 sh[2 * 512];
  __shared__ float4 tq[2 * 256];
  for (int64_t base = (int64_t)blockIdx.x * 512; base < n; base += (int64_t)gridDim.x * 512) {
    const int64_t i0 = base + 2 * threadIdx.x, i1 = i0 + 1;
    const float4 t0 = i0 < n ? pos[i0] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 t1 = i1 < n ? pos[i1] : t0;
    __syncthreads();
    tq[2 * threadIdx.x] = make_float4(m1 * t0.x, m1 * t1.x, m1 * t0.y, m1 * t1.y);
    tq[2 * threadIdx.x + 1] = make_float4(m1 * t0.z, m1 * t1.z, 0.f, 0.f);
    const ulonglong2 ta = *reinterpret_cast<const ulonglong2 *>(&tq[2 * threadIdx.x]);
    const ulonglong2 tb2 = *reinterpret_cast<const ulonglong2 *>(&tq[2 * threadIdx.x + 1]);
    const f2x tx = ta.x, ty = ta.y, tz = tb2.x;
    f2x acc[4] = {0ull, 0ull, 0ull, 0ull};
    for (int64_t j0 = 0; j0 < n; j0 += 512) {
      const int nt = (int)min((int64_t)512, n - j0);
      __syncthreads();
      for (int j = threadIdx.x; j < nt; j += 256) st_src(sh, j, pos[j0 + j]);
      __syncthreads();
      p2p_tile2<true>(sh, nt, 0, 1, tx, ty, tz, acc);
    }
    float2 r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) r[k] = upk(acc[k]);
    if (i0 < n) {
      phi_out[i0] = r[0].x;
      grad_out[3 * i0 + 0] = r[1].x;
      grad_out[3 * i0 + 1] = r[2].x;
      grad_out[3 * i0 + 2] = r[3].x;
    }
    if (i1 < n) {
      phi_out[i1] = r[0].y;
      grad_out[3 * i1 + 0] = r[1].y;
      grad_out[3 * i1 + 1] = r[2].y;
      grad_out[3 * i1 + 2] = r[3].y;
    }
  }
}

void launch_p2p_leaves(const int *leaves, int nleaves, CellsView C, ListsView Ls,
                       const float4 *pos, float4 *acc, int *counter, cudaStream_t st) {
  const int resident = fmm_resident_blocks((const void *)k_p2p_leaves, P2P_WARPS * 32, 0);
  // up to 8 waves of blocks (not a persistent grid): blocks retire continually, so that kernels of
  // a higher-priority stream (the M2L class sort running beside P2P) get SMs early
  const int need = (nleaves + P2P_WARPS - 1) / P2P_WARPS;
  const int b = need < 8 * resident ? (need > 0 ? need : 1) : 8 * resident;
  cudaMemsetAsync(counter, 0, sizeof(int), st);
  k_p2p_leaves<<<b, P2P_WARPS * 32, 0, st>>>(leaves, nleaves, C, Ls, pos, acc, -1.0f, counter);
}

void launch_p2p_direct(int64_t n, const float4 *pos, float *phi, float *grad, cudaStream_t st) {
  int64_t b = (n + 511) / 512;
  if (b > 148 * 64) b = 148 * 64;
  if (b < 1) b = 1;
  k_p2p_direct<<<(int)b, 256, 0, st>>>(n, pos, phi, grad, -1.0f);
}
