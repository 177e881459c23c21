// p2p_core.cuh — the P2P pair arithmetic (packed f32x2, two targets per lane), shared by the
// P2P kernels of p2p.cu and by tools/p2p_micro.cu (the instruction-mix ceiling microbenchmark).
#pragma once
#include <cuda_runtime.h>

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
// 8 sources in flight per lane (more ILP per warp, more registers)
template <bool MASK, int S>
__device__ __forceinline__ void p2p_tile_rawS8(const float4 *__restrict__ sp, int ns, int h,
                                               f2x tx, f2x ty, f2x tz, f2x acc[4]) {
  f2x ph = 0ull, gx = 0ull, gy = 0ull, gz = 0ull;
  f2x ph2 = 0ull, gx2 = 0ull, gy2 = 0ull, gz2 = 0ull;
  const float4 *q = sp + h;
  const float4 *end8 = ns > 7 * S ? sp + ns - 7 * S : sp;
  for (; q < end8; q += 8 * S) {
    const float4 s0 = q[0], s1 = q[S], s2 = q[2 * S], s3 = q[3 * S];
    const float4 s4 = q[4 * S], s5 = q[5 * S], s6 = q[6 * S], s7 = q[7 * S];
    p2p_raw<MASK>(s0, tx, ty, tz, ph, gx, gy, gz);
    p2p_raw<MASK>(s1, tx, ty, tz, ph2, gx2, gy2, gz2);
    p2p_raw<MASK>(s2, tx, ty, tz, ph, gx, gy, gz);
    p2p_raw<MASK>(s3, tx, ty, tz, ph2, gx2, gy2, gz2);
    p2p_raw<MASK>(s4, tx, ty, tz, ph, gx, gy, gz);
    p2p_raw<MASK>(s5, tx, ty, tz, ph2, gx2, gy2, gz2);
    p2p_raw<MASK>(s6, tx, ty, tz, ph, gx, gy, gz);
    p2p_raw<MASK>(s7, tx, ty, tz, ph2, gx2, gy2, gz2);
  }
  for (; q < sp + ns; q += S) p2p_raw<MASK>(q[0], tx, ty, tz, ph, gx, gy, gz);
  acc[0] = add2(acc[0], add2(ph, ph2));
  acc[1] = add2(acc[1], add2(gx, gx2));
  acc[2] = add2(acc[2], add2(gy, gy2));
  acc[3] = add2(acc[3], add2(gz, gz2));
}
#ifdef P2P_UNROLL8
#define P2P_TILE_S p2p_tile_rawS8
#else
#define P2P_TILE_S p2p_tile_rawS
#endif
template <bool MASK>
__device__ __forceinline__ void p2p_tile_raw(const float4 *__restrict__ sp, int ns, int h, int S,
                                             f2x tx, f2x ty, f2x tz, f2x acc[4]) {
  switch (S) {
    case 1: P2P_TILE_S<MASK, 1>(sp, ns, h, tx, ty, tz, acc); break;
    case 2: P2P_TILE_S<MASK, 2>(sp, ns, h, tx, ty, tz, acc); break;
    case 3: P2P_TILE_S<MASK, 3>(sp, ns, h, tx, ty, tz, acc); break;
    case 4: P2P_TILE_S<MASK, 4>(sp, ns, h, tx, ty, tz, acc); break;
    case 5: P2P_TILE_S<MASK, 5>(sp, ns, h, tx, ty, tz, acc); break;
    case 6: P2P_TILE_S<MASK, 6>(sp, ns, h, tx, ty, tz, acc); break;
    case 7: P2P_TILE_S<MASK, 7>(sp, ns, h, tx, ty, tz, acc); break;
    case 8: P2P_TILE_S<MASK, 8>(sp, ns, h, tx, ty, tz, acc); break;
    case 10: P2P_TILE_S<MASK, 10>(sp, ns, h, tx, ty, tz, acc); break;
    case 16: P2P_TILE_S<MASK, 16>(sp, ns, h, tx, ty, tz, acc); break;
    default: P2P_TILE_S<MASK, 32>(sp, ns, h, tx, ty, tz, acc); break;
  }
}


// Four targets per lane (two packed target pairs) against one source: every shared-memory source
// load feeds four pairs, and the two pairs give the scheduler two independent chains per source.
// Accumulates straight into acc (no per-tile partial sums: P2P lists are near-field length).
template <bool MASK, int S, int U>
__device__ __forceinline__ void p2p_tile_quad(const float4 *__restrict__ sp, int ns, int h,
                                              const f2x (&t)[6], f2x (&acc)[8]) {
  const float4 *q = sp + h;
  const float4 *endU = ns > (U - 1) * S ? sp + ns - (U - 1) * S : sp;
  for (; q < endU; q += U * S) {
    float4 s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) s[u] = q[u * S];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      p2p_raw<MASK>(s[u], t[0], t[1], t[2], acc[0], acc[1], acc[2], acc[3]);
      p2p_raw<MASK>(s[u], t[3], t[4], t[5], acc[4], acc[5], acc[6], acc[7]);
    }
  }
  for (; q < sp + ns; q += S) {
    const float4 s0 = q[0];
    p2p_raw<MASK>(s0, t[0], t[1], t[2], acc[0], acc[1], acc[2], acc[3]);
    p2p_raw<MASK>(s0, t[3], t[4], t[5], acc[4], acc[5], acc[6], acc[7]);
  }
}

// The same with a run-time slice count S (the CTA-wide lane pool of k_p2p_tma: S = 128 / Q for Q
// target quads takes many values): two sources per unrolled step, the second one S float4 further.
__device__ __forceinline__ float4 lds128(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
template <bool MASK>
__device__ __forceinline__ void p2p_tile_quad_rt(const float4 *__restrict__ sp, int ns, int h, int S,
                                                 const f2x (&t)[6], f2x (&acc)[8]) {
  // 32-bit shared addresses (ptxas still forms them with two IMAD-immediates per step)
  const unsigned base = (unsigned)__cvta_generic_to_shared(sp);
  const unsigned sb = 16u * (unsigned)S, sb2 = 2u * sb;
  unsigned a = base + 16u * (unsigned)h;
  const unsigned end = base + 16u * (unsigned)ns;
  const unsigned end2 = ns > S ? end - sb : base;
  for (; a < end2; a += sb2) {
    const float4 s0 = lds128(a), s1 = lds128(a + sb);
    p2p_raw<MASK>(s0, t[0], t[1], t[2], acc[0], acc[1], acc[2], acc[3]);
    p2p_raw<MASK>(s0, t[3], t[4], t[5], acc[4], acc[5], acc[6], acc[7]);
    p2p_raw<MASK>(s1, t[0], t[1], t[2], acc[0], acc[1], acc[2], acc[3]);
    p2p_raw<MASK>(s1, t[3], t[4], t[5], acc[4], acc[5], acc[6], acc[7]);
  }
  if (a < end) {
    const float4 s0 = lds128(a);
    p2p_raw<MASK>(s0, t[0], t[1], t[2], acc[0], acc[1], acc[2], acc[3]);
    p2p_raw<MASK>(s0, t[3], t[4], t[5], acc[4], acc[5], acc[6], acc[7]);
  }
}
