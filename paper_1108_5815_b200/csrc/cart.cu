// cart.cu — Cartesian Taylor expansions on the device (PAPER.md:60
// "capability to switch to Cartesian expansions ... key to achieving high performance for
// low-accuracy"). Operators of total order p (reading R17), in the power-of-two
// scaled form of the spherical path (r = cell half-width; every scale factor exact):
//
//   P2M  Mh_k    = sum_i q_i u_i^k,                 u = (y - c) / r
//   M2M  Mh_k(P) = sum_C sum_{j <= k} C(k, j) 2^-|k| s_C^(k-j) Mh_j(C),   s_C = octant signs
//   M2L  Lh_n    = sum_{|k| <= p-|n|} (-1)^|k| C(k+n, n) rho^|k| Mh_k a_{k+n}(u),
//                  u = (c_t - c_s) / r_t, rho = r_s / r_t
//   L2L  Lh_n(C) = sum_{m >= n} C(m, n) s_C^(m-n) 2^-(|m|+1) Lh_m(P)
//   L2P  phi = (1/r) sum_n Lh_n u^n,  grad_a = (1/r^2) sum_n Lh_n n_a u^(n - e_a)
//   M2P  phi = (1/r_s) sum_k (-1)^|k| Mh_k a_k(xi),  grad_a = (1/r_s^2) sum_k (-1)^|k| Mh_k
//        (k_a + 1) a_{k+e_a}(xi),  xi = (x - c_s) / r_s
//
// a_m(d) = (1/m!) d^m (1/|d|) by |m| |d|^2 a_m + (2|m|-1) sum_a d_a a_{m-e_a} +
// (|m|-1) sum_a a_{m-2e_a} = 0. Multi-indices are enumerated by order, then kx, ky descending
// (the oracle's order, cartesian.c). All index tables are constexpr: every loop over them is
// fully unrolled, so the coefficient arrays stay in registers.
//
// The M2L runs on CUDA cores, one warp per target cell over its list (deterministic: fixed lane
// assignment and a fixed butterfly reduction), because at p <= 4 the whole translation is ~210
// FMAs -- the tensor-core class GEMM would pad 35 dofs to 64 and do 20x the work.
#include "common.cuh"
#include "kernels.cuh"

namespace {

__host__ __device__ constexpr int ccount(int P) { return (P + 1) * (P + 2) * (P + 3) / 6; }
__host__ __device__ constexpr int cindex(int kx, int ky, int kz) {
  return (kx + ky + kz) * (kx + ky + kz + 1) * (kx + ky + kz + 2) / 6 +
         (ky + kz) * (ky + kz + 1) / 2 + kz;
}
struct MI {
  int x, y, z;
};
// the multi-index table of order P as a constexpr aggregate: a local `constexpr CT<P> T{}` read
// with the (unrolled, hence constant) loop index folds to immediates -- no local-memory arrays
template <int P>
struct CT {
  int x[ccount(P)], y[ccount(P)], z[ccount(P)];
  constexpr CT() : x(), y(), z() {
    for (int s = 0; s <= P; ++s)
      for (int kx = s; kx >= 0; --kx)
        for (int ky = s - kx; ky >= 0; --ky) {
          const int i = cindex(kx, ky, s - kx - ky);
          x[i] = kx;
          y[i] = ky;
          z[i] = s - kx - ky;
        }
  }
  constexpr MI operator[](int i) const { return MI{x[i], y[i], z[i]}; }
  constexpr int ord(int i) const { return x[i] + y[i] + z[i]; }
};
__host__ __device__ constexpr float cbinom(int m, int n) {
  float b = 1.f;
  for (int i = 1; i <= n; ++i) b = b * (float)(m - n + i) / (float)i;
  return b;
}
__host__ __device__ constexpr bool cle(MI a, MI b) { return a.x <= b.x && a.y <= b.y && a.z <= b.z; }

// flattened operator tables (one fully unrolled loop each; a nested 35 x 35 loop with skipped
// entries is not unrolled completely and would index the register arrays dynamically)
__host__ __device__ constexpr int m2l_entries(int P) {
  int e = 0;
  for (int sn = 0; sn <= P; ++sn)
    for (int sk = 0; sn + sk <= P; ++sk) e += (sn + 1) * (sn + 2) / 2 * ((sk + 1) * (sk + 2) / 2);
  return e;
}
// M2L: acc[n] += c * mk[k] * a[m], m = k + n, c = C(k + n, n) (the sign / rho^|k| are in mk)
template <int P>
struct M2LT {
  int n[m2l_entries(P)], k[m2l_entries(P)], m[m2l_entries(P)];
  float c[m2l_entries(P)];
  constexpr M2LT() : n(), k(), m(), c() {
    CT<P> T{};
    int e = 0;
    for (int in = 0; in < ccount(P); ++in)
      for (int ik = 0; ik < ccount(P); ++ik) {
        const MI N = T[in], K = T[ik];
        if (T.ord(in) + T.ord(ik) > P) continue;
        n[e] = in;
        k[e] = ik;
        m[e] = cindex(K.x + N.x, K.y + N.y, K.z + N.z);
        c[e] = cbinom(K.x + N.x, N.x) * cbinom(K.y + N.y, N.y) * cbinom(K.z + N.z, N.z);
        ++e;
      }
  }
};
__host__ __device__ constexpr int shift_entries(int P) {
  int e = 0;
  for (int kx = 0; kx <= P; ++kx)
    for (int ky = 0; kx + ky <= P; ++ky)
      for (int kz = 0; kx + ky + kz <= P; ++kz) e += (kx + 1) * (ky + 1) * (kz + 1);
  return e;
}
// M2M / L2L shifts: pairs (hi, lo) with lo <= hi componentwise; c = C(hi, lo); d = hi - lo parity
// bits (x | y << 1 | z << 2) for the octant sign s^(hi - lo); o = |hi| (M2M) for the 2^-|.| factor
template <int P>
struct ShT {
  int hi[shift_entries(P)], lo[shift_entries(P)], d[shift_entries(P)], o[shift_entries(P)];
  float c[shift_entries(P)];
  constexpr ShT() : hi(), lo(), d(), o(), c() {
    CT<P> T{};
    int e = 0;
    for (int ih = 0; ih < ccount(P); ++ih)
      for (int il = 0; il < ccount(P); ++il) {
        const MI H = T[ih], L = T[il];
        if (!cle(L, H)) continue;
        hi[e] = ih;
        lo[e] = il;
        d[e] = ((H.x - L.x) & 1) | (((H.y - L.y) & 1) << 1) | (((H.z - L.z) & 1) << 2);
        o[e] = T.ord(ih);
        c[e] = cbinom(H.x, L.x) * cbinom(H.y, L.y) * cbinom(H.z, L.z);
        ++e;
      }
  }
};
// the sign s^(hi - lo) of an octant with signs (sx, sy, sz) = +-1, from the parity bits
__device__ __forceinline__ float oct_sign(int d, float sx, float sy, float sz) {
  return ((d & 1) ? sx : 1.f) * ((d & 2) ? sy : 1.f) * ((d & 4) ? sz : 1.f);
}

// a[0 .. ccount(P)) = a_m(u), |m| <= P (u in registers, results in registers)
template <int P>
__device__ __forceinline__ void cart_derivs(float ux, float uy, float uz, float (&a)[ccount(P)]) {
  const float r2 = ux * ux + uy * uy + uz * uz;
  const float ir2 = 1.f / r2;
  a[0] = rsqrtf(r2);
  constexpr CT<P> T{};
#pragma unroll
  for (int i = 1; i < ccount(P); ++i) {
    const MI m = T[i];
    const int s = m.x + m.y + m.z;
    float t1 = 0.f, t2 = 0.f;
    if (m.x >= 1) t1 += ux * a[cindex(m.x - 1, m.y, m.z)];
    if (m.y >= 1) t1 += uy * a[cindex(m.x, m.y - 1, m.z)];
    if (m.z >= 1) t1 += uz * a[cindex(m.x, m.y, m.z - 1)];
    if (m.x >= 2) t2 += a[cindex(m.x - 2, m.y, m.z)];
    if (m.y >= 2) t2 += a[cindex(m.x, m.y - 2, m.z)];
    if (m.z >= 2) t2 += a[cindex(m.x, m.y, m.z - 2)];
    a[i] = -((2.f * s - 1.f) * t1 + (s - 1.f) * t2) * (ir2 / (float)s);
  }
}

// monomials u^k, |k| <= P
template <int P>
__device__ __forceinline__ void cart_monos(float ux, float uy, float uz, float (&mo)[ccount(P)]) {
  float px[P + 1], py[P + 1], pz[P + 1];
  px[0] = py[0] = pz[0] = 1.f;
#pragma unroll
  for (int e = 1; e <= P; ++e) {
    px[e] = px[e - 1] * ux;
    py[e] = py[e - 1] * uy;
    pz[e] = pz[e - 1] * uz;
  }
  constexpr CT<P> T{};
#pragma unroll
  for (int i = 0; i < ccount(P); ++i) {
    const MI k = T[i];
    mo[i] = px[k.x] * py[k.y] * pz[k.z];
  }
}

template <int N>
__device__ __forceinline__ void warp_sum_all(float (&v)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
}

}  // namespace

int cart_stride(int p) { return (ccount(p) + 3) & ~3; }
int cart_count(int p) { return ccount(p); }

// ---- P2M: warp per leaf, lane per particle -----------------------------------------------------
template <int P>
__global__ void __launch_bounds__(128) k_cart_p2m(const int *__restrict__ leaves, int nleaves,
                                                  CellsView C, const float4 *__restrict__ pos,
                                                  float *__restrict__ M) {
  constexpr int NK = ccount(P), CS = (NK + 3) & ~3;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int li = gw; li < nleaves; li += nw) {
    const int leaf = leaves[li];
    const float4 g = C.geo[leaf];
    const float rinv = 1.f / g.w;
    const int b = C.beg[leaf], cnt = C.cnt[leaf];
    float acc[NK];
#pragma unroll
    for (int i = 0; i < NK; ++i) acc[i] = 0.f;
    for (int c0 = 0; c0 < cnt; c0 += WARP) {
      const bool valid = c0 + lane < cnt;
      const float4 y = valid ? pos[b + c0 + lane] : make_float4(g.x, g.y, g.z, 0.f);
      float mo[NK];
      cart_monos<P>((y.x - g.x) * rinv, (y.y - g.y) * rinv, (y.z - g.z) * rinv, mo);
#pragma unroll
      for (int i = 0; i < NK; ++i) acc[i] += y.w * mo[i];
    }
    warp_sum_all(acc);
    float *row = M + (size_t)leaf * CS;
#pragma unroll
    for (int i = 0; i < NK; ++i)
      if (lane == (i & 31)) row[i] = acc[i];
  }
}

// ---- M2M (one level): warp per parent, lanes over output coefficients ---------------------------
template <int P>
__global__ void __launch_bounds__(128) k_cart_m2m(int c0, int nl, CellsView C, float *__restrict__ M) {
  constexpr int NK = ccount(P), CS = (NK + 3) & ~3;
  constexpr CT<P> T{};
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int w = gw; w < nl; w += nw) {
    const int par = c0 + w;
    const int nch = C.nchild[par], ch0 = C.child0[par];
    if (nch == 0) continue;
    const int4 gp = C.grid[par];
    float out[(NK + 31) / 32];
#pragma unroll
    for (int q = 0; q < (NK + 31) / 32; ++q) out[q] = 0.f;
    for (int ch = 0; ch < nch; ++ch) {
      const int c = ch0 + ch;
      const int4 gc = C.grid[c];
      const float sx = gc.x > gp.x ? 1.f : -1.f, sy = gc.y > gp.y ? 1.f : -1.f,
                  sz = gc.z > gp.z ? 1.f : -1.f;
      const float *Mc = M + (size_t)c * CS;
      float mc[NK];
#pragma unroll
      for (int i = 0; i < NK; ++i) mc[i] = Mc[i];
      constexpr ShT<P> S{};
      float o[NK];
#pragma unroll
      for (int i = 0; i < NK; ++i) o[i] = 0.f;
#pragma unroll
      for (int e = 0; e < shift_entries(P); ++e)  // Mh_hi(P) += C(hi, lo) s^(hi-lo) Mh_lo(C)
        o[S.hi[e]] += S.c[e] * oct_sign(S.d[e], sx, sy, sz) * mc[S.lo[e]];
#pragma unroll
      for (int k = 0; k < NK; ++k)
        if (lane == (k & 31)) out[k >> 5] += o[k] * ldexpf(1.f, -T.ord(k));
    }
    float *Mp = M + (size_t)par * CS;
#pragma unroll
    for (int q = 0; q < (NK + 31) / 32; ++q)
      if (q * 32 + lane < NK) Mp[q * 32 + lane] = out[q];
  }
}

// ---- M2L: warp per target cell, lanes over its list; writes every cell's Lh --------------------
template <int P>
__global__ void __launch_bounds__(128) k_cart_m2l(int ncells, CellsView C, ListsView Ls,
                                                  const float *__restrict__ M,
                                                  float *__restrict__ L) {
  constexpr int NK = ccount(P), CS = (NK + 3) & ~3;
  constexpr CT<P> T{};
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < ncells; t += nw) {
    const int off = Ls.off[0][t], cnt = Ls.cnt[0][t];
    float acc[NK];
#pragma unroll
    for (int i = 0; i < NK; ++i) acc[i] = 0.f;
    if (cnt > 0) {
      const int4 gt = C.grid[t];
      const float rt_inv = ldexpf(1.f, -(FMM_LEVELS - gt.w));
      for (int e = lane; e < cnt; e += WARP) {
        const unsigned s = Ls.src[0][off + e];
        const int4 gs = C.grid[s];
        const float ux = (float)(gt.x - gs.x) * rt_inv, uy = (float)(gt.y - gs.y) * rt_inv,
                    uz = (float)(gt.z - gs.z) * rt_inv;
        const float rho = ldexpf(1.f, gt.w - gs.w);
        float a[NK];
        cart_derivs<P>(ux, uy, uz, a);
        // (-1)^|k| rho^|k| Mh_k
        float mk[NK];
        const float *Ms = M + (size_t)s * CS;
        float rp[P + 1];
        rp[0] = 1.f;
#pragma unroll
        for (int o = 1; o <= P; ++o) rp[o] = -rp[o - 1] * rho;
#pragma unroll
        for (int k = 0; k < NK; ++k) mk[k] = rp[T.ord(k)] * Ms[k];
        constexpr M2LT<P> E{};
#pragma unroll
        for (int e = 0; e < m2l_entries(P); ++e) acc[E.n[e]] += E.c[e] * mk[E.k[e]] * a[E.m[e]];
      }
      warp_sum_all(acc);
    }
    float *row = L + (size_t)t * CS;
#pragma unroll
    for (int i = 0; i < NK; ++i)
      if (lane == (i & 31)) row[i] = acc[i];
  }
}

// ---- L2L (one level): warp per child, lanes over output coefficients ----------------------------
template <int P>
__global__ void __launch_bounds__(128) k_cart_l2l(int c0, int nl, CellsView C, float *__restrict__ L) {
  constexpr int NK = ccount(P), CS = (NK + 3) & ~3;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  constexpr CT<P> T{};
  for (int w = gw; w < nl; w += nw) {
    const int c = c0 + w, par = C.parent[c];
    const int4 gc = C.grid[c], gp = C.grid[par];
    const float sx = gc.x > gp.x ? 1.f : -1.f, sy = gc.y > gp.y ? 1.f : -1.f,
                sz = gc.z > gp.z ? 1.f : -1.f;
    const float *Lp = L + (size_t)par * CS;
    float lp[NK];
#pragma unroll
    for (int i = 0; i < NK; ++i) lp[i] = Lp[i];
    float *Lc = L + (size_t)c * CS;
    constexpr ShT<P> S{};
    float o[NK];
#pragma unroll
    for (int i = 0; i < NK; ++i) o[i] = 0.f;
#pragma unroll
    for (int e = 0; e < shift_entries(P); ++e)  // Lh_lo(C) += C(hi, lo) s^(hi-lo) 2^-(|hi|+1) Lh_hi(P)
      o[S.lo[e]] += S.c[e] * ldexpf(1.f, -(S.o[e] + 1)) * oct_sign(S.d[e], sx, sy, sz) * lp[S.hi[e]];
#pragma unroll
    for (int n = 0; n < NK; ++n)
      if (lane == (n & 31)) Lc[n] += o[n];
  }
}

// ---- L2P + combine + un-permute: warp per leaf, lane per particle (as k_l2p) -------------------
template <int P>
__global__ void __launch_bounds__(128) k_cart_l2p(const int *__restrict__ leaves, int nleaves,
                                                  CellsView C, const float4 *__restrict__ pos,
                                                  const float *__restrict__ L,
                                                  const float4 *__restrict__ acc,
                                                  const unsigned *__restrict__ perm,
                                                  float *__restrict__ phi_out,
                                                  float *__restrict__ grad_out, int use_local) {
  constexpr int NK = ccount(P), CS = (NK + 3) & ~3;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int li = gw; li < nleaves; li += nw) {
    const int leaf = leaves[li];
    const int b = C.beg[leaf], cnt = C.cnt[leaf];
    const float4 g = C.geo[leaf];
    const float rinv = 1.f / g.w;
    float l[NK];
    const float *Lr = L + (size_t)leaf * CS;
#pragma unroll
    for (int i = 0; i < NK; ++i) l[i] = use_local ? Lr[i] : 0.f;
    for (int c0 = 0; c0 < cnt; c0 += WARP) {
      if (c0 + lane >= cnt) continue;
      const int i = b + c0 + lane;
      const float4 x = pos[i];
      float4 out = acc[i];
      if (use_local) {
        float mo[NK];
        cart_monos<P>((x.x - g.x) * rinv, (x.y - g.y) * rinv, (x.z - g.z) * rinv, mo);
        float ph = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
        constexpr CT<P> T{};
#pragma unroll
        for (int n = 0; n < NK; ++n) {
          const MI N = T[n];
          ph += l[n] * mo[n];
          if (N.x) gx += (float)N.x * l[n] * mo[cindex(N.x - 1, N.y, N.z)];
          if (N.y) gy += (float)N.y * l[n] * mo[cindex(N.x, N.y - 1, N.z)];
          if (N.z) gz += (float)N.z * l[n] * mo[cindex(N.x, N.y, N.z - 1)];
        }
        const float r2i = rinv * rinv;
        out.x += ph * rinv;
        out.y += gx * r2i;
        out.z += gy * r2i;
        out.w += gz * r2i;
      }
      const size_t o = perm[i];
      phi_out[o] = out.x;
      grad_out[3 * o + 0] = out.y;
      grad_out[3 * o + 1] = out.z;
      grad_out[3 * o + 2] = out.w;
    }
  }
}

// ---- M2P: warp per leaf (dynamic queue), lanes = targets; M2P lists of the leaf and ancestors ----
template <int P>
__global__ void __launch_bounds__(128) k_cart_m2p(const int *__restrict__ leaves, int nleaves,
                                                  CellsView C, ListsView Ls,
                                                  const float4 *__restrict__ pos,
                                                  const float *__restrict__ M,
                                                  float4 *__restrict__ acc, int *next_leaf) {
  constexpr int NK = ccount(P), NK1 = ccount(P + 1), CS = (NK + 3) & ~3;
  const int lane = threadIdx.x & 31;
  for (;;) {
    int li = 0;
    if (lane == 0) li = atomicAdd(next_leaf, 1);
    li = __shfl_sync(0xffffffffu, li, 0);
    if (li >= nleaves) break;
    const int leaf = leaves[li];
    bool any = false;
    for (int a = leaf; a >= 0; a = C.parent[a]) any |= Ls.cnt[1][a] > 0;
    if (!any) continue;
    const int b = C.beg[leaf], cnt = C.cnt[leaf];
    for (int c0 = 0; c0 < cnt; c0 += WARP) {
      const bool valid = c0 + lane < cnt;
      const int i = b + c0 + lane;
      const float4 x = valid ? pos[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      float phi = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
      for (int a = leaf; a >= 0; a = C.parent[a]) {
        const int off = Ls.off[1][a], n_s = Ls.cnt[1][a];
        for (int e = 0; e < n_s; ++e) {
          const int s = Ls.src[1][off + e];
          const float4 g = C.geo[s];
          const float rinv = 1.f / g.w;
          float d[NK1];
          cart_derivs<P + 1>((x.x - g.x) * rinv, (x.y - g.y) * rinv, (x.z - g.z) * rinv, d);
          const float *Ms = M + (size_t)s * CS;
          float ph = 0.f, dx = 0.f, dy = 0.f, dz = 0.f;
          constexpr CT<P> T{};
#pragma unroll
          for (int k = 0; k < NK; ++k) {
            const MI K = T[k];
            const float mk = ((K.x + K.y + K.z) & 1) ? -Ms[k] : Ms[k];
            ph += mk * d[k];
            dx += mk * (float)(K.x + 1) * d[cindex(K.x + 1, K.y, K.z)];
            dy += mk * (float)(K.y + 1) * d[cindex(K.x, K.y + 1, K.z)];
            dz += mk * (float)(K.z + 1) * d[cindex(K.x, K.y, K.z + 1)];
          }
          phi += ph * rinv;
          const float r2i = rinv * rinv;
          gx += dx * r2i;
          gy += dy * r2i;
          gz += dz * r2i;
        }
      }
      if (valid) {
        float4 v = acc[i];
        acc[i] = make_float4(v.x + phi, v.y + gx, v.z + gy, v.w + gz);
      }
    }
  }
}

// ---- launchers ----------------------------------------------------------------------------------
static int cart_grid(int64_t warps) {
  int64_t b = (warps + 3) / 4;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}
#define CART_DISPATCH(p, CALL)                 \
  switch (p) {                                 \
    case 1: { constexpr int P_ = 1; CALL; } break; \
    case 2: { constexpr int P_ = 2; CALL; } break; \
    case 3: { constexpr int P_ = 3; CALL; } break; \
    default: { constexpr int P_ = 4; CALL; } break; \
  }

bool cart_supported(int p) { return p >= 1 && p <= CART_PMAX; }
void launch_cart_p2m(int p, const int *leaves, int nleaves, CellsView C, const float4 *pos,
                     float *M, cudaStream_t st) {
  if (nleaves <= 0) return;
  CART_DISPATCH(p, (k_cart_p2m<P_><<<cart_grid(nleaves), 128, 0, st>>>(leaves, nleaves, C, pos, M)));
}
void launch_cart_m2m(int p, int c0, int nl, CellsView C, float *M, cudaStream_t st) {
  if (nl <= 0) return;
  CART_DISPATCH(p, (k_cart_m2m<P_><<<cart_grid(nl), 128, 0, st>>>(c0, nl, C, M)));
}
void launch_cart_m2l(int p, int ncells, CellsView C, ListsView Ls, const float *M, float *L,
                     cudaStream_t st) {
  if (ncells <= 0) return;
  CART_DISPATCH(p, (k_cart_m2l<P_><<<cart_grid(ncells), 128, 0, st>>>(ncells, C, Ls, M, L)));
}
void launch_cart_l2l(int p, int c0, int nl, CellsView C, float *L, cudaStream_t st) {
  if (nl <= 0) return;
  CART_DISPATCH(p, (k_cart_l2l<P_><<<cart_grid(nl), 128, 0, st>>>(c0, nl, C, L)));
}
void launch_cart_l2p(int p, const int *leaves, int nleaves, CellsView C, const float4 *pos,
                     const float *L, const float4 *acc, const unsigned *perm, float *phi,
                     float *grad, int use_local, cudaStream_t st) {
  if (nleaves <= 0) return;
  CART_DISPATCH(p, (k_cart_l2p<P_><<<cart_grid(nleaves), 128, 0, st>>>(
                       leaves, nleaves, C, pos, L, acc, perm, phi, grad, use_local)));
}
void launch_cart_m2p(int p, const int *leaves, int nleaves, CellsView C, ListsView Ls,
                     const float4 *pos, const float *M, float4 *acc, int *counter,
                     cudaStream_t st) {
  if (nleaves <= 0) return;
  cudaMemsetAsync(counter, 0, sizeof(int), st);
  CART_DISPATCH(p, (k_cart_m2p<P_><<<148 * 8, 128, 0, st>>>(leaves, nleaves, C, Ls, pos, M, acc,
                                                             counter)));
}
