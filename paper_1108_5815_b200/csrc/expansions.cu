// expansions.cu — P2M, M2M, M2L, L2L, M2P and L2P on CUDA cores (sm_100a), FP32.
//
// Expansions (DESIGN.md §3 R1): R_n^m = r^n P_n^m e^{im phi}/(n+m)!,
// I_n^m = (n-m)! P_n^m e^{im phi}/r^{n+1}, evaluated with trig-free recurrences. They are stored
// power-of-two SCALED by the cell half-width r: Mhat_n^m = M_n^m / r^n,
// Lhat_n^m = L_n^m r^{n+1}, so FP32 never overflows at p <= 16 (unscaled I up to degree 2p
// would reach 1e54). Only orders m >= 0 are stored; m < 0 follows from A_n^{-m} = (-1)^m conj(A).
//
//   P2M  Mhat_n^m   = sum_i q_i conj(R_n^m((y_i - c)/r))
//   M2M  Mhat_n^m(P) = sum_{j,k} Mhat_j^k(C) 2^-j conj(R_{n-j}^{m-k}(b/r_P))
//   M2L  Lhat_j^k(t) = (-1)^{j+k} sum_{n<=p,m} Mhat_n^m(s) rho^n I_{n+j}^{m-k}(u)
//        u = (c_t - c_s)/r_t, rho = r_s/r_t   [for rho > 1 the same sum is formed at
//        v = u/rho with M unscaled and the result times rho^-(j+1): identical, in FP32 range]
//   L2L  Lhat_n^m(C) += 2^-(n+1) sum_{j>=n,k} Lhat_j^k(P) R_{j-n}^{k-m}(e/r_P)
//   M2P  phi += (1/r_s) sum Mhat I(xi), grad from I_{n+1} (d/dz I = -I_{n+1}, (dx+idy) I =
//        I_{n+1}^{m+1})
//   L2P  phi += (1/r) sum Lhat R(xi), grad from R_{n-1}
#include "common.cuh"
#include "kernels.cuh"

#include <cstdlib>

__constant__ short2 c_nm[nc_of(FMM_PMAX)];  // coefficient index -> (n, m) (also used by m2l.cu)

static bool upload_nm_table() {
  short2 h[nc_of(FMM_PMAX)];
  for (int n = 0; n <= FMM_PMAX; ++n)
    for (int m = 0; m <= n; ++m) h[cidx(n, m)] = make_short2((short)n, (short)m);
  return cudaMemcpyToSymbol(c_nm, h, sizeof(h)) == cudaSuccess;
}
// __constant__ memory is per device context: uploaded once per device (thread-safe)
void ensure_nm_table() { fmm_once_per_device((const void *)&c_nm, upload_nm_table); }

__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }

// Regular harmonics R_n^m(x), n <= P, m >= 0, into tab[cidx(n,m)]; lanes take columns m.
__device__ void regular_table(float x, float y, float z, int P, float2 *tab, int lane) {
  const float r2 = x * x + y * y + z * z;
  for (int m = lane; m <= P; m += WARP) {
    float2 Rmm = make_float2(1.f, 0.f);
    for (int k = 1; k <= m; ++k) Rmm = cscale(cmul(Rmm, make_float2(x, y)), -1.f / (2.f * k));
    tab[cidx(m, m)] = Rmm;
    float2 R2 = make_float2(0.f, 0.f), R1 = Rmm;
    for (int n = m + 1; n <= P; ++n) {
      float2 Rn;
      if (n == m + 1) Rn = cscale(Rmm, z);
      else {
        const float inv = 1.f / ((float)(n - m) * (float)(n + m));
        Rn = make_float2(((2 * n - 1) * z * R1.x - r2 * R2.x) * inv, ((2 * n - 1) * z * R1.y - r2 * R2.y) * inv);
      }
      tab[cidx(n, m)] = Rn;
      R2 = R1;
      R1 = Rn;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// P2M: warp per leaf; lane = particle. Each lane accumulates q conj(R(xi)) of its particles in
// registers (all NC coefficients, templated p), then the warp sums the 32 lane vectors through a
// padded shared-memory transpose (fixed order: deterministic).
#ifndef P2M_MINB
#define P2M_MINB 1
#endif
template <int p>
__global__ void __launch_bounds__(128, P2M_MINB) k_p2m(const int *__restrict__ leaves, int nleaves,
                                             CellsView C, const float4 *__restrict__ pos,
                                             float2 *__restrict__ M) {
  constexpr int NC = nc_of(p), NCS = nc_stride(p), RS = 2 * NC + 1;  // odd row stride
  extern __shared__ float sh_p2m[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float *red = sh_p2m + wib * 32 * RS;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int li = gw; li < nleaves; li += nw) {
    const int leaf = leaves[li];
    const float4 g = C.geo[leaf];
    const float rinv = 1.f / g.w;
    const int b = C.beg[leaf], cnt = C.cnt[leaf];
    float acc[2 * NC];
#pragma unroll
    for (int o = 0; o < 2 * NC; ++o) acc[o] = 0.f;
    for (int c0 = 0; c0 < cnt; c0 += WARP) {
      const bool valid = c0 + lane < cnt;
      const float4 y = valid ? pos[b + c0 + lane] : make_float4(g.x, g.y, g.z, 0.f);
      const float x = (y.x - g.x) * rinv, yy = (y.y - g.y) * rinv, z = (y.z - g.z) * rinv;
      const float q = y.w;
      const float r2 = x * x + yy * yy + z * z;
      float2 Rmm = make_float2(1.f, 0.f);
#pragma unroll
      for (int m = 0; m <= p; ++m) {
        if (m > 0) Rmm = cscale(cmul(Rmm, make_float2(x, yy)), -1.f / (2.f * m));
        float2 R2 = make_float2(0.f, 0.f), R1 = Rmm;
#pragma unroll
        for (int n = m; n <= p; ++n) {
          float2 Rn;
          if (n == m) Rn = Rmm;
          else if (n == m + 1) Rn = cscale(Rmm, z);
          else {
            const float inv = 1.f / ((float)(n - m) * (float)(n + m));
            Rn = make_float2(((2 * n - 1) * z * R1.x - r2 * R2.x) * inv,
                             ((2 * n - 1) * z * R1.y - r2 * R2.y) * inv);
          }
          if (n > m) {
            R2 = R1;
            R1 = Rn;
          }
          acc[2 * cidx(n, m)] += q * Rn.x;       // q conj(R)
          acc[2 * cidx(n, m) + 1] -= q * Rn.y;
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int o = 0; o < 2 * NC; ++o) red[lane * RS + o] = acc[o];
    __syncwarp();
    for (int o = lane; o < 2 * NC; o += WARP) {
      float s = 0.f;
      for (int l = 0; l < 32; ++l) s += red[l * RS + o];
      reinterpret_cast<float *>(M + (size_t)leaf * NCS)[o] = s;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------------------------
// P2M, round 2: the same sums in groups of order columns m in [M0, M1) holding <= P2M_GROUP
// complex coefficients, so the per-lane accumulators fit a small register budget (the one-pass
// kernel above needs 2 NC accumulators: 255 registers, 8 warps per SM at p = 10). Per group the
// lanes (one particle each) accumulate q conj(R_n^m) for its columns, then a padded shared-memory
// transpose sums the 32 lanes in lane order (deterministic) and writes the group's coefficients.
#ifndef P2M_GROUP
#define P2M_GROUP 24
#endif
__host__ __device__ constexpr int p2m_group_end(int P, int m0) {
  int m1 = m0, c = 0;
  while (m1 <= P && (c + (P - m1 + 1) <= P2M_GROUP || m1 == m0)) {
    c += P - m1 + 1;
    ++m1;
  }
  return m1;
}
__host__ __device__ constexpr int p2m_group_coeffs(int P, int m0, int m1) {
  int c = 0;
  for (int m = m0; m < m1; ++m) c += P - m + 1;
  return c;
}
template <int P, int M0, int M1>
__device__ __forceinline__ void p2m_group(int leaf, const float4 g, float rinv, int b, int cnt,
                                          const float4 *__restrict__ pos, float2 *__restrict__ M,
                                          float *red, int lane, int sl, int W) {
  constexpr int G = p2m_group_coeffs(P, M0, M1), RS = 2 * G + 1, NCS = nc_stride(P);
  float acc[2 * G];
#pragma unroll
  for (int o = 0; o < 2 * G; ++o) acc[o] = 0.f;
  for (int c0 = 0; c0 < cnt; c0 += W) {
    const bool valid = c0 + sl < cnt;
    const float4 y = valid ? pos[b + c0 + sl] : make_float4(g.x, g.y, g.z, 0.f);
    const float x = (y.x - g.x) * rinv, yy = (y.y - g.y) * rinv, z = (y.z - g.z) * rinv;
    const float q = y.w;
    const float r2 = x * x + yy * yy + z * z;
    float2 Rmm = make_float2(1.f, 0.f);
#pragma unroll
    for (int m = 1; m <= M0; ++m) Rmm = cscale(cmul(Rmm, make_float2(x, yy)), -1.f / (2.f * m));
    int o = 0;
#pragma unroll
    for (int m = M0; m < M1; ++m) {
      if (m > M0) Rmm = cscale(cmul(Rmm, make_float2(x, yy)), -1.f / (2.f * m));
      float2 R2 = make_float2(0.f, 0.f), R1 = Rmm;
#pragma unroll
      for (int n = m; n <= P; ++n) {
        float2 Rn;
        if (n == m) Rn = Rmm;
        else if (n == m + 1) Rn = cscale(Rmm, z);
        else {
          const float inv = 1.f / ((float)(n - m) * (float)(n + m));
          Rn = make_float2(((2 * n - 1) * z * R1.x - r2 * R2.x) * inv,
                           ((2 * n - 1) * z * R1.y - r2 * R2.y) * inv);
        }
        if (n > m) {
          R2 = R1;
          R1 = Rn;
        }
        acc[o] += q * Rn.x;  // q conj(R)
        acc[o + 1] -= q * Rn.y;
        o += 2;
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int o = 0; o < 2 * G; ++o) red[lane * RS + o] = acc[o];
  __syncwarp();
  const int base = lane - sl;  // first row of this leaf's lanes
  for (int o = sl; o < 2 * G; o += W) {
    float sum = 0.f;
    for (int l = 0; l < W; ++l) sum += red[(base + l) * RS + o];
    // group-local float o -> (m, n): columns m0.., each n = m..P, re/im
    int c = o >> 1, m = M0;
    while (c > P - m) {
      c -= P - m + 1;
      ++m;
    }
    const int n = m + c;
    reinterpret_cast<float *>(M + (size_t)leaf * NCS)[2 * cidx(n, m) + (o & 1)] = sum;
  }
  __syncwarp();
}
template <int P, int M0>
struct P2MGroups {
  static constexpr int M1 = p2m_group_end(P, M0);
  __device__ static void run(int leaf, const float4 g, float rinv, int b, int cnt,
                             const float4 *pos, float2 *M, float *red, int lane, int sl, int W) {
    p2m_group<P, M0, M1>(leaf, g, rinv, b, cnt, pos, M, red, lane, sl, W);
    if constexpr (M1 <= P) P2MGroups<P, M1>::run(leaf, g, rinv, b, cnt, pos, M, red, lane, sl, W);
  }
};
__host__ __device__ constexpr int p2m_max_group(int P) {
  int best = 0;
  for (int m0 = 0; m0 <= P; m0 = p2m_group_end(P, m0)) {
    const int c = p2m_group_coeffs(P, m0, p2m_group_end(P, m0));
    best = c > best ? c : best;
  }
  return best;
}
#ifndef P2MG_MINB
#define P2MG_MINB 4
#endif
template <int p>
__global__ void __launch_bounds__(128, P2MG_MINB) k_p2m_g(const int *__restrict__ leaves, int nleaves,
                                                         CellsView C, const float4 *__restrict__ pos,
                                                         float2 *__restrict__ M) {
  constexpr int RS = 2 * p2m_max_group(p) + 1;
  extern __shared__ float sh_p2mg[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float *red = sh_p2mg + wib * 32 * RS;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  // one leaf on W lanes: a whole warp, or a half-warp each of two leaves of <= 16 particles
  auto leaf_body = [&](int leaf, int sl, int W) {
    const float4 g = C.geo[leaf];
    const float rinv = 1.f / g.w;
    const int b = C.beg[leaf], cnt = C.cnt[leaf];
    FMM_DCHECK(FMM_IN(leaf, g_fmm_chk.rows) && b >= 0 && (long long)b + cnt <= g_fmm_chk.pos,
               "P2M leaf / particle range");
    P2MGroups<p, 0>::run(leaf, g, rinv, b, cnt, pos, M, red, lane, sl, W);
  };
  const int npairs = (nleaves + 1) / 2;
  for (int pk = gw; pk < npairs; pk += nw) {
    const int la = leaves[2 * pk], lb = 2 * pk + 1 < nleaves ? leaves[2 * pk + 1] : -1;
    if (lb >= 0 && C.cnt[la] <= 16 && C.cnt[lb] <= 16) {
      leaf_body((lane >> 4) ? lb : la, lane & 15, 16);
    } else {
      leaf_body(la, lane, 32);
      if (lb >= 0) leaf_body(lb, lane, 32);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// M2M: one CTA of 8 warps per parent cell of one level; warp w shifts child w (b/r_P is exactly
// (+-1/2, +-1/2, +-1/2)) and the 8 contributions are summed in child order in shared memory
// (deterministic). Eight warps per parent keep the few-parent top levels from being latency-bound.
template <int p>
__global__ void __launch_bounds__(256) k_m2m(int c0, int nl, CellsView C, float2 *__restrict__ M) {
  constexpr int NC = nc_of(p), NCS = nc_stride(p);
  __shared__ float2 Mc[8][NC], Rb[8][NC], part[8][NC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = blockIdx.x; k < nl; k += gridDim.x) {
    const int P = c0 + k;
    const int nch = C.nchild[P];
    if (nch == 0) continue;  // block-uniform
    if (w < nch) {
      const int4 gp = C.grid[P];
      const float rP = (float)(1 << (FMM_LEVELS - gp.w));
      const int Cc = C.child0[P] + w;
      const int4 gc = C.grid[Cc];
      for (int o = lane; o < NC; o += WARP) Mc[w][o] = M[(size_t)Cc * NCS + o];
      regular_table((gc.x - gp.x) / rP, (gc.y - gp.y) / rP, (gc.z - gp.z) / rP, p, Rb[w], lane);
      __syncwarp();
      for (int o = lane; o < NC; o += WARP) {
        const int n = c_nm[o].x, m = c_nm[o].y;
        float2 a = make_float2(0.f, 0.f);
        float sc = 1.f;
        for (int j = 0; j <= n; ++j, sc *= 0.5f) {
          const int klo = max(-j, m - (n - j)), khi = min(j, m + (n - j));
          float2 pa = make_float2(0.f, 0.f);
          for (int kk = klo; kk <= khi; ++kk)
            pa = cadd(pa, cmul(sget(Mc[w], j, kk), cconj(sget(Rb[w], n - j, m - kk))));
          a = cadd(a, cscale(pa, sc));
        }
        part[w][o] = a;
      }
    }
    __syncthreads();
    for (int o = threadIdx.x; o < NC; o += blockDim.x) {
      float2 acc = part[0][o];
      for (int c = 1; c < nch; ++c) acc = cadd(acc, part[c][o]);
      M[(size_t)P * NCS + o] = acc;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// L2L: warp per child cell of one level; adds the parent's local expansion shifted by
// e/r_P = (+-1/2, +-1/2, +-1/2).
template <int p>
__global__ void __launch_bounds__(128) k_l2l(int c0, int nl, CellsView C, float2 *__restrict__ L) {
  constexpr int NC = nc_of(p), NCS = nc_stride(p);
  __shared__ float2 sh[4][2][NC];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float2 *Lp = sh[wib][0], *Re = sh[wib][1];
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int k = gw; k < nl; k += nw) {
    const int Cc = c0 + k;
    const int P = C.parent[Cc];
    const int4 gp = C.grid[P], gc = C.grid[Cc];
    const float rP = (float)(1 << (FMM_LEVELS - gp.w));
    __syncwarp();
    for (int o = lane; o < NC; o += WARP) Lp[o] = L[(size_t)P * NCS + o];
    regular_table((gc.x - gp.x) / rP, (gc.y - gp.y) / rP, (gc.z - gp.z) / rP, p, Re, lane);
    __syncwarp();
    for (int o = lane; o < NC; o += WARP) {
      const int n = c_nm[o].x, m = c_nm[o].y;
      float2 a = make_float2(0.f, 0.f);
      for (int j = n; j <= p; ++j) {
        const int klo = max(-j, m - (j - n)), khi = min(j, m + (j - n));
        for (int kk = klo; kk <= khi; ++kk) a = cadd(a, cmul(sget(Lp, j, kk), sget(Re, j - n, kk - m)));
      }
      const float sc = ldexpf(1.f, -(n + 1));
      const float2 old = L[(size_t)Cc * NCS + o];
      L[(size_t)Cc * NCS + o] = make_float2(old.x + sc * a.x, old.y + sc * a.y);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// M2P: warp per leaf, lanes = target particles; sources = M2P lists of the leaf and its ancestors.
template <int p>
__global__ void __launch_bounds__(128) k_m2p(const int *__restrict__ leaves, int nleaves,
                                             CellsView C, ListsView Ls,
                                             const float4 *__restrict__ pos,
                                             const float2 *__restrict__ M,
                                             float4 *__restrict__ acc, int *next_leaf) {
  extern __shared__ float2 sh_m2p[];
  constexpr int NC = nc_of(p), NCS = nc_stride(p);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float2 *Ms = sh_m2p + wib * NC;
  for (;;) {
    int li = 0;
    if (lane == 0) li = atomicAdd(next_leaf, 1);  // dynamic leaf queue (load balance)
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
          __syncwarp();
          for (int o = lane; o < NC; o += WARP) Ms[o] = M[(size_t)s * NCS + o];
          __syncwarp();
          const float4 g = C.geo[s];
          const float rinv = 1.f / g.w;
          const float xx = (x.x - g.x) * rinv, yy = (x.y - g.y) * rinv, zz = (x.z - g.z) * rinv;
          const float ir2 = 1.f / (xx * xx + yy * yy + zz * zz);
          float ph = 0.f, dz = 0.f;
          float2 dxy = make_float2(0.f, 0.f);
          float2 Imm = make_float2(sqrtf(ir2), 0.f);
#pragma unroll
          for (int mm = 0; mm <= p + 1; ++mm) {
            if (mm > 0) Imm = cscale(cmul(Imm, make_float2(xx, yy)), -(2.f * mm - 1.f) * ir2);
            float2 I2 = make_float2(0.f, 0.f), I1 = Imm;
            const float w = mm ? 2.f : 1.f;
#pragma unroll
            for (int a2 = mm; a2 <= p + 1; ++a2) {
              float2 Ia;
              if (a2 == mm) Ia = Imm;
              else if (a2 == mm + 1) Ia = cscale(Imm, (2.f * mm + 1.f) * zz * ir2);
              else {
                const float c1 = (2.f * a2 - 1.f) * zz, c2 = (float)(a2 + mm - 1) * (float)(a2 - mm - 1);
                Ia = make_float2((c1 * I1.x - c2 * I2.x) * ir2, (c1 * I1.y - c2 * I2.y) * ir2);
              }
              if (a2 > mm) {
                I2 = I1;
                I1 = Ia;
              }
              // phi: M_a^mm I_a^mm (a <= p)
              if (a2 <= p && mm <= p) {
                const float2 mv = Ms[cidx(a2, mm)];
                ph += w * (mv.x * Ia.x - mv.y * Ia.y);
              }
              // d/dz: -M_n^mm I_{n+1}^mm, n = a2 - 1
              if (a2 >= 1 && a2 - 1 >= mm && a2 - 1 <= p) {
                const float2 mv = Ms[cidx(a2 - 1, mm)];
                dz -= w * (mv.x * Ia.x - mv.y * Ia.y);
              }
              // (dx + i dy): + M_n^{mm-1} I_{n+1}^{mm}, n = a2 - 1 >= mm - 1
              if (mm >= 1 && a2 - 1 <= p) {
                const float2 r = cmul(Ms[cidx(a2 - 1, mm - 1)], Ia);
                dxy.x += r.x;
                dxy.y += r.y;
              }
              // (dx + i dy): - conj(M_n^{mm+1} I_{n+1}^{mm}), n = a2 - 1 >= mm + 1
              if (a2 - 1 >= mm + 1 && a2 - 1 <= p) {
                const float2 r = cmul(Ms[cidx(a2 - 1, mm + 1)], Ia);
                dxy.x -= r.x;
                dxy.y += r.y;
              }
            }
          }
          phi += ph * rinv;
          const float r2i = rinv * rinv;
          gx += dxy.x * r2i;
          gy += dxy.y * r2i;
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

// ---------------------------------------------------------------------------------------------
// L2P + combine + un-permute: warp per leaf, lanes = particles. out = acc (+ L2P if use_local),
// written to the caller's order: phi[perm[i]], grad[3 perm[i] + a].
template <int p>
#ifndef L2P_MINB
#define L2P_MINB 5  // 96 registers, no spills (round 2: C4 downward 3.28 -> 3.17 ms vs 6 blocks at 80)
#endif
__global__ void __launch_bounds__(128, L2P_MINB) k_l2p(const int *__restrict__ leaves, int nleaves,
                                             CellsView C, const float4 *__restrict__ pos,
                                             const float2 *__restrict__ L,
                                             const float4 *__restrict__ acc,
                                             const unsigned *__restrict__ perm,
                                             float *__restrict__ phi_out,
                                             float *__restrict__ grad_out, int use_local) {
  extern __shared__ float2 sh_l2p[];
  constexpr int NC = nc_of(p), NCS = nc_stride(p);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float2 *Ll = sh_l2p + wib * NC;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int li = gw; li < nleaves; li += nw) {
    const int leaf = leaves[li];
    const int b = C.beg[leaf], cnt = C.cnt[leaf];
    FMM_DCHECK(FMM_IN(leaf, g_fmm_chk.rows) && b >= 0 && (long long)b + cnt <= g_fmm_chk.pos,
               "L2P leaf / particle range");
    const float4 g = C.geo[leaf];
    const float rinv = 1.f / g.w;
    __syncwarp();
    if (use_local)
      for (int o = lane; o < NC; o += WARP) Ll[o] = L[(size_t)leaf * NCS + o];
    __syncwarp();
    for (int c0 = 0; c0 < cnt; c0 += WARP) {
      const bool valid = c0 + lane < cnt;
      if (!valid) continue;
      const int i = b + c0 + lane;
      const float4 x = pos[i];
      float4 out = acc[i];
      if (use_local) {
        const float xx = (x.x - g.x) * rinv, yy = (x.y - g.y) * rinv, zz = (x.z - g.z) * rinv;
        const float r2 = xx * xx + yy * yy + zz * zz;
        float ph = 0.f, dz = 0.f;
        float2 dxy = make_float2(0.f, 0.f);
        float2 Rmm = make_float2(1.f, 0.f);
#pragma unroll
        for (int mm = 0; mm <= p; ++mm) {
          if (mm > 0) Rmm = cscale(cmul(Rmm, make_float2(xx, yy)), -1.f / (2.f * mm));
          float2 R2 = make_float2(0.f, 0.f), R1 = Rmm;
          const float w = mm ? 2.f : 1.f;
#pragma unroll
          for (int a2 = mm; a2 <= p; ++a2) {
            float2 Ra;
            if (a2 == mm) Ra = Rmm;
            else if (a2 == mm + 1) Ra = cscale(Rmm, zz);
            else {
              const float inv = 1.f / ((float)(a2 - mm) * (float)(a2 + mm));
              const float c1 = (2.f * a2 - 1.f) * zz;
              Ra = make_float2((c1 * R1.x - r2 * R2.x) * inv, (c1 * R1.y - r2 * R2.y) * inv);
            }
            if (a2 > mm) {
              R2 = R1;
              R1 = Ra;
            }
            {  // phi: L_a^mm R_a^mm
              const float2 lv = Ll[cidx(a2, mm)];
              ph += w * (lv.x * Ra.x - lv.y * Ra.y);
            }
            if (a2 + 1 <= p) {
              // d/dz: L_{a+1}^mm R_a^mm
              const float2 lz = Ll[cidx(a2 + 1, mm)];
              dz += w * (lz.x * Ra.x - lz.y * Ra.y);
              // (dx + i dy): + L_{a+1}^{mm-1} R_a^{mm}
              if (mm >= 1) {
                const float2 r = cmul(Ll[cidx(a2 + 1, mm - 1)], Ra);
                dxy.x += r.x;
                dxy.y += r.y;
              }
              // (dx + i dy): - conj(L_{a+1}^{mm+1} R_a^{mm})
              if (mm + 1 <= a2 + 1) {
                const float2 r = cmul(Ll[cidx(a2 + 1, mm + 1)], Ra);
                dxy.x -= r.x;
                dxy.y += r.y;
              }
            }
          }
        }
        const float r2i = rinv * rinv;
        out.x += ph * rinv;
        out.y += dxy.x * r2i;
        out.z += dxy.y * r2i;
        out.w += dz * r2i;
      }
      const size_t o = perm[i];
      phi_out[o] = out.x;
      grad_out[3 * o + 0] = out.y;
      grad_out[3 * o + 1] = out.z;
      grad_out[3 * o + 2] = out.w;
    }
  }
}

// ---------------------------------------------------------------------------------------------
static int warp_grid(int64_t nitems, int warps_per_block) {
  int64_t b = (nitems + warps_per_block - 1) / warps_per_block;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

M2LTiles make_m2l_tiles(int p) {
  M2LTiles T;
  T.ntiles = 0;
  for (int j = 0; j <= p; ++j)
    for (int k0 = 0; k0 <= j; k0 += 3) {
      const int K = (j - k0 + 1) < 3 ? (j - k0 + 1) : 3;
      T.tile[T.ntiles++] = j | (k0 << 8) | (K << 16);
    }
  return T;
}

#define FMM_DISPATCH_P(p, CALL)                                                      \
  switch (p) {                                                                       \
    case 1: { constexpr int P_ = 1; CALL; } break;                                   \
    case 2: { constexpr int P_ = 2; CALL; } break;                                   \
    case 3: { constexpr int P_ = 3; CALL; } break;                                   \
    case 4: { constexpr int P_ = 4; CALL; } break;                                   \
    case 5: { constexpr int P_ = 5; CALL; } break;                                   \
    case 6: { constexpr int P_ = 6; CALL; } break;                                   \
    case 7: { constexpr int P_ = 7; CALL; } break;                                   \
    case 8: { constexpr int P_ = 8; CALL; } break;                                   \
    case 9: { constexpr int P_ = 9; CALL; } break;                                   \
    case 10: { constexpr int P_ = 10; CALL; } break;                                 \
    case 11: { constexpr int P_ = 11; CALL; } break;                                 \
    case 12: { constexpr int P_ = 12; CALL; } break;                                 \
    case 13: { constexpr int P_ = 13; CALL; } break;                                 \
    case 14: { constexpr int P_ = 14; CALL; } break;                                 \
    case 15: { constexpr int P_ = 15; CALL; } break;                                 \
    default: { constexpr int P_ = 16; CALL; } break;                                 \
  }

void launch_p2m(int p, const int *leaves, int nleaves, CellsView C, const float4 *pos, float2 *M,
                cudaStream_t st) {
  ensure_nm_table();
  static const bool one_pass = getenv("FMM_P2M_ONEPASS") != nullptr;  // A/B: round-1 kernel
  if (one_pass) {
    FMM_DISPATCH_P(p, ({
      const size_t smem = 4 * 32 * (2 * nc_of(P_) + 1) * sizeof(float);
      fmm_smem_optin((const void *)k_p2m<P_>, smem);
      k_p2m<P_><<<warp_grid(nleaves, 4), 128, smem, st>>>(leaves, nleaves, C, pos, M);
    }));
    return;
  }
  // column groups (k_p2m_g). Measured at C4 (ncu, serialised): one-pass 2.65 ms, column groups
  // 1.90 ms; a 2-D (particle slot x column pair) lane map 3.77 ms (divergent column loops)
  FMM_DISPATCH_P(p, ({
    const size_t smem = 4 * 32 * (2 * p2m_max_group(P_) + 1) * sizeof(float);
    fmm_smem_optin((const void *)k_p2m_g<P_>, smem);
    k_p2m_g<P_><<<warp_grid((nleaves + 1) / 2, 4), 128, smem, st>>>(leaves, nleaves, C, pos, M);
  }));
}
void launch_m2m(int p, int c0, int nl, CellsView C, float2 *M, cudaStream_t st) {
  ensure_nm_table();
  const int blocks = nl < 148 * 8 ? (nl > 0 ? nl : 1) : 148 * 8;
  FMM_DISPATCH_P(p, (k_m2m<P_><<<blocks, 256, 0, st>>>(c0, nl, C, M)));
}
void launch_l2l(int p, int c0, int nl, CellsView C, float2 *L, cudaStream_t st) {
  ensure_nm_table();
  FMM_DISPATCH_P(p, (k_l2l<P_><<<warp_grid(nl, 4), 128, 0, st>>>(c0, nl, C, L)));
}
void launch_m2p(int p, const int *leaves, int nleaves, CellsView C, ListsView Ls,
                const float4 *pos, const float2 *M, float4 *acc, int *counter, cudaStream_t st) {
  ensure_nm_table();
  cudaMemsetAsync(counter, 0, sizeof(int), st);
  FMM_DISPATCH_P(p, (k_m2p<P_><<<148 * 8, 128, 4 * nc_of(P_) * sizeof(float2), st>>>(
                        leaves, nleaves, C, Ls, pos, M, acc, counter)));
}
void launch_l2p(int p, const int *leaves, int nleaves, CellsView C, const float4 *pos,
                const float2 *L, const float4 *acc, const unsigned *perm, float *phi, float *grad,
                int use_local, cudaStream_t st) {
  ensure_nm_table();
  FMM_DISPATCH_P(p, (k_l2p<P_><<<warp_grid(nleaves, 4), 128, 4 * nc_of(P_) * sizeof(float2), st>>>(
                        leaves, nleaves, C, pos, L, acc, perm, phi, grad, use_local)));
}

FMM_CHK_DEFINE_SETTER(fmm_chk_set_expansions)
