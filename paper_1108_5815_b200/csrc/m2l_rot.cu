// m2l_rot.cu — rotation-based O(p^3) M2L (PAPER.md:122 / P:153 / P:169 name
// the choice of translation scheme, P:205 the O(p^4) cell-cell kernel it replaces).
//
// The translation of a class (level difference, centre offset) is factorised as
//     rotate the source multipole so that the offset d points along +z,
//     translate along z (the only non-zero irregular harmonics on the axis are I_a^0(|d| z) =
//     a! / |d|^(a+1): L'_j^k = (-1)^(j+k) sum_{n >= |k|} M'_n^k rho^n (n+j)! / |u|^(n+j+1)),
//     rotate the local expansion back,
// in the power-of-two scaled form of the other M2L paths (u = d / r_t, rho = r_s / r_t). With
// Q = Ry(-theta) Rz(-phi) (Q d = |d| z), the regular harmonics of this build's convention rotate
// as R_n^m(Q y) = sum_m' A^n_{m m'} R_n^m'(y), A^n_{m m'} = d^n_{m m'}(-theta) c_m' / c_m
// e^{-i m' phi}, c_m = sqrt((n - m)! (n + m)!) (d = Wigner's small-d, explicit sum in FP64), so
//     M'_n = conj(A^n) M_n,   L_j = L'_j A^j
// (checked against the direct translation to 1e-15 in FP64 while deriving, and against the
// oracle's direct M2L through the whole method in tests/test_gpu_rotation.py). Per degree the
// rotations are real (2n+1) x (2n+1) maps of the real degrees of freedom of a real field (dof
// order of common.cuh), built once per class: sum_n (2n+1)^2 + the axial table instead of the
// (p+1)^4 dense class matrix.
//
// Execution: the pairs are the class-sorted work items of the class GEMM path (m2l.cu); one CTA
// per item loads the item's class operators into shared memory and its 8 warps take one pair at
// a time, the lanes over output dofs (fwd rotation, axial, back rotation: ~3 (p+1)^3 MACs per
// pair instead of (p+1)^4). Results go into the pair's Y slot (dof order, deterministic mode) or
// are added into the target's local expansion with float reductions in L2 (accumulate mode).
#include "common.cuh"
#include "kernels.cuh"

namespace {

__host__ __device__ constexpr int rot_block_floats(int p) {  // sum_{n <= p} (2n+1)^2
  return (p + 1) * (2 * p + 1) * (2 * p + 3) / 3;
}
__host__ __device__ constexpr int rot_class_floats(int p) {  // Rf | Rb | Z, 16-byte rows
  return (2 * rot_block_floats(p) + (p + 1) * (p + 1) + 3) & ~3;
}
__device__ __forceinline__ int rot_base(int n) { return n * (2 * n - 1) * (2 * n + 1) / 3; }  // sum_{n' < n}

__device__ double dfact(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= i;
  return f;
}
// Wigner small-d d^n_{mp m}(beta), explicit sum (FP64: ~1e-12 for n <= 16)
__device__ double wigner_d(int n, int mp, int m, double beta) {
  const double c = cos(0.5 * beta), s = sin(0.5 * beta);
  const double pre = sqrt(dfact(n + mp)) * sqrt(dfact(n - mp)) * sqrt(dfact(n + m)) * sqrt(dfact(n - m));
  double tot = 0.0;
  for (int k = 0; k <= 2 * n; ++k) {
    const int a1 = n + m - k, a3 = mp - m + k, a4 = n - mp - k;
    if (a1 < 0 || a3 < 0 || a4 < 0) continue;
    const double t = pre / (dfact(a1) * dfact(k) * dfact(a3) * dfact(a4)) *
                     pow(c, 2 * n + m - mp - 2 * k) * pow(s, mp - m + 2 * k);
    tot += ((mp - m + k) & 1) ? -t : t;
  }
  return tot;
}

__device__ __forceinline__ int dof_degree(int d) {  // floor(sqrt(d)), exact for d < 2^22
  int n = (int)sqrtf((float)d);
  n += (n + 1) * (n + 1) <= d;
  n -= n * n > d;
  return n;
}
// dof d -> float index in an (m >= 0, complex) row (common.cuh dof_to_float, closed form)
__device__ __forceinline__ int dof_float(int d) {
  const int n = dof_degree(d), r = d - n * n;
  if (r == 0) return n * (n + 1);
  const int m = (r + 1) >> 1;
  return 2 * (n * (n + 1) / 2 + m) + ((r + 1) & 1);
}
// dof (degree-local offset r, 0 .. 2n) -> (m, part): r = 0 (0, Re); r = 2m - 1 (m, Re); r = 2m (m, Im)
__device__ __forceinline__ void r_to_mp(int r, int &m, int &part) {
  m = (r + 1) >> 1;
  part = r ? ((r + 1) & 1) : 0;
}

}  // namespace

bool m2l_rot_supported(int p) { return p >= 1 && p <= FMM_PMAX; }
size_t m2l_rot_class_floats(int p) { return (size_t)rot_class_floats(p); }

// one block per class (grid-stride): Rf[n][in][out], Rb[n][in][out], Z[j][n]
__global__ void __launch_bounds__(256) k_m2l_rot_build(int p, const int *__restrict__ counters,
                                                       const unsigned *__restrict__ class_rep,
                                                       const int *__restrict__ pair_t,
                                                       const unsigned *__restrict__ src, CellsView C,
                                                       float *__restrict__ R) {
  const int ng = counters[3];
  const int RB = rot_block_floats(p);
  for (int gid = blockIdx.x; gid < ng; gid += gridDim.x) {
    const int rep = class_rep[gid];
    const int4 gt = C.grid[pair_t[rep]], gs = C.grid[src[rep]];
    const double rt = (double)(1 << (FMM_LEVELS - gt.w));
    const double ux = (gt.x - gs.x) / rt, uy = (gt.y - gs.y) / rt, uz = (gt.z - gs.z) / rt;
    const double ur = sqrt(ux * ux + uy * uy + uz * uz);
    const double theta = acos(fmin(1.0, fmax(-1.0, uz / ur))), phi = atan2(uy, ux);
    const double beta = -theta, gamma = -phi;
    const double rho = ldexp(1.0, gt.w - gs.w);
    float *Rf = R + (size_t)gid * rot_class_floats(p), *Rb = Rf + RB, *Z = Rb + RB;
    // rotation blocks: entry (n, in, out) -> thread
    for (int e = threadIdx.x; e < RB; e += blockDim.x) {
      int n = 0;
      while (rot_base(n + 1) <= e) ++n;
      const int w = 2 * n + 1, loc = e - rot_base(n), in = loc / w, out = loc - in * w;
      int mi, pi, mo, po;
      r_to_mp(in, mi, pi);
      r_to_mp(out, mo, po);
      const double cf = sqrt(dfact(n - mo) * dfact(n + mo));
      // A[m][m'] = d(m, m') c_m' / c_m e^{i m' gamma}
      auto A = [&](int m, int mp, double &re, double &im) {
        const double v = wigner_d(n, m, mp, beta) * sqrt(dfact(n - mp) * dfact(n + mp)) /
                         sqrt(dfact(n - m) * dfact(n + m));
        re = v * cos(mp * gamma);
        im = v * sin(mp * gamma);
      };
      // input basis vector X: X^mi = 1 or i; X^-mi = (-1)^mi conj(X^mi) (mi > 0)
      const double xr = pi ? 0.0 : 1.0, xi = pi ? 1.0 : 0.0;
      const double sgn = (mi & 1) ? -1.0 : 1.0;
      // forward: out^mo = sum_m' conj(A[mo][m']) X^m'
      double fr = 0.0, fi = 0.0, ar, ai;
      A(mo, mi, ar, ai);
      fr += ar * xr + ai * xi;  // conj(a) x = (ar - i ai)(xr + i xi)
      fi += ar * xi - ai * xr;
      if (mi > 0) {
        A(mo, -mi, ar, ai);
        const double yr = sgn * xr, yi = -sgn * xi;
        fr += ar * yr + ai * yi;
        fi += ar * yi - ai * yr;
      }
      Rf[rot_base(n) + in * w + out] = (float)(po ? fi : fr);
      // back: out^ko = sum_k Y^k A[k][ko], Y^mi = X^mi, Y^-mi = (-1)^mi conj(Y^mi)
      double br = 0.0, bi = 0.0;
      A(mi, mo, ar, ai);
      br += xr * ar - xi * ai;
      bi += xr * ai + xi * ar;
      if (mi > 0) {
        A(-mi, mo, ar, ai);
        const double yr = sgn * xr, yi = -sgn * xi;
        br += yr * ar - yi * ai;
        bi += yr * ai + yi * ar;
      }
      Rb[rot_base(n) + in * w + out] = (float)(po ? bi : br);
      (void)cf;
    }
    // axial: Z[j][n] = (-1)^j rho^n (n + j)! / |u|^(n + j + 1)   (the (-1)^k is applied per k)
    for (int e = threadIdx.x; e < (p + 1) * (p + 1); e += blockDim.x) {
      const int j = e / (p + 1), n = e - j * (p + 1);
      const double v = pow(rho, n) * dfact(n + j) / pow(ur, n + j + 1);
      Z[e] = (float)((j & 1) ? -v : v);
    }
  }
}

// Persistent CTAs over the class-sorted work items (x = first sorted position, y = count,
// w = class); 8 warps, one pair per warp at a time.
#define ROT_WARPS 8
__global__ void __launch_bounds__(ROT_WARPS * 32) k_m2l_rot(int p, const int4 *__restrict__ items,
                                                            const int *__restrict__ counters,
                                                            int *queue,
                                                            const unsigned *__restrict__ yslot,
                                                            const unsigned *__restrict__ ssrc,
                                                            const float *__restrict__ R,
                                                            const float *__restrict__ M,
                                                            float *__restrict__ Y,
                                                            float *__restrict__ Lacc) {
  extern __shared__ __align__(16) float sh_rot[];
  const int KD = dof_of(p), RB = rot_block_floats(p), RCF = rot_class_floats(p);
  const int MROW = 2 * nc_stride(p), YSD = dof_stride(p);
  float *cls = sh_rot;                                   // Rf | Rb | Z of the item's class
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float *vin = sh_rot + RCF + warp * 3 * 256, *vmid = vin + 256, *vax = vmid + 256;
  const float *Rf = cls, *Rb = cls + RB, *Z = cls + 2 * RB;
  __shared__ int item_sh;
  const int nitems = counters[1];
  for (;;) {
    __syncthreads();  // the previous item's class data is no longer read
    if (threadIdx.x == 0) item_sh = atomicAdd(queue, 1);
    __syncthreads();
    const int it = item_sh;
    if (it >= nitems) break;
    const int4 item = items[it];
    const float4 *g4 = reinterpret_cast<const float4 *>(R + (size_t)item.w * RCF);
    for (int i = threadIdx.x; i < RCF / 4; i += blockDim.x) reinterpret_cast<float4 *>(cls)[i] = g4[i];
    __syncthreads();
    for (int pr = warp; pr < item.y; pr += ROT_WARPS) {
      const int pos = item.x + pr;
      const unsigned s = ssrc[pos], ys = yslot[pos];
      const float *Mrow = M + (size_t)s * MROW;
      for (int d = lane; d < KD; d += 32) vin[d] = Mrow[dof_float(d)];
      __syncwarp();
      // forward rotation, per degree
      for (int d = lane; d < KD; d += 32) {
        const int n = dof_degree(d), w = 2 * n + 1, o = d - n * n;
        const float *Rn = Rf + rot_base(n) + o;
        const float *vn = vin + n * n;
        float acc = 0.f;
        for (int i = 0; i < w; ++i) acc = fmaf(Rn[i * w], vn[i], acc);
        vmid[d] = acc;
      }
      __syncwarp();
      // axial translation along z: L'_(j,k,part) = (-1)^k sum_{n >= k} Z[j][n] M'_(n,k,part)
      for (int d = lane; d < KD; d += 32) {
        const int j = dof_degree(d), r = d - j * j;
        const int k = (r + 1) >> 1, off = r;  // M'_(n,k,part) sits at n^2 + r (same r for all n)
        const float *zj = Z + j * (p + 1);
        float acc = 0.f;
        for (int n = k; n <= p; ++n) acc = fmaf(zj[n], vmid[n * n + off], acc);
        vax[d] = (k & 1) ? -acc : acc;
      }
      __syncwarp();
      // back rotation; the result in dof order (Y slot) or in float order for the reductions
      for (int d = lane; d < KD; d += 32) {
        const int n = dof_degree(d), w = 2 * n + 1, o = d - n * n;
        const float *Rn = Rb + rot_base(n) + o;
        const float *vn = vax + n * n;
        float acc = 0.f;
        for (int i = 0; i < w; ++i) acc = fmaf(Rn[i * w], vn[i], acc);
        if (Lacc) vin[dof_float(d)] = acc;
        else Y[(size_t)ys * YSD + d] = acc;
      }
      if (Lacc) {
        __syncwarp();
        // (the Im part of each m = 0 coefficient is zero in every row)
        for (int n = lane; n <= p; n += 32) vin[n * (n + 1) + 1] = 0.f;
        for (int f = 2 * nc_of(p); f < MROW; ++f)
          if (lane == 0) vin[f] = 0.f;
        __syncwarp();
        float *dst = Lacc + (size_t)ys * MROW;
        for (int q4 = lane; q4 < MROW / 4; q4 += 32) {
          const float4 v = reinterpret_cast<const float4 *>(vin)[q4];
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * q4), "f"(v.x),
                       "f"(v.y), "f"(v.z), "f"(v.w)
                       : "memory");
        }
      }
      __syncwarp();
    }
  }
}

cudaError_t m2l_rot_build(int p, const M2LWork &W, int ngclass, float *R, cudaStream_t st) {
  if (ngclass <= 0) return cudaSuccess;
  k_m2l_rot_build<<<std::min(ngclass, 148 * 8), 256, 0, st>>>(p, W.counters, W.class_rep, W.pair_t,
                                                              W.src, W.C, R);
  return cudaGetLastError();
}
cudaError_t m2l_rot_apply(int p, const M2LWork &W, const float *R, const float2 *M,
                          cudaStream_t st, float2 *Lacc) {
  const size_t smem = sizeof(float) * ((size_t)rot_class_floats(p) + (size_t)ROT_WARPS * 3 * 256);
  fmm_smem_optin((const void *)k_m2l_rot, smem);
  const int grid = fmm_resident_blocks((const void *)k_m2l_rot, ROT_WARPS * 32, smem);
  cudaMemsetAsync(W.counters + 4, 0, sizeof(int), st);
  k_m2l_rot<<<grid, ROT_WARPS * 32, smem, st>>>(p, W.items, W.counters, W.counters + 4,
                                                Lacc ? W.stgt : W.sidx, W.ssrc, R,
                                                reinterpret_cast<const float *>(M), W.Y,
                                                reinterpret_cast<float *>(Lacc));
  return cudaGetLastError();
}
