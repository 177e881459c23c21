// p2p.cu — particle-particle direct summation ("a direct summation is performed
// between all particles in the cells"; P:67 target-parallel GPU N-body).
//
//   phi_i  += sum_j q_j / r_ij          grad_i += sum_j q_j (x_j - x_i) / r_ij^3
//
// Target-parallel: one lane per target particle, sources staged through shared memory in tiles
// and read back as broadcast LDS.128; rsqrt on the MUFU pipe, the rest FP32 FMA. Pairs with r = 0
// (the particle itself, coincident particles) contribute nothing; they only occur when the source
// cell IS the target leaf, so only that case pays for the mask. Accumulation is tile-blocked:
// each tile's sum is formed separately and then added to the running total (keeps the FP32 error
// of long sums at ~1e-7, SURVEY §8(a) a12 accumulation rule).
#include "common.cuh"
#include "kernels.cuh"

#define P2P_TILE 128
#define P2P_WARPS 8

template <bool MASK>
__device__ __forceinline__ void p2p_tile(const float4 *__restrict__ sp, int ns, float4 t,
                                         float &phi, float &gx, float &gy, float &gz) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 8
  for (int j = 0; j < ns; ++j) {
    const float4 s = sp[j];
    const float dx = s.x - t.x, dy = s.y - t.y, dz = s.z - t.z;
    const float r2 = dx * dx + dy * dy + dz * dz;
    float rinv = rsqrtf(r2);
    if (MASK) rinv = r2 > 0.f ? rinv : 0.f;
    const float qr = s.w * rinv;
    const float qr3 = qr * rinv * rinv;
    a0 += qr;
    a1 += qr3 * dx;
    a2 += qr3 * dy;
    a3 += qr3 * dz;
  }
  phi += a0;
  gx += a1;
  gy += a2;
  gz += a3;
}

// Warp per (leaf, chunk of 32 targets); sources = P2P lists of the leaf and all its ancestors
// (a P2P pair with a non-leaf target applies to every particle under it).
__global__ void __launch_bounds__(P2P_WARPS * 32) k_p2p_leaves(const int *__restrict__ leaves,
                                                               int nleaves, CellsView C,
                                                               ListsView Ls,
                                                               const float4 *__restrict__ pos,
                                                               float4 *__restrict__ acc) {
  __shared__ float4 sh[P2P_WARPS][P2P_TILE];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float4 *sp = sh[wib];
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int li = gw; li < nleaves; li += nw) {
    const int leaf = leaves[li];
    const int tb = C.beg[leaf], tn = C.cnt[leaf];
    for (int c0 = 0; c0 < tn; c0 += WARP) {
      const bool valid = c0 + lane < tn;
      const int i = tb + c0 + lane;
      const float4 t = valid ? pos[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      float phi = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
      for (int a = leaf; a >= 0; a = C.parent[a]) {
        const int off = Ls.off[2][a], ncell = Ls.cnt[2][a];
        for (int e = 0; e < ncell; ++e) {
          const int s = Ls.src[2][off + e];
          const int sb = C.beg[s], sn = C.cnt[s];
          const bool self = (s == leaf);
          for (int j0 = 0; j0 < sn; j0 += P2P_TILE) {
            const int nt = min(P2P_TILE, sn - j0);
            __syncwarp();
            for (int j = lane; j < nt; j += WARP) sp[j] = pos[sb + j0 + j];
            __syncwarp();
            if (self)
              p2p_tile<true>(sp, nt, t, phi, gx, gy, gz);
            else
              p2p_tile<false>(sp, nt, t, phi, gx, gy, gz);
          }
        }
      }
      if (valid) acc[i] = make_float4(phi, gx, gy, gz);
    }
  }
}

// FMM_DIRECT: all N targets against all N sources in caller order (no tree). Block of 256 targets,
// source tiles of 256 staged by the whole block.
__global__ void __launch_bounds__(256) k_p2p_direct(int64_t n, const float4 *__restrict__ pos,
                                                    float *__restrict__ phi_out,
                                                    float *__restrict__ grad_out) {
  __shared__ float4 sh[256];
  for (int64_t base = (int64_t)blockIdx.x * 256; base < n; base += (int64_t)gridDim.x * 256) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < n;
    const float4 t = valid ? pos[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    float phi = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
    for (int64_t j0 = 0; j0 < n; j0 += 256) {
      const int nt = (int)min((int64_t)256, n - j0);
      __syncthreads();
      if (threadIdx.x < nt) sh[threadIdx.x] = pos[j0 + threadIdx.x];
      __syncthreads();
      p2p_tile<true>(sh, nt, t, phi, gx, gy, gz);
    }
    if (valid) {
      phi_out[i] = phi;
      grad_out[3 * i + 0] = gx;
      grad_out[3 * i + 1] = gy;
      grad_out[3 * i + 2] = gz;
    }
  }
}

void launch_p2p_leaves(const int *leaves, int nleaves, CellsView C, ListsView Ls,
                       const float4 *pos, float4 *acc, cudaStream_t st) {
  int64_t b = (nleaves + P2P_WARPS - 1) / P2P_WARPS;
  if (b > 148 * 8) b = 148 * 8;
  if (b < 1) b = 1;
  k_p2p_leaves<<<(int)b, P2P_WARPS * 32, 0, st>>>(leaves, nleaves, C, Ls, pos, acc);
}

void launch_p2p_direct(int64_t n, const float4 *pos, float *phi, float *grad, cudaStream_t st) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 64) b = 148 * 64;
  if (b < 1) b = 1;
  k_p2p_direct<<<(int)b, 256, 0, st>>>(n, pos, phi, grad);
}
