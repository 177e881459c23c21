// dist.cu — device kernels of the multi-GPU evaluation ("domain
// decomposition ... local essential tree"). The host pipeline is in fmm_api.cu (dist_build_tree,
// dist_let, dist_return); the collectives are in comm.cu.
//
// Decomposition used here:
//   * the GLOBAL tree is built on every rank without moving particles: per level, each rank
//     binary-searches its own sorted keys and one allreduce sums the child bounds (tree.cu k_split);
//   * ranks own contiguous runs of global leaves (Morton order), balanced by particle count;
//   * cells whose particle range crosses a rank boundary ("straddling") get their multipoles by an
//     allreduce of the per-rank partial sums (M2M is linear);
//   * every rank traverses the global tree for its own targets, then requests exactly the remote
//     multipoles (M2L / M2P sources) and particle ranges (P2P sources) its lists name: a
//     receiver-driven local essential tree.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.cuh"

__global__ void k_iota(unsigned *a, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[i] = (unsigned)i;
}

__global__ void k_gather4(const float4 *__restrict__ src, const unsigned *__restrict__ perm, int n,
                          float4 *__restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}

// Rank boundaries at leaf starts: boundary r (1 <= r < R) = first particle of the leaf that holds
// global sorted index floor(r * N / R); K[r] = that leaf's first Morton key.
__global__ void k_partition(const int *__restrict__ leaves, int nleaves, CellsView C,
                            const uint64_t *__restrict__ prefix, int N, int R, int *off,
                            uint64_t *K) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    off[0] = 0;
    K[0] = 0;
    off[R] = N;
    K[R] = ~0ull;
  }
  if (i >= nleaves) return;
  const int c = leaves[i];
  const int b = C.beg[c], n = C.cnt[c];
  for (int r = 1; r < R; ++r) {
    const int t = (int)(((int64_t)r * N) / R);
    if (b <= t && t < b + n) {
      off[r] = b;
      const int lev = C.grid[c].w;
      K[r] = prefix[c] << (3 * (FMM_LEVELS - lev));
    }
  }
}

// lb[r] = number of local sorted keys < K[r]
__global__ void k_key_bounds(const uint64_t *__restrict__ keys, int n, const uint64_t *__restrict__ K,
                             int R, int *lb) {
  const int r = threadIdx.x;
  if (r > R) return;
  const uint64_t k = K[r];
  int l = 0, h = n;
  if (r == R) l = n;
  while (l < h) {
    const int m = (l + h) >> 1;
    if (keys[m] < k) l = m + 1;
    else h = m;
  }
  lb[r] = l;
}

// own leaves: lo <= begin < hi (ranks own whole leaves)
__global__ void k_range_leaf_flags(int ncells, CellsView C, int lo, int hi, int *flag) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const int b = C.beg[c];
  flag[c] = C.nchild[c] == 0 && b >= lo && b < hi;
}

__device__ __forceinline__ bool straddles(int b, int n, const int *off, int R) {
  for (int r = 1; r < R; ++r)
    if (b < off[r] && off[r] < b + n) return true;
  return false;
}

__global__ void k_straddle_flags(int ncells, CellsView C, const int *__restrict__ off, int R,
                                 int *flag) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  flag[c] = straddles(C.beg[c], C.cnt[c], off, R);
}

// one warp per row
__global__ void k_rows(const float2 *__restrict__ src, float2 *__restrict__ dst, int stride,
                       const unsigned *__restrict__ ids, int n, int to_ids) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = w; i < n; i += nw) {
    const size_t a = (size_t)ids[i] * stride, b = (size_t)i * stride;
    for (int e = lane; e < stride; e += 32) {
      if (to_ids) dst[a + e] = src[b + e];
      else dst[b + e] = src[a + e];
    }
  }
}

// Remote data named by this rank's lists. A multipole is locally complete when the cell lies in
// [lo, hi) or straddles (allreduced); a P2P source range needs the particles outside [lo, hi).
__global__ void k_need_flags(ListsView Ls, int n_m2l, int n_m2p, int n_p2p, CellsView C,
                             const int *__restrict__ strad, int lo, int hi, int *needM, int *needP) {
  const int total = n_m2l + n_m2p + n_p2p;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    if (e < n_m2l + n_m2p) {
      const unsigned s = e < n_m2l ? Ls.src[0][e] : Ls.src[1][e - n_m2l];
      const int b = C.beg[s], n = C.cnt[s];
      if (!(b >= lo && b + n <= hi) && !strad[s]) needM[s] = 1;
    } else {
      const int k = e - n_m2l - n_m2p;
      const int2 r = Ls.p2p_rng[k];
      if (!(r.x >= lo && r.x + r.y <= hi)) needP[Ls.src[2][k]] = 1;
    }
  }
}

__device__ __forceinline__ int owner_of(int b, const int *off, int R) {
  int r = 0;
  while (r + 1 < R && off[r + 1] <= b) ++r;
  return r;
}

__global__ void k_owner_of_cells(const unsigned *__restrict__ ids, int n, CellsView C,
                                 const int *__restrict__ off, int R, unsigned *owner) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) owner[i] = (unsigned)owner_of(C.beg[ids[i]], off, R);
}

// pieces of P2P source ranges outside this rank: one per overlapped remote rank
__global__ void k_piece_count(const unsigned *__restrict__ ids, int n, CellsView C,
                              const int *__restrict__ off, int R, int me, int *cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = C.beg[ids[i]], e = b + C.cnt[ids[i]];
  int k = 0;
  for (int r = 0; r < R; ++r)
    if (r != me && max(b, off[r]) < min(e, off[r + 1])) ++k;
  cnt[i] = k;
}
__global__ void k_piece_write(const unsigned *__restrict__ ids, int n, CellsView C,
                              const int *__restrict__ off, int R, int me, const int *__restrict__ excl,
                              unsigned *owner, unsigned *pidx, int2 *rng) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = C.beg[ids[i]], e = b + C.cnt[ids[i]];
  int k = excl[i];
  for (int r = 0; r < R; ++r) {
    const int lo = max(b, off[r]), hi = min(e, off[r + 1]);
    if (r != me && lo < hi) {
      owner[k] = (unsigned)r;
      pidx[k] = (unsigned)k;
      rng[k] = make_int2(lo, hi);
      ++k;
    }
  }
}

__global__ void k_gather_int2(const int2 *__restrict__ src, const unsigned *__restrict__ idx, int n,
                              int2 *__restrict__ dst, int *__restrict__ size) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int2 r = src[idx[i]];
  dst[i] = r;
  size[i] = r.y - r.x;
}

__global__ void k_range_sizes(const int2 *__restrict__ rng, int n, int *__restrict__ size) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) size[i] = rng[i].y - rng[i].x;
}

__global__ void k_owner_hist(const unsigned *__restrict__ owner, int n, int *counts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&counts[owner[i]], 1);
}

// particles of ranges [lo, hi) (global sorted index) <-> a packed buffer at roff[i]; warp per range
__global__ void k_range_copy(float4 *__restrict__ pos, const int2 *__restrict__ rng,
                             const int *__restrict__ roff, int n, float4 *__restrict__ buf,
                             int to_pos) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = w; i < n; i += nw) {
    const int2 r = rng[i];
    const int o = roff[i];
    for (int j = lane; j < r.y - r.x; j += 32) {
      if (to_pos) pos[r.x + j] = buf[o + j];
      else buf[o + j] = pos[r.x + j];
    }
  }
}

__global__ void k_scatter_results(const float *__restrict__ rphi, const float *__restrict__ rgrad,
                                  const unsigned *__restrict__ perm, int n, float *__restrict__ phi,
                                  float *__restrict__ grad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned o = perm[i];
    phi[o] = rphi[i];
    grad[3 * (size_t)o] = rgrad[3 * (size_t)i];
    grad[3 * (size_t)o + 1] = rgrad[3 * (size_t)i + 1];
    grad[3 * (size_t)o + 2] = rgrad[3 * (size_t)i + 2];
  }
}

// ---- launchers ----------------------------------------------------------------------------------
static int blocks_for(int64_t n, int bs) {
  int64_t g = (n + bs - 1) / bs;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

void launch_iota(unsigned *a, int n, cudaStream_t st) {
  if (n > 0) k_iota<<<blocks_for(n, 256), 256, 0, st>>>(a, n);
}
void launch_gather4(const float4 *src, const unsigned *perm, int n, float4 *dst, cudaStream_t st) {
  if (n > 0) k_gather4<<<blocks_for(n, 256), 256, 0, st>>>(src, perm, n, dst);
}
void launch_partition(const int *leaves, int nleaves, CellsView C, const uint64_t *prefix, int N,
                      int R, int *off, uint64_t *K, cudaStream_t st) {
  k_partition<<<blocks_for(std::max(nleaves, 1), 256), 256, 0, st>>>(leaves, nleaves, C, prefix,
                                                                      N, R, off, K);
}
void launch_key_bounds(const uint64_t *keys, int n, const uint64_t *K, int R, int *lb,
                       cudaStream_t st) {
  k_key_bounds<<<1, 64, 0, st>>>(keys, n, K, R, lb);
}
void launch_range_leaf_flags(int ncells, CellsView C, int lo, int hi, int *flag, cudaStream_t st) {
  k_range_leaf_flags<<<blocks_for(ncells, 256), 256, 0, st>>>(ncells, C, lo, hi, flag);
}
void launch_straddle_flags(int ncells, CellsView C, const int *off, int R, int *flag,
                           cudaStream_t st) {
  k_straddle_flags<<<blocks_for(ncells, 256), 256, 0, st>>>(ncells, C, off, R, flag);
}
void launch_rows(const float2 *src, float2 *dst, int stride, const unsigned *ids, int n,
                 bool to_ids, cudaStream_t st) {
  if (n > 0) k_rows<<<blocks_for((int64_t)n * 32, 256), 256, 0, st>>>(src, dst, stride, ids, n, to_ids);
}
void launch_need_flags(ListsView Ls, int n_m2l, int n_m2p, int n_p2p, CellsView C,
                       const int *strad, int lo, int hi, int *needM, int *needP, cudaStream_t st) {
  const int total = n_m2l + n_m2p + n_p2p;
  if (total > 0)
    k_need_flags<<<blocks_for(total, 256), 256, 0, st>>>(Ls, n_m2l, n_m2p, n_p2p, C, strad, lo, hi,
                                                         needM, needP);
}
void launch_owner_of_cells(const unsigned *ids, int n, CellsView C, const int *off, int R,
                           unsigned *owner, cudaStream_t st) {
  if (n > 0) k_owner_of_cells<<<(n + 255) / 256, 256, 0, st>>>(ids, n, C, off, R, owner);
}
void launch_piece_count(const unsigned *ids, int n, CellsView C, const int *off, int R, int me,
                        int *cnt, cudaStream_t st) {
  if (n > 0) k_piece_count<<<(n + 255) / 256, 256, 0, st>>>(ids, n, C, off, R, me, cnt);
}
void launch_piece_write(const unsigned *ids, int n, CellsView C, const int *off, int R, int me,
                        const int *excl, unsigned *owner, unsigned *pidx, int2 *rng,
                        cudaStream_t st) {
  if (n > 0)
    k_piece_write<<<(n + 255) / 256, 256, 0, st>>>(ids, n, C, off, R, me, excl, owner, pidx, rng);
}
void launch_gather_int2(const int2 *src, const unsigned *idx, int n, int2 *dst, int *size,
                        cudaStream_t st) {
  if (n > 0) k_gather_int2<<<(n + 255) / 256, 256, 0, st>>>(src, idx, n, dst, size);
}
void launch_range_sizes(const int2 *rng, int n, int *size, cudaStream_t st) {
  if (n > 0) k_range_sizes<<<(n + 255) / 256, 256, 0, st>>>(rng, n, size);
}
void launch_owner_hist(const unsigned *owner, int n, int *counts, cudaStream_t st) {
  if (n > 0) k_owner_hist<<<(n + 255) / 256, 256, 0, st>>>(owner, n, counts);
}
void launch_range_copy(float4 *pos, const int2 *rng, const int *roff, int n, float4 *buf,
                       bool to_pos, cudaStream_t st) {
  if (n > 0)
    k_range_copy<<<blocks_for((int64_t)n * 32, 256), 256, 0, st>>>(pos, rng, roff, n, buf, to_pos);
}
void launch_scatter_results(const float *rphi, const float *rgrad, const unsigned *perm, int n,
                            float *phi, float *grad, cudaStream_t st) {
  if (n > 0) k_scatter_results<<<blocks_for(n, 256), 256, 0, st>>>(rphi, rgrad, perm, n, phi, grad);
}
cudaError_t sort_owner_pairs(void *tmp, size_t &tmp_bytes, const unsigned *kin, unsigned *kout,
                             const unsigned *vin, unsigned *vout, int n, int bits,
                             cudaStream_t st) {
  return cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, vin, vout, n, 0, bits, st);
}
