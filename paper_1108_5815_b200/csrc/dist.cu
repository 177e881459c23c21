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

#include <climits>

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


// ---- sender-side local essential tree (PAPER.md:89, P:114 overlap) --------
// Every rank decides, from the global skeleton alone, what every other rank's traversal might read
// from it, right after its upward sweep -- so the exchange runs while the local traversal does.
// Geometry is in doubled-grid integer units (exact): centre c~, half-width r~ = 2^(21 - level).
//
// Receiver r's traversal splits a source cell S only in a pair (T, S) whose MAC fails with
// r_T <= r_S (or T a leaf). T intersects r's particle range, so T contains one of r's leaves L:
// either T is inside L (c_T in B_r, the box of r's leaf cubes) or L inside T (c_T within sqrt(3) r_T
// of B_r). With R(T, S) < (r_T + r_S) / theta this gives the conservative opening test
//     dist(c_S, B_r) < max(2 r_S / theta + sqrt(3) r_S, (rleafmax_r + r_S) / theta)
// (the second term: a leaf T with r_T > r_S is one of r's own leaves, c_T in B_r). The test is
// monotone up the tree (a parent is open whenever a child is), so the cells r can ever touch are
// the children of open cells ("visible"). r needs the multipole of every visible cell that is mine
// (not straddling: those are allreduced everywhere) and the particles (my part of the range) of
// every visible cell it might P2P with: an open leaf (a rejected leaf-leaf pair), or -- hybrid
// mode -- any visible cell with t_pp n_S < t_mp (an accepted pair takes P2P only then).
// box[LETB r + 0..8] = min x, y, z, max x, y, z of r's leaf cubes, largest leaf half-width,
// smallest leaf particle count, largest half-width of r's target cells with <= kmax particles
#define LETB 9
__global__ void k_let_box_init(int R, int *box) {
  const int i = threadIdx.x;
  if (i < R * LETB) {
    const int k = i % LETB;
    box[i] = k < 3 || k == 7 ? INT_MAX : (k < 6 ? INT_MIN : 0);
  }
}
// slot 8: target cells of r (cells intersecting r's range) that could take a P2P by cost
__global__ void k_let_small_cells(int ncells, CellsView C, const int *__restrict__ off, int R,
                                  int kmax, int *box) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const int b = C.beg[c], n = C.cnt[c];
  if (n > kmax) return;
  const int h = 1 << (FMM_LEVELS - C.grid[c].w);
  for (int r = 0; r < R; ++r)
    if (b < off[r + 1] && b + n > off[r]) atomicMax(box + LETB * r + 8, h);
}
__global__ void k_let_boxes(const int *__restrict__ leaves, int nleaves, CellsView C,
                            const int *__restrict__ off, int R, int *box) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nleaves) return;
  const int c = leaves[i];
  const int r = owner_of(C.beg[c], off, R);
  const int4 g = C.grid[c];
  const int h = 1 << (FMM_LEVELS - g.w);
  int *b = box + LETB * r;
  atomicMin(b + 7, C.cnt[c]);
  atomicMin(b + 0, g.x - h);
  atomicMin(b + 1, g.y - h);
  atomicMin(b + 2, g.z - h);
  atomicMax(b + 3, g.x + h);
  atomicMax(b + 4, g.y + h);
  atomicMax(b + 5, g.z + h);
  atomicMax(b + 6, h);
}
// bit r of open[c]: receiver r's traversal may split c. Bit r of near[c]: c lies close enough
// to r for an ACCEPTED pair (T, c) of r's traversal to exist with T small enough for a P2P by
// cost: the pair's parent pair (T0, S0) failed the MAC and the split cell is the larger, so
// R(T, c) < (r_T0 + r_S0) / theta + sqrt(3) max(r_T0, r_S0) with the split radius twice the
// child's; with c_T within sqrt(3) r_T of B_r this bounds dist(c, B_r) by
// max(4 r_c / theta + 4 sqrt(3) r_c, 4 r_big / theta + 3 sqrt(3) r_big), r_big = slot 8.
__global__ void k_let_open(int ncells, CellsView C, const int *__restrict__ box, int R, int me,
                           double theta, unsigned *open, unsigned *near) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const int4 g = C.grid[c];
  const double rs = (double)(1 << (FMM_LEVELS - g.w));
  unsigned m = 0, nm = 0;
  for (int r = 0; r < R; ++r) {
    const int *b = box + LETB * r;
    if (r == me || b[6] == 0) continue;  // (a rank without leaves never traverses)
    const long long dx = max(0, max(b[0] - g.x, g.x - b[3]));
    const long long dy = max(0, max(b[1] - g.y, g.y - b[4]));
    const long long dz = max(0, max(b[2] - g.z, g.z - b[5]));
    const double d = sqrt((double)(dx * dx + dy * dy + dz * dz));
    const double thr = fmax(2.0 * rs / theta + 1.7320508075688772 * rs, ((double)b[6] + rs) / theta);
    if (d < thr * (1.0 + 1e-9) + 1.0) m |= 1u << r;
    const double rb = (double)b[8];
    const double thn = fmax(4.0 * rs / theta + 6.928203230275509 * rs,
                            4.0 * rb / theta + 5.196152422706632 * rb);
    if (d < thn * (1.0 + 1e-9) + 1.0) nm |= 1u << r;
  }
  open[c] = m;
  near[c] = nm;
}
// flags[(kind * R + r) * ncells + c], kind 0 = multipole, 1 = particles
__global__ void k_let_flags(int ncells, CellsView C, const unsigned *__restrict__ open,
                            const unsigned *__restrict__ near, const int *__restrict__ box,
                            const int *__restrict__ off, int R, int me, double t_pp, double t_mp,
                            double t_ml, int *flags) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const int b = C.beg[c], n = C.cnt[c];
  const int lo = off[me], hi = off[me + 1];
  const int par = C.parent[c];
  const unsigned vis = par < 0 ? ~0u : open[par];
  const bool mine = b >= lo && b + n <= hi && !straddles(b, n, off, R);
  const bool touches = b < hi && b + n > lo;
  const bool leaf = C.nchild[c] == 0;
  for (int r = 0; r < R; ++r) {
    const bool v = r != me && ((vis >> r) & 1u);
    const bool theirs = b >= off[r] && b + n <= off[r + 1];
    // an accepted pair (T, c) of r is P2P only if t_pp n_T n_c < t_mp n_T and < t_ml, with
    // n_T >= r's smallest leaf count (t_pp = 0: FMM / treecode mode, never)
    const double ntmin = (double)max(box[LETB * r + 7], 1);
    const bool cheap = t_pp > 0.0 && ((near[c] >> r) & 1u) &&
                       t_pp * n < t_mp * (1.0 + 1e-9) &&       // (margins: the
                       t_pp * n * ntmin < t_ml * (1.0 + 1e-9);  // traversal's rounding)
    flags[(size_t)r * ncells + c] = v && mine;
    flags[(size_t)(R + r) * ncells + c] =
        v && touches && !theirs && ((leaf && ((open[c] >> r) & 1u)) || cheap);
  }
}
// per compacted particle entry: [begin, end) (global sorted index) of my part of the cell's range
__global__ void k_let_prange(const unsigned *__restrict__ ids, int n, CellsView C, int lo, int hi,
                             int2 *__restrict__ rng, int *__restrict__ size) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = ids[i];
  const int b = max(C.beg[c], lo), e = min(C.beg[c] + C.cnt[c], hi);
  rng[i] = make_int2(b, e);  // [lo, hi), as k_range_copy reads it
  size[i] = e - b;
}
// records sent with the particles: (global begin, count, offset in the sender's buffer segment
// for that receiver, 0); seg0[r] = first particle entry of receiver r's segment
__global__ void k_let_precords(const int2 *__restrict__ rng, const int *__restrict__ excl, int n,
                               const int *__restrict__ seg0, int R, int4 *__restrict__ rec) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int r = 0;
  while (r + 1 < R && seg0[r + 1] <= i) ++r;
  rec[i] = make_int4(rng[i].x, rng[i].y - rng[i].x, excl[i] - excl[seg0[r]], 0);
}
// receiver: particles of the records of one sender into their global positions (warp per record)
__global__ void k_let_punpack(const int4 *__restrict__ rec, int n, const float4 *__restrict__ data,
                              float4 *__restrict__ pos, int *__restrict__ have) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = w; i < n; i += nw) {
    const int4 r = rec[i];
    for (int j = lane; j < r.y; j += 32) {
      pos[r.x + j] = data[r.z + j];
      if (have) have[r.x + j] = 1;
    }
  }
}
__global__ void k_let_mark(const unsigned *__restrict__ ids, int n, int *__restrict__ have) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) have[ids[i]] = 1;
}
// LET check (tests): every remote multipole / particle this rank's lists name was received
__global__ void k_let_verify(ListsView Ls, int n_m2l, int n_m2p, int n_p2p, CellsView C,
                             const int *__restrict__ strad, int lo, int hi,
                             const int *__restrict__ haveM, const int *__restrict__ haveP,
                             int *missing) {
  const int total = n_m2l + n_m2p + n_p2p;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    if (e < n_m2l + n_m2p) {
      const unsigned s = e < n_m2l ? Ls.src[0][e] : Ls.src[1][e - n_m2l];
      const int b = C.beg[s], n = C.cnt[s];
      if (!(b >= lo && b + n <= hi) && !strad[s] && !haveM[s]) atomicAdd(missing, 1);
    } else {
      const int2 r = Ls.p2p_rng[e - n_m2l - n_m2p];
      for (int j = r.x; j < r.x + r.y; ++j)
        if ((j < lo || j >= hi) && !haveP[j]) {
          atomicAdd(missing + 1, 1);
          break;
        }
    }
  }
}
// compaction of segment-major flags: ids[excl[i]] = i mod nc (the cell) for every set flag
__global__ void k_seg_scatter(const int *__restrict__ flags, const int *__restrict__ excl,
                              int64_t n, int nc, unsigned *__restrict__ ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flags[i]) ids[excl[i]] = (unsigned)(i % nc);
}
// counts of the 2R flag segments from the exclusive scan: cnt[k] = excl[(k+1) nc] - excl[k nc]
__global__ void k_seg_counts(const int *__restrict__ flags, const int *__restrict__ excl, int nseg,
                             int nc, int *cnt) {
  const int k = threadIdx.x;
  if (k >= nseg) return;
  const size_t a = (size_t)k * nc, b = (size_t)(k + 1) * nc - 1;
  cnt[k] = nc > 0 ? excl[b] + flags[b] - excl[a] : 0;
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

int let_box_ints(int R) { return LETB * R; }
void launch_let_boxes(const int *leaves, int nleaves, int ncells, CellsView C, const int *off,
                      int R, int kmax, int *box, cudaStream_t st) {
  k_let_box_init<<<1, 512, 0, st>>>(R, box);
  if (nleaves > 0) k_let_boxes<<<(nleaves + 255) / 256, 256, 0, st>>>(leaves, nleaves, C, off, R, box);
  if (kmax > 0) k_let_small_cells<<<blocks_for(ncells, 256), 256, 0, st>>>(ncells, C, off, R, kmax, box);
}
void launch_let_flags(int ncells, CellsView C, const int *box, const int *off, int R, int me,
                      double theta, double t_pp, double t_mp, double t_ml, unsigned *open,
                      unsigned *near, int *flags, cudaStream_t st) {
  k_let_open<<<blocks_for(ncells, 256), 256, 0, st>>>(ncells, C, box, R, me, theta, open, near);
  k_let_flags<<<blocks_for(ncells, 256), 256, 0, st>>>(ncells, C, open, near, box, off, R, me,
                                                       t_pp, t_mp, t_ml, flags);
}
void launch_seg_counts(const int *flags, const int *excl, int nseg, int nc, int *cnt,
                       cudaStream_t st) {
  k_seg_counts<<<1, 64, 0, st>>>(flags, excl, nseg, nc, cnt);
}
void launch_seg_scatter(const int *flags, const int *excl, int64_t n, int nc, unsigned *ids,
                        cudaStream_t st) {
  if (n > 0) k_seg_scatter<<<blocks_for(n, 256), 256, 0, st>>>(flags, excl, n, nc, ids);
}
void launch_let_prange(const unsigned *ids, int n, CellsView C, int lo, int hi, int2 *rng,
                       int *size, cudaStream_t st) {
  if (n > 0) k_let_prange<<<(n + 255) / 256, 256, 0, st>>>(ids, n, C, lo, hi, rng, size);
}
void launch_let_precords(const int2 *rng, const int *excl, int n, const int *seg0, int R,
                         int4 *rec, cudaStream_t st) {
  if (n > 0) k_let_precords<<<(n + 255) / 256, 256, 0, st>>>(rng, excl, n, seg0, R, rec);
}
void launch_let_punpack(const int4 *rec, int n, const float4 *data, float4 *pos, int *have,
                        cudaStream_t st) {
  if (n > 0) k_let_punpack<<<blocks_for((int64_t)n * 32, 256), 256, 0, st>>>(rec, n, data, pos, have);
}
void launch_let_mark(const unsigned *ids, int n, int *have, cudaStream_t st) {
  if (n > 0) k_let_mark<<<(n + 255) / 256, 256, 0, st>>>(ids, n, have);
}
void launch_let_verify(ListsView Ls, int n_m2l, int n_m2p, int n_p2p, CellsView C,
                       const int *strad, int lo, int hi, const int *haveM, const int *haveP,
                       int *missing, cudaStream_t st) {
  const int total = n_m2l + n_m2p + n_p2p;
  if (total > 0)
    k_let_verify<<<blocks_for(total, 256), 256, 0, st>>>(Ls, n_m2l, n_m2p, n_p2p, C, strad, lo, hi,
                                                         haveM, haveP, missing);
}
