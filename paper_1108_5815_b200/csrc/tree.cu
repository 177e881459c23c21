// tree.cu — root cube, Morton keys, sort/gather and the level-synchronous adaptive octree.
//
// SURVEY §8(a) a1-a5. The paper builds the tree on the host even in its GPU runs;
// here every step runs on the device. The key is a pure function of the float32 input
// (power-of-two root cube, exact FP64 scaling with explicit _rn intrinsics so nothing is
// contracted into an FMA), so the tree equals the one defined in DESIGN.md §3 bit for bit.
#include <cub/cub.cuh>

#include "common.cuh"
#include <algorithm>
#include <cstdlib>
#include "kernels.cuh"

// ---- a1: bounding box + non-finite check ---------------------------------------------------
__device__ __forceinline__ unsigned f2ord(float f) {
  unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__global__ void k_bbox_init(unsigned *mm, RootInfo *root) {
  if (threadIdx.x < 3) mm[threadIdx.x] = 0xffffffffu;
  else if (threadIdx.x < 6) mm[threadIdx.x] = 0u;
  if (threadIdx.x == 0) root->nonfinite = 0;
}

__global__ void __launch_bounds__(256) k_bbox(const float *__restrict__ xyz,
                                              const float *__restrict__ q, int64_t n,
                                              unsigned *mm, RootInfo *root) {
  unsigned lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0, 0, 0};
  unsigned bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float v = xyz[3 * i + a];
      bad |= !isfinite(v);
      const unsigned o = f2ord(v);
      lo[a] = min(lo[a], o);
      hi[a] = max(hi[a], o);
    }
    bad |= !isfinite(q[i]);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    for (int s = 16; s > 0; s >>= 1) {
      lo[a] = min(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], s));
      hi[a] = max(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], s));
    }
  }
  bad = __any_sync(0xffffffffu, bad);
  // block reduction, then one atomic per block and value (not per warp: contention)
  __shared__ unsigned slo[3][8], shi[3][8], sbad[8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      slo[a][w] = lo[a];
      shi[a][w] = hi[a];
    }
    sbad[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    const int a = threadIdx.x;
    unsigned l = slo[a][0], h = shi[a][0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      l = min(l, slo[a][k]);
      h = max(h, shi[a][k]);
    }
    atomicMin(&mm[a], l);
    atomicMax(&mm[3 + a], h);
  } else if (threadIdx.x == 3) {
    unsigned b = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) b |= sbad[k];
    if (b) atomicOr(&root->nonfinite, 1u);
  }
}

// Root cube: centre of the bbox, side L = 2^ceil(log2 extent) (1 if the extent is 0).
__global__ void k_root(const unsigned *mm, RootInfo *root) {
  if (root->nonfinite) {  // the host reports FMM_E_NONFINITE; keep the cube finite meanwhile
    for (int a = 0; a < 3; ++a) root->origin[a] = 0.0;
    root->L = 1.0;
    root->scale = 2097152.0;
    return;
  }
  double mn[3], mx[3], ext = 0.0;
  for (int a = 0; a < 3; ++a) {
    mn[a] = (double)ord2f(mm[a]);
    mx[a] = (double)ord2f(mm[3 + a]);
    const double e = __dsub_rn(mx[a], mn[a]);
    if (e > ext) ext = e;
  }
  double side = 1.0;
  if (ext > 0.0) {
    while (side < ext) side *= 2.0;
    while (side * 0.5 >= ext) side *= 0.5;
  }
  for (int a = 0; a < 3; ++a)
    root->origin[a] = __dsub_rn(__dmul_rn(0.5, __dadd_rn(mn[a], mx[a])), __dmul_rn(0.5, side));
  root->L = side;
  root->scale = 2097152.0 / side;
}

// ---- a2: Morton keys -------------------------------------------------------------------------
__device__ __forceinline__ uint64_t spread3(uint64_t v) {  // 21 bits -> every third bit
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

__global__ void __launch_bounds__(256) k_keys(const float *__restrict__ xyz, int64_t n,
                                              const RootInfo *__restrict__ root,
                                              uint64_t *__restrict__ keys,
                                              unsigned *__restrict__ idx) {
  const double o0 = root->origin[0], o1 = root->origin[1], o2 = root->origin[2],
               sc = root->scale;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double o[3] = {o0, o1, o2};
    uint64_t g[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double t = floor(__dmul_rn(__dsub_rn((double)xyz[3 * i + a], o[a]), sc));
      t = fmin(fmax(t, 0.0), 2097151.0);
      g[a] = (uint64_t)t;
    }
    keys[i] = (spread3(g[0]) << 2) | (spread3(g[1]) << 1) | spread3(g[2]);
    idx[i] = (unsigned)i;
  }
}

// ---- a3: gather into Morton-sorted SoA float4 ------------------------------------------------
__global__ void __launch_bounds__(256) k_gather(const float *__restrict__ xyz,
                                                const float *__restrict__ q,
                                                const unsigned *__restrict__ perm, int64_t n,
                                                float4 *__restrict__ pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned o = perm ? perm[i] : (unsigned)i;
    pos[i] = make_float4(xyz[3 * (int64_t)o], xyz[3 * (int64_t)o + 1], xyz[3 * (int64_t)o + 2], q[o]);
  }
}

// ---- a4/a5: level-synchronous adaptive octree -------------------------------------------------
__device__ __forceinline__ void cell_geometry(uint64_t prefix, int level, const RootInfo *root,
                                              int4 *grid, float4 *geo) {
  // de-interleave the level-bit prefix into integer cell coordinates
  unsigned g[3] = {0, 0, 0};
  for (int b = 0; b < level; ++b) {
    g[0] |= (unsigned)((prefix >> (3 * b + 2)) & 1) << b;
    g[1] |= (unsigned)((prefix >> (3 * b + 1)) & 1) << b;
    g[2] |= (unsigned)((prefix >> (3 * b + 0)) & 1) << b;
  }
  const int unit = 1 << (FMM_LEVELS - level);
  *grid = make_int4((2 * (int)g[0] + 1) * unit, (2 * (int)g[1] + 1) * unit,
                    (2 * (int)g[2] + 1) * unit, level);
  const double w = root->L / (double)(1u << level);  // exact: power of two
  *geo = make_float4((float)(root->origin[0] + ((double)g[0] + 0.5) * w),
                     (float)(root->origin[1] + ((double)g[1] + 0.5) * w),
                     (float)(root->origin[2] + ((double)g[2] + 0.5) * w), (float)(0.5 * w));
}

__global__ void k_root_cell(int64_t n, const RootInfo *root, CellsView C, uint64_t *prefix) {
  C.beg[0] = 0;
  C.cnt[0] = (int)n;
  C.parent[0] = -1;
  C.child0[0] = -1;
  C.nchild[0] = 0;
  prefix[0] = 0;
  cell_geometry(0, 0, root, &C.grid[0], &C.geo[0]);
}

// For each cell of level `level` (ids [c0, c0 + nl)): child sub-ranges by binary search on the
// sorted keys. A cell is split iff count > ncrit and level < 21. One thread
// per (cell, octant o): bnd[8k + o] = first index of the cell whose child prefix is >= base + o
// (8 independent searches instead of 8 sequential ones per cell: short latency chains at the top
// levels where there are few cells and long ranges).
// Distributed build (nloc >= 0): the keys are this rank's locally sorted shard and the search runs
// over all of it, so bnd = the number of LOCAL keys below the child's first key; the sum of bnd
// over the ranks (one allreduce per level) is the global sorted index of the child's first key,
// i.e. exactly what a single-GPU build over the union would find. Unsplit cells write 0.
__device__ __forceinline__ bool split_cell(int n, int ncrit, int level) {
  return n > ncrit && level < FMM_LEVELS;
}

__global__ void __launch_bounds__(256) k_split(int c0, int nl, int level, int ncrit,
                                               const uint64_t *__restrict__ keys, int nloc,
                                               CellsView C, const uint64_t *__restrict__ prefix,
                                               int *__restrict__ bnd) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= 8 * nl) return;
  const int k = id >> 3, o = id & 7;
  const int c = c0 + k;
  const int b = C.beg[c], n = C.cnt[c];
  if (!split_cell(n, ncrit, level)) {
    bnd[id] = 0;
    return;
  }
  const int shift = 3 * (FMM_LEVELS - (level + 1));
  const uint64_t tgt = prefix[c] * 8 + (uint64_t)o;
  int l = nloc >= 0 ? 0 : b, r = nloc >= 0 ? nloc : b + n;
  while (l < r) {
    const int m = (l + r) >> 1;
    if ((keys[m] >> shift) < tgt) l = m + 1;
    else r = m;
  }
  bnd[id] = l;
}

// child ranges from the 8 boundaries of each cell (non-empty octants, Morton order)
__global__ void __launch_bounds__(256) k_split_ranges(int c0, int nl, int level, int ncrit,
                                                      CellsView C, const int *__restrict__ bnd,
                                                      int *__restrict__ nch,
                                                      int2 *__restrict__ crange) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nl) return;
  int cnt = 0;
  const int c = c0 + k;
  if (split_cell(C.cnt[c], ncrit, level)) {
    const int end = C.beg[c] + C.cnt[c];
    for (int o = 0; o < 8; ++o) {
      const int lo = bnd[8 * k + o], hi = o < 7 ? bnd[8 * k + o + 1] : end;
      if (hi > lo) crange[8 * k + cnt++] = make_int2(lo, (hi - lo) | (o << 28));
    }
  }
  nch[k] = cnt;
}

__global__ void __launch_bounds__(256) k_emit(int c0, int nl, int next0, int level,
                                              const int *__restrict__ nch,
                                              const int *__restrict__ excl,
                                              const int2 *__restrict__ crange,
                                              const RootInfo *__restrict__ root, CellsView C,
                                              uint64_t *__restrict__ prefix) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nl) return;
  const int c = c0 + k;
  const int m = nch[k];
  const int first = next0 + excl[k];
  C.nchild[c] = m;
  C.child0[c] = m ? first : -1;
  const uint64_t pp = prefix[c];
  for (int j = 0; j < m; ++j) {
    const int2 r = crange[8 * k + j];
    const int id = first + j;
    const int oct = (r.y >> 28) & 7;
    C.beg[id] = r.x;
    C.cnt[id] = r.y & 0x0fffffff;
    C.parent[id] = c;
    C.child0[id] = -1;
    C.nchild[id] = 0;
    const uint64_t cp = pp * 8 + (uint64_t)oct;
    prefix[id] = cp;
    cell_geometry(cp, level + 1, root, &C.grid[id], &C.geo[id]);
  }
}

__global__ void k_level_total(const int *nch, const int *excl, int nl, int *out) {
  *out = nl ? excl[nl - 1] + nch[nl - 1] : 0;
}

// Leaves (nchild == 0) in cell order.
__global__ void __launch_bounds__(256) k_leaf_flags(int ncells, const int *__restrict__ nchild,
                                                    int *__restrict__ flag) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < ncells) flag[c] = nchild[c] == 0;
}
__global__ void __launch_bounds__(256) k_leaf_scatter(int ncells, const int *__restrict__ flag,
                                                      const int *__restrict__ excl,
                                                      int *__restrict__ leaves) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < ncells && flag[c]) leaves[excl[c]] = c;
}

// Morton partition of the targets (multi-GPU): a leaf belongs to part floor(begin * nparts / n).
// flag = leaf of part `part`; the part's sorted particle range [lo, hi) via atomics into lohi.
__global__ void __launch_bounds__(256) k_part_flags(int ncells, CellsView C, int64_t n,
                                                    int nparts, int part, int *__restrict__ flag,
                                                    int *__restrict__ lohi) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  int f = 0;
  if (C.nchild[c] == 0) {
    const int b = C.beg[c];
    f = (int)(((int64_t)b * nparts) / n) == part;
    if (f) {
      atomicMin(&lohi[0], b);
      atomicMax(&lohi[1], b + C.cnt[c]);
    }
  }
  flag[c] = f;
}
__global__ void k_part_init(int *lohi, int n) {
  lohi[0] = n;
  lohi[1] = 0;
}
__global__ void __launch_bounds__(256) k_part_indices(int lo, int cnt,
                                                      const unsigned *__restrict__ perm,
                                                      int64_t *__restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
    out[i] = perm[lo + i];
}

// ---- a3 short sort: radix passes over the key bits [SORT_LOW_BITS, 63) + a tie fix-up ---------
// Keys that agree in bits SORT_LOW_BITS..62 form runs that the stable radix pass left in index
// order; each run is put in full-key order (ties in the full key keep the index order, so the
// result is exactly the stable 63-bit sort): runs of <= SORT_RUN_MAX by one thread (insertion
// sort), runs of <= SORT_BLOCK_MAX by one CTA (bitonic sort of (key, original index) pairs in
// shared memory), longer runs flag the caller, which then sorts all 63 bits. The caller picks
// SORT_LOW_BITS (a run-time argument) from the previous tree's depth D: the bits of levels
// 0..D+2, so the runs are particles sharing a cell two levels below the deepest leaf (C2, D = 5:
// 21 bits, 3 passes; C4, D = 7: 27 bits, 4 passes; C3, D = 12: 42 bits, 6 passes).
#define SORT_RUN_MAX 64
#define SORT_BLOCK_MAX 4096
__global__ void k_sort_fixup(uint64_t *__restrict__ keys, unsigned *__restrict__ vals, int64_t n,
                             int *flag, int2 *__restrict__ runs, int *nruns, int runs_cap,
                             int SORT_LOW_BITS) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i + 1 < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t hi = keys[i] >> SORT_LOW_BITS;
    if ((keys[i + 1] >> SORT_LOW_BITS) != hi) continue;          // not inside a run
    if (i > 0 && (keys[i - 1] >> SORT_LOW_BITS) == hi) continue;  // not the run's first element
    int64_t e = i + 1;
    while (e < n && (keys[e] >> SORT_LOW_BITS) == hi && e - i <= SORT_BLOCK_MAX) ++e;
    if (e - i > SORT_RUN_MAX) {  // a CTA sorts it (k_sort_fixup_block), or the caller redoes all
      const int r = e - i <= SORT_BLOCK_MAX ? atomicAdd(nruns, 1) : runs_cap;
      if (r < runs_cap)
        runs[r] = make_int2((int)i, (int)(e - i));
      else
        atomicOr(flag, 1);
      continue;
    }
    for (int64_t a = i + 1; a < e; ++a) {  // insertion sort by the full key (stable)
      const uint64_t k = keys[a];
      const unsigned v = vals[a];
      int64_t b = a - 1;
      while (b >= i && keys[b] > k) {
        keys[b + 1] = keys[b];
        vals[b + 1] = vals[b];
        --b;
      }
      keys[b + 1] = k;
      vals[b + 1] = v;
    }
  }
}
// one CTA per long run: bitonic sort of (full key, original index) -- a total order, so the
// result equals the stable sort's
__global__ void __launch_bounds__(512) k_sort_fixup_block(uint64_t *__restrict__ keys,
                                                          unsigned *__restrict__ vals,
                                                          const int2 *__restrict__ runs,
                                                          const int *__restrict__ nruns) {
  __shared__ uint64_t sk[SORT_BLOCK_MAX];
  __shared__ unsigned sv[SORT_BLOCK_MAX];
  const int nr = *nruns;
  for (int r = blockIdx.x; r < nr; r += gridDim.x) {
    const int2 run = runs[r];
    int P = 64;
    while (P < run.y) P <<= 1;
    __syncthreads();
    for (int t = threadIdx.x; t < P; t += blockDim.x) {
      sk[t] = t < run.y ? keys[run.x + t] : ~0ull;
      sv[t] = t < run.y ? vals[run.x + t] : ~0u;
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = threadIdx.x; t < P; t += blockDim.x) {
          const int u = t ^ j;
          if (u > t) {
            const uint64_t a = sk[t], b = sk[u];
            const unsigned va = sv[t], vb = sv[u];
            const bool gt = a > b || (a == b && va > vb);
            if (((t & k) == 0) == gt) {
              sk[t] = b;
              sk[u] = a;
              sv[t] = vb;
              sv[u] = va;
            }
          }
        }
        __syncthreads();
      }
    for (int t = threadIdx.x; t < run.y; t += blockDim.x) {
      keys[run.x + t] = sk[t];
      vals[run.x + t] = sv[t];
    }
  }
}

// ---- a4/a5 in one cooperative kernel (single GPU) ------------------------------------------------
// The level loop of build_levels on the device: per level, the 8 child bounds of every cell by
// binary search, the child counts, a grid-wide exclusive scan (block segments + one block scanning
// the block totals) and the emission of the next level, separated by grid syncs -- no host round
// trip per level. st[] (device): [0] total cells, [1] overflow (capacity), [2] depth,
// [3] leaves, [8 + l] level offsets, [32 + l] level counts.
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#define TREE_BLOCK 256
__device__ __forceinline__ int block_excl_scan(int v, int *ws, int &total) {
  // exclusive scan of one value per thread across the block; ws: 32 ints of shared memory
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < nw ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) ws[lane] = t;
  }
  __syncthreads();
  total = ws[nw - 1];
  const int r = x - v + (w ? ws[w - 1] : 0);
  __syncthreads();
  return r;
}
__global__ void __launch_bounds__(TREE_BLOCK) k_tree_coop(const uint64_t *__restrict__ keys, int n,
                                                          int ncrit, const RootInfo *__restrict__ root,
                                                          CellsView C, uint64_t *__restrict__ prefix,
                                                          int cap, int *__restrict__ bnd,
                                                          int *__restrict__ nch, int2 *__restrict__ crange,
                                                          int *__restrict__ blk, int *__restrict__ st,
                                                          int *__restrict__ leaves) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int ws[32];
  const int G = gridDim.x, b = blockIdx.x;
  const int gtid = b * blockDim.x + threadIdx.x, gthreads = G * blockDim.x;
  if (gtid == 0) {
    C.beg[0] = 0;
    C.cnt[0] = n;
    C.parent[0] = -1;
    C.child0[0] = -1;
    C.nchild[0] = 0;
    prefix[0] = 0;
    cell_geometry(0, 0, root, &C.grid[0], &C.geo[0]);
    st[1] = 0;
    st[8] = 0;
    st[32] = 1;
  }
  // Two grid syncs per level: (1) every block takes a contiguous segment of the level's cells,
  // finds each cell's 8 child bounds by binary search (8 lanes per cell, the next octant's bound
  // by a shuffle), counts and compacts the non-empty children and publishes its segment's child
  // total; (2) after the sync every block sums the totals of the blocks before it (its offset) and
  // of all blocks (the next level's size) itself -- no serial scan by one block, no extra sync --
  // and emits its children in cell order (deterministic).
  auto prefix_of = [&](int upto, int &all) {  // sum of blk[0, upto) and of blk[0, G), block-wide
    int a = 0, t = 0;
    for (int j = threadIdx.x; j < G; j += blockDim.x) {
      const int v = blk[j];
      t += v;
      if (j < upto) a += v;
    }
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
      ws[threadIdx.x >> 5] = a;
      ws[16 + (threadIdx.x >> 5)] = t;
    }
    __syncthreads();
    a = 0;
    t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += ws[w];
      t += ws[16 + w];
    }
    __syncthreads();
    all = t;
    return a;
  };
  int c0 = 0, nl = 1, total = 1, level = 0;
  for (;; ++level) {
    grid.sync();
    const int shift = 3 * (FMM_LEVELS - (level + 1));
    const int seg = (nl + G - 1) / G, s0 = min(b * seg, nl), s1 = min(s0 + seg, nl);
    int bsum = 0;
    for (int base = s0 * 8; base < s1 * 8; base += blockDim.x) {
      const int id = base + threadIdx.x;
      const bool live = id < s1 * 8;
      const int k = id >> 3, o = id & 7, c = c0 + k;
      int lo = 0, end = 0;
      bool split = false;
      if (live) {
        const int cb = C.beg[c], cn = C.cnt[c];
        end = cb + cn;
        lo = cb;
        split = split_cell(cn, ncrit, level);
        if (split) {
          const uint64_t tgt = prefix[c] * 8 + (uint64_t)o;
          int r = end;
          while (lo < r) {
            const int m = (lo + r) >> 1;
            if ((keys[m] >> shift) < tgt) lo = m + 1;
            else r = m;
          }
        }
      }
      const int nxt = __shfl_down_sync(0xffffffffu, lo, 1);  // the next octant's bound
      const int hi = o < 7 ? nxt : end;
      const bool ne = live && split && hi > lo;
      const unsigned bal = __ballot_sync(0xffffffffu, ne);
      const unsigned grp = (bal >> (threadIdx.x & 24)) & 0xffu;  // this cell's 8 lanes
      if (ne) {
        const int pos = __popc(grp & ((1u << o) - 1u));
        crange[8 * k + pos] = make_int2(lo, (hi - lo) | (o << 28));
      }
      if (live && o == 0) {
        nch[k] = __popc(grp);
        bsum += __popc(grp);
      }
    }
    for (int o = 16; o > 0; o >>= 1) bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = bsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
      blk[b] = t;
    }
    __syncthreads();
    grid.sync();
    int nnext = 0;
    int run = total + prefix_of(b, nnext);
    if (total + nnext > cap) {
      if (gtid == 0) st[1] = 1;
      break;  // every block takes the same decision
    }
    if (nnext == 0) break;
    // emit the children: block-local exclusive scan of the segment + the block's offset
    for (int k0 = s0; k0 < s1; k0 += blockDim.x) {
      const int k = k0 + threadIdx.x;
      const int m = k < s1 ? nch[k] : 0;
      int tot;
      const int e = block_excl_scan(m, ws, tot);
      if (k < s1) {
        const int c = c0 + k, first = run + e;
        C.nchild[c] = m;
        C.child0[c] = m ? first : -1;
        const uint64_t pp = prefix[c];
        for (int j = 0; j < m; ++j) {
          const int2 r = crange[8 * k + j];
          const int id = first + j, oct = (r.y >> 28) & 7;
          C.beg[id] = r.x;
          C.cnt[id] = r.y & 0x0fffffff;
          C.parent[id] = c;
          C.child0[id] = -1;
          C.nchild[id] = 0;
          const uint64_t cp = pp * 8 + (uint64_t)oct;
          prefix[id] = cp;
          cell_geometry(cp, level + 1, root, &C.grid[id], &C.geo[id]);
        }
      }
      run += tot;
    }
    c0 = total;
    nl = nnext;
    total += nnext;
    if (gtid == 0) {
      st[8 + level + 1] = c0;
      st[32 + level + 1] = nl;
    }
  }
  // leaves in cell order (flag, grid-wide scan, scatter): the same segment scheme
  grid.sync();
  if (st[1]) return;
  const int seg = (total + G - 1) / G, s0 = min(b * seg, total), s1 = min(s0 + seg, total);
  int cnt = 0;
  for (int c = s0 + threadIdx.x; c < s1; c += blockDim.x) cnt += C.nchild[c] == 0;
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    blk[b] = t;
  }
  __syncthreads();
  grid.sync();
  int nleaves = 0;
  int run = prefix_of(b, nleaves);
  if (gtid == 0) {
    st[0] = total;
    st[2] = level;
    st[3] = nleaves;
  }
  for (int c0l = s0; c0l < s1; c0l += blockDim.x) {
    const int c = c0l + threadIdx.x;
    const int f = c < s1 ? (C.nchild[c] == 0) : 0;
    int tot;
    const int e = block_excl_scan(f, ws, tot);
    if (f) leaves[run + e] = c;
    run += tot;
  }
}

// ---- host launchers --------------------------------------------------------------------------
static int grid_for(int64_t n, int bs) {
  int64_t g = (n + bs - 1) / bs;
  if (g > 148 * 32) g = 148 * 32;
  return (int)(g < 1 ? 1 : g);
}

void launch_bbox(const float *xyz, const float *q, int64_t n, unsigned *mm, RootInfo *root,
                 cudaStream_t st) {
  k_bbox_init<<<1, 32, 0, st>>>(mm, root);
  k_bbox<<<grid_for(n, 256), 256, 0, st>>>(xyz, q, n, mm, root);
  k_root<<<1, 1, 0, st>>>(mm, root);
}
// distributed bbox: the local min/max (and the non-finite flag in mm[6]) before the allreduce,
// then the root cube from the reduced values
__global__ void k_nonfinite_to_mm(unsigned *mm, RootInfo *root) { mm[6] = root->nonfinite; }
__global__ void k_mm_to_nonfinite(const unsigned *mm, RootInfo *root) { root->nonfinite = mm[6]; }
void launch_bbox_local(const float *xyz, const float *q, int64_t n, unsigned *mm, RootInfo *root,
                       cudaStream_t st) {
  k_bbox_init<<<1, 32, 0, st>>>(mm, root);
  if (n > 0) k_bbox<<<grid_for(n, 256), 256, 0, st>>>(xyz, q, n, mm, root);
  k_nonfinite_to_mm<<<1, 1, 0, st>>>(mm, root);
}
void launch_root_from_mm(const unsigned *mm, RootInfo *root, cudaStream_t st) {
  k_mm_to_nonfinite<<<1, 1, 0, st>>>(mm, root);
  k_root<<<1, 1, 0, st>>>(mm, root);
}
void launch_keys(const float *xyz, int64_t n, const RootInfo *root, uint64_t *keys, unsigned *idx,
                 cudaStream_t st) {
  k_keys<<<grid_for(n, 256), 256, 0, st>>>(xyz, n, root, keys, idx);
}
void launch_gather(const float *xyz, const float *q, const unsigned *perm, int64_t n, float4 *pos,
                   cudaStream_t st) {
  k_gather<<<grid_for(n, 256), 256, 0, st>>>(xyz, q, perm, n, pos);
}
cudaError_t sort_keys(void *tmp, size_t &tmp_bytes, const uint64_t *kin, uint64_t *kout,
                      const unsigned *vin, unsigned *vout, int64_t n, cudaStream_t st) {
  return cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, vin, vout, (int)n, 0, 63, st);
}
// bits [low_bits, 63) only (3-6 onesweep passes instead of 8), then the tie fix-up; *flag set
// => the caller must redo the full sort. runs: scratch of runs_cap entries, flag[1] their count.
int sort_runs_cap(int64_t n) { return (int)(n / (SORT_RUN_MAX + 1)) + 1; }
cudaError_t sort_keys_short(void *tmp, size_t &tmp_bytes, const uint64_t *kin, uint64_t *kout,
                            const unsigned *vin, unsigned *vout, int64_t n, int *flag,
                            int2 *runs, int low_bits, cudaStream_t st) {
  cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, vin, vout, (int)n,
                                                  low_bits, 63, st);
  if (e || !tmp || n < 2) return e;
  cudaMemsetAsync(flag + 1, 0, sizeof(int), st);
  k_sort_fixup<<<grid_for(n, 256), 256, 0, st>>>(kout, vout, n, flag, runs, flag + 1,
                                                 sort_runs_cap(n), low_bits);
  k_sort_fixup_block<<<148 * 2, 512, 0, st>>>(kout, vout, runs, flag + 1);
  return cudaGetLastError();
}
// the cooperative tree build: grid size for this device (all blocks co-resident)
int tree_coop_grid() {
  const int res = fmm_resident_blocks((const void *)k_tree_coop, TREE_BLOCK, 0);
  static const int per_sm = getenv("FMM_TREE_GRID") ? atoi(getenv("FMM_TREE_GRID")) : 0;
  return per_sm > 0 ? std::min(res, 148 * per_sm) : res;  // (A/B knob: blocks per SM)
}
cudaError_t launch_tree_coop(const uint64_t *keys, int n, int ncrit, const RootInfo *root,
                             CellsView C, uint64_t *prefix, int cap, int *bnd, int *nch,
                             int2 *crange, int *blk, int *st_dev, int *leaves, int grid,
                             cudaStream_t st) {
  void *args[] = {(void *)&keys, (void *)&n, (void *)&ncrit, (void *)&root, (void *)&C,
                  (void *)&prefix, (void *)&cap, (void *)&bnd, (void *)&nch, (void *)&crange,
                  (void *)&blk, (void *)&st_dev, (void *)&leaves};
  return cudaLaunchCooperativeKernel((const void *)k_tree_coop, grid, TREE_BLOCK, args, 0, st);
}
cudaError_t exclusive_scan(void *tmp, size_t &tmp_bytes, const int *in, int *out, int n,
                           cudaStream_t st) {
  return cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in, out, n, st);
}
void launch_root_cell(int64_t n, const RootInfo *root, CellsView C, uint64_t *prefix,
                      cudaStream_t st) {
  k_root_cell<<<1, 1, 0, st>>>(n, root, C, prefix);
}
void launch_split(int c0, int nl, int level, int ncrit, const uint64_t *keys, CellsView C,
                  const uint64_t *prefix, int *nch, int2 *crange, int *bnd, cudaStream_t st) {
  launch_split_bounds(c0, nl, level, ncrit, keys, -1, C, prefix, bnd, st);
  launch_split_ranges(c0, nl, level, ncrit, C, bnd, nch, crange, st);
}
void launch_split_bounds(int c0, int nl, int level, int ncrit, const uint64_t *keys, int nloc,
                         CellsView C, const uint64_t *prefix, int *bnd, cudaStream_t st) {
  k_split<<<(8 * nl + 255) / 256, 256, 0, st>>>(c0, nl, level, ncrit, keys, nloc, C, prefix, bnd);
}
void launch_split_ranges(int c0, int nl, int level, int ncrit, CellsView C, const int *bnd,
                         int *nch, int2 *crange, cudaStream_t st) {
  k_split_ranges<<<(nl + 255) / 256, 256, 0, st>>>(c0, nl, level, ncrit, C, bnd, nch, crange);
}
void launch_emit(int c0, int nl, int next0, int level, const int *nch, const int *excl,
                 const int2 *crange, const RootInfo *root, CellsView C, uint64_t *prefix,
                 cudaStream_t st) {
  k_emit<<<(nl + 255) / 256, 256, 0, st>>>(c0, nl, next0, level, nch, excl, crange, root, C,
                                            prefix);
}
void launch_level_total(const int *nch, const int *excl, int nl, int *total, cudaStream_t st) {
  k_level_total<<<1, 1, 0, st>>>(nch, excl, nl, total);
}
void launch_part_flags(int ncells, CellsView C, int64_t n, int nparts, int part, int *flag,
                       int *lohi, cudaStream_t st) {
  k_part_init<<<1, 1, 0, st>>>(lohi, (int)n);
  k_part_flags<<<(ncells + 255) / 256, 256, 0, st>>>(ncells, C, n, nparts, part, flag, lohi);
}
void launch_part_indices(int lo, int cnt, const unsigned *perm, int64_t *out, cudaStream_t st) {
  const int b = (cnt + 255) / 256 < 148 * 8 ? (cnt + 255) / 256 : 148 * 8;
  k_part_indices<<<b > 0 ? b : 1, 256, 0, st>>>(lo, cnt, perm, out);
}
void launch_leaf_flags(int ncells, const int *nchild, int *flag, cudaStream_t st) {
  k_leaf_flags<<<(ncells + 255) / 256, 256, 0, st>>>(ncells, nchild, flag);
}
void launch_leaf_scatter(int ncells, const int *flag, const int *excl, int *leaves,
                         cudaStream_t st) {
  k_leaf_scatter<<<(ncells + 255) / 256, 256, 0, st>>>(ncells, flag, excl, leaves);
}

// ---- distinct target / source sets --------------------------------------------
__global__ void k_target_flags(const unsigned *__restrict__ perm, int n, int nt, int *flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    flag[i] = perm[i] < (unsigned)nt;
}
__global__ void k_cell_targets(int ncells, CellsView C, const int *__restrict__ excl,
                               const int *__restrict__ flag, int n, int *ntgt, int *leafflag) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const int b = C.beg[c], e = b + C.cnt[c];
  const int hi = e < n ? excl[e] : excl[n - 1] + flag[n - 1];
  const int k = hi - excl[b];
  ntgt[c] = k;
  leafflag[c] = C.nchild[c] == 0 && k > 0;
}
void launch_target_flags(const unsigned *perm, int n, int nt, int *flag, cudaStream_t st) {
  k_target_flags<<<grid_for(n, 256), 256, 0, st>>>(perm, n, nt, flag);
}
void launch_cell_targets(int ncells, CellsView C, const int *excl, const int *flag, int n,
                         int *ntgt, int *leafflag, cudaStream_t st) {
  k_cell_targets<<<(ncells + 255) / 256, 256, 0, st>>>(ncells, C, excl, flag, n, ntgt, leafflag);
}
