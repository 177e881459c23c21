// common.cuh — device-side data layout shared by the sm_100a kernels of libfmm.so.
//
// HBM layout:
//   pos4   float4[N]        Morton-sorted (x, y, z, q)
//   perm   uint32[N]        sorted index -> caller index
//   keys   uint64[N]        sorted 63-bit Morton keys (21 levels, x bit most significant)
//   cells  SoA, BFS order (level-major, Morton order inside a level):
//            cbeg/ccnt int32, cparent int32, cchild0/cnchild int32,
//            cgrid int4 (doubled-grid centre cx~,cy~,cz~ = (2g+1)*2^(21-l), level) — exact MAC,
//            cgeo float4 (centre x, y, z in FP32, half-width r)
//   Mhat / Lhat float2[ncells][nc_stride(p)]  power-of-two scaled expansions, orders m >= 0 only
//   lists  per target cell (off, cnt) into uint32 source-cell arrays, one array per kind
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define FMM_LEVELS 21
#define FMM_PMAX 16
#define WARP 32

// Number of stored coefficients (m >= 0) for order p, and the index of (n, m >= 0).
__host__ __device__ __forceinline__ constexpr int nc_of(int p) { return (p + 1) * (p + 2) / 2; }
__host__ __device__ __forceinline__ constexpr int cidx(int n, int m) { return n * (n + 1) / 2 + m; }
// Per-cell row stride (complex entries) of the Mhat / Lhat arrays: NC rounded up to even, so
// every row starts 16-byte aligned (TMA bulk copies); the pad entry is kept at zero.
__host__ __device__ __forceinline__ constexpr int nc_stride(int p) { return (nc_of(p) + 1) & ~1; }

// Real degrees of freedom of an expansion (the tensor-core paths): (p+1)^2 of them, ordered for
// n = 0..p as (n,0,Re), then for m = 1..n: (n,m,Re), (n,m,Im). The Im part of m = 0 is zero.
__host__ __device__ constexpr int dof_of(int p) { return (p + 1) * (p + 1); }
__host__ __device__ constexpr int dof_stride(int p) { return (dof_of(p) + 3) & ~3; }  // Y rows
// dof d -> float index inside an (m >= 0, complex) expansion row
__host__ __device__ constexpr int dof_to_float(int d) {
  int n = 0;
  while ((n + 1) * (n + 1) <= d) ++n;
  const int r = d - n * n;                      // 0 .. 2n
  if (r == 0) return 2 * (n * (n + 1) / 2);     // Re of (n, 0)
  const int m = (r + 1) / 2, im = (r + 1) & 1;  // r = 2m-1 -> Re, r = 2m -> Im
  return 2 * (n * (n + 1) / 2 + m) + im;
}
// float index f -> dof, or -1 for the (zero) Im part of an m = 0 coefficient
__host__ __device__ constexpr int float_to_dof(int f) {
  const int c = f / 2, part = f & 1;
  int n = 0;
  while ((n + 1) * (n + 2) / 2 <= c) ++n;
  const int m = c - n * (n + 1) / 2;
  if (m == 0) return part ? -1 : n * n;
  return n * n + 2 * m - 1 + part;
}

struct RootInfo {
  double origin[3];
  double L;       // power-of-two side of the root cube
  double scale;   // 2^21 / L
  unsigned int nonfinite;
  int pad;
};

// Cell arrays (device pointers) passed by value to kernels.
struct CellsView {
  int *beg, *cnt, *parent, *child0, *nchild;
  int4 *grid;    // (cx~, cy~, cz~, level)
  float4 *geo;   // (cx, cy, cz, r)
};

struct ListsView {
  int *off[3];       // per target cell, per kind (M2L, M2P, P2P)
  int *cnt[3];
  unsigned *src[3];  // source cell ids
  int2 *p2p_rng;     // (begin, count) of every P2P source cell, parallel to src[2]
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }

// Signed-order access into m >= 0 storage of a real field: A_n^{-m} = (-1)^m conj(A_n^m).
__device__ __forceinline__ float2 sget(const float2 *A, int n, int m) {
  if (m >= 0) return A[cidx(n, m)];
  float2 v = A[cidx(n, -m)];
  return (m & 1) ? make_float2(-v.x, v.y) : make_float2(v.x, -v.y);
}

#define CUDA_OK(x) ((x) == cudaSuccess)

// Per-device, thread-safe one-time setup (host side). Function attributes and __constant__
// tables belong to a device context, so a second handle on another device (or an in-process
// group thread) must not see a process-wide "already configured" flag.
// Raise the dynamic shared-memory limit of `func` on the current device to at least `bytes`.
void fmm_smem_optin(const void *func, size_t bytes);
// Run `fn` once per (key, current device); `fn` returns whether it succeeded (retried otherwise).
bool fmm_once_per_device(const void *key, bool (*fn)());
// Resident blocks per SM x SMs for `func` at `threads` threads and `smem` dynamic bytes on the
// current device (cached per device).
int fmm_resident_blocks(const void *func, int threads, size_t smem);

// ---- FMM_CHECK builds: device-side bounds checks of the data-dependent indices ----------------
// (compute-sanitizer is not available on the GPU pool; tests/test_gpu_check.py builds the library
// with -DFMM_CHECK and runs the small all-kernel workload of tools/sanitize_run.py.) The bounds are
// the capacities (elements) of the handle's buffers, published per evaluation to every
// translation unit's copy (fmm_check_publish). A failed check prints the site and traps.
struct FmmChk {
  long long pos;    // particles in the sorted position / accumulator arrays (incl. LET copies)
  long long cells;  // cell records
  long long rows;   // expansion rows of M and L
  long long yrows;  // per-pair result slots (deterministic M2L)
  long long lists;  // entries of each interaction list
};
#ifdef FMM_CHECK
#include <cstdio>
static __device__ FmmChk g_fmm_chk;
// the bounds only grow (atomicMax, stream-ordered): handles of an in-process group publish on
// their own streams, and a plain copy from one could land after a later, larger one of another
#define FMM_CHK_DEFINE_SETTER(name)                                                             \
  static __global__ void k_chk_max_##name(FmmChk c) {                                           \
    atomicMax(&g_fmm_chk.pos, c.pos);                                                           \
    atomicMax(&g_fmm_chk.cells, c.cells);                                                       \
    atomicMax(&g_fmm_chk.rows, c.rows);                                                         \
    atomicMax(&g_fmm_chk.yrows, c.yrows);                                                       \
    atomicMax(&g_fmm_chk.lists, c.lists);                                                       \
  }                                                                                             \
  void name(const FmmChk &c, cudaStream_t st) { k_chk_max_##name<<<1, 1, 0, st>>>(c); }
#define FMM_DCHECK(cond, what)                                                                  \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("FMM_CHECK failed: %s [%s] at %s:%d (block %d thread %d)\n", what, #cond, __FILE__, \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                      \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#define FMM_IN(i, bound) ((long long)(i) >= 0 && (long long)(i) < (long long)(bound))
#else
#define FMM_CHK_DEFINE_SETTER(name) \
  void name(const FmmChk &, cudaStream_t) {}
#define FMM_DCHECK(cond, what) \
  do {                         \
  } while (0)
#define FMM_IN(i, bound) true
#endif
// one setter per translation unit that checks (their g_fmm_chk copies are separate)
void fmm_chk_set_p2p(const FmmChk &, cudaStream_t);
void fmm_chk_set_m2l_tc(const FmmChk &, cudaStream_t);
void fmm_chk_set_m2l(const FmmChk &, cudaStream_t);
void fmm_chk_set_traverse(const FmmChk &, cudaStream_t);
void fmm_chk_set_expansions(const FmmChk &, cudaStream_t);
