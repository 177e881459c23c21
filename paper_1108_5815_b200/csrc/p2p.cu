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

#include <algorithm>
#include <cstdlib>

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

#include "p2p_core.cuh"

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


// ================================================================================================
// k_p2p_tma — the same pairs, CTA-cooperative and warp-specialised (round 2).
//
// One CTA works on one target chunk (<= 64 particles of a leaf) at a time, pulled from the
// dynamic leaf queue. Warp 4 (the producer) walks the P2P lists of the leaf and its ancestors and
// streams the source particle ranges -- contiguous in Morton order -- into a ring of P2Q_STAGES
// shared-memory tiles with one TMA bulk copy (cp.async.bulk ... complete_tx) per range piece,
// signalling a `full` mbarrier per tile; the leaf itself comes first, in tiles of its own flagged
// for the r = 0 mask. Warps 0-3 (the consumers) do nothing but the packed-FP32 inner loop: each
// takes a quarter of every tile (the 2-D lane map of k_p2p_leaves inside the warp: G target
// pairs x S source slices), releases the tile through an `empty` mbarrier, and at the chunk's
// last tile the slices and the four warps are reduced in a fixed order (deterministic) and the
// chunk is written once. Compared with k_p2p_leaves the consumers never walk lists, issue copies
// or wait on their own loads, so the FMA pipe stays fed.
// ================================================================================================
// Tile size and depth measured on the B200 (C2 / C3 / C4 P2P ms, bench.py): 768 x 3 stages
// 1.33 / 6.84 / 30.1; 512 x 4: 1.31 / 7.01 / 30.6; 384 x 6: 1.39 / 7.85 / 33.4; 2 consumer
// warps per CTA (384 x 3, 8 CTAs per SM): 1.36 / 7.87 / 32.7; per-lane cp.async instead of TMA
// bulk copies: 1.37 / 6.84 / 31.4; round-1 k_p2p_leaves: 1.32 / 7.33 / 31.6.
#ifndef P2Q_TILE
#if defined(P2Q_LASTRED) && P2Q_LASTRED == 1
#define P2Q_TILE 640  // 4 CTAs per SM with the P2Q_STAGES reduction buffers of the last-warp reduction
#else
#define P2Q_TILE 816  // the largest with 4 CTAs per SM (quad-lane consumers; 768: C4 P2P +0.8%)
#endif
#endif
#ifndef P2Q_STAGES
#define P2Q_STAGES 3
#endif
#ifndef P2Q_CWARPS
#define P2Q_CWARPS 4  // consumer warps per CTA (they split every tile)
#endif
#define P2Q_THREADS (32 * (P2Q_CWARPS + 1))
#ifndef P2Q_MINB
#define P2Q_MINB 4  // 90 registers, 4 CTAs = 16 consumer warps per SM (6 CTAs at 64 registers
                    // measured slower although tools/p2p_micro's bare loop gains 57% -> 59%)
#endif
#ifndef P2Q_CPASYNC
#define P2Q_CPASYNC 0  // producer copies with per-lane cp.async (1) or one TMA bulk copy per range (0)
#endif
#ifndef P2Q_QUAD
#define P2Q_QUAD 1  // consumers: CTA-wide pool of 128 lanes x 4 targets (1) or per-warp 32 x 2 (0)
#endif
#if P2Q_QUAD
#define P2Q_CHUNK 128  // most targets per chunk: the pool's 128 lanes x 4 targets, >= 1 slice each
#else
#define P2Q_CHUNK 64  // most targets per chunk: 32 lanes x 2 packed targets
#endif
// Ring of reduction buffers. A warp finishes a chunk's reduction before it releases the chunk's
// last tile, and the producer reopens a stage only after all four warps released it: so when a
// warp reaches the end of chunk j, every warp has released the tile P2Q_STAGES tiles back, hence
// finished the reductions of all chunks ending there or earlier. Each chunk has >= 1 tile, so
// P2Q_STAGES buffers suffice.
#define P2Q_RED P2Q_STAGES
#define P2Q_BATCH 8   // leaves per queue atomic

// Targets of the next chunk of a leaf with `rem` targets left. A chunk of k targets keeps
// k * S(k) of the 64 lane slots busy (S(k) = floor(32 / ceil(k / 2)) source slices), so 33..48
// targets go as 32 + rest (e.g. 40: 32 at S = 2 and 8 at S = 8 -> 0.625 of the slot-steps of one
// 40-target chunk at S = 1); from 49 on one chunk costs no more than two.
__device__ __forceinline__ int p2q_chunk(int rem) {
#if P2Q_QUAD
  return min(rem, P2Q_CHUNK);
#else
  return rem >= 49 ? min(rem, P2Q_CHUNK) : (rem > 32 ? 32 : rem);
#endif
}

enum { QF_FIRST = 1, QF_LAST = 2, QF_MASK = 4, QF_END = 8 };
// desc.w bits: [0, 30) list count, 30: the list is the raw P2P list (else the merged runs of
// k_p2p_merge), 31: a proper ancestor has a P2P list the producer must walk
#define P2Q_RAW 0x40000000
#define P2Q_CNT(w) ((w) & 0x3fffffff)

#ifdef P2Q_TRACE  // tools-only build: a timeline of CTA 0's ring (device printf, globaltimer ns)
__device__ __forceinline__ unsigned long long q_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#include <cstdio>
#ifndef P2Q_TRACE_K0
#define P2Q_TRACE_K0 0
#endif
__device__ unsigned long long g_q_tr[5][6][P2Q_TRACE];
__device__ int g_q_trv[5][6][P2Q_TRACE];
#define Q_TRACE(who_, ev_, k_, v_)                                                              \
  do {                                                                                          \
    if (blockIdx.x == 0 && (k_) >= P2Q_TRACE_K0 && (k_) < P2Q_TRACE_K0 + P2Q_TRACE) {          \
      const int w_ = (who_) == 9 ? 4 : (who_);                                                  \
      g_q_tr[w_][ev_][(k_) - P2Q_TRACE_K0] = q_now();                                           \
      g_q_trv[w_][ev_][(k_) - P2Q_TRACE_K0] = (int)(v_);                                        \
    }                                                                                           \
  } while (0)
__global__ void k_q_trace_dump() {
  for (int w = 0; w < 5; ++w)
    for (int e = 0; e < 6; ++e)
      for (int k = 0; k < P2Q_TRACE; ++k)
        if (g_q_tr[w][e][k])
          printf("TR %d %d %d %d %llu\n", w == 4 ? 9 : w, e, k, g_q_trv[w][e][k], g_q_tr[w][e][k]);
  for (int w = 0; w < 5; ++w)
    for (int e = 0; e < 6; ++e)
      for (int k = 0; k < P2Q_TRACE; ++k) g_q_tr[w][e][k] = 0;
}
#else
#define Q_TRACE(who_, ev_, k_, v_) \
  do {                         \
  } while (0)
#endif

__device__ __forceinline__ unsigned q_saddr(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void q_mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(q_saddr(bar)), "r"(count));
}
__device__ __forceinline__ void q_mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(q_saddr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void q_mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(q_saddr(bar)) : "memory");
}
__device__ __forceinline__ void q_mbar_wait(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n Q_WAIT:\n"
      " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra Q_DONE;\n bra Q_WAIT;\n Q_DONE:\n }" ::"r"(q_saddr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void q_cpasync_arrive(unsigned long long *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(q_saddr(bar)) : "memory");
}
__device__ __forceinline__ void q_bulk_g2s(void *dst, const void *src, unsigned bytes,
                                           unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          q_saddr(dst)),
      "l"(src), "r"(bytes), "r"(q_saddr(bar))
      : "memory");
}

__global__ void __launch_bounds__(P2Q_THREADS, P2Q_MINB)
    k_p2p_tma(const int *__restrict__ leaves, int nleaves, CellsView C, ListsView Ls,
              const float4 *__restrict__ pos, float4 *__restrict__ acc_out, float m1,
              int *next_leaf, const int4 *__restrict__ desc, const int2 *__restrict__ mrg) {
  extern __shared__ __align__(128) float4 p2q_dyn[];  // [P2Q_STAGES][P2Q_TILE] source tiles
  float4(*tile)[P2Q_TILE] = reinterpret_cast<float4(*)[P2Q_TILE]>(p2q_dyn);
  __shared__ int4 meta[P2Q_STAGES];  // (leaf begin, count, flags, chunk start | size << 16)
  __shared__ __align__(8) unsigned long long full[P2Q_STAGES], empty[P2Q_STAGES];
#if P2Q_QUAD
  // per-lane partial sums of the chunk's last tile: [buffer][slot = slice * Q + quad][target]
#ifndef P2Q_LASTRED
#define P2Q_LASTRED 0  // 1: the last consumer warp to finish a chunk reduces it, no barrier (with
                       // 640-particle tiles for the buffers: C4 P2P 28.4 ms vs 27.5, slower)
#endif
#if P2Q_LASTRED == 2
#define P2Q_REDBUF 2  // two buffers, reuse guarded by a per-buffer generation count
#elif P2Q_LASTRED
#define P2Q_REDBUF P2Q_STAGES  // see P2Q_RED
#elif defined(P2Q_ONEBUF) && P2Q_ONEBUF
#define P2Q_REDBUF 1  // one buffer, a second consumer barrier after the reduction (8 KB for tiles)
#else
#define P2Q_REDBUF 2  // the 4 consumer warps meet at a named barrier, then reduce together
#endif
  __shared__ __align__(16) float4 red[P2Q_REDBUF][32 * P2Q_CWARPS][4];
  __shared__ int red_cnt[P2Q_REDBUF];
  __shared__ int red_gen[P2Q_REDBUF];  // reductions completed on each buffer (P2Q_LASTRED == 2)
#else
  __shared__ __align__(16) float4 red[P2Q_RED][P2Q_CWARPS][P2Q_CHUNK];
  __shared__ int red_cnt[P2Q_RED];
#endif
  const int lane = threadIdx.x & 31;
#ifndef P2Q_PROD_ROT
#define P2Q_PROD_ROT 0  // 1: the producer is warp blockIdx % 4 (measured: C4 P2P 27.9 -> 31.7 ms;
                        // with warp 4 the 4 CTAs of an SM already put one producer on each SMSP)
#endif
  // role: the producer warp, and the consumers' pool rank 0..P2Q_CWARPS-1 (`warp` below)
  const int wraw = threadIdx.x >> 5, prod = P2Q_PROD_ROT ? (int)(blockIdx.x & 3) : P2Q_CWARPS;
  const int warp = wraw == prod ? P2Q_CWARPS : (wraw < prod ? wraw : wraw - 1);
  if (threadIdx.x == 0) {
    for (int b = 0; b < (int)(sizeof(red_cnt) / sizeof(int)); ++b) red_cnt[b] = red_gen[b] = 0;
    for (int s = 0; s < P2Q_STAGES; ++s) {
      q_mbar_init(&full[s], P2Q_CPASYNC ? 33 : 1);  // (32 producer lanes' copies +) the meta
      q_mbar_init(&empty[s], P2Q_CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == P2Q_CWARPS) {
    // ------------------------------------------------------------------ producer warp
    unsigned k = 0;     // tiles opened so far (tile k uses stage k % P2Q_STAGES)
    int fill = 0;       // sources in the open tile
    bool open = false;
    int flags_pending = 0;
    auto open_tile = [&]() {
      if (lane == 0) Q_TRACE(9, 0, k, 0);
      if (k >= P2Q_STAGES) q_mbar_wait(&empty[k % P2Q_STAGES], ((k / P2Q_STAGES) + 1) & 1);
      if (lane == 0) Q_TRACE(9, 1, k, 0);
      fill = 0;
      open = true;
    };
    auto close_tile = [&](int leaf, int flags, int c0) {
#if P2Q_CPASYNC
      q_cpasync_arrive(&full[k % P2Q_STAGES]);  // fires when this lane's copies have landed
#endif
      __syncwarp();  // every lane's expect_tx precedes the arrive
      if (lane == 0) {
        Q_TRACE(9, 2, k, fill);
        meta[k % P2Q_STAGES] = make_int4(leaf, fill, flags, c0);
        q_mbar_arrive(&full[k % P2Q_STAGES]);
      }
      __syncwarp();
      ++k;
      open = false;
    };
    // lanes hold one particle range each (cnt = 0: none); append them in lane order
    auto emit = [&](int beg, int cnt, int leaf, int c0, bool self = false) {
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      const int lo = incl - cnt;
      int done = 0;
      while (done < total) {
        if (!open) open_tile();
        const int take = min(P2Q_TILE - fill, total - done);
        const int a = max(lo, done), e = min(lo + cnt, done + take);
#if P2Q_CPASYNC
        // each lane copies its own range piece, 16 B per cp.async (LDGSTS); completion is tracked
        // by the lanes' cp.async.mbarrier.arrive at close_tile
        {
          float4 *dst = &tile[k % P2Q_STAGES][fill - done];
          const float4 *src = pos + beg - lo;
          for (int x = a; x < e; ++x) cp_async16(dst + x, src + x);
        }
#else
        if (a < e) {  // one TMA bulk copy per range piece
          FMM_DCHECK(beg + (a - lo) >= 0 && (long long)beg + (e - lo) <= g_fmm_chk.pos,
                     "P2P source range");
          unsigned long long *fb = &full[k % P2Q_STAGES];
          q_mbar_expect_tx(fb, (unsigned)(e - a) * 16u);
          q_bulk_g2s(&tile[k % P2Q_STAGES][fill + (a - done)], pos + beg + (a - lo),
                     (unsigned)(e - a) * 16u, fb);
        }
#endif
        fill += take;
        done += take;
        if (fill == P2Q_TILE) {
          close_tile(leaf, flags_pending, c0);
          // the next tile holds no own particle once the leaf's own range has been emitted
          flags_pending &= self ? ~QF_FIRST : ~(QF_FIRST | QF_MASK);
        }
      }
    };
#ifndef P2Q_MERGE
#define P2Q_MERGE 0  // per-batch sort + merge in the producer (superseded by k_p2p_merge)
#endif
    // A batch of (up to) 32 source ranges, one per lane, sorted by begin (bitonic, in registers)
    // and merged where contiguous: the cells of a P2P list are largely Morton-contiguous runs
    // (siblings), and a merged run is one bulk copy instead of several (the producer's copy issue
    // is serialised over the lanes, and small leaves have many small ranges)
    auto emit_rng = [&](int2 r, int tb, int cw) {
#if P2Q_MERGE
      int key = r.y > 0 ? r.x : 0x7fffffff, cnt = r.y > 0 ? r.y : 0;
#pragma unroll
      for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
          const int pkey = __shfl_xor_sync(0xffffffffu, key, j);
          const int pcnt = __shfl_xor_sync(0xffffffffu, cnt, j);
          const bool lower = (lane & j) == 0, up = (lane & kk) == 0;
          if (lower == up ? pkey < key : pkey > key) {
            key = pkey;
            cnt = pcnt;
          }
        }
      }
      const bool valid = cnt > 0;
      const int pend = __shfl_up_sync(0xffffffffu, key + cnt, 1);
      const bool head = valid && (lane == 0 || pend != key);
      const unsigned heads = __ballot_sync(0xffffffffu, head);
      const int nvalid = __popc(__ballot_sync(0xffffffffu, valid));
      const unsigned later = heads & ~(0xffffffffu >> (31 - lane));  // heads above this lane
      const int last = (later ? __ffs(later) - 1 : nvalid) - 1;       // last lane of this run
      const int rend = __shfl_sync(0xffffffffu, key + cnt, last < 0 ? 0 : last);
      emit(key, head ? rend - key : 0, tb, cw);
#else
      emit(r.x, r.y, tb, cw);
#endif
    };
    // Leaves in batches of P2Q_BATCH per queue atomic; lane j holds the descriptor of leaf j of
    // the batch. Every global load is issued one step ahead of its use so that the producer does
    // not stall the ring on L2 latency: the next batch is claimed (and its descriptors loaded)
    // while this one is emitted, the next leaf's first 32 source ranges are loaded while this
    // leaf is emitted, and range batch e0 + 32 while batch e0 is emitted.
    auto claim = [&](int &bb, int &nb) {
      int bs = 1;
      if (lane == 0) {  // guided: P2Q_BATCH leaves while many remain, single leaves for the tail
        const int seen = *(volatile int *)next_leaf;
        bs = nleaves - seen > 4 * P2Q_BATCH * (int)gridDim.x ? P2Q_BATCH : 1;
        bb = atomicAdd(next_leaf, bs);
      }
      bb = __shfl_sync(0xffffffffu, bb, 0);
      bs = __shfl_sync(0xffffffffu, bs, 0);
      nb = bb < nleaves ? min(bs, nleaves - bb) : 0;
    };
    auto lane_desc = [&](int4 d, int j) {
      return make_int4(__shfl_sync(0xffffffffu, d.x, j), __shfl_sync(0xffffffffu, d.y, j),
                       __shfl_sync(0xffffffffu, d.z, j), __shfl_sync(0xffffffffu, d.w, j));
    };
    // the leaf's own list: its merged source ranges (k_p2p_merge); ancestors' lists: raw ranges
    auto load_rng = [&](int off, int dw, int e0) {  // dw: the leaf's desc.w
      const int ncell = P2Q_CNT(dw);
      if (e0 + lane >= ncell) return make_int2(0, 0);
      return (dw & P2Q_RAW) ? Ls.p2p_rng[off + e0 + lane] : mrg[off + e0 + lane];
    };
    auto load_rng_raw = [&](int off, int ncell, int e0) {
      return e0 + lane < ncell ? Ls.p2p_rng[off + e0 + lane] : make_int2(0, 0);
    };
    int b0 = 0, nb0 = 0, b1 = 0, nb1 = 0;
    claim(b0, nb0);
    int4 dl0 = lane < nb0 ? desc[b0 + lane] : make_int4(0, 0, 0, 0);
    claim(b1, nb1);
    int4 dl1 = lane < nb1 ? desc[b1 + lane] : make_int4(0, 0, 0, 0);
    int2 rfirst = make_int2(0, 0);  // first range batch of the current leaf (prefetched)
    if (nb0 > 0) {
      const int4 d = lane_desc(dl0, 0);
      rfirst = load_rng(d.z, d.w, 0);
    }
    while (nb0 > 0) {
      for (int j = 0; j < nb0; ++j) {
        const int4 d = lane_desc(dl0, j);
        const int4 dn = j + 1 < nb0 ? lane_desc(dl0, j + 1)
                                    : (nb1 > 0 ? lane_desc(dl1, 0) : make_int4(0, 0, 0, 0));
        const int tb = d.x, tn = d.y, off = d.z, ncell = P2Q_CNT(d.w);
        const bool anc = d.w < 0;
        int2 rnext_leaf = make_int2(0, 0);
        for (int c0 = 0, nt = 0; c0 < tn; c0 += nt) {
          nt = p2q_chunk(tn - c0);
          const bool last_chunk = c0 + nt >= tn;
          const int cw = c0 | (nt << 16);  // chunk start | chunk size
          int2 r = c0 == 0 ? rfirst : load_rng(off, d.w, 0);
          if (last_chunk) rnext_leaf = load_rng(dn.z, dn.w, 0);
          // (1) the leaf itself first: the chunk's first tile starts with the leaf's own
          // particles (the consumers read their targets there) and is evaluated with the r = 0
          // mask, like every tile that holds own particles
          flags_pending = QF_FIRST | QF_MASK;
          emit(tb, lane == 0 ? tn : 0, tb, cw, true);
          if (!open) flags_pending &= ~QF_MASK;  // the own range ended on a tile boundary
          // (2) the leaf's P2P list, then (rare) those of its ancestors: a P2P pair with a
          // non-leaf target applies to every particle under it
          for (int e0 = 0; e0 < ncell; e0 += 32) {
            const int2 rn = e0 + 32 < ncell ? load_rng(off, d.w, e0 + 32) : make_int2(0, 0);
            if (r.x == tb) r.y = 0;  // the leaf itself: done above, masked
            emit_rng(r, tb, cw);
            r = rn;
          }
          if (anc) {
            for (int a = C.parent[leaves[b0 + j]]; a >= 0; a = C.parent[a]) {
              const int aoff = Ls.off[2][a], an = Ls.cnt[2][a];
              for (int e0 = 0; e0 < an; e0 += 32) emit_rng(load_rng_raw(aoff, an, e0), tb, cw);
            }
          }
          if (!open) open_tile();  // the chunk's last tile (possibly empty) carries QF_LAST
          close_tile(tb, flags_pending | QF_LAST, cw);
        }
        rfirst = rnext_leaf;
      }
      b0 = b1;
      nb0 = nb1;
      dl0 = dl1;
      if (nb0 > 0) {
        claim(b1, nb1);
        dl1 = lane < nb1 ? desc[b1 + lane] : make_int4(0, 0, 0, 0);
      } else {
        nb1 = 0;
      }
    }
    open_tile();
    close_tile(-1, QF_END, 0);
    return;
  }

  // -------------------------------------------------------------------- consumer warps 0..3
#if P2Q_QUAD
  // The four consumer warps form one pool of 128 lanes. A chunk of nt targets is held as
  // Q = ceil(nt / 4) quads (4 targets per lane in two packed pairs: every shared-memory source
  // load feeds four pairs and two independent chains); the pool's lanes are Q quads x
  // S = 128 / Q source slices (lane L: quad L % Q, slice L / Q takes sources L / Q, + S, ... of
  // every tile). At the chunk's end the 4 consumer warps meet at a named barrier, each lane
  // deposits its partial sums, and thread i sums target i's slices in slice order
  // (deterministic).
  {
    const int L = 32 * warp + lane;  // 0 .. 32 * P2Q_CWARPS - 1
    unsigned k = 0, chunk = 0;
    f2x t[6];
    f2x acc[8];
    int Q = 1, S = 1, g = 0, h = 0, nt = 0, tb = 0, c0 = 0;
    bool active = false;
    for (;;) {
      const int st = k % P2Q_STAGES;
      if ((L & 31) == 0) Q_TRACE(L >> 5, 3, k, 0);
      q_mbar_wait(&full[st], (k / P2Q_STAGES) & 1);
      const int4 m = meta[st];
      if ((L & 31) == 0) Q_TRACE(L >> 5, 4, k, m.y | ((m.w >> 16) << 16));
      if (m.z & QF_END) break;
      if (m.z & QF_FIRST) {
        tb = m.x;
        c0 = m.w & 0xffff;
        nt = m.w >> 16;
        FMM_DCHECK(tb >= 0 && (long long)tb + c0 + nt <= g_fmm_chk.pos && nt <= P2Q_CHUNK,
                   "P2P target chunk");
        Q = (nt + 3) >> 2;
        S = (32 * P2Q_CWARPS) / Q;
        g = L % Q;
        h = L / Q;
        active = h < S;
        const float4 *src = m.y > c0 + nt - 1 ? tile[st] : pos + tb;
        float4 tv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = 4 * g + e;
          tv[e] = src[c0 + (i < nt ? i : 4 * g)];
        }
        t[0] = pk(m1 * tv[0].x, m1 * tv[1].x);
        t[1] = pk(m1 * tv[0].y, m1 * tv[1].y);
        t[2] = pk(m1 * tv[0].z, m1 * tv[1].z);
        t[3] = pk(m1 * tv[2].x, m1 * tv[3].x);
        t[4] = pk(m1 * tv[2].y, m1 * tv[3].y);
        t[5] = pk(m1 * tv[2].z, m1 * tv[3].z);
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = 0ull;
      }
      const int n = active ? m.y : 0;
      if (m.z & QF_MASK)
        p2p_tile_quad_rt<true>(tile[st], n, h, S, t, acc);
      else
        p2p_tile_quad_rt<false>(tile[st], n, h, S, t, acc);
      if ((L & 31) == 0) Q_TRACE(L >> 5, 5, k, m.z);
      ++k;
      if (m.z & QF_LAST) {
        float4(*rb)[4] = red[chunk % P2Q_REDBUF];
#if P2Q_LASTRED == 2
        // buffer chunk % 2 was last used by chunk - 2: wait (rarely) until that reduction is done
        if (chunk >= 2)
          while (*(volatile int *)&red_gen[chunk % 2] < (int)(chunk >> 1)) {
          }
        __syncwarp();
#endif
        ++chunk;
        if (active) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const float2 ph = upk(acc[4 * c]), gx = upk(acc[4 * c + 1]), gy = upk(acc[4 * c + 2]),
                         gz = upk(acc[4 * c + 3]);
            rb[h * Q + g][2 * c] = make_float4(ph.x, gx.x, gy.x, gz.x);
            rb[h * Q + g][2 * c + 1] = make_float4(ph.y, gx.y, gy.y, gz.y);
          }
        }
        auto reduce = [&](int first, int step) {  // target i: its S slices in slice order
          for (int i = first; i < nt; i += step) {
            const int gi = i >> 2, e = i & 3;
            float4 v = rb[gi][e];
            for (int hh = 1; hh < S; ++hh) {
              const float4 u = rb[hh * Q + gi][e];
              v.x += u.x;
              v.y += u.y;
              v.z += u.z;
              v.w += u.w;
            }
            acc_out[tb + c0 + i] = v;
          }
        };
#if P2Q_LASTRED
        // lock-free: the last of the consumer warps to deposit its partials reduces the chunk,
        // the others go on (a buffer is reused P2Q_STAGES chunks later, after every warp has
        // released the tile that ended this chunk -- see P2Q_RED)
        const int b = (chunk - 1) % P2Q_REDBUF;
        __threadfence_block();
        __syncwarp();
        int prev = 0;
        if ((L & 31) == 0) prev = atomicAdd(&red_cnt[b], 1);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == P2Q_CWARPS - 1) {
          __threadfence_block();
          reduce(L & 31, 32);
          __syncwarp();
          if ((L & 31) == 0) {
            red_cnt[b] = 0;
            if (P2Q_LASTRED == 2) {
              __threadfence_block();
              atomicAdd(&red_gen[b], 1);
            }
          }
        }
#else
        asm volatile("bar.sync 2, %0;" ::"n"(32 * P2Q_CWARPS) : "memory");
        reduce(L, 32 * P2Q_CWARPS);
        if (P2Q_REDBUF == 1) asm volatile("bar.sync 2, %0;" ::"n"(32 * P2Q_CWARPS) : "memory");
#endif
      }
      __syncwarp();
      if ((L & 31) == 0) q_mbar_arrive(&empty[st]);
    }
    return;
  }
#else
  unsigned k = 0, chunk = 0;
  f2x tx = 0ull, ty = 0ull, tz = 0ull;
  f2x acc[4] = {0ull, 0ull, 0ull, 0ull};
  int G = 1, S = 1, grp = 0, h = 0, nt = 0, tb = 0, c0 = 0;
  bool active = false;
  for (;;) {
    const int st = k % P2Q_STAGES;
    q_mbar_wait(&full[st], (k / P2Q_STAGES) & 1);
    const int4 m = meta[st];
    if (m.z & QF_END) break;
    if (m.z & QF_FIRST) {
      tb = m.x;
      c0 = m.w & 0xffff;
      nt = m.w >> 16;
      G = (nt + 1) >> 1;
      S = 32 / G;
      grp = lane % G;
      h = lane / G;
      active = h < S;
      const int i0 = c0 + 2 * grp, i1 = i0 + 1;
      // the targets are particles c0.. of the leaf, i.e. of this (first, masked) tile when the
      // whole leaf fits in one tile
      const float4 *src = m.y > c0 + nt - 1 ? tile[st] : pos + tb;
      const float4 t0 = 2 * grp < nt ? src[i0] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 t1 = 2 * grp + 1 < nt ? src[i1] : t0;
      tx = pk(m1 * t0.x, m1 * t1.x);
      ty = pk(m1 * t0.y, m1 * t1.y);
      tz = pk(m1 * t0.z, m1 * t1.z);
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[c] = 0ull;
    }
    // this warp's quarter of the tile
    const int n = m.y;
    const int a = (warp * n) / P2Q_CWARPS, e = ((warp + 1) * n) / P2Q_CWARPS;
    if (m.z & QF_MASK)
      p2p_tile_raw<true>(tile[st] + a, active ? e - a : 0, h, S, tx, ty, tz, acc);
    else
      p2p_tile_raw<false>(tile[st] + a, active ? e - a : 0, h, S, tx, ty, tz, acc);
    ++k;
    if (!(m.z & QF_LAST)) {
      __syncwarp();
      if (lane == 0) q_mbar_arrive(&empty[st]);
    } else {
      // slices of this warp in slice order; the last of the four warps to finish sums the warps
      // in warp order and writes the chunk (deterministic, and nobody waits at a barrier)
      float2 r[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) r[c] = upk(acc[c]);
      float2 tot[4] = {r[0], r[1], r[2], r[3]};
      for (int sl = 1; sl < S; ++sl) {
        const int from = grp + sl * G;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          tot[c].x += __shfl_sync(0xffffffffu, r[c].x, from);
          tot[c].y += __shfl_sync(0xffffffffu, r[c].y, from);
        }
      }
      const int b = chunk % P2Q_RED;
      ++chunk;
      if (h == 0) {
        if (2 * grp < nt) red[b][warp][2 * grp] = make_float4(tot[0].x, tot[1].x, tot[2].x, tot[3].x);
        if (2 * grp + 1 < nt)
          red[b][warp][2 * grp + 1] = make_float4(tot[0].y, tot[1].y, tot[2].y, tot[3].y);
      }
      __threadfence_block();
      __syncwarp();
      int prev = 0;
      if (lane == 0) prev = atomicAdd(&red_cnt[b], 1);
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev == P2Q_CWARPS - 1) {
        __threadfence_block();
        for (int i = lane; i < nt; i += 32) {
          float4 v = red[b][0][i];
#pragma unroll
          for (int w = 1; w < P2Q_CWARPS; ++w) {
            const float4 u = red[b][w][i];
            v.x += u.x;
            v.y += u.y;
            v.z += u.z;
            v.w += u.w;
          }
          acc_out[tb + c0 + i] = v;
        }
        __syncwarp();
        if (lane == 0) red_cnt[b] = 0;
      }
      __syncwarp();
      if (lane == 0) q_mbar_arrive(&empty[st]);  // after the reduction (see P2Q_RED)
    }
  }
#endif
}

// per target leaf: (begin, count, own P2P list offset, own list count | 1 << 31 when a proper
// ancestor has a non-empty P2P list)
__global__ void k_p2p_desc(const int *__restrict__ leaves, int nleaves, CellsView C, ListsView Ls,
                           int4 *__restrict__ desc, int raw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nleaves) return;
  const int leaf = leaves[i];
  bool anc = false;
  for (int a = C.parent[leaf]; a >= 0 && !anc; a = C.parent[a]) anc = Ls.cnt[2][a] > 0;
  desc[i] = make_int4(C.beg[leaf], C.cnt[leaf], Ls.off[2][leaf],
                      Ls.cnt[2][leaf] | (anc ? (int)0x80000000u : 0) | raw);
}

// Per target leaf, a warp merges the source ranges of the leaf's own P2P list AND of its
// ancestors' lists (a P2P pair with a non-leaf target applies to every particle under it; in
// hybrid mode a large target against a tiny source cell is P2P) where they are contiguous in
// particle order (the cells of a P2P list are largely Morton-contiguous runs: siblings, the
// children of a split neighbour), leaving the leaf itself out. The runs go to mrg[off ..] (the
// slot of the leaf's own list) and desc.w = their count with the ancestor flag cleared, so the
// producer warp of k_p2p_tma -- the bottleneck on small leaves -- issues fewer, longer bulk copies
// and never walks the tree (measured with the oracle's lists: 88 ranges -> 23 runs per leaf of
// < 20 particles, 109 -> 41 for 20-64). O(n) per list: the begins go into a shared-memory hash
// table, each range finds the range starting at its end (its successor), and each run head (a
// range nobody precedes) sums its chain. Fallback (the producer then walks the ancestors as
// before): more than P2P_MERGE_MAX ranges, or more runs than the own list's slot holds.
#define P2P_MERGE_MAX 256
#ifndef P2P_MERGE_NT
#define P2P_MERGE_NT 16  // leaves of more particles keep their raw ranges (32: C4 +0.4 ms)
#endif
#define P2P_MERGE_HT 512  // hash slots per warp (power of two, >= 2 x P2P_MERGE_MAX)
__global__ void __launch_bounds__(128) k_p2p_merge(const int *__restrict__ leaves, int nleaves,
                                                   CellsView C, ListsView Ls, int4 *__restrict__ desc,
                                                   int2 *__restrict__ mrg) {
  __shared__ int2 rr[4][P2P_MERGE_MAX];           // the ranges (own list, then ancestors')
  __shared__ int ht[4][P2P_MERGE_HT];             // begin -> range index (-1: empty)
  __shared__ short nx[4][P2P_MERGE_MAX];          // successor range (-1: none)
  __shared__ short NX2[4][P2P_MERGE_MAX];         // pointer-jumping double buffer
  __shared__ short hs[4][P2P_MERGE_MAX];          // the slot a range landed in
  __shared__ unsigned char hp[4][P2P_MERGE_MAX];  // has a predecessor
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int2 *R = rr[w];
  int *T = ht[w];
  short *NX = nx[w], *HS = hs[w];
  unsigned char *HP = hp[w];
  for (int e = lane; e < P2P_MERGE_HT; e += 32) T[e] = -1;
  auto slot = [](int key) { return (int)(((unsigned)key * 2654435761u) >> (32 - 9)) & (P2P_MERGE_HT - 1); };
  for (int i = blockIdx.x * 4 + w; i < nleaves; i += gridDim.x * 4) {
    const int leaf = leaves[i];
    const int4 d = desc[i];  // (begin, count, own list offset, own count | ancestor flag)
    const int tb = d.x, off = d.z, n0 = d.w & 0x7fffffff;
    const bool anc = d.w < 0;
    if (d.y > P2P_MERGE_NT) {  // large leaf: its consumers outpace the producer anyway
      if (lane == 0) desc[i].w = d.w | P2Q_RAW;
      continue;
    }
    __syncwarp();
    // gather the ranges: own list, then every ancestor's (none of them is the leaf itself,
    // which lies inside every ancestor's particle range)
    int n = 0;
    bool fits = true;
    auto gather = [&](int loff, int lcnt) {
      if (n + lcnt > P2P_MERGE_MAX) {
        fits = false;
        return;
      }
      for (int e = lane; e < lcnt; e += 32) {
        int2 r = Ls.p2p_rng[loff + e];
        if (r.x == tb) r.y = 0;
        R[n + e] = r;
      }
      n += lcnt;
    };
    gather(off, n0);
    if (anc)
      for (int a = C.parent[leaf]; a >= 0 && fits; a = C.parent[a]) {
        const int ac = Ls.cnt[2][a];
        if (ac > 0) gather(Ls.off[2][a], ac);
      }
    if (!fits) {  // fallback: the raw own list, the producer walks the ancestors
      if (lane == 0) desc[i].w = d.w | P2Q_RAW;
      continue;
    }
    __syncwarp();
    for (int e = lane; e < n; e += 32) {
      const int2 r = R[e];
      NX[e] = -1;
      HP[e] = 0;
      if (r.y > 0) {
        int h = slot(r.x);
        while (atomicCAS(&T[h], -1, e) != -1) h = (h + 1) & (P2P_MERGE_HT - 1);
        HS[e] = (short)h;
      }
    }
    __syncwarp();
    for (int e = lane; e < n; e += 32) {
      const int2 r = R[e];
      if (r.y <= 0) continue;
      const int end = r.x + r.y;
      for (int h = slot(end);; h = (h + 1) & (P2P_MERGE_HT - 1)) {
        const int j = T[h];
        if (j < 0) break;
        if (R[j].x == end) {
          NX[e] = (short)j;
          HP[j] = 1;
          break;
        }
      }
    }
    __syncwarp();
    int m = 0;
    for (int e0 = 0; e0 < n; e0 += 32) {
      const int e = e0 + lane;
      const bool head = e < n && R[e].y > 0 && !HP[e];
      m += __popc(__ballot_sync(0xffffffffu, head));
    }
    const bool merged = m <= n0;  // the runs fit the own list's slot of mrg
    if (merged) {
      // last range of every chain by pointer jumping (NX[e] -> the chain's last range, in
      // log2(run length) rounds, no divergent walks)
      for (int e = lane; e < n; e += 32)
        if (NX[e] < 0) NX[e] = (short)e;
      __syncwarp();
      short *A = NX, *B = NX2[w];
      for (;;) {
        bool changed = false;
        for (int e = lane; e < n; e += 32) {
          const short v = A[A[e]];
          B[e] = v;
          changed |= v != A[e];
        }
        __syncwarp();
        short *t = A;
        A = B;
        B = t;
        if (!__any_sync(0xffffffffu, changed)) break;
      }
      int mo = 0;
      for (int e0 = 0; e0 < n; e0 += 32) {
        const int e = e0 + lane;
        bool head = false;
        int2 run = make_int2(0, 0);
        if (e < n) {
          run = R[e];
          head = run.y > 0 && !HP[e];
          if (head) {
            const int2 last = R[A[e]];
            run.y = last.x + last.y - run.x;
          }
        }
        const unsigned hb = __ballot_sync(0xffffffffu, head);
        if (head) mrg[off + mo + __popc(hb & ((1u << lane) - 1u))] = run;
        mo += __popc(hb);
      }
      FMM_DCHECK((long long)off + m <= g_fmm_chk.lists, "P2P merged runs");
    if (lane == 0) desc[i].w = m;  // ancestors folded in: flag cleared
    } else if (lane == 0) {
      desc[i].w = d.w | P2Q_RAW;
    }
    __syncwarp();
    for (int e = lane; e < n; e += 32)  // clear the used slots for the next leaf
      if (R[e].y > 0) T[HS[e]] = -1;
  }
}

void launch_p2p_leaves(const int *leaves, int nleaves, CellsView C, ListsView Ls,
                       const float4 *pos, float4 *acc, int *counter, int4 *desc, int2 *mrg,
                       cudaStream_t st, cudaEvent_t ev_main) {
  static const bool legacy = getenv("FMM_P2P_LEGACY") != nullptr;  // A/B: round-1 kernel
  if (!legacy) {
    const size_t dyn = sizeof(float4) * P2Q_STAGES * P2Q_TILE;
    fmm_smem_optin((const void *)k_p2p_tma, dyn);
    const int res = fmm_resident_blocks((const void *)k_p2p_tma, P2Q_THREADS, dyn);
    if (nleaves <= 0) return;
#ifndef P2Q_MERGE_PASS
#define P2Q_MERGE_PASS 1
#endif
    k_p2p_desc<<<(nleaves + 255) / 256, 256, 0, st>>>(leaves, nleaves, C, Ls, desc,
                                                       P2Q_MERGE_PASS ? 0 : P2Q_RAW);
    if (P2Q_MERGE_PASS)
      k_p2p_merge<<<std::min((nleaves + 3) / 4, 148 * 16), 128, 0, st>>>(leaves, nleaves, C, Ls, desc, mrg);
    const int b = std::max(1, std::min(res, (nleaves + P2Q_BATCH - 1) / P2Q_BATCH));
    cudaMemsetAsync(counter, 0, sizeof(int), st);
    if (ev_main) cudaEventRecord(ev_main, st);  // the main kernel alone (bench roofline)
    k_p2p_tma<<<b, P2Q_THREADS, dyn, st>>>(leaves, nleaves, C, Ls, pos, acc, -1.0f, counter, desc, mrg);
#ifdef P2Q_TRACE
    k_q_trace_dump<<<1, 1, 0, st>>>();
#endif
    return;
  }
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

FMM_CHK_DEFINE_SETTER(fmm_chk_set_p2p)
